// Instantiates the phase-only kernels (hier_kernel MODE != full) for int32
// (LL protocol, as the all-reduce uses for int32).
#include "nvrar_kernels.cuh"

namespace nvrar {
template <bool EMU>
static KernelFn phase_pick_i32(int mode, int nodes) {
  switch (mode) {
    case kModeRS: return hier_kernel<I32, false, 1, EMU, kModeRS>;
    case kModeAG: return hier_kernel<I32, false, 1, EMU, kModeAG>;
    case kModeRD: return phase_for<I32, false, EMU, kModeRD>(nodes);
    default: return nullptr;
  }
}
KernelFn kernel_phase_i32(int mode, int nodes, bool emu) {
  return emu ? phase_pick_i32<true>(mode, nodes) : phase_pick_i32<false>(mode, nodes);
}
}  // namespace nvrar
