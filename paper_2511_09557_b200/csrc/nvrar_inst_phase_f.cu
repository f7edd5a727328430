// Instantiates the phase-only kernels (hier_kernel MODE != full) for the
// floating-point dtypes, default protocol (Lamport). The intra-only phases do
// not depend on the node count; rd_inter does.
#include "nvrar_kernels.cuh"

namespace nvrar {
template <class E, bool EMU>
static KernelFn phase_pick(int mode, int nodes) {
  switch (mode) {
    case kModeRS: return hier_kernel<E, true, 1, EMU, kModeRS>;
    case kModeAG: return hier_kernel<E, true, 1, EMU, kModeAG>;
    case kModeRD:
      if constexpr (E::kBytes == 4) return phase_for<E, true, EMU, kModeRD>(nodes);
      return nullptr;
    default: return nullptr;
  }
}
KernelFn kernel_phase_f32(int mode, int nodes, bool emu) {
  return emu ? phase_pick<F32, true>(mode, nodes) : phase_pick<F32, false>(mode, nodes);
}
KernelFn kernel_phase_bf16(int mode, int nodes, bool emu) {
  return emu ? phase_pick<BF16, true>(mode, nodes) : phase_pick<BF16, false>(mode, nodes);
}
}  // namespace nvrar
