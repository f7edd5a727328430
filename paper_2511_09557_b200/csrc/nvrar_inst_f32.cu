// Instantiates the F32 kernels (split per dtype so nvcc builds them in parallel).
#include "nvrar_kernels.cuh"

namespace nvrar {
KernelFn kernel_f32(bool flat, int nodes, bool emu, bool lamport) {
  return lamport ? kernel_for<F32, true>(flat, nodes, emu) : kernel_for<F32, false>(flat, nodes, emu);
}
KernelFn kernel_direct_f32(int nodes) { return direct_for<F32>(nodes); }
}  // namespace nvrar
