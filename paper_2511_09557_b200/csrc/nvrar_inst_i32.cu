// Instantiates the I32 kernels (split per dtype so nvcc builds them in parallel).
#include "nvrar_kernels.cuh"

namespace nvrar {
KernelFn kernel_i32(bool flat, int nodes, bool emu, bool lamport) {
  (void)lamport;  // int32 has no spare bit pattern: always LL
  return kernel_for<I32, false>(flat, nodes, emu);
}
KernelFn kernel_direct_i32(int nodes) { return direct_for<I32>(nodes); }
}  // namespace nvrar
