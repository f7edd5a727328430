// Instantiates the I32 flat kernels (LL protocol only: int32 has no spare bit
// pattern for the Lamport empty marker).
#include "nvrar_kernels.cuh"

namespace nvrar {
KernelFn kernel_flat_i32(int nodes, int gpus, bool emu, bool lamport) {
  (void)lamport;
  return flat_kernel_for<I32, false>(nodes, gpus, emu);
}
}  // namespace nvrar
