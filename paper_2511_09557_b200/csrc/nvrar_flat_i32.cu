// Instantiates the I32 flat kernels (LL protocol only: int32 has no spare bit
// pattern for the Lamport empty marker).
#include "nvrar_kernels.cuh"

namespace nvrar {
KernelFn kernel_flat_i32(int nodes, int gpus, bool emu, bool lamport, bool fast) {
  return lamport ? flat_kernel_for<I32, true>(nodes, gpus, emu, fast)
                 : flat_kernel_for<I32, false>(nodes, gpus, emu, fast);
}
}  // namespace nvrar
