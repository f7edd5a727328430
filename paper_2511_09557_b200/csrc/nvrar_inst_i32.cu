// Instantiates the I32 hierarchical and direct kernels (flat: nvrar_flat_i32.cu).
#include "nvrar_kernels.cuh"

namespace nvrar {
KernelFn kernel_hier_i32(int nodes, int gpus, bool emu, bool lamport) {
  (void)lamport;  // int32 has no spare bit pattern: always LL
  return hier_kernel_for<I32, false>(nodes, gpus, emu);
}
KernelFn kernel_direct_i32(int nodes, int gpus) { return direct_for<I32>(nodes, gpus); }
}  // namespace nvrar
