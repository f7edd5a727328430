// Instantiates the BF16 hierarchical and direct kernels (the flat ones are in
// nvrar_flat_bf16.cu: one file per group so nvcc builds them in parallel).
#include "nvrar_kernels.cuh"

namespace nvrar {
KernelFn kernel_hier_bf16(int nodes, int gpus, bool emu, bool lamport) {
  return lamport ? hier_kernel_for<BF16, true>(nodes, gpus, emu)
                 : hier_kernel_for<BF16, false>(nodes, gpus, emu);
}
KernelFn kernel_direct_bf16(int nodes, int gpus) { return direct_for<BF16>(nodes, gpus); }
}  // namespace nvrar
