// Instantiates the F32 hierarchical and direct kernels (the flat ones are in
// nvrar_flat_f32.cu: one file per group so nvcc builds them in parallel).
#include "nvrar_kernels.cuh"

namespace nvrar {
KernelFn kernel_hier_f32(int nodes, int gpus, bool emu, bool lamport) {
  return lamport ? hier_kernel_for<F32, true>(nodes, gpus, emu)
                 : hier_kernel_for<F32, false>(nodes, gpus, emu);
}
KernelFn kernel_direct_f32(int nodes, int gpus) { return direct_for<F32>(nodes, gpus); }
}  // namespace nvrar
