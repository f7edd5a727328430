// Instantiates the registered-buffer one-shot kernels (nvrar_allreduce_registered).
#include "nvrar_kernels.cuh"

namespace nvrar {
KernelFn kernel_pull_f32(int nodes, int gpus) { return pull_for<F32>(nodes, gpus); }
KernelFn kernel_pull_bf16(int nodes, int gpus) { return pull_for<BF16>(nodes, gpus); }
KernelFn kernel_pull_i32(int nodes, int gpus) { return pull_for<I32>(nodes, gpus); }
}  // namespace nvrar
