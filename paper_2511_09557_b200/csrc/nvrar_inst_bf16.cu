// Instantiates the BF16 kernels (split per dtype so nvcc builds them in parallel).
#include "nvrar_kernels.cuh"

namespace nvrar {
KernelFn kernel_bf16(bool flat, int nodes, bool emu) { return kernel_for<BF16>(flat, nodes, emu); }
}  // namespace nvrar
