// Instantiates the I32 kernels (split per dtype so nvcc builds them in parallel).
#include "nvrar_kernels.cuh"

namespace nvrar {
KernelFn kernel_i32(bool flat, int nodes, bool emu) { return kernel_for<I32>(flat, nodes, emu); }
}  // namespace nvrar
