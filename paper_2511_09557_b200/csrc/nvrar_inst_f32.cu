// Instantiates the F32 kernels (split per dtype so nvcc builds them in parallel).
#include "nvrar_kernels.cuh"

namespace nvrar {
KernelFn kernel_f32(bool flat, int nodes, bool emu) { return kernel_for<F32>(flat, nodes, emu); }
}  // namespace nvrar
