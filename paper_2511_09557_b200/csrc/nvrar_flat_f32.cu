// Instantiates the F32 flat kernels (one-shot / two-shot), specialised on
// (nodes, MAXG), both protocols, device and virtual-rank launches.
#include "nvrar_kernels.cuh"

namespace nvrar {
KernelFn kernel_flat_f32(int nodes, int gpus, bool emu, bool lamport, bool fast) {
  return lamport ? flat_kernel_for<F32, true>(nodes, gpus, emu, fast)
                 : flat_kernel_for<F32, false>(nodes, gpus, emu, fast);
}
}  // namespace nvrar
