// Instantiates the F32 flat kernels (one-shot / two-shot), specialised on
// (nodes, MAXG), both protocols, device and virtual-rank launches.
#include "nvrar_kernels.cuh"

namespace nvrar {
KernelFn kernel_flat_f32(int nodes, int gpus, bool emu, bool lamport) {
  return lamport ? flat_kernel_for<F32, true>(nodes, gpus, emu)
                 : flat_kernel_for<F32, false>(nodes, gpus, emu);
}
}  // namespace nvrar
