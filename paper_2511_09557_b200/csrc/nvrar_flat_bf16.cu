// Instantiates the BF16 flat kernels (one-shot / two-shot), specialised on
// (nodes, MAXG), both protocols, device and virtual-rank launches.
#include "nvrar_kernels.cuh"

namespace nvrar {
KernelFn kernel_flat_bf16(int nodes, int gpus, bool emu, bool lamport) {
  return lamport ? flat_kernel_for<BF16, true>(nodes, gpus, emu)
                 : flat_kernel_for<BF16, false>(nodes, gpus, emu);
}
}  // namespace nvrar
