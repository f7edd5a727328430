// Instantiates the BF16 kernels (split per dtype so nvcc builds them in parallel).
#include "nvrar_kernels.cuh"

namespace nvrar {
KernelFn kernel_bf16(bool flat, int nodes, bool emu, bool lamport) {
  return lamport ? kernel_for<BF16, true>(flat, nodes, emu) : kernel_for<BF16, false>(flat, nodes, emu);
}
KernelFn kernel_direct_bf16(int nodes) { return direct_for<BF16>(nodes); }
}  // namespace nvrar
