// Kernel dispatch plus the two small kernels: the count == 0 sequence bump and
// the NVLink signal-latency probe (alpha_signal of the roofline).
#include "nvrar_kernels.cuh"

namespace nvrar {

// n == 0 still consumes a sequence number (nvrar.hpp:93-96).
__global__ void seq_bump_kernel(const __grid_constant__ LaunchParams lp) {
  const RankDesc& d = *lp.desc[blockIdx.y];
  pdl_wait();
  if (ld_volatile32(&d.state->err.code) != 0u) return;
  const uint32_t s = ld_volatile32(&d.state->seq[0]) + 1u;
  __syncthreads();
  for (int i = threadIdx.x; i < kSeqSlots; i += blockDim.x) d.state->seq[i] = s;
}

// Flag ping-pong between this rank and `peer` through the diag words of the
// symmetric regions: the initiator stores base+i into the peer's word and
// waits for the echo in its own. Round trip / 2 = one-way signal latency.
__global__ void pingpong_kernel(const __grid_constant__ LaunchParams lp, int peer, int iters,
                                uint64_t base, int initiator, uint64_t* out_ns) {
  const RankDesc& d = lp.d0;
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  uint64_t* mine = diag_word(d, d.rank);
  uint64_t* theirs = diag_word(d, peer);
  const uint64_t t_limit = globaltimer() + d.timeout_ns;
  const uint64_t t0 = globaltimer();
  uint64_t t_last_send = 0, t_last_recv = 0;
  for (int i = 1; i <= iters; ++i) {
    const uint64_t v = base + static_cast<uint64_t>(i);
    if (initiator) {
      t_last_send = globaltimer();
      st_volatile64(theirs, v);
    }
    while (ld_volatile64(mine) != v) {
      if (globaltimer() > t_limit) {
        *out_ns = ~0ull;
        return;
      }
    }
    t_last_recv = globaltimer();
    if (!initiator) st_volatile64(theirs, v);
  }
  // [0] initiator's elapsed ns; [1] last send (initiator) / last echo time
  // (responder); [2] last receive — absolute %globaltimer values, which let the
  // host estimate the clock offset between the two GPUs.
  out_ns[0] = globaltimer() - t0;
  out_ns[1] = initiator ? t_last_send : t_last_recv;
  out_ns[2] = t_last_recv;
}

KernelFn select_kernel(int dtype, bool flat, int nodes, int gpus, bool emu, bool lamport) {
  switch (dtype) {
    case 0: return flat ? kernel_flat_i32(nodes, gpus, emu, false) : kernel_hier_i32(nodes, gpus, emu, false);
    case 1: return flat ? kernel_flat_f32(nodes, gpus, emu, lamport) : kernel_hier_f32(nodes, gpus, emu, lamport);
    case 2: return flat ? kernel_flat_bf16(nodes, gpus, emu, lamport) : kernel_hier_bf16(nodes, gpus, emu, lamport);
    default: return nullptr;
  }
}

KernelFn select_direct(int dtype, int nodes, int gpus) {
  switch (dtype) {
    case 0: return kernel_direct_i32(nodes, gpus);
    case 1: return kernel_direct_f32(nodes, gpus);
    case 2: return kernel_direct_bf16(nodes, gpus);
    default: return nullptr;
  }
}

KernelFn select_phase(int dtype, int mode, int nodes, bool emu) {
  switch (dtype) {
    case 0: return kernel_phase_i32(mode, nodes, emu);
    case 1: return kernel_phase_f32(mode, nodes, emu);
    case 2: return kernel_phase_bf16(mode, nodes, emu);
    default: return nullptr;
  }
}

KernelFn select_pull(int dtype, int nodes, int gpus) {
  switch (dtype) {
    case 0: return kernel_pull_i32(nodes, gpus);
    case 1: return kernel_pull_f32(nodes, gpus);
    case 2: return kernel_pull_bf16(nodes, gpus);
    default: return nullptr;
  }
}

KernelFn bump_kernel() { return seq_bump_kernel; }

using PingFn = void (*)(LaunchParams, int, int, uint64_t, int, uint64_t*);
PingFn pingpong_fn() { return pingpong_kernel; }

int flat_max_gpus(int nodes) {
  switch (nodes) {
    case 1: return 8;
    case 2: return 8;
    case 4: return 4;
    case 8: return 2;
    default: return 0;
  }
}

}  // namespace nvrar
