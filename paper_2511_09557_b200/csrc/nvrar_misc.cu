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

// Word-atomicity canary (acceptance_test.cpp:338-364, criterion 7, on the GPU
// transport): the writer streams 16-byte fused cells {i*K, base+i, i*K, base+i}
// into the peer's canary cell with seeded delays between stores; the reader
// polls its own cell and checks every observation: both flags equal and each
// data word the function of its flag. A torn cell (a mix of two stores) breaks
// the relation. out[0] = torn observations (reader) / 0 (writer), ~0 = timeout.
__global__ void canary_kernel(const __grid_constant__ LaunchParams lp, int peer, int iters,
                              int writer, uint32_t base, uint32_t jitter_ns, uint32_t seed,
                              uint32_t* out) {
  const RankDesc& d = lp.d0;
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  constexpr uint32_t K = 2654435761u;
  const uint64_t t_limit = globaltimer() + d.timeout_ns;
  if (writer) {
    uint4* theirs = canary_cell(d, peer);
    for (int i = 1; i <= iters; ++i) {
      const uint32_t f = base + static_cast<uint32_t>(i);
      st_volatile16(theirs, f * K, f, f * K, f);
      if (jitter_ns) __nanosleep(mix32(seed ^ mix32(static_cast<uint32_t>(i))) % jitter_ns);
    }
    out[0] = 0;
    return;
  }
  const uint4* mine = canary_cell(d, d.rank);
  uint32_t torn = 0;
  const uint32_t last = base + static_cast<uint32_t>(iters);
  for (uint32_t spins = 0;; ++spins) {
    const uint4 v = ld_volatile16(mine);
    const bool empty = (v.x & v.y & v.z & v.w) == 0xFFFFFFFFu;
    if (!empty && (v.y != v.w || v.x != v.y * K || v.z != v.w * K)) ++torn;
    // done at this run's last flag — or past it: the writer does not wait for
    // the reader, so it may already be streaming its next run's cells (flags
    // grow run to run; those observations are checked the same way)
    if (!empty && v.y == v.w && static_cast<int32_t>(v.y - last) >= 0) break;
    if (jitter_ns) __nanosleep(mix32(seed ^ spins) % jitter_ns);
    if ((spins & 255u) == 0u && globaltimer() > t_limit) {
      out[0] = ~0u;
      return;
    }
  }
  out[0] = torn;
}

using CanaryFn = void (*)(LaunchParams, int, int, int, uint32_t, uint32_t, uint32_t, uint32_t*);
CanaryFn canary_fn() { return canary_kernel; }

KernelFn select_kernel(int dtype, bool flat, int nodes, int gpus, bool emu, bool lamport,
                       bool fast) {
  switch (dtype) {
    case 0: return flat ? kernel_flat_i32(nodes, gpus, emu, false, fast) : kernel_hier_i32(nodes, gpus, emu, false);
    case 1: return flat ? kernel_flat_f32(nodes, gpus, emu, lamport, fast) : kernel_hier_f32(nodes, gpus, emu, lamport);
    case 2: return flat ? kernel_flat_bf16(nodes, gpus, emu, lamport, fast) : kernel_hier_bf16(nodes, gpus, emu, lamport);
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
