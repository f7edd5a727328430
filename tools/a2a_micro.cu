// One-shot exchange floor on P GPUs (one process, peer access): every GPU
// pushes `bytes` of Lamport cells to each of the P-1 others (slot per source)
// and polls its P-1 incoming slots — the communication of a one-shot
// all-reduce with nothing else. Stamps %globaltimer; reports the time from the
// earliest send start to the last arrival over all GPUs (timer offsets from a
// ping-pong with GPU0).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/a2a_micro tools/a2a_micro.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

constexpr int kMaxP = 8;

struct Peers {
  uint4* slot[kMaxP];  // slot[p] = my slot inside GPU p's buffer (for my pushes)
  uint4* in[kMaxP];    // my buffer's slot for source p
  volatile uint32_t* ready;     // on GPU0: ready[g]
  volatile uint32_t* go[kMaxP]; // go word on each GPU
};

__device__ __forceinline__ uint64_t gt() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void exch(Peers pr, int me, int P, uint64_t cells, uint32_t val, uint64_t* stamps,
                     int sleep_ns, int leader, int bulk) {
  extern __shared__ uint4 stage[];
  // start barrier across GPUs so launch skew does not count
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) pr.ready[me] = val;
    if (me == 0 && blockIdx.x == 0) {
      for (int g = 0; g < P; ++g)
        while (pr.ready[g] != val) {
        }
      for (int g = 0; g < P; ++g) *pr.go[g] = val;
    }
    while (*pr.go[me] != val) {
    }
    stamps[3 * blockIdx.x] = gt();
  }
  __syncthreads();
  if (bulk) {
    // TMA bulk copy: this CTA's contiguous range, staged once in shared memory,
    // one cp.async.bulk per peer (large NVLink writes instead of 16-byte stores)
    const uint64_t c0 = cells * blockIdx.x / gridDim.x, c1 = cells * (blockIdx.x + 1) / gridDim.x;
    for (uint64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) stage[i - c0] = make_uint4(val, val, val, val);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0 && c1 > c0) {
      const uint32_t sm = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
      for (int j = 1; j < P; ++j) {
        const int q = (me + j) % P;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(pr.slot[q] + c0),
                     "r"(sm), "r"(static_cast<uint32_t>((c1 - c0) * 16)) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
  } else if (bulk == 2) {
    // 32-byte stores (sm_100 STG.256): two cells per store
    for (uint64_t i = 2 * (blockIdx.x * blockDim.x + threadIdx.x); i < cells;
         i += 2ull * gridDim.x * blockDim.x) {
      for (int j = 1; j < P; ++j) {
        const int q = (me + j) % P;
        asm volatile("st.volatile.global.v8.u32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(pr.slot[q] + i),
                     "r"(val));
      }
    }
  } else {
  for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cells;
       i += (uint64_t)gridDim.x * blockDim.x) {
    for (int j = 1; j < P; ++j) {
      const int q = (me + j) % P;
      asm volatile("st.volatile.global.v4.u32 [%0], {%1,%1,%1,%1};" ::"l"(pr.slot[q] + i),
                   "r"(val));
    }
  }
  }
  if (threadIdx.x == 0) stamps[3 * blockIdx.x + 1] = gt();
  for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cells;
       i += (uint64_t)gridDim.x * blockDim.x) {
    for (int j = 1; j < P; ++j) {
      const int q = (me + j) % P;
      if (leader) {
        // lane 31's cell first (one poller per warp), then every lane checks its own
        const uint64_t last = i - (threadIdx.x & 31) + 31;
        if ((threadIdx.x & 31) == 31 || last >= cells) {
        }
        if ((threadIdx.x & 31) == 0 && last < cells) {
          while (true) {
            uint4 v;
            asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "l"(pr.in[q] + last));
            if (v.x == val && v.w == val) break;
            if (sleep_ns) __nanosleep(sleep_ns);
          }
        }
        __syncwarp();
      }
      while (true) {
        uint4 v;
        asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(pr.in[q] + i));
        if (v.x == val && v.w == val) break;
        if (sleep_ns) __nanosleep(sleep_ns);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) stamps[3 * blockIdx.x + 2] = gt();
}

__global__ void ping(volatile uint64_t* mine, volatile uint64_t* theirs, int iters, int init,
                     uint64_t* out) {
  uint64_t s = 0, r = 0;
  for (int i = 1; i <= iters; ++i) {
    if (init) {
      s = gt();
      *theirs = i;
    }
    while (*mine != (uint64_t)i) {
    }
    r = gt();
    if (!init) *theirs = i;
  }
  out[0] = s;
  out[1] = r;
}

int main() {
  int P = 0;
  CK(cudaGetDeviceCount(&P));
  P = std::min(P, kMaxP);
  if (P < 2) return 0;
  const uint64_t slot_bytes = 4ull << 20;
  std::vector<uint4*> buf(P);
  std::vector<uint64_t*> st(P), flag(P), out(P);
  std::vector<uint32_t*> gow(P);
  uint32_t* ready = nullptr;
  std::vector<cudaStream_t> s(P);
  for (int g = 0; g < P; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < P; ++h)
      if (h != g) CK(cudaDeviceEnablePeerAccess(h, 0));
    CK(cudaMalloc(&buf[g], slot_bytes * P));
    CK(cudaMalloc(&st[g], 1 << 16));
    CK(cudaMalloc(&flag[g], 64));
    CK(cudaMalloc(&out[g], 64));
    CK(cudaMemset(flag[g], 0, 64));
    CK(cudaStreamCreateWithFlags(&s[g], cudaStreamNonBlocking));
    CK(cudaMalloc(&gow[g], 64));
    CK(cudaMemset(gow[g], 0, 64));
    if (g == 0) {
      CK(cudaMalloc(&ready, 256));
      CK(cudaMemset(ready, 0, 256));
    }
  }
  // timer offsets vs GPU0
  std::vector<double> off(P, 0.0);
  for (int g = 1; g < P; ++g) {
    CK(cudaSetDevice(g));
    ping<<<1, 1, 0, s[g]>>>(flag[g], flag[0], 100, 0, out[g]);
    CK(cudaSetDevice(0));
    ping<<<1, 1, 0, s[0]>>>(flag[0], flag[g], 100, 1, out[0]);
    CK(cudaStreamSynchronize(s[0]));
    CK(cudaSetDevice(g));
    CK(cudaStreamSynchronize(s[g]));
    uint64_t a[2], b[2];
    CK(cudaMemcpy(a, out[0], 16, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b, out[g], 16, cudaMemcpyDeviceToHost));
    off[g] = (double)b[1] - ((double)a[0] + (double)a[1]) / 2.0;
    CK(cudaSetDevice(0));
    CK(cudaMemset(flag[0], 0, 64));
    CK(cudaSetDevice(g));
    CK(cudaMemset(flag[g], 0, 64));
  }
  printf("P=%d\n", P);
  uint32_t val = 0x40000000u;
  for (int g = 0; g < P; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaFuncSetAttribute(exch, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10));
  }
  // variant 6 (32-byte STG.256 pushes) faults: 256-bit stores to peer memory
  // are an illegal access on B200 (measured); kept selectable for reference.
  for (int variant : {1, 5}) {
  const int sleep_ns = variant == 0 ? 0 : variant == 1 ? 32 : variant == 2 ? 256 : variant == 3 ? 1000 : 32;
  const int leader = variant == 4;
  const int bulk = variant == 5 ? 1 : variant == 6 ? 2 : 0;
  printf("-- poll sleep %d ns%s%s\n", sleep_ns, leader ? ", warp-leader poll" : "",
         bulk == 1 ? ", TMA bulk pushes" : bulk == 2 ? ", 32-byte stores" : "");
  for (uint64_t bytes : {16ull, 512ull, 4ull << 10, 16ull << 10, 128ull << 10, 512ull << 10,
                         2048ull << 10}) {
    for (int grid : {32, 128}) {
      std::vector<double> tot, iss, lat;
      for (int rep = 0; rep < 5; ++rep) {
        ++val;
        for (int g = 0; g < P; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaMemset(buf[g], 0xFF, slot_bytes * P));
          CK(cudaDeviceSynchronize());
        }
        for (int g = 0; g < P; ++g) {
          Peers pr{};
          for (int q = 0; q < P; ++q) {
            pr.slot[q] = reinterpret_cast<uint4*>(reinterpret_cast<char*>(buf[q]) + g * slot_bytes);
            pr.in[q] = reinterpret_cast<uint4*>(reinterpret_cast<char*>(buf[g]) + q * slot_bytes);
          }
          pr.ready = ready;
          for (int q = 0; q < P; ++q) pr.go[q] = gow[q];
          CK(cudaSetDevice(g));
          const size_t smem = bulk == 1 ? ((bytes / 16 + grid - 1) / grid) * 16 : 0;
          exch<<<grid, 512, smem, s[g]>>>(pr, g, P, bytes / 16, val, st[g], sleep_ns, leader && !bulk, bulk);
        }
        double t0 = 1e30, t_end = 0, iss_end = 0, t0_last = 0;
        for (int g = 0; g < P; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaStreamSynchronize(s[g]));
          std::vector<uint64_t> h(3 * grid);
          CK(cudaMemcpy(h.data(), st[g], 24 * grid, cudaMemcpyDeviceToHost));
          for (int b = 0; b < grid; ++b) {
            t0 = std::min(t0, (double)h[3 * b] - off[g]);
            t0_last = std::max(t0_last, (double)h[3 * b] - off[g]);
            iss_end = std::max(iss_end, (double)h[3 * b + 1] - off[g]);
            t_end = std::max(t_end, (double)h[3 * b + 2] - off[g]);
          }
        }
        tot.push_back((t_end - t0) / 1e3);
        iss.push_back((iss_end - t0) / 1e3);
        lat.push_back((t_end - t0_last) / 1e3);
      }
      std::sort(tot.begin(), tot.end());
      std::sort(iss.begin(), iss.end());
      std::sort(lat.begin(), lat.end());
      printf("bytes/peer=%8llu grid=%4d : pushes issued by %.3f us, all arrived by %.3f us, "
             "last start -> last arrival %.3f us (p50)\n",
             (unsigned long long)bytes, grid, iss[2], tot[2], lat[2]);
    }
  }
  }
  return 0;
}
