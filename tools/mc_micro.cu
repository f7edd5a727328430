// NVSwitch multicast (NVLS) vs unicast pushes for the one-shot exchange on P
// GPUs of one process: every GPU sends `bytes` of 16-byte Lamport cells to all
// others — either P-1 unicast st.v4 per cell (today's kernels) or ONE
// multimem.st.v4 per cell to a multicast mapping that the switch replicates to
// every GPU's copy — and polls its P-1 inbound slots. Reports last sender
// start -> last arrival (timer offsets from a ping-pong with GPU0).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mc_micro tools/mc_micro.cu -lcuda
#include <cuda.h>
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
#define CU(x)                                                  \
  do {                                                         \
    CUresult r = (x);                                          \
    if (r != CUDA_SUCCESS) {                                   \
      const char* s = nullptr;                                 \
      cuGetErrorString(r, &s);                                 \
      printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, s);   \
      return 1;                                                \
    }                                                          \
  } while (0)

constexpr int kMaxP = 8;

struct Args {
  uint4* uc[kMaxP];  // unicast view of each GPU's region (peer-mapped)
  uint4* mc;         // multicast view (stores reach every GPU's region)
  volatile uint32_t* ready;
  volatile uint32_t* go[kMaxP];
};

__device__ __forceinline__ uint64_t gt() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// region layout: [P sources][slot cells]
__global__ void exch(Args a, int me, int P, uint64_t cells, uint64_t slot, uint32_t val,
                     uint64_t* stamps, int multicast) {
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) a.ready[me] = val;
    if (me == 0 && blockIdx.x == 0) {
      for (int g = 0; g < P; ++g)
        while (a.ready[g] != val) {
        }
      for (int g = 0; g < P; ++g) *a.go[g] = val;
    }
    while (*a.go[me] != val) {
    }
    stamps[3 * blockIdx.x] = gt();
  }
  __syncthreads();
  const float fv = __uint_as_float(val);
  for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cells;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (multicast) {
      asm volatile("multimem.st.global.v4.f32 [%0], {%1,%1,%1,%1};" ::"l"(a.mc + me * slot + i),
                   "f"(fv)
                   : "memory");
    } else {
      for (int j = 1; j < P; ++j) {
        const int q = (me + j) % P;
        asm volatile("st.volatile.global.v4.u32 [%0], {%1,%1,%1,%1};" ::"l"(a.uc[q] + me * slot + i),
                     "r"(val));
      }
    }
  }
  if (threadIdx.x == 0) stamps[3 * blockIdx.x + 1] = gt();
  for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cells;
       i += (uint64_t)gridDim.x * blockDim.x) {
    for (int j = 1; j < P; ++j) {
      const int q = (me + j) % P;
      while (true) {
        uint4 v;
        asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(a.uc[me] + q * slot + i));
        if (v.x == val && v.w == val) break;
        __nanosleep(32);
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
  CU(cuInit(0));
  std::vector<CUdevice> dev(P);
  for (int g = 0; g < P; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaFree(nullptr));
    CU(cuDeviceGet(&dev[g], g));
    for (int h = 0; h < P; ++h)
      if (h != g) CK(cudaDeviceEnablePeerAccess(h, 0));
  }
  const uint64_t slot_bytes = 4ull << 20;
  CUmulticastObjectProp mp{};
  mp.numDevices = P;
  mp.handleTypes = 0;
  size_t gran = 0;
  mp.size = slot_bytes * P;
  CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t size = (slot_bytes * P + gran - 1) / gran * gran;
  mp.size = size;
  CUmemGenericAllocationHandle mc;
  CU(cuMulticastCreate(&mc, &mp));
  for (int g = 0; g < P; ++g) CU(cuMulticastAddDevice(mc, dev[g]));
  std::vector<CUmemGenericAllocationHandle> mem(P);
  std::vector<CUdeviceptr> uc(P);
  std::vector<CUmemAccessDesc> acc(P);
  for (int g = 0; g < P; ++g) {
    acc[g].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc[g].location.id = g;
    acc[g].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  }
  for (int g = 0; g < P; ++g) {
    CK(cudaSetDevice(g));
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = g;
    CU(cuMemCreate(&mem[g], size, &ap, 0));
    CU(cuMemAddressReserve(&uc[g], size, gran, 0, 0));
    CU(cuMemMap(uc[g], size, 0, mem[g], 0));
    CU(cuMemSetAccess(uc[g], size, acc.data(), P));
  }
  for (int g = 0; g < P; ++g) CU(cuMulticastBindMem(mc, 0, mem[g], 0, size, 0));
  CUdeviceptr mcva;
  CU(cuMemAddressReserve(&mcva, size, gran, 0, 0));
  CU(cuMemMap(mcva, size, 0, mc, 0));
  CU(cuMemSetAccess(mcva, size, acc.data(), P));

  std::vector<uint64_t*> st(P), flag(P), out(P);
  std::vector<uint32_t*> gow(P);
  uint32_t* ready = nullptr;
  std::vector<cudaStream_t> s(P);
  for (int g = 0; g < P; ++g) {
    CK(cudaSetDevice(g));
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
  }
  printf("P=%d multicast granularity %zu\n", P, gran);
  uint32_t val = 0x40000000u;
  for (int multicast = 0; multicast < 2; ++multicast) {
    printf("-- %s\n", multicast ? "multimem.st to the multicast mapping (switch replicates)"
                                 : "P-1 unicast st.v4 per cell");
    for (uint64_t bytes : {16ull, 4ull << 10, 16ull << 10, 64ull << 10, 256ull << 10,
                           1024ull << 10, 2048ull << 10}) {
      for (int grid : {32, 128}) {
        std::vector<double> lat, tot;
        for (int rep = 0; rep < 7; ++rep) {
          ++val;
          for (int g = 0; g < P; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaMemset(reinterpret_cast<void*>(uc[g]), 0xFF, size));
            CK(cudaDeviceSynchronize());
          }
          Args a{};
          for (int q = 0; q < P; ++q) a.uc[q] = reinterpret_cast<uint4*>(uc[q]);
          a.mc = reinterpret_cast<uint4*>(mcva);
          a.ready = ready;
          for (int q = 0; q < P; ++q) a.go[q] = gow[q];
          for (int g = 0; g < P; ++g) {
            CK(cudaSetDevice(g));
            exch<<<grid, 512, 0, s[g]>>>(a, g, P, bytes / 16, slot_bytes / 16, val, st[g],
                                         multicast);
          }
          double t0 = 1e30, t0_last = 0, t_end = 0;
          for (int g = 0; g < P; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaStreamSynchronize(s[g]));
            std::vector<uint64_t> h(3 * grid);
            CK(cudaMemcpy(h.data(), st[g], 24 * grid, cudaMemcpyDeviceToHost));
            for (int b = 0; b < grid; ++b) {
              t0 = std::min(t0, (double)h[3 * b] - off[g]);
              t0_last = std::max(t0_last, (double)h[3 * b] - off[g]);
              t_end = std::max(t_end, (double)h[3 * b + 2] - off[g]);
            }
          }
          lat.push_back((t_end - t0_last) / 1e3);
          tot.push_back((t_end - t0) / 1e3);
        }
        std::sort(lat.begin(), lat.end());
        std::sort(tot.begin(), tot.end());
        printf("bytes/peer=%8llu grid=%4d : first start -> last arrival %.3f us, last start -> last arrival %.3f us (p50)\n",
               (unsigned long long)bytes, grid, tot[3], lat[3]);
      }
    }
  }
  return 0;
}
