// NVLink push-latency microbenchmark (one process, two GPUs, peer access).
// GPU0 CTAs store `bytes` of Lamport cells (16 B, never all-ones) into a buffer
// on GPU1; GPU1 CTAs poll their share of cells until all arrived. Both sides
// stamp %globaltimer; the offset between the two GPUs' timers comes from a
// flag ping-pong. Reports, per configuration, send-issue time and the time the
// last receiver CTA saw its last cell, relative to the send start.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvlink_micro tools/nvlink_micro.cu
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

__device__ __forceinline__ uint64_t gt() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void sender(uint4* dst, uint64_t cells, uint32_t val, uint64_t* stamps) {
  if (threadIdx.x == 0) stamps[2 * blockIdx.x] = gt();
  for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cells;
       i += (uint64_t)gridDim.x * blockDim.x) {
    asm volatile("st.volatile.global.v4.u32 [%0], {%1,%1,%1,%1};" ::"l"(dst + i), "r"(val));
  }
  __syncthreads();
  if (threadIdx.x == 0) stamps[2 * blockIdx.x + 1] = gt();
}

__global__ void receiver(const uint4* src, uint64_t cells, uint32_t val, uint64_t* stamps,
                         int sleep_ns) {
  for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cells;
       i += (uint64_t)gridDim.x * blockDim.x) {
    while (true) {
      uint4 v;
      asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "l"(src + i));
      if (v.x == val && v.w == val) break;
      if (sleep_ns) __nanosleep(sleep_ns);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) stamps[blockIdx.x] = gt();
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
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("need 2 GPUs\n");
    return 0;
  }
  const uint64_t cap = 64ull << 20;
  uint4* buf1;
  uint64_t *st0, *st1, *f0, *f1, *o0, *o1;
  CK(cudaSetDevice(1));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaMalloc(&buf1, cap));
  CK(cudaMalloc(&st1, 1 << 16));
  CK(cudaMalloc(&f1, 64));
  CK(cudaMalloc(&o1, 64));
  CK(cudaMemset(f1, 0, 64));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&st0, 1 << 16));
  CK(cudaMalloc(&f0, 64));
  CK(cudaMalloc(&o0, 64));
  CK(cudaMemset(f0, 0, 64));
  cudaStream_t s0, s1;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaSetDevice(1));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));

  // clock offset (GPU1 - GPU0) via ping-pong
  CK(cudaSetDevice(1));
  ping<<<1, 1, 0, s1>>>(f1, f0, 100, 0, o1);
  CK(cudaSetDevice(0));
  ping<<<1, 1, 0, s0>>>(f0, f1, 100, 1, o0);
  CK(cudaStreamSynchronize(s0));
  CK(cudaSetDevice(1));
  CK(cudaStreamSynchronize(s1));
  uint64_t h0[2], h1[2];
  CK(cudaMemcpy(h0, o0, 16, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h1, o1, 16, cudaMemcpyDeviceToHost));
  const double offset = (double)h1[1] - ((double)h0[0] + (double)h0[1]) / 2.0;
  printf("clock offset gpu1-gpu0 = %.0f ns, last round trip = %llu ns\n", offset,
         (unsigned long long)(h0[1] - h0[0]));

  uint32_t val = 0x40000000u;
  for (int sleep_ns : {0, 64}) {
    for (uint64_t bytes : {16ull << 10, 128ull << 10, 384ull << 10, 1536ull << 10}) {
      for (int grid : {1, 8, 32, 128}) {
        std::vector<double> sent, got;
        for (int rep = 0; rep < 5; ++rep) {
          ++val;
          const uint64_t cells = bytes / 16;
          CK(cudaSetDevice(1));
          CK(cudaMemset(buf1, 0xFF, bytes));
          CK(cudaDeviceSynchronize());
          receiver<<<grid, 512, 0, s1>>>(buf1, cells, val, st1, sleep_ns);
          CK(cudaSetDevice(0));
          // let the receiver start polling first
          sender<<<grid, 512, 0, s0>>>(buf1, cells, val, st0);
          CK(cudaStreamSynchronize(s0));
          CK(cudaSetDevice(1));
          CK(cudaStreamSynchronize(s1));
          std::vector<uint64_t> a(2 * grid), b(grid);
          CK(cudaMemcpy(a.data(), st0, 16 * grid, cudaMemcpyDeviceToHost));
          CK(cudaMemcpy(b.data(), st1, 8 * grid, cudaMemcpyDeviceToHost));
          uint64_t s_start = ~0ull, s_end = 0, r_end = 0;
          for (int i = 0; i < grid; ++i) {
            s_start = std::min(s_start, a[2 * i]);
            s_end = std::max(s_end, a[2 * i + 1]);
            r_end = std::max(r_end, b[i]);
          }
          sent.push_back((double)(s_end - s_start) / 1e3);
          got.push_back(((double)r_end - offset - (double)s_start) / 1e3);
        }
        std::sort(sent.begin(), sent.end());
        std::sort(got.begin(), got.end());
        printf("sleep=%2d bytes=%8llu grid=%4d : send issue %.3f us, last arrival %.3f us (p50)\n",
               sleep_ns, (unsigned long long)bytes, grid, sent[2], got[2]);
      }
    }
  }
  return 0;
}
