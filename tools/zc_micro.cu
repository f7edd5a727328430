// Zero-copy PCIe micro-benchmark for the N=1 e2e step's shape: 8 ranks x 1 MB
// fp32 of pinned host input, summed per 16-byte unit, written to 8 x 1 MB of
// pinned host output — split into its read half and write half to see which
// bounds the host path (nvrar_allreduce_local_host's direct schedule).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/zc_micro tools/zc_micro.cu
//   tools/zc_micro            # prints one line per (mode, CTAs, threads)
//
// modes: R  host in  -> device out      (the read half)
//        W  device in -> host out       (the write half)
//        RW host in  -> host out        (the e2e kernel's shape)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#define CK(x)                                                               \
  do {                                                                      \
    cudaError_t e_ = (x);                                                   \
    if (e_ != cudaSuccess) {                                                \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      return 1;                                                             \
    }                                                                       \
  } while (0)

constexpr int kRanks = 8;
struct Ptrs {
  const uint4* in[kRanks];
  uint4* out[kRanks];
};

// CTA b of rank slice y walks its contiguous range of units, warps coalesced
// (the direct kernel's layout: blockIdx.y = the rank slice of the outputs)
__global__ void zc_kernel(Ptrs p, unsigned units) {
  const unsigned slice = (units + gridDim.y - 1) / gridDim.y;
  const unsigned s0 = min(slice * blockIdx.y, units), s1 = min(s0 + slice, units);
  const unsigned ub = s0 + (unsigned)((unsigned long long)(s1 - s0) * blockIdx.x / gridDim.x);
  const unsigned ue = s0 + (unsigned)((unsigned long long)(s1 - s0) * (blockIdx.x + 1) / gridDim.x);
  for (unsigned u = ub + threadIdx.x; u < ue; u += blockDim.x) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int r = 0; r < kRanks; ++r) {
      const uint4 v = p.in[r][u];
      acc.x += __uint_as_float(v.x);
      acc.y += __uint_as_float(v.y);
      acc.z += __uint_as_float(v.z);
      acc.w += __uint_as_float(v.w);
    }
    const uint4 o = make_uint4(__float_as_uint(acc.x), __float_as_uint(acc.y), __float_as_uint(acc.z),
                               __float_as_uint(acc.w));
#pragma unroll
    for (int r = 0; r < kRanks; ++r) p.out[r][u] = o;
  }
}

int main() {
  const size_t bytes = 1 << 20;
  const unsigned units = bytes / 16;
  std::vector<void*> hin(kRanks), hout(kRanks), din(kRanks), dout(kRanks);
  for (int r = 0; r < kRanks; ++r) {
    CK(cudaHostAlloc(&hin[r], bytes, cudaHostAllocDefault));
    CK(cudaHostAlloc(&hout[r], bytes, cudaHostAllocDefault));
    CK(cudaMalloc(&din[r], bytes));
    CK(cudaMalloc(&dout[r], bytes));
    CK(cudaMemset(din[r], 0, bytes));
    std::fill_n(static_cast<float*>(hin[r]), bytes / 4, 1.0f);
  }
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const char* modes[] = {"R", "W", "RW"};
  const int grids[] = {1, 2, 4, 8, 16, 37};
  const int threads[] = {128, 256, 512};
  for (int m = 0; m < 3; ++m) {
    Ptrs p;
    for (int r = 0; r < kRanks; ++r) {
      p.in[r] = static_cast<const uint4*>(m == 1 ? din[r] : hin[r]);
      p.out[r] = static_cast<uint4*>(m == 0 ? dout[r] : hout[r]);
    }
    for (int g : grids) {
      for (int t : threads) {
        dim3 grid(g, kRanks);
        zc_kernel<<<grid, t, 0, s>>>(p, units);
        CK(cudaStreamSynchronize(s));
        std::vector<float> ts;
        for (int rep = 0; rep < 9; ++rep) {
          CK(cudaEventRecord(e0, s));
          zc_kernel<<<grid, t, 0, s>>>(p, units);
          CK(cudaEventRecord(e1, s));
          CK(cudaEventSynchronize(e1));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          ts.push_back(ms * 1e3f);
        }
        std::sort(ts.begin(), ts.end());
        const double us = ts[ts.size() / 2];
        const double moved = (m == 2 ? 2.0 : 1.0) * kRanks * bytes;
        printf("mode=%-2s ctas_per_rank=%-3d threads=%-4d units_per_thread=%-6.1f us=%8.1f GB/s=%6.1f\n",
               modes[m], g, t, (double)units / (g * kRanks * t), us, moved / us / 1e3);
      }
    }
  }
  if (static_cast<float*>(hout[0])[0] != 8.0f) {
    fprintf(stderr, "wrong sum %f\n", static_cast<float*>(hout[0])[0]);
    return 1;
  }
  return 0;
}
