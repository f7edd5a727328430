// Launch-overhead microbenchmarks on B200 (sm_100a): per-kernel time inside a
// CUDA graph of back-to-back launches, for the building blocks of the NVRAR
// kernel prologue. Build + run (GPU box):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/launch_micro tools/launch_micro.cu
//   ./tools/launch_micro
#include <cuda_runtime.h>
#include <cstdlib>

#ifndef PAD_BYTES
#define PAD_BYTES 8
#endif

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

struct Args {
  const uint4* in;
  uint4* out;
  uint64_t per_call_elems;  // uint4 per call
  int calls;
  unsigned* state;
  int mode;  // bit0: pdl wait/trigger, bit1: state load+sync, bit2: copy,
             // bit3: state load as ld.relaxed.gpu (else ld.volatile = STRONG.SYS),
             // bit4: state store right after the load (else at the end)
  unsigned char pad[PAD_BYTES];  // parameter-block size experiment
};

__global__ void k_main(const __grid_constant__ Args a, int call) {
  if (a.mode & 1) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  __shared__ unsigned s;
  if (a.mode & 2) {
    if (threadIdx.x == 0) {
      unsigned v;
      if (a.mode & 8) {
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.state + blockIdx.x) : "memory");
      } else {
        asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(a.state + blockIdx.x) : "memory");
      }
      s = v;
      if (a.mode & 16) a.state[blockIdx.x] = v + 1;
    }
    __syncthreads();
  }
  if (a.mode & 4) {
    const uint64_t base = static_cast<uint64_t>(call % a.calls) * a.per_call_elems;
    for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.per_call_elems;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
      uint4 v = a.in[base + i];
      if (a.mode & 2) v.x += s;
      a.out[base + i] = v;
    }
  }
  if ((a.mode & 2) && !(a.mode & 16) && threadIdx.x == 0) a.state[blockIdx.x] = s + 1;
}

int run(const char* name, int mode, int grid, int block, bool pdl, uint64_t bytes, const uint4* in,
        uint4* out, unsigned* state, int ncalls_rot) {
  Args a{in, out, bytes / 16, ncalls_rot, state, mode, {}};
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const int calls = 100;
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
  for (int c = 0; c < calls; ++c) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, k_main, a, c));
  }
  CK(cudaStreamEndCapture(st, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  for (int w = 0; w < 3; ++w) CK(cudaGraphLaunch(ge, st));
  CK(cudaStreamSynchronize(st));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::vector<float> ms;
  for (int r = 0; r < 7; ++r) {
    CK(cudaEventRecord(e0, st));
    CK(cudaGraphLaunch(ge, st));
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float t;
    CK(cudaEventElapsedTime(&t, e0, e1));
    ms.push_back(t);
  }
  std::sort(ms.begin(), ms.end());
  printf("%-44s grid=%4d block=%4d pdl=%d bytes=%8llu : %7.3f us/launch\n", name, grid, block,
         pdl ? 1 : 0, (unsigned long long)bytes, ms[3] * 1e3 / calls);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(st);
  return 0;
}

#include <algorithm>

int main() {
  const uint64_t rot = 160ull << 20;  // > L2
  uint4 *in, *out;
  unsigned* state;
  CK(cudaMalloc(&in, rot));
  CK(cudaMalloc(&out, rot));
  CK(cudaMalloc(&state, 4096));
  CK(cudaMemset(in, 1, rot));
  CK(cudaMemset(state, 0, 4096));
  if (getenv("LM_VARIANTS")) {
    // round 2: where the fixed per-call cost of a state-reading kernel goes
    printf("param block %d bytes\n", (int)sizeof(Args));
    for (int grid : {64}) {
      run("empty", 1, grid, 512, true, 0, in, out, state, 1);
      run("state: volatile load + sync, store at end", 1 | 2, grid, 512, true, 0, in, out, state, 1);
      run("state: relaxed.gpu load + sync, store at end", 1 | 2 | 8, grid, 512, true, 0, in, out, state, 1);
      run("state: volatile load + sync, store early", 1 | 2 | 16, grid, 512, true, 0, in, out, state, 1);
      run("state: relaxed.gpu load + sync, store early", 1 | 2 | 8 | 16, grid, 512, true, 0, in, out, state, 1);
      const int rc = static_cast<int>(rot / (128ull << 10) / 2);
      run("copy 128K", 1 | 4, grid, 512, true, 128ull << 10, in, out, state, rc);
      run("state(volatile) + copy 128K", 1 | 2 | 4, grid, 512, true, 128ull << 10, in, out, state, rc);
      run("state(relaxed.gpu, early store) + copy 128K", 1 | 2 | 4 | 8 | 16, grid, 512, true,
          128ull << 10, in, out, state, rc);
    }
    return 0;
  }
  for (int pdl = 0; pdl < 2; ++pdl) {
    for (int grid : {32, 128}) {
      run("empty", pdl ? 1 : 0, grid, 512, pdl, 0, in, out, state, 1);
      run("state load + syncthreads", (pdl ? 1 : 0) | 2, grid, 512, pdl, 0, in, out, state, 1);
      for (uint64_t bytes : {128ull << 10, 1ull << 20}) {
        const int rc = static_cast<int>(rot / bytes / 2);
        run("copy (rotating, > L2)", (pdl ? 1 : 0) | 4, grid, 512, pdl, bytes, in, out, state, rc);
        run("state + copy (rotating)", (pdl ? 1 : 0) | 6, grid, 512, pdl, bytes, in, out, state, rc);
        run("state + copy (same buffer, L2-hot)", (pdl ? 1 : 0) | 6, grid, 512, pdl, bytes, in,
            out, state, 1);
      }
    }
  }
  run("empty 1x32", 0, 1, 32, false, 0, in, out, state, 1);
  run("empty 1x32 pdl", 1, 1, 32, true, 0, in, out, state, 1);
  return 0;
}
