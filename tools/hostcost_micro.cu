// Host-side cost of one host-buffer all-reduce call's bookkeeping: the
// pointer-kind queries (16 per N=1 call: 8 inputs + 8 outputs), cudaSetDevice
// and a kernel launch — which of them the ~9 us per call is.
//
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/hostcost_micro \
//        tools/hostcost_micro.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>

__global__ void empty_kernel(int) {}

template <class F>
static double per_call_us(F f, int reps = 20000) {
  for (int i = 0; i < 100; ++i) f();
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) f();
  const auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
}

int main() {
  constexpr int kPtrs = 16;
  void* h[kPtrs];
  for (auto& p : h) {
    if (cudaHostAlloc(&p, 1 << 20, cudaHostAllocDefault) != cudaSuccess) return 1;
  }
  cudaStream_t s;
  cudaStreamCreate(&s);
  printf("cudaPointerGetAttributes x16: %.2f us\n", per_call_us([&] {
           for (auto p : h) {
             cudaPointerAttributes a{};
             cudaPointerGetAttributes(&a, p);
           }
         }));
  printf("cuPointerGetAttribute(DEVICE_POINTER) x16: %.2f us\n", per_call_us([&] {
           for (auto p : h) {
             CUdeviceptr d = 0;
             cuPointerGetAttribute(&d, CU_POINTER_ATTRIBUTE_DEVICE_POINTER,
                                   reinterpret_cast<CUdeviceptr>(p));
           }
         }));
  printf("cuPointerGetAttribute(MEMORY_TYPE) x16: %.2f us\n", per_call_us([&] {
           for (auto p : h) {
             unsigned t = 0;
             cuPointerGetAttribute(&t, CU_POINTER_ATTRIBUTE_MEMORY_TYPE,
                                   reinterpret_cast<CUdeviceptr>(p));
           }
         }));
  printf("cudaHostGetDevicePointer x16: %.2f us\n", per_call_us([&] {
           for (auto p : h) {
             void* d = nullptr;
             cudaHostGetDevicePointer(&d, p, 0);
           }
         }));
  printf("cudaSetDevice: %.2f us\n", per_call_us([&] { cudaSetDevice(0); }));
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(8, 8);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  printf("cudaLaunchKernelEx (PDL attr, async): %.2f us\n", per_call_us([&] {
           cudaLaunchKernelEx(&cfg, empty_kernel, 0);
         }, 5000));
  cudaStreamSynchronize(s);
  return 0;
}
