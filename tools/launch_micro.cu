// What makes a short launch of the task GEMM cost ~25 us on the GPU?  Isolate: big
// __grid_constant__ params vs large dynamic shared memory.
#include <cstdio>
#include <cuda_runtime.h>
struct Big { double x[160]; };   // 1.3 KB
__global__ void k_small(double* o) { if (threadIdx.x == 0) o[blockIdx.x] = 1.0; }
__global__ void k_big(const __grid_constant__ Big b, double* o) { if (threadIdx.x == 0) o[blockIdx.x] = b.x[blockIdx.x & 127]; }
__global__ void k_smem(double* o) { extern __shared__ double s[]; s[threadIdx.x] = threadIdx.x; __syncthreads(); if (threadIdx.x == 0) o[blockIdx.x] = s[5]; }
template <class F> float t(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize(); cudaEventRecord(a);
  for (int i = 0; i < 50; ++i) f();
  cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms * 1000 / 50;
}
int main() {
  double* o; cudaMalloc(&o, 1 << 20);
  Big big{};
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  printf("small: %.1f us\n", t([&] { k_small<<<8, 256>>>(o); }));
  printf("big param: %.1f us\n", t([&] { k_big<<<8, 256>>>(big, o); }));
  printf("smem 200KB: %.1f us\n", t([&] { k_smem<<<8, 256, 200 * 1024>>>(o); }));
  printf("smem 40KB: %.1f us\n", t([&] { k_smem<<<8, 256, 40 * 1024>>>(o); }));
  printf("smem 200KB x148: %.1f us\n", t([&] { k_smem<<<148, 256, 200 * 1024>>>(o); }));
  return 0;
}
