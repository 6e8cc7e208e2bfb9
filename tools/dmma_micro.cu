// DMMA microbenchmarks: what does the FP64 tensor pipe need to stay busy on sm_100a?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_micro dmma_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

// register-only outer product MF x NF per warp
template <int MF, int NF>
__global__ void outer_reg(double* out, int iters) {
  double acc[MF][NF][2] = {};
  double fa[MF], fb[NF];
#pragma unroll
  for (int i = 0; i < MF; ++i) fa[i] = 1.0 + i * 1e-3 + threadIdx.x * 1e-9;
#pragma unroll
  for (int j = 0; j < NF; ++j) fb[j] = 1.0 - j * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < MF; ++i)
#pragma unroll
      for (int j = 0; j < NF; ++j) dmma(acc[i][j], fa[i], fb[j]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < MF; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 1.2345) out[threadIdx.x] = s;
}

// outer product with fragments re-read from shared memory every k4 step (no barriers)
template <int MF, int NF>
__global__ void outer_lds(double* out, int iters) {
  __shared__ double sa[16 * 132], sb[16 * 132];
  for (int i = threadIdx.x; i < 16 * 132; i += blockDim.x) { sa[i] = 1.0 + i * 1e-6; sb[i] = 1.0 - i * 1e-6; }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
  const int wm = (warp & 1) * 64, wn = (warp >> 1) * 32;
  double acc[MF][NF][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kq = 0; kq < 4; ++kq) {
      double fa[MF], fb[NF];
#pragma unroll
      for (int i = 0; i < MF; ++i) fa[i] = sa[(kq * 4 + q) * 132 + ((wm + i * 8 + g) & 127)];
#pragma unroll
      for (int j = 0; j < NF; ++j) fb[j] = sb[(kq * 4 + q) * 132 + ((wn + j * 8 + g) & 127)];
#pragma unroll
      for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) dmma(acc[i][j], fa[i], fb[j]);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < MF; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 1.2345) out[threadIdx.x] = s;
}

template <class F>
float timeit(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  float best = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  double* out; cudaMalloc(&out, 1 << 20);
  int sms = 148;
  const int iters = 4096;
#define RUN(K, MF, NF, TH, BPS)                                                                 \
  {                                                                                             \
    float ms = timeit([&] { K<MF, NF><<<sms * BPS, TH>>>(out, iters); });                        \
    double fl = (double)sms * BPS * (TH / 32) * iters * MF * NF * 512.0 * (#K[6] == 'l' ? 4 : 1); \
    printf("%-10s MF=%d NF=%d threads=%d blocks/SM=%d: %.2f TF/s\n", #K, MF, NF, TH, BPS, fl / ms / 1e9); \
  }
  RUN(outer_reg, 8, 4, 256, 1);
  RUN(outer_reg, 4, 4, 256, 1);
  RUN(outer_reg, 4, 4, 512, 1);
  RUN(outer_reg, 8, 4, 128, 1);
  RUN(outer_reg, 2, 2, 256, 1);
  RUN(outer_reg, 1, 8, 256, 1);
  RUN(outer_lds, 8, 4, 256, 1);
  RUN(outer_lds, 4, 4, 512, 1);
  RUN(outer_lds, 4, 4, 256, 1);
  cudaError_t e = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(e));
  return 0;
}
