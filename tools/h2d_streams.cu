// H2D bandwidth of 8 MB strided tile copies (cudaMemcpy2DAsync from pinned host memory,
// 1024 columns of 8 KB at ld 16384 doubles) with 1, 2 or 4 concurrent streams.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/h2d_streams tools/h2d_streams.cu
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t ld = 16384, rows = 1024, cols = 1024, ntiles = 128;
  double* host;
  cudaMallocHost(&host, ld * cols * 16 * sizeof(double));   // 16 row-tiles x 1024 cols
  double* dev;
  cudaMalloc(&dev, ntiles * rows * cols * sizeof(double));
  cudaStream_t st[4];
  for (int i = 0; i < 4; ++i) cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int ns : {1, 2, 4}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(a, st[0]);
      for (int s = 1; s < ns; ++s) cudaStreamWaitEvent(st[s], a, 0);
      for (size_t t = 0; t < ntiles; ++t) {
        const double* src = host + (t % 16) * rows + ((t / 16) % 1) * cols * ld;
        cudaMemcpy2DAsync(dev + t * rows * cols, rows * 8, src, ld * 8, rows * 8, cols,
                          cudaMemcpyHostToDevice, st[t % ns]);
      }
      for (int s = 1; s < ns; ++s) { cudaEvent_t e; cudaEventCreate(&e); cudaEventRecord(e, st[s]); cudaStreamWaitEvent(st[0], e, 0); }
      cudaEventRecord(b, st[0]);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("%d stream(s): %.1f GB/s\n", ns, ntiles * rows * cols * 8 / (ms * 1e6));
    }
  }
  return 0;
}
