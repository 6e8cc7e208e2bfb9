// Host enqueue cost and link bandwidth of strided tile copies: one cudaMemcpy2DAsync per
// tile vs one cudaMemcpy3DBatchAsync per batch (CUDA 12.8+), H2D from pinned host memory
// and D2D (same GPU, as a stand-in for the peer lane).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/batch_copy_micro tools/batch_copy_micro.cu
#include <chrono>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

int main() {
  const size_t ld = 16384, rows = 1024, cols = 1024;   // 8 MB tiles of a 16384-row matrix
  const int ntiles = 64;
  double* host;
  CK(cudaMallocHost(&host, ld * cols * 4 * sizeof(double)));   // 16 row tiles x 4 col tiles
  double *dev, *dev2;
  CK(cudaMalloc(&dev, (size_t)ntiles * rows * cols * sizeof(double)));
  CK(cudaMalloc(&dev2, (size_t)ntiles * rows * cols * sizeof(double)));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto src_of = [&](int t) { return host + (t % 16) * rows + ((t / 16) % 4) * cols * ld; };
  for (int mode = 0; mode < 4; ++mode) {      // 0: 2D H2D, 1: batch H2D, 2: 2D D2D, 3: batch D2D
    const bool batch = mode & 1, d2d = mode >= 2;
    double best_us = 1e30, best_gbs = 0;
    for (int rep = 0; rep < 4; ++rep) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a, st));
      auto t0 = std::chrono::high_resolution_clock::now();
      if (!batch) {
        for (int t = 0; t < ntiles; ++t) {
          const void* src = d2d ? (const void*)(dev2 + (size_t)t * rows * cols) : (const void*)src_of(t);
          const size_t spitch = d2d ? rows * 8 : ld * 8;
          CK(cudaMemcpy2DAsync(dev + (size_t)t * rows * cols, rows * 8, src, spitch, rows * 8, cols,
                               d2d ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
        }
      } else {
        std::vector<cudaMemcpy3DBatchOp> ops(ntiles);
        for (int t = 0; t < ntiles; ++t) {
          cudaMemcpy3DBatchOp& o = ops[t];
          memset(&o, 0, sizeof(o));
          o.src.type = cudaMemcpyOperandTypePointer;
          o.src.op.ptr.ptr = d2d ? (void*)(dev2 + (size_t)t * rows * cols) : (void*)src_of(t);
          o.src.op.ptr.rowLength = d2d ? rows * 8 : ld * 8;
          o.src.op.ptr.layerHeight = cols;
          o.dst.type = cudaMemcpyOperandTypePointer;
          o.dst.op.ptr.ptr = dev + (size_t)t * rows * cols;
          o.dst.op.ptr.rowLength = rows * 8;
          o.dst.op.ptr.layerHeight = cols;
          o.extent = make_cudaExtent(rows * 8, cols, 1);
          o.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
        }
        size_t fail = 0;
        CK(cudaMemcpy3DBatchAsync(ntiles, ops.data(), &fail, 0, st));
      }
      auto t1 = std::chrono::high_resolution_clock::now();
      CK(cudaEventRecord(b, st));
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double us = std::chrono::duration<double, std::micro>(t1 - t0).count();
      if (us < best_us) best_us = us;
      const double gbs = (double)ntiles * rows * cols * 8 / (ms * 1e6);
      if (gbs > best_gbs) best_gbs = gbs;
    }
    printf("%s %s: host enqueue %.1f us for %d tiles (%.2f us/tile), %.1f GB/s\n", d2d ? "D2D" : "H2D",
           batch ? "cudaMemcpy3DBatchAsync" : "cudaMemcpy2DAsync x N", best_us, ntiles, best_us / ntiles, best_gbs);
  }
  return 0;
}
