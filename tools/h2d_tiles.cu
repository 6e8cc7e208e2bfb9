// H2D / D2H bandwidth of strided tile copies (cudaMemcpy2DAsync, pinned host memory) per tile
// shape and number of concurrent copy streams: is a 512-tile of a 2048-row matrix (512
// columns of 4 KB at a 16 KB pitch, cfg1) as fast over the host link as a 1024-tile of a
// 16384-row matrix (8 KB columns at 128 KB pitch, cfg2)?  Also: the whole column panel as
// one contiguous copy, and tiles issued as 1-column-per-call vs 2-d.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/h2d_tiles tools/h2d_tiles.cu
#include <cstdio>
#include <cuda_runtime.h>

static double run(double* dev, double* host, size_t ld, size_t rows, size_t cols, int ntiles, int ns,
                  cudaStream_t* st, bool d2h) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaDeviceSynchronize();
    cudaEventRecord(a, st[0]);
    for (int s = 1; s < ns; ++s) cudaStreamWaitEvent(st[s], a, 0);
    const size_t row_tiles = ld / rows;
    for (int t = 0; t < ntiles; ++t) {
      double* hp = host + (t % row_tiles) * rows + ((t / row_tiles) * cols) * ld;
      double* dp = dev + (size_t)t * rows * cols;
      if (d2h)
        cudaMemcpy2DAsync(hp, ld * 8, dp, rows * 8, rows * 8, cols, cudaMemcpyDeviceToHost, st[t % ns]);
      else
        cudaMemcpy2DAsync(dp, rows * 8, hp, ld * 8, rows * 8, cols, cudaMemcpyHostToDevice, st[t % ns]);
    }
    for (int s = 1; s < ns; ++s) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, st[s]);
      cudaStreamWaitEvent(st[0], e, 0);
    }
    cudaEventRecord(b, st[0]);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return (double)ntiles * rows * cols * 8 / (best * 1e6);
}

int main() {
  struct Shape { size_t ld, rows, cols; int ntiles; const char* name; };
  Shape shapes[] = {
      {2048, 512, 512, 48, "cfg1 tile 512 of ld 2048 (4 KB columns), 48 tiles = one call's H2D"},
      {2048, 2048, 512, 12, "cfg1 column panel 2048x512 (contiguous 8 MB), 12 panels"},
      {16384, 1024, 1024, 48, "cfg2 tile 1024 of ld 16384 (8 KB columns), 48 tiles"},
      {16384, 512, 512, 96, "tile 512 of ld 16384 (4 KB columns), 96 tiles"},
      {4096, 256, 256, 96, "tile 256 of ld 4096 (2 KB columns), 96 tiles"},
  };
  size_t host_elems = 0, dev_elems = 0;
  for (auto& s : shapes) {
    size_t need = s.ld * s.cols * ((s.ntiles + s.ld / s.rows - 1) / (s.ld / s.rows));
    if (need > host_elems) host_elems = need;
    if ((size_t)s.ntiles * s.rows * s.cols > dev_elems) dev_elems = (size_t)s.ntiles * s.rows * s.cols;
  }
  double *host, *dev;
  cudaMallocHost(&host, host_elems * 8);
  cudaMalloc(&dev, dev_elems * 8);
  for (size_t i = 0; i < host_elems; ++i) host[i] = 1.0;
  cudaStream_t st[4];
  for (int i = 0; i < 4; ++i) cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
  for (auto& s : shapes) {
    for (int d2h = 0; d2h < 2; ++d2h)
      for (int ns : {1, 2, 4})
        printf("%s %s, %d stream(s): %.1f GB/s\n", d2h ? "D2H" : "H2D", s.name, ns,
               run(dev, host, s.ld, s.rows, s.cols, s.ntiles, ns, st, d2h));
  }
  // per-call cost: 48 x 2 MB tiles issued back to back, time from first issue to the host
  // returning (enqueue cost), single stream
  return 0;
}
