// Peak probe for the roofline denominators this repo needs and MEASURED_PEAKS.json lacks:
// FP64 DMMA (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4), FP64 DFMA, pinned host<->device
// tile-copy bandwidth (cudaMemcpy2DAsync of 8 MiB column-major tiles, the transfer
// shape of the tile engine), and device-to-device copy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_peaks probe_peaks.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int CH>
__global__ void dmma_loop(double* out, int iters) {
  double acc[CH][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < CH; ++c) { acc[c][0] = 0; acc[c][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int CH>
__global__ void dfma_loop(double* out, int iters) {
  double acc[CH];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.0) out[threadIdx.x] = s;
}

static float time_kernel(void (*launch)(cudaStream_t), cudaStream_t st, int reps) {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  launch(st); CK(cudaStreamSynchronize(st));
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0, st)); launch(st); CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
  }
  return best;
}

static double* g_out; static int g_sms; static int g_iters; static int g_blocks_per_sm; static int g_threads;
static void l_dmma(cudaStream_t s) { dmma_loop<8><<<g_sms * g_blocks_per_sm, g_threads, 0, s>>>(g_out, g_iters); }
static void l_dfma(cudaStream_t s) { dfma_loop<8><<<g_sms * g_blocks_per_sm, g_threads, 0, s>>>(g_out, g_iters); }

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  g_sms = p.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d,\n", p.name, g_sms, clk_khz);
  CK(cudaMalloc(&g_out, 1 << 20));
  cudaStream_t st; CK(cudaStreamCreate(&st));
  // DMMA sweep over warps per SM
  printf(" \"dmma\": [");
  int cfgs[][2] = {{1, 128}, {1, 256}, {2, 256}, {1, 512}, {4, 256}};
  for (int c = 0; c < 5; ++c) {
    g_blocks_per_sm = cfgs[c][0]; g_threads = cfgs[c][1]; g_iters = 4096;
    float ms = time_kernel(l_dmma, st, 5);
    double flops = (double)g_sms * g_blocks_per_sm * (g_threads / 32) * g_iters * 8 * 512.0;
    printf("%s{\"blocks_per_sm\": %d, \"threads\": %d, \"ms\": %.4f, \"tflops\": %.3f}", c ? ", " : "",
           g_blocks_per_sm, g_threads, ms, flops / ms / 1e9);
  }
  printf("],\n \"dfma\": [");
  for (int c = 0; c < 5; ++c) {
    g_blocks_per_sm = cfgs[c][0]; g_threads = cfgs[c][1]; g_iters = 4096;
    float ms = time_kernel(l_dfma, st, 5);
    double flops = (double)g_sms * g_blocks_per_sm * g_threads * g_iters * 8 * 2.0;
    printf("%s{\"blocks_per_sm\": %d, \"threads\": %d, \"ms\": %.4f, \"tflops\": %.3f}", c ? ", " : "",
           g_blocks_per_sm, g_threads, ms, flops / ms / 1e9);
  }
  printf("],\n"); fflush(stdout);
  // sustained DMMA: ~3 s back-to-back
  {
    g_blocks_per_sm = 1; g_threads = 256; g_iters = 65536;
    cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    l_dmma(st); CK(cudaStreamSynchronize(st));
    CK(cudaEventRecord(e0, st));
    int n = 0; float ms = 0;
    for (n = 0; n < 400; ++n) { l_dmma(st); }
    CK(cudaEventRecord(e1, st)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = (double)g_sms * 8 * g_iters * 8 * 512.0 * n;
    printf(" \"dmma_sustained\": {\"ms\": %.1f, \"tflops\": %.3f},\n", ms, flops / ms / 1e9);
  }
  // Host link: 8 MiB tiles (1024 x 1024 f64) out of a 16384-row column-major host matrix.
  {
    size_t ld = 16384 + 3, cols = 1024 * 16;
    size_t host_bytes = ld * cols * 8;
    double* h; CK(cudaMallocHost(&h, host_bytes));
    for (size_t i = 0; i < host_bytes / 8; i += 512) h[i] = (double)i;
    double* d; size_t tiles = 8; CK(cudaMalloc(&d, tiles * 1024 * 1024 * 8));
    cudaStream_t s2; CK(cudaStreamCreate(&s2));
    cudaEvent_t e0, e1, e2, e3; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1)); CK(cudaEventCreate(&e2)); CK(cudaEventCreate(&e3));
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaEventRecord(e0, st));
      for (size_t t = 0; t < tiles; ++t)
        CK(cudaMemcpy2DAsync(d + t * 1024 * 1024, 1024 * 8, h + (t % 16) * 1024 + t * 1024 * ld, ld * 8, 1024 * 8, 1024, cudaMemcpyHostToDevice, st));
      CK(cudaEventRecord(e1, st)); CK(cudaEventSynchronize(e1));
    }
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double h2d = tiles * 8.0 * 1024 * 1024 / ms / 1e6;
    CK(cudaEventRecord(e0, st));
    for (size_t t = 0; t < tiles; ++t)
      CK(cudaMemcpy2DAsync(h + (t % 16) * 1024 + t * 1024 * ld, ld * 8, d + t * 1024 * 1024, 1024 * 8, 1024 * 8, 1024, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(e1, st)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double d2h = tiles * 8.0 * 1024 * 1024 / ms / 1e6;
    // concurrent: H2D on st, D2H on s2
    CK(cudaEventRecord(e0, st)); CK(cudaEventRecord(e2, s2));
    for (size_t t = 0; t < tiles / 2; ++t) {
      CK(cudaMemcpy2DAsync(d + t * 1024 * 1024, 1024 * 8, h + t * 1024 * ld, ld * 8, 1024 * 8, 1024, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpy2DAsync(h + (8 + t) * 1024 * ld, ld * 8, d + (4 + t) * 1024 * 1024, 1024 * 8, 1024 * 8, 1024, cudaMemcpyDeviceToHost, s2));
    }
    CK(cudaEventRecord(e1, st)); CK(cudaEventRecord(e3, s2)); CK(cudaEventSynchronize(e1)); CK(cudaEventSynchronize(e3));
    float ms1, ms2; CK(cudaEventElapsedTime(&ms1, e0, e1)); CK(cudaEventElapsedTime(&ms2, e2, e3));
    double dup = (tiles * 8.0 * 1024 * 1024) / (ms1 > ms2 ? ms1 : ms2) / 1e6;
    // contiguous 1-D 64 MiB
    CK(cudaEventRecord(e0, st));
    CK(cudaMemcpyAsync(d, h, 64ull << 20, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(e1, st)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    double h2d1 = 64.0 * (1 << 20) / ms / 1e6;
    // d2d
    double* d2; CK(cudaMalloc(&d2, 1ull << 30)); double* d3; CK(cudaMalloc(&d3, 1ull << 30));
    CK(cudaMemcpyAsync(d3, d2, 1ull << 30, cudaMemcpyDeviceToDevice, st));
    CK(cudaEventRecord(e0, st));
    CK(cudaMemcpyAsync(d3, d2, 1ull << 30, cudaMemcpyDeviceToDevice, st));
    CK(cudaEventRecord(e1, st)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    double d2d = 2.0 * (1ull << 30) / ms / 1e6;
    printf(" \"h2d_tile_gbs\": %.2f, \"d2h_tile_gbs\": %.2f, \"duplex_tile_gbs_total\": %.2f, \"h2d_1d_64MiB_gbs\": %.2f, \"d2d_copy_rw_gbs\": %.1f,\n",
           h2d, d2h, dup, h2d1, d2d);
    int ndev = 0; CK(cudaGetDeviceCount(&ndev));
    printf(" \"device_count\": %d}\n", ndev);
  }
  return 0;
}
