// Micro-benchmark of the tcgen05 GEMM ring handshake (no TMA, no MMA): producer lane
// waits "empty", arrives "full"; MMA lane waits "full", releases "empty" either with
// tcgen05.commit (mode 0) or a plain mbarrier arrive (mode 1); mode 2 issues one real
// tcgen05.mma (128x256x8 tf32 on garbage smem) per stage before the commit.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ring_micro tools/ring_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n"
               ::"r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su(b)) : "memory");
}

template <int STAGES>
__global__ void ring(int iters, int mode, long long* out) {
  __shared__ __align__(1024) uint8_t sm[32 * 1024];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  __shared__ uint32_t tslot;
  __shared__ uint64_t done;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(&empty[s])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  const bool spin = mode >= 3;
  if (mode >= 3) mode -= 3;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(su(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot;
  long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    for (int it = 0; it < iters; ++it) {
      const int st = it % STAGES;
      if (it >= STAGES) wait(&empty[st], ((it / STAGES) - 1) & 1);
      arrive(&full[st]);
    }
  } else if (warp >= 2 && spin) {
    wait(&done, 0);       // epilogue warps parked on the accumulator barrier (all lanes)
  } else if (warp == 1 && lane == 0) {
    uint64_t desc = 0;
    desc |= (uint64_t)((su(sm) >> 4) & 0x3FFF);
    desc |= (uint64_t)1 << 16;
    desc |= (uint64_t)(1024 >> 4) << 32;
    desc |= (uint64_t)1 << 46;
    desc |= (uint64_t)2 << 61;
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
    for (int it = 0; it < iters; ++it) {
      const int st = it % STAGES;
      wait(&full[st], (it / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      if (mode == 2) {
        for (int k = 0; k < 4; ++k)
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem), "l"(desc), "l"(desc), "r"(idesc), "r"(1));
      }
      if (mode == 1) arrive(&empty[st]);
      else asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                        ::"r"(su(&empty[st])) : "memory");
    }
    arrive(&done);
  }
  __syncwarp();
  long long t1 = clock64();
  if (lane == 0 && warp == 1) out[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  long long h[148];
  const int iters = 4096;
  for (int mode = 0; mode < 6; ++mode) {
    for (int st : {2, 4, 8}) {
      auto k = st == 2 ? ring<2> : st == 4 ? ring<4> : ring<8>;
      k<<<148, 192>>>(iters, mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      k<<<148, 192>>>(iters, mode, d);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148;
      printf("mode %d (%s) stages %d: %.1f clk/iter (clock64), %.1f ns/iter (events)\n", mode,
             (mode % 3) == 0 ? (mode >= 3 ? "commit + 4 waiting warps" : "commit") : (mode % 3) == 1 ? (mode >= 3 ? "arrive + 4 waiting warps" : "arrive") : (mode >= 3 ? "4 mma + commit + 4 waiting warps" : "4 mma + commit"), st, avg / iters, ms * 1e6 / iters);
    }
  }
  return 0;
}
