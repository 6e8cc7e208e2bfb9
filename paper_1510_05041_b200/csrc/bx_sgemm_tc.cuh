// SGEMM tile task on the 5th-generation tensor cores: tcgen05.mma.kind::tf32 with the
// accumulator in TMEM, operands streamed into 128B-swizzled shared memory by TMA
// (cp.async.bulk.tensor) under an mbarrier full/empty ring.
//
// Same task contract as the FP64 kernel (bx_gemm_dmma.cuh):
//     C[h x w] = alpha * sum_s op_s(A_s) op_s(B_s) + beta * C      (fp32 storage)
// The reference has no single-precision path (/root/reference/pkg/src/tileblas/tiling.py:
// 57-60 rejects float32); this kernel serves the cfg5 SGEMM workload.  tcgen05 has no
// fp32 kind: kind::tf32 rounds the inputs to 10-bit mantissas and accumulates in fp32.
//
// Warp roles (192 threads, 1 CTA per SM):
//   warp 0      TMA producer (one elected lane)
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers, alpha/beta, coalesced stores
// CTA tile BM=128 x BN=256, BK=32 fp32 (one 128-B swizzle row), 4 stages (192 KB).
// Operand major-ness per step: A is MN-major when stored untransposed (column-major
// M x K), K-major when transposed; B is K-major untransposed, MN-major transposed.
#pragma once
#include <cuda.h>
#include <cstdint>
#include <cuda_runtime.h>

namespace bx {

constexpr int S_BM = 128, S_BN = 256, S_BK = 32, S_STAGES = 4, S_THREADS = 192;
constexpr int S_MAX_STEPS = 16;
constexpr int S_A_BYTES = S_BM * S_BK * 4;            // 16 KB
constexpr int S_B_BYTES = S_BN * S_BK * 4;            // 32 KB
constexpr int S_STAGE_BYTES = S_A_BYTES + S_B_BYTES;
constexpr int S_SMEM_BYTES = S_STAGES * S_STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int S_TMEM_COLS = 256;

struct SgemmStep {
  CUtensorMap map_a;   // 64-B aligned by declaration
  CUtensorMap map_b;
  int d;               // reduction extent of the step
  int pad_[31];
};

struct SgemmTask {
  SgemmStep steps[S_MAX_STEPS];
  float* c;
  int ldc, h, w, nsteps;
  int ta, tb;          // operand stored transposed
  float alpha, beta;
  int mn_lbo, mn_sbo;  // MN-major descriptor strides (bytes)
  int dbg;             // diagnostic ablation (bx_set_sgemm_debug): 1 no TMA after the first
                       // ring fill, 2 no MMA (results are garbage; timing only)
  int a3d, b3d;        // MN-major operand loaded by ONE 3-d TMA box {32, BK, groups} instead
                       // of one 2-d box per 32-wide group (extent a multiple of 32)
  int group_m;         // persistent kernel: m-tiles per raster group
};

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void s_mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(s_u32(b)), "r"(n));
}
__device__ __forceinline__ void s_mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n}\n" ::"r"(s_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void s_mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void s_tma_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n"
      ::"r"(s_u32(dst)), "l"((uint64_t)map), "r"(s_u32(bar)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void s_tma_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n"
      ::"r"(s_u32(dst)), "l"((uint64_t)map), "r"(s_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void s_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void s_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// Epilogue: 16 consecutive columns of one output row (lane = row, so each store
// instruction of a warp writes 32 consecutive floats).  With beta != 0 the 16 C loads are
// all issued before the first store: one memory round trip per 16 columns instead of 16
// dependent ones (which made a beta = 1 epilogue longer than the mainloop of a K = 8192
// pair tile).
__device__ __forceinline__ void s_store16(const SgemmTask& t, const uint32_t* v, int row, int col0) {
  float* base = t.c + (size_t)col0 * t.ldc + row;
  float cv[16];
  if (t.beta != 0.0f) {
#pragma unroll
    for (int i = 0; i < 16; ++i) cv[i] = col0 + i < t.w ? base[(size_t)i * t.ldc] : 0.0f;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (col0 + i < t.w) {
      float r = t.alpha * __uint_as_float(v[i]);
      if (t.beta != 0.0f) r = fmaf(t.beta, cv[i], r);
      base[(size_t)i * t.ldc] = r;
    }
  }
}

// shared-memory matrix descriptor (sm100 "version 1").  layout 2 = SWIZZLE_128B (K-major
// operands, 8 rows x 128 B atoms); layout 1 = SWIZZLE_128B_BASE32B (32-bit MN-major
// operands: 4 k-rows x 128 B atoms, 32-B swizzle granules — TMA's SWIZZLE_128B_ATOM_32B).
__device__ __forceinline__ uint64_t s_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;          // version = 1 (Blackwell)
  d |= (uint64_t)layout << 61;
  return d;
}

// instruction descriptor: D f32, A/B tf32, M=128, N=BN, per-operand major-ness
__host__ __device__ constexpr uint32_t s_idesc(int a_mn_major, int b_mn_major) {
  uint32_t d = 0;
  d |= 1u << 4;                    // c_format F32
  d |= 2u << 7;                    // a_format TF32
  d |= 2u << 10;                   // b_format TF32
  d |= (uint32_t)a_mn_major << 15;
  d |= (uint32_t)b_mn_major << 16;
  d |= (uint32_t)(S_BN >> 3) << 17;
  d |= (uint32_t)(S_BM >> 4) << 24;
  return d;
}

// Operand major-ness is a template parameter (TA: A stored transposed, TB: B stored
// transposed) so the MMA issue loop is branch-free: its descriptors are the per-kernel
// base descriptors plus compile-time offsets (stage, k-slice), and the ring is unrolled
// over the stages.  The single MMA-issuing thread is on the critical path of the tensor
// pipe (4 MMAs of 128 cycles per stage), so every instruction it spends on address
// arithmetic is tensor time lost.
template <int TA, int TB>
__global__ void __launch_bounds__(S_THREADS, 1) sgemm_tc_kernel(const __grid_constant__ SgemmTask t) {
  extern __shared__ __align__(1024) uint8_t s_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)s_raw + 1023) & ~(uintptr_t)1023);   // SW128 needs 1 KB
  uint64_t* full = (uint64_t*)(smem + S_STAGES * S_STAGE_BYTES);
  uint64_t* empty = full + S_STAGES;
  uint64_t* accum = empty + S_STAGES;
  uint32_t* tmem_slot = (uint32_t*)(accum + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grouped rasterisation: consecutive CTAs sweep GROUP_M m-tiles before moving along n,
  // so the CTAs in flight share A and B panels in L2 instead of streaming all of A per
  // column of tiles (22x DRAM re-reads without it)
  constexpr int GROUP_M = 8;
  const int tiles_m = (t.h + S_BM - 1) / S_BM, tiles_n = (t.w + S_BN - 1) / S_BN;
  const int per_group = GROUP_M * tiles_n;
  const int first_m = (blockIdx.x / per_group) * GROUP_M;
  const int gsize = min(tiles_m - first_m, GROUP_M);
  const int m0 = (first_m + (blockIdx.x % per_group) % gsize) * S_BM;
  const int n0 = ((blockIdx.x % per_group) / gsize) * S_BN;

  int total = 0;
  for (int s = 0; s < t.nsteps; ++s) total += (t.steps[s].d + S_BK - 1) / S_BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S_STAGES; ++s) { s_mbar_init(&full[s], 1); s_mbar_init(&empty[s], 1); }
    s_mbar_init(accum, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(s_u32(tmem_slot)), "n"(S_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  s_fence_before();
  __syncthreads();
  s_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int step = 0, k0 = 0;
      int dcur = t.nsteps > 0 ? t.steps[0].d : 0;
      const CUtensorMap* ma = &t.steps[0].map_a;
      const CUtensorMap* mb = &t.steps[0].map_b;
      for (int it = 0; it < total; ++it) {
        const int st = it % S_STAGES;
        if (it >= S_STAGES) s_mbar_wait(&empty[st], ((it / S_STAGES) - 1) & 1);
        uint8_t* sa = smem + st * S_STAGE_BYTES;
        uint8_t* sb = sa + S_A_BYTES;
        if ((t.dbg & 1) && it >= S_STAGES) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(s_u32(&full[st])) : "memory");
        } else {
          s_mbar_expect_tx(&full[st], S_STAGE_BYTES);
          if (TA) {
            // A stored K x M (K contiguous): K-major, one box {BK, BM}
            s_tma_2d(sa, ma, &full[st], k0, m0);
          } else {
            // A stored M x K (M contiguous): MN-major, boxes {32 M, BK} stacked every 4 KB
            if (t.a3d) {
              s_tma_3d(sa, ma, &full[st], 0, k0, m0 / 32);
            } else {
#pragma unroll
              for (int i = 0; i < S_BM / 32; ++i) s_tma_2d(sa + i * 4096, ma, &full[st], m0 + 32 * i, k0);
            }
          }
          if (!TB) {
            // B stored K x N (K contiguous): K-major, one box {BK, BN}
            s_tma_2d(sb, mb, &full[st], k0, n0);
          } else if (t.b3d) {
            s_tma_3d(sb, mb, &full[st], 0, k0, n0 / 32);
          } else {
#pragma unroll
            for (int i = 0; i < S_BN / 32; ++i) s_tma_2d(sb + i * 4096, mb, &full[st], n0 + 32 * i, k0);
          }
        }
        k0 += S_BK;
        if (k0 >= dcur) {
          k0 = 0;
          if (++step < t.nsteps) {
            dcur = t.steps[step].d;
            ma = &t.steps[step].map_a;
            mb = &t.steps[step].map_b;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = s_idesc(!TA, TB);
      // K-major: the k-slice advances 32 B along the swizzled 128-B row (SBO = 8 rows x
      // 128 B); MN-major: it advances 8 k-rows (1 KB), SBO = 4 k-rows (512 B) between k
      // groups, LBO = 4 KB between the 32-wide MN groups (one TMA box each)
      const uint32_t sbase = s_u32(smem);
      const uint64_t da0 = TA ? s_desc(sbase, 16, 1024, 2) : s_desc(sbase, t.mn_lbo, t.mn_sbo, 1);
      const uint64_t db0 = TB ? s_desc(sbase + S_A_BYTES, t.mn_lbo, t.mn_sbo, 1)
                              : s_desc(sbase + S_A_BYTES, 16, 1024, 2);
      constexpr uint32_t AK = TA ? 32 / 16 : 1024 / 16;     // descriptor units (16 B)
      constexpr uint32_t BKS = TB ? 1024 / 16 : 32 / 16;
      constexpr uint32_t SU = S_STAGE_BYTES / 16;
      const bool do_mma = !(t.dbg & 2);
      for (int it0 = 0; it0 < total; it0 += S_STAGES) {
        const uint32_t par = (it0 / S_STAGES) & 1;
#pragma unroll
        for (int st = 0; st < S_STAGES; ++st) {
          if (it0 + st >= total) break;
          s_mbar_wait(&full[st], par);
          s_fence_after();
          if (do_mma) {
#pragma unroll
            for (int kk = 0; kk < S_BK / 8; ++kk) {
              const uint32_t acc = (it0 + st + kk) != 0;
              asm volatile(
                  "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                  " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                  ::"r"(tmem), "l"(da0 + (uint64_t)(st * SU + kk * AK)), "l"(db0 + (uint64_t)(st * SU + kk * BKS)),
                    "n"(idesc), "r"(acc));
            }
          }
          // frees the stage once these MMAs have read it
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                       ::"r"(s_u32(&empty[st])) : "memory");
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                   ::"r"(s_u32(accum)) : "memory");
    }
  } else {
    // epilogue warps 2..5: TMEM lanes 32*(warp%4) .. +31  <->  tile rows
    const int q = warp & 3;
    const int row = m0 + 32 * q + lane;
    if (total > 0) {
      s_mbar_wait(accum, 0);
      s_fence_after();
    }
    for (int c0 = 0; c0 < S_BN; c0 += 16) {
      uint32_t v[16];
      if (total > 0) {
        const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0u;
      }
      if (row < t.h && !(t.dbg & 8)) {
        s_store16(t, v, row, n0 + c0);
      }
    }
  }
  s_fence_before();
  __syncthreads();
  if (warp == 1) {
    s_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(S_TMEM_COLS));
  }
}

}  // namespace bx

// ---------------------------------------------------------------------------------------
// 2-SM variant: a cluster of two CTAs (one TPC) runs tcgen05.mma.cta_group::2 with
// M = 256 (each CTA owns 128 rows of A and of the accumulator) and N = 256 (each CTA
// stages 128 columns of B; the MMA reads both halves).  Per pair and k-slab 64 KB are
// loaded for 256x256x32 MACs — 1.5x less L2 traffic per flop than the 1-SM 128x256 tile,
// which ran out of L2 bandwidth.  Both CTAs' TMA loads complete on the leader's "full"
// barrier (peer bit cleared from the cluster address); the leader's commit multicasts to
// both CTAs' "empty" and "accum" barriers.
// ---------------------------------------------------------------------------------------
namespace bx {

constexpr int P_BM = 256, P_BN = 256, P_BK = 32, P_STAGES = 6, P_THREADS = 192;
constexpr int P_A_BYTES = 128 * P_BK * 4;                 // this CTA's 128 rows of A
constexpr int P_B_BYTES = 128 * P_BK * 4;                 // this CTA's 128 columns of B
constexpr int P_STAGE_BYTES = P_A_BYTES + P_B_BYTES;      // 32 KB
constexpr int P_SMEM_BYTES = P_STAGES * P_STAGE_BYTES + 1024 + 256;
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;               // leader CTA's copy of a smem address

__device__ __forceinline__ uint32_t p_cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void p_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void p_mbar_wait(uint64_t* b, uint32_t parity) {
  // bounded spin during bring-up: trap instead of hanging the GPU on a protocol bug
  asm volatile(
      "{\n .reg .pred p;\n .reg .u32 n;\n mov.u32 n, 0;\n W_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @p bra D_%=;\n add.u32 n, n, 1;\n setp.gt.u32 p, n, 200000000;\n @p trap;\n bra W_%=;\n D_%=:\n}\n"
      ::"r"(s_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void p_tma_2d_pair(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n"
      ::"r"(s_u32(dst)), "l"((uint64_t)map), "r"(s_u32(bar) & PEER_MASK), "r"(c0), "r"(c1) : "memory");
}

__device__ __forceinline__ void p_tma_3d_pair(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n"
      ::"r"(s_u32(dst)), "l"((uint64_t)map), "r"(s_u32(bar) & PEER_MASK), "r"(c0), "r"(c1), "r"(c2) : "memory");
}

template <int TA, int TB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(P_THREADS, 1)
    sgemm_tc2_kernel(const __grid_constant__ SgemmTask t) {
  extern __shared__ __align__(1024) uint8_t s_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)s_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + P_STAGES * P_STAGE_BYTES);
  uint64_t* empty = full + P_STAGES;
  uint64_t* accum = empty + P_STAGES;
  uint32_t* tmem_slot = (uint32_t*)(accum + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = p_cluster_rank();
  const int pair = blockIdx.x >> 1;
  const int GROUP_M = t.group_m > 0 ? t.group_m : 4;
  const int tiles_m = (t.h + P_BM - 1) / P_BM, tiles_n = (t.w + P_BN - 1) / P_BN;
  const int per_group = GROUP_M * tiles_n;
  const int first_m = (pair / per_group) * GROUP_M;
  const int gsize = min(tiles_m - first_m, GROUP_M);
  const int m0 = (first_m + (pair % per_group) % gsize) * P_BM;
  const int n0 = ((pair % per_group) / gsize) * P_BN;
  const int my_m0 = m0 + 128 * (int)rank;   // rows of A / accumulator held by this CTA
  const int my_n0 = n0 + 128 * (int)rank;   // columns of B staged by this CTA

  int total = 0;
  for (int s = 0; s < t.nsteps; ++s) total += (t.steps[s].d + P_BK - 1) / P_BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < P_STAGES; ++s) { s_mbar_init(&full[s], 1); s_mbar_init(&empty[s], 1); }
    s_mbar_init(accum, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(s_u32(tmem_slot)), "n"(S_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  s_fence_before();
  p_cluster_sync();
  s_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int step = 0, k0 = 0;
      int dcur = t.nsteps > 0 ? t.steps[0].d : 0;
      const CUtensorMap* ma = &t.steps[0].map_a;
      const CUtensorMap* mb = &t.steps[0].map_b;
      for (int it = 0; it < total; ++it) {
        const int st = it % P_STAGES;
        if (it >= P_STAGES) p_mbar_wait(&empty[st], ((it / P_STAGES) - 1) & 1);
        uint8_t* sa = smem + st * P_STAGE_BYTES;
        uint8_t* sb = sa + P_A_BYTES;
        // the leader's barrier expects both CTAs' bytes
        if (rank == 0) s_mbar_expect_tx(&full[st], 2 * P_STAGE_BYTES);
        if (TA) {
          p_tma_2d_pair(sa, ma, &full[st], k0, my_m0);
        } else if (t.a3d) {
          p_tma_3d_pair(sa, ma, &full[st], 0, k0, my_m0 / 32);
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) p_tma_2d_pair(sa + i * 4096, ma, &full[st], my_m0 + 32 * i, k0);
        }
        if (!TB) {
          p_tma_2d_pair(sb, mb, &full[st], k0, my_n0);
        } else if (t.b3d) {
          p_tma_3d_pair(sb, mb, &full[st], 0, k0, my_n0 / 32);
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) p_tma_2d_pair(sb + i * 4096, mb, &full[st], my_n0 + 32 * i, k0);
        }
        k0 += P_BK;
        if (k0 >= dcur) {
          k0 = 0;
          if (++step < t.nsteps) {
            dcur = t.steps[step].d;
            ma = &t.steps[step].map_a;
            mb = &t.steps[step].map_b;
          }
        }
      }
      // producer tail: wait for the leader's last multicast commits on this CTA's "empty"
      // barriers, so no arrival can land in this SM's shared memory after the CTA exits
      // (the next CTA scheduled on the SM would see it on its own barriers)
      for (int it = total > P_STAGES ? total - P_STAGES : 0; it < total; ++it)
        p_mbar_wait(&empty[it % P_STAGES], (it / P_STAGES) & 1);
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = (s_idesc(!TA, TB) & ~(0x1Fu << 24)) | ((uint32_t)(P_BM >> 4) << 24);  // M = 256
      const uint32_t sbase = s_u32(smem);
      const uint64_t da0 = TA ? s_desc(sbase, 16, 1024, 2) : s_desc(sbase, t.mn_lbo, t.mn_sbo, 1);
      const uint64_t db0 = TB ? s_desc(sbase + P_A_BYTES, t.mn_lbo, t.mn_sbo, 1)
                              : s_desc(sbase + P_A_BYTES, 16, 1024, 2);
      constexpr uint32_t AK = TA ? 32 / 16 : 1024 / 16;
      constexpr uint32_t BKS = TB ? 1024 / 16 : 32 / 16;
      constexpr uint32_t SU = P_STAGE_BYTES / 16;
      for (int it0 = 0; it0 < total; it0 += P_STAGES) {
        const uint32_t par = (it0 / P_STAGES) & 1;
#pragma unroll
        for (int st = 0; st < P_STAGES; ++st) {
          if (it0 + st >= total) break;
          p_mbar_wait(&full[st], par);
          s_fence_after();
#pragma unroll
          for (int kk = 0; kk < P_BK / 8; ++kk) {
            const uint32_t acc = (it0 + st + kk) != 0;
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                " tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                ::"r"(tmem), "l"(da0 + (uint64_t)(st * SU + kk * AK)), "l"(db0 + (uint64_t)(st * SU + kk * BKS)),
                  "n"(idesc), "r"(acc));
          }
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                       ::"r"(s_u32(&empty[st])), "h"((uint16_t)3) : "memory");
        }
      }
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                   ::"r"(s_u32(accum)), "h"((uint16_t)3) : "memory");
    }
  } else {
    const int q = warp & 3;
    const int row = my_m0 + 32 * q + lane;
    if (total > 0) {
      p_mbar_wait(accum, 0);
      s_fence_after();
    }
    for (int c0 = 0; c0 < P_BN; c0 += 16) {
      uint32_t v[16];
      if (total > 0) {
        const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0u;
      }
      if (row < t.h) {
        s_store16(t, v, row, n0 + c0);
      }
    }
  }
  s_fence_before();
  p_cluster_sync();
  if (warp == 1) {
    s_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(S_TMEM_COLS));
  }
}

}  // namespace bx

// ---------------------------------------------------------------------------------------
// Persistent 2-SM variant (bx_set_sgemm_variant(2)): one 2-CTA cluster per TPC loops over
// pair tiles (static round robin in the grouped raster order).  TMEM holds two 256-column
// accumulators, so the MMA thread starts tile t+1 while the epilogue warps drain tile t:
// the tensor pipe no longer idles through the per-tile epilogue, cluster teardown, CTA
// launch, TMEM allocation and ring refill of the one-tile-per-cluster kernel.  The stage
// ring (full/empty) runs on across tiles.  tfull[b] (MMA -> epilogue, multicast commit to
// both CTAs) and tempty[b] (epilogue -> MMA: the 8 epilogue warps of the pair arrive on
// the leader's barrier through its cluster address) hand accumulator b back and forth.
// ---------------------------------------------------------------------------------------
namespace bx {

__device__ __forceinline__ uint32_t p_leader_addr(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(r) : "r"(s_u32(p)));
  return r;
}
__device__ __forceinline__ void p_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}

template <int TA, int TB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(P_THREADS, 1)
    sgemm_tc2p_kernel(const __grid_constant__ SgemmTask t) {
  extern __shared__ __align__(1024) uint8_t s_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)s_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + P_STAGES * P_STAGE_BYTES);
  uint64_t* empty = full + P_STAGES;
  uint64_t* tfull = empty + P_STAGES;      // [2]
  uint64_t* tempty = tfull + 2;            // [2] (used in the leader CTA)
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = p_cluster_rank();
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int GROUP_M = t.group_m > 0 ? t.group_m : 4;
  const int tiles_m = (t.h + P_BM - 1) / P_BM, tiles_n = (t.w + P_BN - 1) / P_BN;
  const int ntiles = tiles_m * tiles_n;
  const int per_group = GROUP_M * tiles_n;
  auto tile_origin = [&](int tile, int& m0, int& n0) {
    const int first_m = (tile / per_group) * GROUP_M;
    const int gsize = min(tiles_m - first_m, GROUP_M);
    m0 = (first_m + (tile % per_group) % gsize) * P_BM;
    n0 = ((tile % per_group) / gsize) * P_BN;
  };

  int kslabs = 0;
  for (int s = 0; s < t.nsteps; ++s) kslabs += (t.steps[s].d + P_BK - 1) / P_BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < P_STAGES; ++s) { s_mbar_init(&full[s], 1); s_mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { s_mbar_init(&tfull[b], 1); s_mbar_init(&tempty[b], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(s_u32(tmem_slot)), "n"(2 * S_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  s_fence_before();
  p_cluster_sync();
  s_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0 && kslabs > 0) {
      int it = 0;
      for (int tile = cluster; tile < ntiles; tile += nclusters) {
        int m0, n0;
        tile_origin(tile, m0, n0);
        const int my_m0 = m0 + 128 * (int)rank, my_n0 = n0 + 128 * (int)rank;
        int step = 0, k0 = 0, dcur = t.steps[0].d;
        const CUtensorMap* ma = &t.steps[0].map_a;
        const CUtensorMap* mb = &t.steps[0].map_b;
        for (int ks = 0; ks < kslabs; ++ks, ++it) {
          const int st = it % P_STAGES;
          if (it >= P_STAGES) p_mbar_wait(&empty[st], ((it / P_STAGES) - 1) & 1);
          uint8_t* sa = smem + st * P_STAGE_BYTES;
          uint8_t* sb = sa + P_A_BYTES;
          if (rank == 0) s_mbar_expect_tx(&full[st], 2 * P_STAGE_BYTES);
          if (TA) {
            p_tma_2d_pair(sa, ma, &full[st], k0, my_m0);
          } else if (t.a3d) {
            p_tma_3d_pair(sa, ma, &full[st], 0, k0, my_m0 / 32);
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) p_tma_2d_pair(sa + i * 4096, ma, &full[st], my_m0 + 32 * i, k0);
          }
          if (!TB) {
            p_tma_2d_pair(sb, mb, &full[st], k0, my_n0);
          } else if (t.b3d) {
            p_tma_3d_pair(sb, mb, &full[st], 0, k0, my_n0 / 32);
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) p_tma_2d_pair(sb + i * 4096, mb, &full[st], my_n0 + 32 * i, k0);
          }
          k0 += P_BK;
          if (k0 >= dcur) {
            k0 = 0;
            if (++step < t.nsteps) {
              dcur = t.steps[step].d;
              ma = &t.steps[step].map_a;
              mb = &t.steps[step].map_b;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0 && kslabs > 0) {
      constexpr uint32_t idesc = (s_idesc(!TA, TB) & ~(0x1Fu << 24)) | ((uint32_t)(P_BM >> 4) << 24);
      const uint32_t sbase = s_u32(smem);
      const uint64_t da0 = TA ? s_desc(sbase, 16, 1024, 2) : s_desc(sbase, t.mn_lbo, t.mn_sbo, 1);
      const uint64_t db0 = TB ? s_desc(sbase + P_A_BYTES, t.mn_lbo, t.mn_sbo, 1)
                              : s_desc(sbase + P_A_BYTES, 16, 1024, 2);
      constexpr uint32_t AK = TA ? 32 / 16 : 1024 / 16;
      constexpr uint32_t BKS = TB ? 1024 / 16 : 32 / 16;
      constexpr uint32_t SU = P_STAGE_BYTES / 16;
      int it = 0, n = 0;
      for (int tile = cluster; tile < ntiles; tile += nclusters, ++n) {
        const int b = n & 1;
        if (n >= 2) p_mbar_wait(&tempty[b], ((n >> 1) - 1) & 1);   // epilogue drained acc b
        s_fence_after();
        const uint32_t acc_tm = tmem + (uint32_t)(b * S_TMEM_COLS);
        for (int ks = 0; ks < kslabs; ++ks, ++it) {
          const int st = it % P_STAGES;
          p_mbar_wait(&full[st], (it / P_STAGES) & 1);
          s_fence_after();
          const uint64_t so = (uint64_t)(st * SU);
#pragma unroll
          for (int kk = 0; kk < P_BK / 8; ++kk) {
            const uint32_t acc = (ks + kk) != 0;
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                " tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                ::"r"(acc_tm), "l"(da0 + so + kk * AK), "l"(db0 + so + kk * BKS), "n"(idesc), "r"(acc));
          }
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                       ::"r"(s_u32(&empty[st])), "h"((uint16_t)3) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                     ::"r"(s_u32(&tfull[b])), "h"((uint16_t)3) : "memory");
      }
    }
  } else {
    const int q = warp & 3;
    const uint32_t lead_tempty[2] = {p_leader_addr(&tempty[0]), p_leader_addr(&tempty[1])};
    int n = 0;
    for (int tile = cluster; tile < ntiles; tile += nclusters, ++n) {
      const int b = n & 1;
      int m0, n0;
      tile_origin(tile, m0, n0);
      const int row = m0 + 128 * (int)rank + 32 * q + lane;
      if (kslabs > 0) {
        p_mbar_wait(&tfull[b], (n >> 1) & 1);
        s_fence_after();
      }
      for (int c0 = 0; c0 < P_BN; c0 += 16) {
        uint32_t v[16];
        if (kslabs > 0) {
          const uint32_t taddr = tmem + (uint32_t)(b * S_TMEM_COLS) + ((uint32_t)(32 * q) << 16) + (uint32_t)c0;
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0u;
        }
        if (c0 + 16 >= P_BN && kslabs > 0) {
          // every TMEM read of accumulator b by this warp is done: hand it back to the MMA
          s_fence_before();
          __syncwarp();
          if (lane == 0) p_arrive_cluster(lead_tempty[b]);
        }
        if (row < t.h) {
          s_store16(t, v, row, n0 + c0);
        }
      }
    }
  }
  s_fence_before();
  p_cluster_sync();
  if (warp == 1) {
    s_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(2 * S_TMEM_COLS));
  }
}

}  // namespace bx

// ---------------------------------------------------------------------------------------
// Persistent 2-SM variant with cluster launch control (bx_set_sgemm_variant(3)).  The grid
// is the full one-cluster-per-pair-tile grid of variant 1; a running cluster finishes its
// own tile and then *cancels* the next not-yet-launched cluster (clusterlaunchcontrol.
// try_cancel) and computes that cluster's tile instead.  The hardware hands out clusters
// in launch order, so the in-flight tiles stay the contiguous raster window of variant 1
// (no drift, no extra DRAM traffic — the failure of the round-robin variant 2) while the
// double-buffered TMEM accumulators of variant 2 overlap tile t's epilogue with tile
// t+1's MMAs.  Warp 6 of the leader CTA is the scheduler: it keeps up to two responses
// ahead in a 2-slot ring (cfull: the response landed, multicast to both CTAs with 16
// bytes of transaction each; cempty: all 11 consumers of the pair — 2 producers, the MMA
// thread, 8 epilogue warps — read it, counted on the leader's barrier).  A failed cancel
// (no cluster left) ends every role after its current tile; no query follows a failure.
// ---------------------------------------------------------------------------------------
namespace bx {

constexpr int C_THREADS = 224;             // P_THREADS + the scheduler warp
constexpr int C_CONSUMERS = 11;            // 2 producers + 1 MMA + 8 epilogue warps

__device__ __forceinline__ uint32_t p_rank_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(s_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void p_arrive_expect_tx_cluster(uint32_t cluster_addr, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;\n"
               ::"r"(cluster_addr), "r"(bytes) : "memory");
}
// cancel the next unlaunched cluster; the 16-byte response lands in every CTA of this
// cluster at `resp`'s offset and completes 16 bytes of transaction on each CTA's `bar`
__device__ __forceinline__ void clc_try_cancel(void* resp, uint64_t* bar) {
  asm volatile(
      "clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.multicast::cluster::all.b128 [%0], [%1];\n"
      ::"r"(s_u32(resp)), "r"(s_u32(bar)) : "memory");
}
// ctaid.x of the first CTA of the cancelled cluster, or -1 (nothing left to cancel)
__device__ __forceinline__ int clc_first_ctaid(const void* resp) {
  uint32_t x = 0, ok = 0;
  asm volatile(
      "{\n .reg .pred p;\n .reg .b128 r;\n ld.shared.b128 r, [%2];\n"
      " clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p, r;\n selp.u32 %1, 1, 0, p;\n"
      " @p clusterlaunchcontrol.query_cancel.get_first_ctaid.v4.b32.b128 {%0, _, _, _}, r;\n}\n"
      : "=r"(x), "=r"(ok) : "r"(s_u32(resp)) : "memory");
  // order this generic-proxy read before the next async-proxy write of the slot
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  return ok ? (int)x : -1;
}

template <int TA, int TB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(C_THREADS, 1)
    sgemm_tc2c_kernel(const __grid_constant__ SgemmTask t) {
  extern __shared__ __align__(1024) uint8_t s_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)s_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + P_STAGES * P_STAGE_BYTES);
  uint64_t* empty = full + P_STAGES;
  uint64_t* tfull = empty + P_STAGES;      // [2]
  uint64_t* tempty = tfull + 2;            // [2] (used in the leader CTA)
  uint64_t* cfull = tempty + 2;            // [2] CLC response landed
  uint64_t* cempty = cfull + 2;            // [2] CLC response consumed (leader CTA)
  uint4* resp = (uint4*)(cempty + 2);      // [2] 16-byte CLC responses (16-B aligned)
  uint32_t* tmem_slot = (uint32_t*)(resp + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = p_cluster_rank();
  const int GROUP_M = t.group_m > 0 ? t.group_m : 4;
  const int tiles_m = (t.h + P_BM - 1) / P_BM, tiles_n = (t.w + P_BN - 1) / P_BN;
  const int per_group = GROUP_M * tiles_n;
  auto tile_origin = [&](int tile, int& m0, int& n0) {
    const int first_m = (tile / per_group) * GROUP_M;
    const int gsize = min(tiles_m - first_m, GROUP_M);
    m0 = (first_m + (tile % per_group) % gsize) * P_BM;
    n0 = ((tile % per_group) / gsize) * P_BN;
  };
  const uint32_t lead_cempty[2] = {p_leader_addr(&cempty[0]), p_leader_addr(&cempty[1])};
  // the tile after the j-th: wait for response j, hand the slot back, decode
  auto next_tile = [&](int j, bool release) -> int {
    const int sl = j & 1;
    p_mbar_wait(&cfull[sl], (j >> 1) & 1);
    const int x = clc_first_ctaid(&resp[sl]);
    if (release) p_arrive_cluster(lead_cempty[sl]);
    return x < 0 ? -1 : x >> 1;
  };

  int kslabs = 0;
  for (int s = 0; s < t.nsteps; ++s) kslabs += (t.steps[s].d + P_BK - 1) / P_BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < P_STAGES; ++s) { s_mbar_init(&full[s], 1); s_mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) {
      s_mbar_init(&tfull[b], 1);
      s_mbar_init(&tempty[b], 8);
      s_mbar_init(&cfull[b], 1);
      s_mbar_init(&cempty[b], C_CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(s_u32(tmem_slot)), "n"(2 * S_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  s_fence_before();
  p_cluster_sync();
  s_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 6) {
    if (lane == 0 && rank == 0) {
      const uint32_t peer_cfull[2] = {p_rank_addr(&cfull[0], 1), p_rank_addr(&cfull[1], 1)};
      for (int i = 0;; ++i) {
        const int sl = i & 1;
        if (i >= 2) p_mbar_wait(&cempty[sl], ((i >> 1) - 1) & 1);
        s_mbar_expect_tx(&cfull[sl], 16);
        p_arrive_expect_tx_cluster(peer_cfull[sl], 16);
        clc_try_cancel(&resp[sl], &cfull[sl]);
        p_mbar_wait(&cfull[sl], (i >> 1) & 1);
        if (clc_first_ctaid(&resp[sl]) < 0) break;   // nothing left: never query again
      }
    }
  } else if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int tile = blockIdx.x >> 1, j = 0; tile >= 0; tile = next_tile(j++, true)) {
        if (kslabs == 0) continue;
        int m0, n0;
        tile_origin(tile, m0, n0);
        const int my_m0 = m0 + 128 * (int)rank, my_n0 = n0 + 128 * (int)rank;
        int step = 0, k0 = 0, dcur = t.steps[0].d;
        const CUtensorMap* ma = &t.steps[0].map_a;
        const CUtensorMap* mb = &t.steps[0].map_b;
        for (int ks = 0; ks < kslabs; ++ks, ++it) {
          const int st = it % P_STAGES;
          if (it >= P_STAGES) p_mbar_wait(&empty[st], ((it / P_STAGES) - 1) & 1);
          uint8_t* sa = smem + st * P_STAGE_BYTES;
          uint8_t* sb = sa + P_A_BYTES;
          if (rank == 0) s_mbar_expect_tx(&full[st], 2 * P_STAGE_BYTES);
          if (TA) {
            p_tma_2d_pair(sa, ma, &full[st], k0, my_m0);
          } else if (t.a3d) {
            p_tma_3d_pair(sa, ma, &full[st], 0, k0, my_m0 / 32);
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) p_tma_2d_pair(sa + i * 4096, ma, &full[st], my_m0 + 32 * i, k0);
          }
          if (!TB) {
            p_tma_2d_pair(sb, mb, &full[st], k0, my_n0);
          } else if (t.b3d) {
            p_tma_3d_pair(sb, mb, &full[st], 0, k0, my_n0 / 32);
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) p_tma_2d_pair(sb + i * 4096, mb, &full[st], my_n0 + 32 * i, k0);
          }
          k0 += P_BK;
          if (k0 >= dcur) {
            k0 = 0;
            if (++step < t.nsteps) {
              dcur = t.steps[step].d;
              ma = &t.steps[step].map_a;
              mb = &t.steps[step].map_b;
            }
          }
        }
      }
      // producer tail: the leader's last multicast commits land on this CTA's "empty"
      // barriers before it exits (else they would hit the next CTA on this SM)
      for (int i2 = it > P_STAGES ? it - P_STAGES : 0; i2 < it; ++i2)
        p_mbar_wait(&empty[i2 % P_STAGES], (i2 / P_STAGES) & 1);
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = (s_idesc(!TA, TB) & ~(0x1Fu << 24)) | ((uint32_t)(P_BM >> 4) << 24);
      const uint32_t sbase = s_u32(smem);
      const uint64_t da0 = TA ? s_desc(sbase, 16, 1024, 2) : s_desc(sbase, t.mn_lbo, t.mn_sbo, 1);
      const uint64_t db0 = TB ? s_desc(sbase + P_A_BYTES, t.mn_lbo, t.mn_sbo, 1)
                              : s_desc(sbase + P_A_BYTES, 16, 1024, 2);
      constexpr uint32_t AK = TA ? 32 / 16 : 1024 / 16;
      constexpr uint32_t BKS = TB ? 1024 / 16 : 32 / 16;
      constexpr uint32_t SU = P_STAGE_BYTES / 16;
      int it = 0, n = 0;
      for (int tile = blockIdx.x >> 1, j = 0; tile >= 0; tile = next_tile(j++, true), ++n) {
        if (kslabs == 0) continue;
        const int b = n & 1;
        if (n >= 2) p_mbar_wait(&tempty[b], ((n >> 1) - 1) & 1);   // epilogue drained acc b
        s_fence_after();
        const uint32_t acc_tm = tmem + (uint32_t)(b * S_TMEM_COLS);
        for (int ks = 0; ks < kslabs; ++ks, ++it) {
          const int st = it % P_STAGES;
          p_mbar_wait(&full[st], (it / P_STAGES) & 1);
          s_fence_after();
          const uint64_t so = (uint64_t)(st * SU);
#pragma unroll
          for (int kk = 0; kk < P_BK / 8; ++kk) {
            const uint32_t acc = (ks + kk) != 0;
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                " tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                ::"r"(acc_tm), "l"(da0 + so + kk * AK), "l"(db0 + so + kk * BKS), "n"(idesc), "r"(acc));
          }
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                       ::"r"(s_u32(&empty[st])), "h"((uint16_t)3) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                     ::"r"(s_u32(&tfull[b])), "h"((uint16_t)3) : "memory");
      }
    }
  } else if (warp >= 2 && warp <= 5) {
    const int q = warp & 3;
    const uint32_t lead_tempty[2] = {p_leader_addr(&tempty[0]), p_leader_addr(&tempty[1])};
    int n = 0;
    for (int tile = blockIdx.x >> 1, j = 0; tile >= 0; ++n) {
      const int b = n & 1;
      int m0, n0;
      tile_origin(tile, m0, n0);
      const int row = m0 + 128 * (int)rank + 32 * q + lane;
      if (kslabs > 0) {
        p_mbar_wait(&tfull[b], (n >> 1) & 1);
        s_fence_after();
      }
      for (int c0 = 0; c0 < P_BN; c0 += 16) {
        uint32_t v[16];
        if (kslabs > 0) {
          const uint32_t taddr = tmem + (uint32_t)(b * S_TMEM_COLS) + ((uint32_t)(32 * q) << 16) + (uint32_t)c0;
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0u;
        }
        if (c0 + 16 >= P_BN && kslabs > 0) {
          // every TMEM read of accumulator b by this warp is done: hand it back to the MMA
          s_fence_before();
          __syncwarp();
          if (lane == 0) p_arrive_cluster(lead_tempty[b]);
        }
        if (row < t.h) {
          s_store16(t, v, row, n0 + c0);
        }
      }
      // next tile: every lane reads the response, one arrival per warp
      {
        const int sl = j & 1;
        p_mbar_wait(&cfull[sl], (j >> 1) & 1);
        const int x = clc_first_ctaid(&resp[sl]);
        __syncwarp();
        if (lane == 0) p_arrive_cluster(lead_cempty[sl]);
        ++j;
        tile = x < 0 ? -1 : x >> 1;
      }
    }
  }
  s_fence_before();
  p_cluster_sync();
  if (warp == 1) {
    s_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(2 * S_TMEM_COLS));
  }
}

}  // namespace bx

// ---------------------------------------------------------------------------------------
// 3xTF32 split for the precise SGEMM mode (bx_set_sgemm_precise): x = hi + lo with hi the
// TF32-rounded value (low 13 mantissa bits zero, so the tensor core takes it exactly) and
// lo = x - hi (exact in fp32).  A*B ~= hi_a*hi_b + hi_a*lo_b + lo_a*hi_b restores ~fp32
// accuracy at a third of the TF32 rate.  Strided rows x cols column-major input -> two
// packed (ld = rows rounded up to 4) outputs.
// ---------------------------------------------------------------------------------------
namespace bx {

__global__ void tf32_split_kernel(const float* __restrict__ x, int ldx, int rows, int cols, float* __restrict__ hi,
                                  float* __restrict__ lo, int ldo) {
  const int r = blockIdx.x * 32 + threadIdx.x;
  const int c = blockIdx.y * 8 + threadIdx.y;
  if (r >= rows || c >= cols) return;
  const float v = x[(size_t)c * ldx + r];
  uint32_t u = __float_as_uint(v);
  if ((u & 0x7F800000u) != 0x7F800000u) u = (u + 0x1000u) & 0xFFFFE000u;   // round to 10-bit mantissa
  const float h = __uint_as_float(u);
  hi[(size_t)c * ldo + r] = h;
  lo[(size_t)c * ldo + r] = v - h;
}

}  // namespace bx

