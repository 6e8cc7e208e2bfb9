// FP64 tile-task GEMM on the B200 FP64 tensor path (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4).
//
// One launch computes one output tile task of the BLASX planner
// (reference: /root/reference/pkg/src/tileblas/routines.py:227-380, kernels.py:49-58):
//
//     C[h x w] = alpha * sum_s op_s(A_s)[h x d_s] * op_s(B_s)[d_s x w] + beta * C
//
// over a list of k-steps whose accumulators stay in registers for the whole k-range
// (C is read once and written once per task instead of once per step).  beta == 0
// never reads C (kernels.py:39-41); tri != 0 restricts reads/writes to the stored
// triangle of a diagonal tile (syrk/syr2k_update, kernels.py:67-102) and skips CTAs
// that lie wholly in the unstored half.
//
// Device tile layout (chosen by the transfer engine): column-major,
// leading dimension a multiple of 8 elements, base 256-B aligned.  Operands are staged
// into shared memory with 16-B cp.async (zero-filled past the tile edge) in one of two
// layouts per operand, both bank-conflict free for the DMMA fragment loads (pitch = 4
// mod 16 doubles): "MN-major" sX[k][mn] when mn is the contiguous direction in global
// memory, "K-major" sX[mn][k] when k is.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bx {

constexpr int G_MAX_STEPS = 40;

enum TriMode { TRI_NONE = 0, TRI_LOWER = 1, TRI_UPPER = 2 };
// Triangular operand (per step): a CTA reads only the k-range where the step's triangular
// operand can be non-zero — e.g. X = inv(L) B with inv(L) lower: output row block
// [m0, m0+BM) needs k < m0+BM.  Halves the flops of the TRSM diagonal apply and of the
// TRMM diagonal step (op(tri(A)) B); the operand's other triangle holds exact zeros, so a
// kernel that ignores the mode computes the same result.
enum KMode { KM_NONE = 0, KM_A_LOWER = 1, KM_A_UPPER = 2, KM_B_UPPER = 3, KM_B_LOWER = 4 };

__device__ __forceinline__ void step_krange(int d, int kmode, int m0, int n0, int bm, int bn, int& kb, int& ke) {
  kb = 0;
  ke = d;
  if (kmode == KM_A_LOWER) ke = min(d, m0 + bm);
  else if (kmode == KM_A_UPPER) kb = min(d, m0);
  else if (kmode == KM_B_UPPER) ke = min(d, n0 + bn);
  else if (kmode == KM_B_LOWER) kb = min(d, n0);
}

struct GemmStep {
  const double* a;
  const double* b;
  int lda, ldb, d, kmode;
};

struct GemmTask {
  double* c;
  int ldc, h, w, nsteps, tri, group_m;
  double alpha, beta;
  GemmStep steps[G_MAX_STEPS];
};

// Tile configuration: CTA BM x BN x BK, warp tile WM x WN, STAGES-deep cp.async ring.
template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_>
struct GemmCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int MF = WM / 8, NF = WN / 8;
  static constexpr int LD_K = BK + 4;  // K-major pitch (doubles), = 4 mod 16
  static constexpr int A_ELEMS = (BK * (BM + 4) > BM * LD_K) ? BK * (BM + 4) : BM * LD_K;
  static constexpr int B_ELEMS = (BK * (BN + 4) > BN * LD_K) ? BK * (BN + 4) : BN * LD_K;
  static constexpr int SMEM_BYTES = STAGES * (A_ELEMS + B_ELEMS) * 8;
  static_assert((BM + 4) % 16 == 4 && (BN + 4) % 16 == 4 && LD_K % 16 == 4, "pitch");
  static_assert((BM * BK / 2) % THREADS == 0 && (BN * BK / 2) % THREADS == 0, "load split");
};

using CfgWide = GemmCfg<128, 128, 16, 64, 32, 4>;     // 8 warps, 2 warps/SMSP
using CfgDeep = GemmCfg<128, 128, 32, 32, 32, 3>;     // 16 warps, 4 warps/SMSP

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

// Stage one BK-deep slab of op(X) along mn in [mn0, mn0+EXT) into shared memory.
// KCONTIG: k is the contiguous direction in global memory -> K-major smem.
template <class Cfg, int EXT, bool KCONTIG>
__device__ __forceinline__ void load_slab(double* s, const double* g, int ld, int mn0, int mn_ext,
                                          int k0, int d, int tid) {
  constexpr int BK = Cfg::BK;
  constexpr int KCH = BK / 2;      // 16-B chunks per mn row (K-major)
  constexpr int MCH = EXT / 2;     // 16-B chunks per k row (MN-major)
#pragma unroll
  for (int c = 0; c < (EXT * BK / 2) / Cfg::THREADS; ++c) {
    int idx = tid + c * Cfg::THREADS;
    if (KCONTIG) {
      int mn = idx / KCH, k = (idx % KCH) * 2;
      int gm = mn0 + mn, gk = k0 + k;
      int valid = (gm < mn_ext) ? min(max(d - gk, 0), 2) : 0;
      const double* src = valid ? g + (size_t)gm * ld + gk : g;
      cp_async16(s + mn * Cfg::LD_K + k, src, valid * 8);
    } else {
      int k = idx / MCH, mn = (idx % MCH) * 2;
      int gm = mn0 + mn, gk = k0 + k;
      int valid = (gk < d) ? min(max(mn_ext - gm, 0), 2) : 0;
      const double* src = valid ? g + (size_t)gk * ld + gm : g;
      cp_async16(s + k * (EXT + 4) + mn, src, valid * 8);
    }
  }
}

template <class Cfg, int EXT, bool KMAJ>
__device__ __forceinline__ double frag(const double* s, int mn, int k) {
  return KMAJ ? s[mn * Cfg::LD_K + k] : s[k * (EXT + 4) + mn];
}

// TA/TB: operand stored transposed (op = T).  A is K-contiguous iff TA; B iff !TB.
template <class Cfg, bool TA, bool TB>
__global__ void __launch_bounds__(Cfg::THREADS, 1) gemm_task_kernel(const __grid_constant__ GemmTask t) {
  extern __shared__ __align__(128) double smem[];
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES;
  constexpr int MF = Cfg::MF, NF = Cfg::NF;
  constexpr bool A_KMAJ = TA;
  constexpr bool B_KMAJ = !TB;

  // grouped rasterisation of a 1-D grid (L2 reuse when one launch spans many tiles)
  const int tiles_m = (t.h + BM - 1) / BM, tiles_n = (t.w + BN - 1) / BN;
  const int bid = blockIdx.x;
  const int per_group = t.group_m * tiles_n;
  const int first_m = (bid / per_group) * t.group_m;
  const int gsize = min(tiles_m - first_m, t.group_m);
  const int bm = first_m + (bid % per_group) % gsize;
  const int bn = (bid % per_group) / gsize;
  const int m0 = bm * BM, n0 = bn * BN;
  if (t.tri == TRI_LOWER && n0 >= m0 + BM) return;   // wholly above the diagonal
  if (t.tri == TRI_UPPER && m0 >= n0 + BN) return;   // wholly below

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp % Cfg::WARPS_M) * Cfg::WM, wn = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int g = lane >> 2, q = lane & 3;

  int total = 0;
  for (int s = 0; s < t.nsteps; ++s) total += (t.steps[s].d + BK - 1) / BK;

  double* sA = smem;
  double* sB = smem + STAGES * Cfg::A_ELEMS;

  int ld_step = 0, ld_k = 0;   // producer cursor over (step, k)
  auto issue = [&](int stage) {
    const GemmStep& st = t.steps[ld_step];
    load_slab<Cfg, BM, A_KMAJ>(sA + stage * Cfg::A_ELEMS, st.a, st.lda, m0, t.h, ld_k, st.d, tid);
    load_slab<Cfg, BN, B_KMAJ>(sB + stage * Cfg::B_ELEMS, st.b, st.ldb, n0, t.w, ld_k, st.d, tid);
    ld_k += BK;
    if (ld_k >= st.d) { ld_k = 0; ++ld_step; }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < total) issue(s);
    cp_async_commit();
  }

  double acc[MF][NF][2];
#pragma unroll
  for (int i = 0; i < MF; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int it = 0; it < total; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int nxt = it + STAGES - 1;
      if (nxt < total) issue(nxt % STAGES);
      cp_async_commit();
    }
    const double* a = sA + (it % STAGES) * Cfg::A_ELEMS;
    const double* b = sB + (it % STAGES) * Cfg::B_ELEMS;
    double fa[2][MF], fb[2][NF];
#pragma unroll
    for (int i = 0; i < MF; ++i) fa[0][i] = frag<Cfg, BM, A_KMAJ>(a, wm + i * 8 + g, q);
#pragma unroll
    for (int j = 0; j < NF; ++j) fb[0][j] = frag<Cfg, BN, B_KMAJ>(b, wn + j * 8 + g, q);
#pragma unroll
    for (int kq = 0; kq < BK / 4; ++kq) {
      const int cur = kq & 1, nx = cur ^ 1;
      if (kq + 1 < BK / 4) {
#pragma unroll
        for (int i = 0; i < MF; ++i) fa[nx][i] = frag<Cfg, BM, A_KMAJ>(a, wm + i * 8 + g, (kq + 1) * 4 + q);
#pragma unroll
        for (int j = 0; j < NF; ++j) fb[nx][j] = frag<Cfg, BN, B_KMAJ>(b, wn + j * 8 + g, (kq + 1) * 4 + q);
      }
#pragma unroll
      for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) dmma(acc[i][j], fa[cur][i], fb[cur][j]);
    }
  }
  cp_async_wait<0>();

  // epilogue: C = alpha*acc + beta*C  (beta == 0: C never read)
  // epilogue, one fragment row i at a time: with beta != 0 its NF x 2 C loads are all
  // issued before the first store (one memory round trip per row instead of 2 NF
  // dependent ones — the epilogue of a short launch with beta = 1 is otherwise a few % of it)
  const double alpha = t.alpha, beta = t.beta;
#pragma unroll
  for (int i = 0; i < MF; ++i) {
    const int r = m0 + wm + i * 8 + g;
    if (r >= t.h) continue;
    double cv[NF][2];
    bool ok[NF][2];
#pragma unroll
    for (int j = 0; j < NF; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cc = n0 + wn + j * 8 + 2 * q + e;
        ok[j][e] = cc < t.w && !(t.tri == TRI_LOWER && cc > r) && !(t.tri == TRI_UPPER && cc < r);
        cv[j][e] = (beta != 0.0 && ok[j][e]) ? t.c[(size_t)cc * t.ldc + r] : 0.0;
      }
    }
#pragma unroll
    for (int j = 0; j < NF; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (!ok[j][e]) continue;
        const int cc = n0 + wn + j * 8 + 2 * q + e;
        double v = alpha * acc[i][j][e];
        if (beta != 0.0) v = fma(beta, cv[j][e], v);
        t.c[(size_t)cc * t.ldc + r] = v;
      }
    }
  }
}

}  // namespace bx

// ---------------------------------------------------------------------------------------
// Barrier-free variant: every warp is both producer and consumer, but stage hand-off runs
// through mbarriers instead of __syncthreads.  Each thread's cp.async share of a slab
// arrives on the stage's "full" barrier when it lands (cp.async.mbarrier.arrive.noinc);
// each warp releases a stage on its "empty" barrier after its fragment loads.  A warp
// refills a stage only once every warp has finished the slab that lived there, which is
// SLACK+1 slabs behind its own position, so warps drift freely and the FP64 tensor pipe
// never drains at slab boundaries (the __syncthreads of the classic pipeline).
// ---------------------------------------------------------------------------------------
namespace bx {

template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_, int SLACK_, int MINB_ = 1, bool NOLOAD_ = false>
struct MbCfg : GemmCfg<BM_, BN_, BK_, WM_, WN_, STAGES_> {
  using Base = GemmCfg<BM_, BN_, BK_, WM_, WN_, STAGES_>;
  static constexpr bool NOLOAD = NOLOAD_;   // experiment: skip global loads after the first ring
  static constexpr int SLACK = SLACK_;
  static constexpr int MIN_BLOCKS = MINB_;   // CTAs per SM the register budget targets
  static constexpr int DIST = STAGES_ - 1 - SLACK_;   // prefetch distance in slabs
  static constexpr int WARPS = Base::WARPS_M * Base::WARPS_N;
  static constexpr int SMEM_BYTES = Base::SMEM_BYTES + 2 * STAGES_ * 8;
  static_assert(DIST >= 1, "stages");
};

using CfgMb = MbCfg<128, 128, 16, 64, 32, 5, 1>;    // default: 8 warps, 5-stage ring
using CfgMb2 = MbCfg<128, 128, 16, 64, 32, 5, 2>;   // more slack, shorter prefetch
using CfgMb16 = MbCfg<128, 128, 16, 32, 32, 5, 1>;  // 16 warps (4 per SMSP)
// two CTAs per SM (4 warps each): one CTA's stage hand-offs hide behind the other's DMMAs
using CfgMbPair = MbCfg<64, 128, 16, 32, 64, 3, 0, 2>;
using CfgMbK32 = MbCfg<128, 128, 32, 64, 32, 3, 0>;    // BK 32, 3 stages (221 KB)
using CfgMbS0 = MbCfg<128, 128, 16, 64, 32, 5, 0>;     // no slack, prefetch distance 4
using CfgMbNoLoad = MbCfg<128, 128, 16, 64, 32, 5, 1, 1, true>;   // experiment only
using CfgMb16S0 = MbCfg<128, 128, 16, 32, 32, 5, 0>;   // 16 warps, no slack
using CfgMb16S2 = MbCfg<128, 128, 16, 32, 32, 5, 2>;   // 16 warps, slack 2
using CfgMb16K32 = MbCfg<128, 128, 32, 32, 32, 3, 0>;  // 16 warps, BK 32, 3 stages
using CfgMb16x64 = MbCfg<128, 128, 16, 32, 64, 5, 1>;  // 8 warps of 32x64
using CfgMbPairS = MbCfg<64, 128, 16, 32, 64, 3, 1, 2>;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared.b64 st, [%0];\n}\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// one contiguous global -> shared bulk copy whose bytes complete_tx on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];\n" ::"r"(smem_u32(b)) : "memory");
}

__device__ __forceinline__ void cp_async16_full(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

template <class Cfg, int EXT, bool KCONTIG>
__device__ __forceinline__ void fast_slab(double* s, const double* g, int ld, int mn0, int k0, int tid) {
  constexpr int BK = Cfg::BK;
  constexpr int PER = (EXT * BK / 2) / Cfg::THREADS;
  if (KCONTIG) {
    constexpr int KCH = BK / 2;
    constexpr int ROWS = Cfg::THREADS / KCH;       // mn rows covered per pass
    const int mn = tid / KCH, k = (tid % KCH) * 2;
    const double* src = g + (size_t)(mn0 + mn) * ld + k0 + k;
    double* dst = s + mn * Cfg::LD_K + k;
#pragma unroll
    for (int c = 0; c < PER; ++c)
      cp_async16_full(dst + c * ROWS * Cfg::LD_K, src + (size_t)c * ROWS * ld);
  } else {
    constexpr int MCH = EXT / 2;
    constexpr int KR = Cfg::THREADS / MCH;         // k rows covered per pass
    const int k = tid / MCH, mn = (tid % MCH) * 2;
    const double* src = g + (size_t)(k0 + k) * ld + mn0 + mn;
    double* dst = s + k * (EXT + 4) + mn;
#pragma unroll
    for (int c = 0; c < PER; ++c)
      cp_async16_full(dst + c * KR * (EXT + 4), src + (size_t)c * KR * ld);
  }
}

// KM: some step has a triangular operand (per-step k-ranges); the plain instantiation keeps
// the simple step walk of the GEMM hot path (the k-range bookkeeping cost 2 % at 16384^3)
template <class Cfg, bool TA, bool TB, bool KM = false>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MIN_BLOCKS) gemm_task_mb_kernel(const __grid_constant__ GemmTask t) {
  extern __shared__ __align__(128) double smem[];
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES, DIST = Cfg::DIST;
  constexpr int MF = Cfg::MF, NF = Cfg::NF, KQ = BK / 4;
  constexpr bool A_KMAJ = TA;
  constexpr bool B_KMAJ = !TB;
  static_assert(KQ % 2 == 0, "fragment double buffer parity");

  const int tiles_m = (t.h + BM - 1) / BM, tiles_n = (t.w + BN - 1) / BN;
  const int bid = blockIdx.x;
  const int per_group = t.group_m * tiles_n;
  const int first_m = (bid / per_group) * t.group_m;
  const int gsize = min(tiles_m - first_m, t.group_m);
  const int bm = first_m + (bid % per_group) % gsize;
  const int bn = (bid % per_group) / gsize;
  const int m0 = bm * BM, n0 = bn * BN;
  if (t.tri == TRI_LOWER && n0 >= m0 + BM) return;
  if (t.tri == TRI_UPPER && m0 >= n0 + BN) return;

  double* sA = smem;
  double* sB = smem + STAGES * Cfg::A_ELEMS;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * Cfg::B_ELEMS);
  uint64_t* empty = full + STAGES;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // this CTA's slabs: each step's k-range (restricted for triangular operands; the range
  // ends are multiples of BM / BN or the step depth, so slabs stay BK-aligned)
  int total = 0;
  bool kfull = true;
  for (int s = 0; s < t.nsteps; ++s) {
    if constexpr (KM) {
      int kb, ke;
      step_krange(t.steps[s].d, t.steps[s].kmode, m0, n0, BM, BN, kb, ke);
      if (ke > kb) total += (ke - kb + BK - 1) / BK;
    } else {
      total += (t.steps[s].d + BK - 1) / BK;
    }
    kfull = kfull && (t.steps[s].d % BK == 0);
  }
  // Interior CTAs (no tile edge in m, n or any step's k) take an unpredicated cp.async
  // path with no bounds arithmetic; edge CTAs keep the zero-filling path.
  const bool bulk = kfull && m0 + BM <= t.h && n0 + BN <= t.w && !Cfg::NOLOAD;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], Cfg::THREADS);
      mbar_init(&empty[s], Cfg::WARPS);
    }
  }
  __syncthreads();

  int ld_step = KM ? -1 : 0, ld_k = 0, ld_end = 0;
  auto next_step = [&]() {   // advance the loader to the next step with a non-empty range
    do {
      ++ld_step;
      if (ld_step >= t.nsteps) return;
      step_krange(t.steps[ld_step].d, t.steps[ld_step].kmode, m0, n0, BM, BN, ld_k, ld_end);
    } while (ld_end <= ld_k);
  };
  if constexpr (KM) next_step();
  auto produce = [&](int slab) {
    const int stage = slab % STAGES;
    if (slab >= STAGES) mbar_wait(&empty[stage], ((slab / STAGES) - 1) & 1);
    const GemmStep& st = t.steps[ld_step];
    if (bulk) {
      fast_slab<Cfg, BM, A_KMAJ>(sA + stage * Cfg::A_ELEMS, st.a, st.lda, m0, ld_k, tid);
      fast_slab<Cfg, BN, B_KMAJ>(sB + stage * Cfg::B_ELEMS, st.b, st.ldb, n0, ld_k, tid);
      cp_async_arrive_noinc(&full[stage]);
    } else {
      if (!Cfg::NOLOAD || slab < STAGES) {
        load_slab<Cfg, BM, A_KMAJ>(sA + stage * Cfg::A_ELEMS, st.a, st.lda, m0, t.h, ld_k, st.d, tid);
        load_slab<Cfg, BN, B_KMAJ>(sB + stage * Cfg::B_ELEMS, st.b, st.ldb, n0, t.w, ld_k, st.d, tid);
      }
      cp_async_arrive_noinc(&full[stage]);
    }
    ld_k += BK;
    if constexpr (KM) {
      if (ld_k >= ld_end) next_step();
    } else if (ld_k >= st.d) {
      ld_k = 0;
      ++ld_step;
    }
  };
  for (int s = 0; s < DIST && s < total; ++s) produce(s);

  const int wm = (warp % Cfg::WARPS_M) * Cfg::WM, wn = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int g = lane >> 2, q = lane & 3;
  double acc[MF][NF][2];
#pragma unroll
  for (int i = 0; i < MF; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double fa[2][MF], fb[2][NF];
  if (total > 0) {
    mbar_wait(&full[0], 0);
#pragma unroll
    for (int i = 0; i < MF; ++i) fa[0][i] = frag<Cfg, BM, A_KMAJ>(sA, wm + i * 8 + g, q);
#pragma unroll
    for (int j = 0; j < NF; ++j) fb[0][j] = frag<Cfg, BN, B_KMAJ>(sB, wn + j * 8 + g, q);
  }
  for (int it = 0; it < total; ++it) {
    if (it + DIST < total) produce(it + DIST);
    const int stage = it % STAGES;
    const double* a = sA + stage * Cfg::A_ELEMS;
    const double* b = sB + stage * Cfg::B_ELEMS;
#pragma unroll
    for (int kq = 0; kq < KQ; ++kq) {
      const int cur = kq & 1, nx = cur ^ 1;
      if (kq + 1 < KQ) {
#pragma unroll
        for (int i = 0; i < MF; ++i) fa[nx][i] = frag<Cfg, BM, A_KMAJ>(a, wm + i * 8 + g, (kq + 1) * 4 + q);
#pragma unroll
        for (int j = 0; j < NF; ++j) fb[nx][j] = frag<Cfg, BN, B_KMAJ>(b, wn + j * 8 + g, (kq + 1) * 4 + q);
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);   // this warp is done reading the stage
        if (it + 1 < total) {
          const int ns = (it + 1) % STAGES;
          mbar_wait(&full[ns], ((it + 1) / STAGES) & 1);
          const double* a2 = sA + ns * Cfg::A_ELEMS;
          const double* b2 = sB + ns * Cfg::B_ELEMS;
#pragma unroll
          for (int i = 0; i < MF; ++i) fa[nx][i] = frag<Cfg, BM, A_KMAJ>(a2, wm + i * 8 + g, q);
#pragma unroll
          for (int j = 0; j < NF; ++j) fb[nx][j] = frag<Cfg, BN, B_KMAJ>(b2, wn + j * 8 + g, q);
        }
      }
      // serpentine order: consecutive DMMAs share an operand register (operand reuse)
#pragma unroll
      for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int jj = 0; jj < NF; ++jj) {
          const int j = (i & 1) ? NF - 1 - jj : jj;
          dmma(acc[i][j], fa[cur][i], fb[cur][j]);
        }
    }
  }
  cp_async_wait<0>();

  // epilogue, one fragment row i at a time: with beta != 0 its NF x 2 C loads are all
  // issued before the first store (one memory round trip per row instead of 2 NF
  // dependent ones — the epilogue of a short launch with beta = 1 is otherwise a few % of it)
  const double alpha = t.alpha, beta = t.beta;
#pragma unroll
  for (int i = 0; i < MF; ++i) {
    const int r = m0 + wm + i * 8 + g;
    if (r >= t.h) continue;
    double cv[NF][2];
    bool ok[NF][2];
#pragma unroll
    for (int j = 0; j < NF; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cc = n0 + wn + j * 8 + 2 * q + e;
        ok[j][e] = cc < t.w && !(t.tri == TRI_LOWER && cc > r) && !(t.tri == TRI_UPPER && cc < r);
        cv[j][e] = (beta != 0.0 && ok[j][e]) ? t.c[(size_t)cc * t.ldc + r] : 0.0;
      }
    }
#pragma unroll
    for (int j = 0; j < NF; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (!ok[j][e]) continue;
        const int cc = n0 + wn + j * 8 + 2 * q + e;
        double v = alpha * acc[i][j][e];
        if (beta != 0.0) v = fma(beta, cv[j][e], v);
        t.c[(size_t)cc * t.ldc + r] = v;
      }
    }
  }
}

}  // namespace bx

// ---------------------------------------------------------------------------------------
// TMA-fed variant of the FP64 task GEMM (bx_set_gemm_variant(8)).  Same task contract and
// tile shape (CTA 128x128x16, 8 warps of 64x32, DMMA m8n8k4), but the operand slabs are
// staged by the tensor-memory accelerator: one thread issues the bulk tensor copies of a
// stage (128-B swizzled boxes, zero fill past every tile edge, bytes complete on the
// stage's mbarrier), so the other 255 threads spend no issue slots on loads — in the
// cp.async kernel above every thread issues 4 copies, their address arithmetic and an
// arrive per slab.  Fragment loads undo the 128-B swizzle (16-B chunk ^ row % 8).
// ---------------------------------------------------------------------------------------
#include <cuda.h>
namespace bx {

constexpr int T_MAX_STEPS = 16, T_STAGES = 6, T_DIST = 4;
constexpr int T_BM = 128, T_BN = 128, T_BK = 16, T_WM = 64, T_WN = 32, T_THREADS_G = 256;
constexpr int T_A_BYTES = T_BM * T_BK * 8, T_B_BYTES = T_BN * T_BK * 8;   // 16 KB each
constexpr int T_STAGE_BYTES = T_A_BYTES + T_B_BYTES;
constexpr int T_SMEM_BYTES = T_STAGES * T_STAGE_BYTES + 1024 + 2 * T_STAGES * 8;

struct GemmTmaStep {
  CUtensorMap ma;      // A_s: MN-major boxes {16 m, 16 k} or K-major box {16 k, 128 m}
  CUtensorMap mb;      // B_s: K-major box {16 k, 128 n} or MN-major boxes {16 n, 16 k}
  int d;
  int pad_[31];
};

struct GemmTmaTask {
  GemmTmaStep steps[T_MAX_STEPS];
  double* c;
  int ldc, h, w, nsteps, tri, group_m;
  double alpha, beta;
};

__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n"
      ::"r"(dst), "l"((uint64_t)map), "r"(bar), "r"(c0), "r"(c1) : "memory");
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(T_THREADS_G, 1) gemm_task_tma_kernel(const __grid_constant__ GemmTmaTask t) {
  extern __shared__ __align__(1024) uint8_t t_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)t_raw + 1023) & ~(uintptr_t)1023);   // 128-B swizzle atoms
  uint64_t* full = (uint64_t*)(smem + T_STAGES * T_STAGE_BYTES);
  uint64_t* empty = full + T_STAGES;
  constexpr int MF = T_WM / 8, NF = T_WN / 8, KQ = T_BK / 4, WARPS = T_THREADS_G / 32;
  constexpr int WARPS_M = T_BM / T_WM;

  const int tiles_m = (t.h + T_BM - 1) / T_BM, tiles_n = (t.w + T_BN - 1) / T_BN;
  const int bid = blockIdx.x;
  const int per_group = t.group_m * tiles_n;
  const int first_m = (bid / per_group) * t.group_m;
  const int gsize = min(tiles_m - first_m, t.group_m);
  const int m0 = (first_m + (bid % per_group) % gsize) * T_BM;
  const int n0 = ((bid % per_group) / gsize) * T_BN;
  if (t.tri == TRI_LOWER && n0 >= m0 + T_BM) return;
  if (t.tri == TRI_UPPER && m0 >= n0 + T_BN) return;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int total = 0;
  for (int s = 0; s < t.nsteps; ++s) total += (t.steps[s].d + T_BK - 1) / T_BK;
  if (tid == 0) {
    for (int s = 0; s < T_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const uint32_t sbase = smem_u32(smem);
  int ld_step = 0, ld_k = 0, ld_d = t.nsteps > 0 ? t.steps[0].d : 0;
  auto produce = [&](int slab) {
    const int stage = slab % T_STAGES;
    if (slab >= T_STAGES) mbar_wait(&empty[stage], ((slab / T_STAGES) - 1) & 1);
    const uint32_t sa = sbase + stage * T_STAGE_BYTES, sb = sa + T_A_BYTES;
    const uint32_t bar = smem_u32(&full[stage]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(T_STAGE_BYTES) : "memory");
    const GemmTmaStep& st = t.steps[ld_step];
    if (TA) {
      tma2d(sa, &st.ma, bar, ld_k, m0);                    // A stored K x M: one K-major box
    } else {
#pragma unroll
      for (int g = 0; g < T_BM / 16; ++g) tma2d(sa + g * 2048, &st.ma, bar, m0 + 16 * g, ld_k);
    }
    if (!TB) {
      tma2d(sb, &st.mb, bar, ld_k, n0);                    // B stored K x N: one K-major box
    } else {
#pragma unroll
      for (int g = 0; g < T_BN / 16; ++g) tma2d(sb + g * 2048, &st.mb, bar, n0 + 16 * g, ld_k);
    }
    ld_k += T_BK;
    if (ld_k >= ld_d) {
      ld_k = 0;
      if (++ld_step < t.nsteps) ld_d = t.steps[ld_step].d;
    }
  };
  if (tid == 0)
    for (int s = 0; s < T_DIST && s < total; ++s) produce(s);

  const int wm = (warp % WARPS_M) * T_WM, wn = (warp / WARPS_M) * T_WN;
  const int g = lane >> 2, q = lane & 3;
  // per-lane swizzled byte offsets of the fragment loads (see the layout notes above)
  //   K-major  (row = mn, 16-B chunk = k/2):   mn*128 + ((k/2) ^ (mn%8))*16 + (k%2)*8
  //   MN-major (box per 16 mn, row = k):       (mn/16)*2048 + k*128 + (((mn%16)/2) ^ (k%8))*16 + (mn%2)*8
  uint32_t kmaj[KQ], mnmaj[4];
#pragma unroll
  for (int kq = 0; kq < KQ; ++kq) kmaj[kq] = (((2 * kq + (q >> 1)) ^ g) << 4) + (q & 1) * 8;
#pragma unroll
  for (int ih = 0; ih < 2; ++ih)
#pragma unroll
    for (int kh = 0; kh < 2; ++kh)
      mnmaj[ih * 2 + kh] = ((((ih * 4 + (g >> 1)) ^ (kh * 4 + q)) << 4) + (g & 1) * 8 + q * 128);
  auto fa = [&](const uint8_t* a, int i, int kq) -> double {
    const int mn = wm + i * 8;
    if (TA) return *(const double*)(a + (mn + g) * 128 + kmaj[kq]);
    return *(const double*)(a + (mn >> 4) * 2048 + kq * 512 + mnmaj[(i & 1) * 2 + (kq & 1)]);
  };
  auto fb = [&](const uint8_t* b, int j, int kq) -> double {
    const int mn = wn + j * 8;
    if (!TB) return *(const double*)(b + (mn + g) * 128 + kmaj[kq]);
    return *(const double*)(b + (mn >> 4) * 2048 + kq * 512 + mnmaj[(j & 1) * 2 + (kq & 1)]);
  };

  double acc[MF][NF][2];
#pragma unroll
  for (int i = 0; i < MF; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double ra[2][MF], rb[2][NF];
  if (total > 0) {
    mbar_wait(&full[0], 0);
#pragma unroll
    for (int i = 0; i < MF; ++i) ra[0][i] = fa(smem, i, 0);
#pragma unroll
    for (int j = 0; j < NF; ++j) rb[0][j] = fb(smem + T_A_BYTES, j, 0);
  }
  for (int it = 0; it < total; ++it) {
    if (tid == 0 && it + T_DIST < total) produce(it + T_DIST);
    const int stage = it % T_STAGES;
    const uint8_t* a = smem + stage * T_STAGE_BYTES;
    const uint8_t* b = a + T_A_BYTES;
#pragma unroll
    for (int kq = 0; kq < KQ; ++kq) {
      const int cur = kq & 1, nx = cur ^ 1;
      if (kq + 1 < KQ) {
#pragma unroll
        for (int i = 0; i < MF; ++i) ra[nx][i] = fa(a, i, kq + 1);
#pragma unroll
        for (int j = 0; j < NF; ++j) rb[nx][j] = fb(b, j, kq + 1);
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);   // this warp is done reading the stage
        if (it + 1 < total) {
          const int ns = (it + 1) % T_STAGES;
          mbar_wait(&full[ns], ((it + 1) / T_STAGES) & 1);
          const uint8_t* a2 = smem + ns * T_STAGE_BYTES;
          const uint8_t* b2 = a2 + T_A_BYTES;
#pragma unroll
          for (int i = 0; i < MF; ++i) ra[nx][i] = fa(a2, i, 0);
#pragma unroll
          for (int j = 0; j < NF; ++j) rb[nx][j] = fb(b2, j, 0);
        }
      }
#pragma unroll
      for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int jj = 0; jj < NF; ++jj) {
          const int j = (i & 1) ? NF - 1 - jj : jj;
          dmma(acc[i][j], ra[cur][i], rb[cur][j]);
        }
    }
  }

  // epilogue, one fragment row i at a time: with beta != 0 its NF x 2 C loads are all
  // issued before the first store (one memory round trip per row instead of 2 NF
  // dependent ones — the epilogue of a short launch with beta = 1 is otherwise a few % of it)
  const double alpha = t.alpha, beta = t.beta;
#pragma unroll
  for (int i = 0; i < MF; ++i) {
    const int r = m0 + wm + i * 8 + g;
    if (r >= t.h) continue;
    double cv[NF][2];
    bool ok[NF][2];
#pragma unroll
    for (int j = 0; j < NF; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cc = n0 + wn + j * 8 + 2 * q + e;
        ok[j][e] = cc < t.w && !(t.tri == TRI_LOWER && cc > r) && !(t.tri == TRI_UPPER && cc < r);
        cv[j][e] = (beta != 0.0 && ok[j][e]) ? t.c[(size_t)cc * t.ldc + r] : 0.0;
      }
    }
#pragma unroll
    for (int j = 0; j < NF; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (!ok[j][e]) continue;
        const int cc = n0 + wn + j * 8 + 2 * q + e;
        double v = alpha * acc[i][j][e];
        if (beta != 0.0) v = fma(beta, cv[j][e], v);
        t.c[(size_t)cc * t.ldc + r] = v;
      }
    }
  }
}

}  // namespace bx
