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
// into shared memory with 16-B cp.async (zero-filled past the tile edge), in one of two
// layouts per operand so both layouts are bank-conflict free for the DMMA fragment
// loads:  "MN-major" sX[k][mn] (row pitch 132) when mn is the contiguous direction
// in global memory, "K-major" sX[mn][k] (row pitch 20) when k is.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bx {

constexpr int G_BM = 128, G_BN = 128, G_BK = 16, G_STAGES = 4, G_THREADS = 256;
constexpr int G_LD_MN = G_BM + 4;   // 132 doubles: conflict-free frag loads (132 = 4 mod 16)
constexpr int G_LD_K = G_BK + 4;    // 20 doubles
constexpr int G_STAGE_ELEMS = (G_BK * G_LD_MN > G_BM * G_LD_K) ? G_BK * G_LD_MN : G_BM * G_LD_K;
constexpr int G_SMEM_BYTES = G_STAGES * 2 * G_STAGE_ELEMS * 8;
constexpr int G_MAX_STEPS = 40;

enum TriMode { TRI_NONE = 0, TRI_LOWER = 1, TRI_UPPER = 2 };

struct GemmStep {
  const double* a;
  const double* b;
  int lda, ldb, d, pad_;
};

struct GemmTask {
  double* c;
  int ldc, h, w, nsteps, tri, group_m;
  double alpha, beta;
  GemmStep steps[G_MAX_STEPS];
};

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

// Stage one BK-deep slab of op(A) rows [m0, m0+128) (TA: A stored transposed) or
// op(B) cols [n0, n0+128) into shared memory.  `mn_ext` is the tile extent along mn
// (h for A, w for B), `d` the step depth, `k0` the slab start within the step.
// KCONTIG: k is the contiguous direction in global memory -> K-major smem.
template <bool KCONTIG>
__device__ __forceinline__ void load_slab(double* s, const double* g, int ld, int mn0, int mn_ext,
                                          int k0, int d, int tid) {
#pragma unroll
  for (int c = 0; c < (G_BM * G_BK / 2) / G_THREADS; ++c) {
    int idx = tid + c * G_THREADS;
    if (KCONTIG) {
      int mn = idx >> 3, k = (idx & 7) * 2;
      int gm = mn0 + mn, gk = k0 + k;
      int valid = (gm < mn_ext) ? min(max(d - gk, 0), 2) : 0;
      const double* src = valid ? g + (size_t)gm * ld + gk : g;
      cp_async16(s + mn * G_LD_K + k, src, valid * 8);
    } else {
      int k = idx >> 6, mn = (idx & 63) * 2;
      int gm = mn0 + mn, gk = k0 + k;
      int valid = (gk < d) ? min(max(mn_ext - gm, 0), 2) : 0;
      const double* src = valid ? g + (size_t)gk * ld + gm : g;
      cp_async16(s + k * G_LD_MN + mn, src, valid * 8);
    }
  }
}

template <bool KMAJ>
__device__ __forceinline__ double frag(const double* s, int mn, int k) {
  return KMAJ ? s[mn * G_LD_K + k] : s[k * G_LD_MN + mn];
}

// TA/TB: operand stored transposed (op = T).  A is MN-contiguous iff !TA; B is
// K-contiguous iff !TB.
template <bool TA, bool TB>
__global__ void __launch_bounds__(G_THREADS, 1) gemm_task_kernel(const __grid_constant__ GemmTask t) {
  extern __shared__ __align__(128) double smem[];
  constexpr bool A_KMAJ = TA;    // A: (m,k) at a[k + m*lda] when TA -> k contiguous
  constexpr bool B_KMAJ = !TB;   // B: (k,n) at b[k + n*ldb] when !TB -> k contiguous

  // grouped rasterisation of a 1-D grid (L2 reuse when one launch spans many tiles)
  const int tiles_m = (t.h + G_BM - 1) / G_BM, tiles_n = (t.w + G_BN - 1) / G_BN;
  int bid = blockIdx.x;
  int gm = t.group_m;
  int per_group = gm * tiles_n;
  int group = bid / per_group;
  int first_m = group * gm;
  int gsize = min(tiles_m - first_m, gm);
  int bm = first_m + (bid % per_group) % gsize;
  int bn = (bid % per_group) / gsize;
  const int m0 = bm * G_BM, n0 = bn * G_BN;
  if (t.tri == TRI_LOWER && n0 >= m0 + G_BM) return;   // wholly above the diagonal
  if (t.tri == TRI_UPPER && m0 >= n0 + G_BN) return;   // wholly below

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 64, wn = (warp >> 1) * 32;
  const int g = lane >> 2, q = lane & 3;

  // total number of BK slabs over all steps
  int total = 0;
  for (int s = 0; s < t.nsteps; ++s) total += (t.steps[s].d + G_BK - 1) / G_BK;

  double* sA = smem;
  double* sB = smem + G_STAGES * G_STAGE_ELEMS;

  int ld_step = 0, ld_k = 0;   // producer cursor
  auto issue = [&](int stage) {
    const GemmStep& st = t.steps[ld_step];
    load_slab<A_KMAJ>(sA + stage * G_STAGE_ELEMS, st.a, st.lda, m0, t.h, ld_k, st.d, tid);
    load_slab<B_KMAJ>(sB + stage * G_STAGE_ELEMS, st.b, st.ldb, n0, t.w, ld_k, st.d, tid);
    ld_k += G_BK;
    if (ld_k >= st.d) { ld_k = 0; ++ld_step; }
  };

#pragma unroll
  for (int s = 0; s < G_STAGES - 1; ++s) {
    if (s < total) issue(s);
    cp_async_commit();
  }

  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int it = 0; it < total; ++it) {
    cp_async_wait<G_STAGES - 2>();
    __syncthreads();
    {
      int nxt = it + G_STAGES - 1;
      if (nxt < total) issue(nxt % G_STAGES);
      cp_async_commit();
    }
    const double* a = sA + (it % G_STAGES) * G_STAGE_ELEMS;
    const double* b = sB + (it % G_STAGES) * G_STAGE_ELEMS;
    double fa[2][8], fb[2][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) fa[0][i] = frag<A_KMAJ>(a, wm + i * 8 + g, q);
#pragma unroll
    for (int j = 0; j < 4; ++j) fb[0][j] = frag<B_KMAJ>(b, wn + j * 8 + g, q);
#pragma unroll
    for (int kq = 0; kq < G_BK / 4; ++kq) {
      const int cur = kq & 1, nx = cur ^ 1;
      if (kq + 1 < G_BK / 4) {
#pragma unroll
        for (int i = 0; i < 8; ++i) fa[nx][i] = frag<A_KMAJ>(a, wm + i * 8 + g, (kq + 1) * 4 + q);
#pragma unroll
        for (int j = 0; j < 4; ++j) fb[nx][j] = frag<B_KMAJ>(b, wn + j * 8 + g, (kq + 1) * 4 + q);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], fa[cur][i], fb[cur][j]);
    }
  }
  cp_async_wait<0>();

  // epilogue: C = alpha*acc + beta*C  (beta == 0: C never read)
  const double alpha = t.alpha, beta = t.beta;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = m0 + wm + i * 8 + g;
    if (r >= t.h) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cc = n0 + wn + j * 8 + 2 * q + e;
        if (cc >= t.w) continue;
        if (t.tri == TRI_LOWER && cc > r) continue;
        if (t.tri == TRI_UPPER && cc < r) continue;
        double* p = t.c + (size_t)cc * t.ldc + r;
        double v = alpha * acc[i][j][e];
        if (beta != 0.0) v = fma(beta, *p, v);
        *p = v;
      }
    }
  }
}

}  // namespace bx
