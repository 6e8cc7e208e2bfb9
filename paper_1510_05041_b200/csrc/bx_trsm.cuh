// FP64 triangular-solve tile kernel (the diagonal step of a TRSM task,
// reference: /root/reference/pkg/src/tileblas/kernels.py:105-161).
//
// All (side, uplo, trans) variants are reduced to ONE forward substitution on a
// logical lower-triangular L through an index map (the §III.C transpose trick applied
// to the solve):
//     E = op(A);  left:  E X = alpha B        right: X E = alpha B  <=>  E^T X^T = alpha B^T
//     swap = trans ^ right      (L(i,j) reads A(j,i) instead of A(i,j))
//     rev  = left ? eff_upper : !eff_upper     (backward substitution = forward on n-1-i)
// Each CTA owns NR (8/16/32) right-hand sides (columns of B for left, rows for right) for
// the whole triangle order n, holds them in shared memory, and walks the diagonal in
// 32-row blocks: substitution on the 32x32 diagonal block (warps over RHS, division by
// the diagonal exactly like the reference; unit diagonal never read), then the trailing
// rows are updated with DMMA (m8n8k4 f64) against the solved block.  alpha is applied
// once, on load (kernels.py:124-125).  An exact zero on a non-unit diagonal sets the
// device-visible singular flag (kernels.py:105-109) -> SingularMatrixError on the host.
#pragma once
#include <cuda_runtime.h>

namespace bx {

constexpr int T_BLK = 32, T_THREADS = 256, T_NMAX = 2048;

struct TrsmArgs {
  const double* a;
  double* b;
  int lda, ldb, n, nrhs;
  int swap, rev, right, unit;
  double alpha;
  int* flag;
};

__device__ __forceinline__ double trsm_L(const TrsmArgs& t, int i, int j) {
  int ii = t.rev ? t.n - 1 - i : i, jj = t.rev ? t.n - 1 - j : j;
  int r = t.swap ? jj : ii, c = t.swap ? ii : jj;
  return t.a[(size_t)c * t.lda + r];
}
__device__ __forceinline__ double* trsm_Y(const TrsmArgs& t, int i, int col) {
  int ii = t.rev ? t.n - 1 - i : i;
  return t.right ? t.b + (size_t)ii * t.ldb + col : t.b + (size_t)col * t.ldb + ii;
}

// Y row pitch for NR right-hand sides: NR + 4 doubles (== 4 mod 16) keeps the DMMA
// B-fragment reads (4 rows x 8 RHS per half-warp) bank-conflict free.
template <int NR>
struct PanelCfg {
  static constexpr int YP = NR + 4;
  static constexpr int NF = NR / 8;   // 8-wide RHS fragments per DMMA row fragment
};

// NR right-hand sides per CTA.  More RHS per CTA amortise each global load of L in the
// trailing update over NR/8 DMMAs and halve the CTAs (SM time) a solve occupies; the
// substitution phase loops warps over the RHS.
template <int NR>
__global__ void __launch_bounds__(T_THREADS) trsm_panel_kernel(const __grid_constant__ TrsmArgs t) {
  constexpr int YP = PanelCfg<NR>::YP, NF = PanelCfg<NR>::NF;
  extern __shared__ __align__(16) double ys[];      // [n][YP]
  __shared__ double ls[T_BLK * (T_BLK + 1)];         // ls[j*(33)+r] = L(i0+r, i0+j)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int col0 = blockIdx.x * NR;
  const int n = t.n;

  for (int idx = tid; idx < n * NR; idx += T_THREADS) {
    int c = t.right ? idx % NR : idx / n;
    int i = t.right ? idx / NR : idx % n;
    int col = col0 + c;
    ys[i * YP + c] = (col < t.nrhs) ? t.alpha * *trsm_Y(t, i, col) : 0.0;
  }
  __syncthreads();

  const int g = lane >> 2, q = lane & 3;
  // diagonal block i0 is loaded into registers one block step ahead (its global loads
  // overlap the previous step's trailing update) and stored to ls after that step's barrier
  constexpr int DV = T_BLK * T_BLK / T_THREADS;
  double v[DV];
  auto load_diag = [&](int i0) {
    const int nb = min(T_BLK, n - i0);
#pragma unroll
    for (int u = 0; u < DV; ++u) {
      const int idx = tid + u * T_THREADS, j = idx / T_BLK, r = idx % T_BLK;
      v[u] = (r < nb && j < nb && r >= j && !(t.unit && r == j)) ? trsm_L(t, i0 + r, i0 + j) : 0.0;
    }
  };
  load_diag(0);
  for (int i0 = 0; i0 < n; i0 += T_BLK) {
    const int nb = min(T_BLK, n - i0);
#pragma unroll
    for (int u = 0; u < DV; ++u) {
      const int idx = tid + u * T_THREADS;
      ls[(idx / T_BLK) * (T_BLK + 1) + idx % T_BLK] = v[u];
    }
    __syncthreads();
    // Trailing-update operands L(r, i0:i0+nb) do not depend on Y: the first chunk's loads
    // are issued now and land while the substitution below runs.  Row fragments (8 rows)
    // go to warps round-robin, U per warp per chunk, so every warp has work.
    constexpr int U = 4;
    const int rbeg = i0 + nb;
    const int nfr = (n - rbeg + 7) / 8;
    double av[U][T_BLK / 4];
    auto load_frags = [&](int c) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int fr = warp + 8 * (c * U + u);
        const int row = rbeg + fr * 8 + g;
#pragma unroll
        for (int kk = 0; kk < T_BLK / 4; ++kk) {
          const int j = 4 * kk + q;
          av[u][kk] = (fr < nfr && row < n && j < nb) ? trsm_L(t, row, i0 + j) : 0.0;
        }
      }
    };
    load_frags(0);
    {
      // substitution on the diagonal block: warp -> RHS (NR / 8 each), lane -> row; the
      // reference divides by the diagonal (kernels.py:140-159), so do we
      const int r = lane;
      double inv = 1.0;
      if (!t.unit && r < nb) {
        const double dd = ls[r * (T_BLK + 1) + r];
        if (dd == 0.0) atomicOr(t.flag, 1);
        inv = 1.0 / dd;
      }
      double y[NF];
#pragma unroll
      for (int f = 0; f < NF; ++f) y[f] = (r < nb) ? ys[(i0 + r) * YP + warp + 8 * f] : 0.0;
      for (int j = 0; j < nb; ++j) {
        const double l = (r > j) ? ls[j * (T_BLK + 1) + r] : 0.0;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          if (r == j && !t.unit) y[f] *= inv;
          const double x = __shfl_sync(0xffffffffu, y[f], j);
          y[f] = fma(-l, x, y[f]);
        }
      }
#pragma unroll
      for (int f = 0; f < NF; ++f)
        if (r < nb) ys[(i0 + r) * YP + warp + 8 * f] = y[f];
    }
    __syncthreads();
    if (i0 + T_BLK < n) load_diag(i0 + T_BLK);
    // trailing update: Y[r] -= L(r, i0:i0+nb) * Y(i0:i0+nb) for r >= i0+nb (DMMA m8n8k4);
    // one L fragment feeds NF DMMAs, U fragments give 2*U*NF independent accumulators
    for (int c = 0; 8 * c * U < nfr; ++c) {
      if (c > 0) load_frags(c);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int fr = warp + 8 * (c * U + u);
        if (fr >= nfr) break;
        const int row = rbeg + fr * 8 + g;
        double acc[NF][2];
#pragma unroll
        for (int f = 0; f < NF; ++f) acc[f][0] = acc[f][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < T_BLK / 4; ++kk) {
          const int j = 4 * kk + q;
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            const double bv = (j < nb) ? ys[(i0 + j) * YP + 8 * f + g] : 0.0;
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[f][0]), "+d"(acc[f][1]) : "d"(av[u][kk]), "d"(bv));
          }
        }
        if (row < n) {
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            ys[row * YP + 8 * f + 2 * q] -= acc[f][0];
            ys[row * YP + 8 * f + 2 * q + 1] -= acc[f][1];
          }
        }
      }
    }
    __syncthreads();
  }

  for (int idx = tid; idx < n * NR; idx += T_THREADS) {
    int c = t.right ? idx % NR : idx / n;
    int i = t.right ? idx / NR : idx % n;
    int col = col0 + c;
    if (col < t.nrhs) *trsm_Y(t, i, col) = ys[i * YP + c];
  }
}

// ---- small helpers: materialise op(tri(A)) / sym(A) of a diagonal tile, scale --------

// dst = op(tri(A)) (unit diagonal substituted) for TRMM diagonal steps (kernels.py:164-185)
// or sym(A) for SYMM diagonal steps (kernels.py:188-211).  The unstored half of A is
// never read.
__global__ void materialize_kernel(const double* __restrict__ a, int lda, double* __restrict__ dst,
                                   int ldd, int n, int mode_sym, int upper, int trans, int unit) {
  int r = blockIdx.x * 32 + threadIdx.x;
  int c = blockIdx.y * 8 + threadIdx.y;
  if (r >= n || c >= n) return;
  double v;
  if (mode_sym) {
    bool stored = upper ? (r <= c) : (r >= c);
    v = stored ? a[(size_t)c * lda + r] : a[(size_t)r * lda + c];
  } else {
    bool eff_upper = (upper != 0) != (trans != 0);
    bool keep = eff_upper ? (r <= c) : (r >= c);
    if (!keep) v = 0.0;
    else if (unit && r == c) v = 1.0;
    else v = trans ? a[(size_t)r * lda + c] : a[(size_t)c * lda + r];
  }
  dst[(size_t)c * ldd + r] = v;
}

template <typename T>
__global__ void axpy_tile_kernel(T* __restrict__ dst, int ldd, const T* __restrict__ src, int lds, int h, int w,
                                 T beta) {
  const int r = blockIdx.x * 32 + threadIdx.x;
  const int c = blockIdx.y * 8 + threadIdx.y;
  if (r < h && c < w) dst[(size_t)c * ldd + r] += beta * src[(size_t)c * lds + r];
}

__global__ void scale_kernel(double* __restrict__ b, int ld, int h, int w, double alpha) {
  int r = blockIdx.x * 32 + threadIdx.x;
  int c = blockIdx.y * 8 + threadIdx.y;
  if (r < h && c < w) b[(size_t)c * ld + r] *= alpha;
}

// ---------------------------------------------------------------------------------------
// Leaf solve for triangle order n <= 64 with many right-hand sides per warp.
// Lane r of a warp owns logical rows r and r + 32 for LEAF_RHS right-hand sides held in
// registers; the diagonal is walked column by column (right-looking substitution):
// the owner lane divides its LEAF_RHS values by L(j,j) (independent divisions -> ILP),
// the solved row is broadcast with shuffles and every lane below updates its rows with
// one FMA per right-hand side.  Warps are independent (no CTA barrier after staging L),
// so per-SM throughput scales with LEAF_RHS instead of being bound by the serial
// division/shuffle latency of one right-hand side.
// ---------------------------------------------------------------------------------------
constexpr int LEAF_RHS = 16, LEAF_WARPS = 8, LEAF_N = 64;

__global__ void __launch_bounds__(LEAF_WARPS * 32) trsm_leaf_kernel(const __grid_constant__ TrsmArgs t) {
  __shared__ double ls[LEAF_N * (LEAF_N + 1)];   // ls[j*65 + r] = L(r, j)
  const int n = t.n;
  {
    // all loads in flight before the first store (one round trip, not n*n/256)
    constexpr int PER = LEAF_N * LEAF_N / (LEAF_WARPS * 32);
    double v[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int idx = threadIdx.x + q * LEAF_WARPS * 32;
      const int j = idx / LEAF_N, r = idx % LEAF_N;
      v[q] = (r < n && j < n && r >= j && !(t.unit && r == j)) ? trsm_L(t, r, j) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int idx = threadIdx.x + q * LEAF_WARPS * 32;
      ls[(idx / LEAF_N) * (LEAF_N + 1) + idx % LEAF_N] = v[q];
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col0 = (blockIdx.x * LEAF_WARPS + warp) * LEAF_RHS;
  if (col0 >= t.nrhs) return;
  const int r0 = lane, r1 = lane + 32;
  double y0[LEAF_RHS], y1[LEAF_RHS];
#pragma unroll
  for (int c = 0; c < LEAF_RHS; ++c) {
    const int col = col0 + c;
    const bool cv = col < t.nrhs;
    y0[c] = (cv && r0 < n) ? t.alpha * *trsm_Y(t, r0, col) : 0.0;
    y1[c] = (cv && r1 < n) ? t.alpha * *trsm_Y(t, r1, col) : 0.0;
  }
  // reciprocals of the diagonal, computed once per lane off the critical path (a division
  // per solved row per RHS on one lane serialises the whole warp)
  double inv0 = 1.0, inv1 = 1.0;
  if (!t.unit) {
    if (r0 < n) {
      const double d = ls[r0 * (LEAF_N + 1) + r0];
      if (d == 0.0) atomicOr(t.flag, 1);
      inv0 = 1.0 / d;
    }
    if (r1 < n) {
      const double d = ls[r1 * (LEAF_N + 1) + r1];
      if (d == 0.0) atomicOr(t.flag, 1);
      inv1 = 1.0 / d;
    }
  }
  // Branch-free column sweep: the owner lane scales its row by 1/L(j,j) (other lanes
  // multiply by 1), broadcasts it, and every lane subtracts L(r,j) x_j (0 above the
  // diagonal).  Rows 0..31 and 32..63 are separate sweeps so no per-element selects remain.
  const bool nonunit = !t.unit;
  for (int j = 0; j < n && j < 32; ++j) {
    const double sc = (nonunit && lane == j) ? inv0 : 1.0;
    const double l0 = (lane > j) ? ls[j * (LEAF_N + 1) + r0] : 0.0;
    const double l1 = (r1 < n) ? ls[j * (LEAF_N + 1) + r1] : 0.0;
#pragma unroll
    for (int c = 0; c < LEAF_RHS; ++c) {
      y0[c] *= sc;
      const double x = __shfl_sync(0xffffffffu, y0[c], j);
      y0[c] = fma(-l0, x, y0[c]);
      y1[c] = fma(-l1, x, y1[c]);
    }
  }
  for (int j = 32; j < n; ++j) {
    const int owner = j - 32;
    const double sc = (nonunit && lane == owner) ? inv1 : 1.0;
    const double l1 = (lane > owner && r1 < n) ? ls[j * (LEAF_N + 1) + r1] : 0.0;
#pragma unroll
    for (int c = 0; c < LEAF_RHS; ++c) {
      y1[c] *= sc;
      const double x = __shfl_sync(0xffffffffu, y1[c], owner);
      y1[c] = fma(-l1, x, y1[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < LEAF_RHS; ++c) {
    const int col = col0 + c;
    if (col < t.nrhs) {
      if (r0 < n) *trsm_Y(t, r0, col) = y0[c];
      if (r1 < n) *trsm_Y(t, r1, col) = y1[c];
    }
  }
}

}  // namespace bx
