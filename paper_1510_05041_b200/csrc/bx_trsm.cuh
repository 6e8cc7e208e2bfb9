// FP64 triangular-solve tile kernel (the diagonal step of a TRSM task,
// reference: /root/reference/pkg/src/tileblas/kernels.py:105-161).
//
// All (side, uplo, trans) variants are reduced to ONE forward substitution on a
// logical lower-triangular L through an index map (the §III.C transpose trick applied
// to the solve):
//     E = op(A);  left:  E X = alpha B        right: X E = alpha B  <=>  E^T X^T = alpha B^T
//     swap = trans ^ right      (L(i,j) reads A(j,i) instead of A(i,j))
//     rev  = left ? eff_upper : !eff_upper     (backward substitution = forward on n-1-i)
// Each CTA owns 8 right-hand sides (columns of B for left, rows for right) for the whole
// triangle order n, holds them in shared memory, and walks the diagonal in 32-row
// blocks: substitution on the 32x32 diagonal block (one warp per RHS, division by the
// diagonal exactly like the reference; unit diagonal never read), then the trailing
// rows are updated with DMMA (m8n8k4 f64) against the solved block.  alpha is applied
// once, on load (kernels.py:124-125).  An exact zero on a non-unit diagonal sets the
// device-visible singular flag (kernels.py:105-109) -> SingularMatrixError on the host.
#pragma once
#include <cuda_runtime.h>

namespace bx {

constexpr int T_NRHS = 8, T_BLK = 32, T_THREADS = 256, T_YP = 12, T_NMAX = 2048;

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

__global__ void __launch_bounds__(T_THREADS) trsm_panel_kernel(const __grid_constant__ TrsmArgs t) {
  extern __shared__ __align__(16) double ys[];      // [n][T_YP]
  __shared__ double ls[T_BLK * (T_BLK + 1)];         // ls[j*(33)+r] = L(i0+r, i0+j)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int col0 = blockIdx.x * T_NRHS;
  const int n = t.n;

  for (int idx = tid; idx < n * T_NRHS; idx += T_THREADS) {
    int c = t.right ? idx % T_NRHS : idx / n;
    int i = t.right ? idx / T_NRHS : idx % n;
    int col = col0 + c;
    ys[i * T_YP + c] = (col < t.nrhs) ? t.alpha * *trsm_Y(t, i, col) : 0.0;
  }
  __syncthreads();

  const int g = lane >> 2, q = lane & 3;
  for (int i0 = 0; i0 < n; i0 += T_BLK) {
    const int nb = min(T_BLK, n - i0);
    {
      double v[T_BLK * T_BLK / T_THREADS];
#pragma unroll
      for (int q = 0; q < T_BLK * T_BLK / T_THREADS; ++q) {
        const int idx = tid + q * T_THREADS, j = idx / T_BLK, r = idx % T_BLK;
        v[q] = (r < nb && j < nb && r >= j && !(t.unit && r == j)) ? trsm_L(t, i0 + r, i0 + j) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < T_BLK * T_BLK / T_THREADS; ++q) {
        const int idx = tid + q * T_THREADS;
        ls[(idx / T_BLK) * (T_BLK + 1) + idx % T_BLK] = v[q];
      }
    }
    __syncthreads();
    {
      // substitution on the diagonal block: warp -> RHS, lane -> row
      const int r = lane;
      double y = (r < nb) ? ys[(i0 + r) * T_YP + warp] : 0.0;
      double inv = 1.0;
      if (!t.unit && r < nb) {
        const double dd = ls[r * (T_BLK + 1) + r];
        if (dd == 0.0) atomicOr(t.flag, 1);
        inv = 1.0 / dd;
      }
      for (int j = 0; j < nb; ++j) {
        if (r == j && !t.unit) y *= inv;
        double x = __shfl_sync(0xffffffffu, y, j);
        if (r > j) y = y - ls[j * (T_BLK + 1) + r] * x;
      }
      if (r < nb) ys[(i0 + r) * T_YP + warp] = y;
    }
    __syncthreads();
    // trailing update: Y[r] -= L(r, i0:i0+nb) * Y(i0:i0+nb) for r >= i0+nb (DMMA m8n8k4)
    const int rbeg = i0 + nb;
    const int nfr = (n - rbeg + 7) / 8;
    for (int f = warp; f < nfr; f += T_THREADS / 32) {
      const int r0 = rbeg + f * 8;
      const int row = r0 + g;
      double acc[2] = {0.0, 0.0};
#pragma unroll 4
      for (int kk = 0; kk < T_BLK; kk += 4) {
        const int j = kk + q;
        double av = (row < n && j < nb) ? trsm_L(t, row, i0 + j) : 0.0;
        double bv = (j < nb) ? ys[(i0 + j) * T_YP + g] : 0.0;
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[0]), "+d"(acc[1]) : "d"(av), "d"(bv));
      }
      if (row < n) {
        ys[row * T_YP + 2 * q] -= acc[0];
        ys[row * T_YP + 2 * q + 1] -= acc[1];
      }
    }
    __syncthreads();
  }

  for (int idx = tid; idx < n * T_NRHS; idx += T_THREADS) {
    int c = t.right ? idx % T_NRHS : idx / n;
    int i = t.right ? idx / T_NRHS : idx % n;
    int col = col0 + c;
    if (col < t.nrhs) *trsm_Y(t, i, col) = ys[i * T_YP + c];
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
