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
    for (int idx = tid; idx < T_BLK * T_BLK; idx += T_THREADS) {
      int j = idx / T_BLK, r = idx % T_BLK;
      double v = 0.0;
      if (r < nb && j < nb && r >= j && !(t.unit && r == j)) v = trsm_L(t, i0 + r, i0 + j);
      ls[j * (T_BLK + 1) + r] = v;
    }
    __syncthreads();
    {
      // substitution on the diagonal block: warp -> RHS, lane -> row
      const int r = lane;
      double y = (r < nb) ? ys[(i0 + r) * T_YP + warp] : 0.0;
      for (int j = 0; j < nb; ++j) {
        if (r == j && !t.unit) {
          double dd = ls[j * (T_BLK + 1) + j];
          if (dd == 0.0) atomicOr(t.flag, 1);
          y = y / dd;
        }
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

__global__ void scale_kernel(double* __restrict__ b, int ld, int h, int w, double alpha) {
  int r = blockIdx.x * 32 + threadIdx.x;
  int c = blockIdx.y * 8 + threadIdx.y;
  if (r < h && c < w) b[(size_t)c * ld + r] *= alpha;
}

}  // namespace bx
