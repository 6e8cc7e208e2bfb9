"""North-star normwise parity bounds (TEST INFRASTRUCTURE).

BASELINE.json ``north_star``:
  GEMM-type:  ||C - C_ref||_F / (|alpha|*||A||_F*||B||_F*k*eps + |beta|*||C0||_F*eps) <= 10
  TRSM:       the same bound on the residual,
              ||op(tri(A)) X - alpha*B0||_F / ((||tri(A)||_F*||X||_F*m + |alpha|*||B0||_F)*eps) <= 10
              (SURVEY.md §8c), plus the GEMM-type bound between X and X_ref.
eps = numpy.finfo(dtype).eps of the arithmetic type (2^-52 for f64, 2^-23 for f32).
"""

from __future__ import annotations

import numpy as np

BOUND = 10.0


def gemm_ratio(c, c_ref, *, a_norm, b_norm, k, alpha, beta, c0_norm, eps):
    """Ratio of ||C - C_ref||_F to the north-star scale; parity iff <= BOUND."""
    num = float(np.linalg.norm(np.asarray(c, np.float64) - np.asarray(c_ref, np.float64)))
    den = abs(alpha) * a_norm * b_norm * k * eps + abs(beta) * c0_norm * eps
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return num / den


def trsm_residual_ratio(tri_a, x, b0, alpha, side, eps):
    """Residual bound for op(tri(A)) X = alpha B (left) / X op(tri(A)) = alpha B (right);
    ``tri_a`` is the materialised op(tri(A)) (unit diagonal already substituted)."""
    r = tri_a @ x - alpha * b0 if side == "left" else x @ tri_a - alpha * b0
    m = tri_a.shape[0]
    den = (np.linalg.norm(tri_a) * np.linalg.norm(x) * m + abs(alpha) * np.linalg.norm(b0)) * eps
    return float(np.linalg.norm(r) / den) if den else 0.0


def routine_ratio(kind, out, ref, *, a, b, c0, alpha, beta, k, eps):
    """Dispatch the GEMM-type bound with the operand norms each routine implies.

    syrk: ||A||·||A||; syr2k: 2·||A||·||B||; symm/trmm/gemm: ||A||·||B||
    (for trmm/trsm B is the input c0)."""
    an = float(np.linalg.norm(a))
    if kind == "syrk":
        bn = an
    elif kind == "syr2k":
        bn = 2.0 * float(np.linalg.norm(b))
    elif kind in ("trmm", "trsm"):
        bn = float(np.linalg.norm(c0))
    else:
        bn = float(np.linalg.norm(b))
    c0n = 0.0 if kind in ("trmm", "trsm") else float(np.linalg.norm(c0))
    return gemm_ratio(out, ref, a_norm=an, b_norm=bn, k=k, alpha=alpha,
                      beta=beta, c0_norm=c0n, eps=eps)
