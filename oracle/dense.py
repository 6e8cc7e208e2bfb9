"""Whole-matrix references (TEST INFRASTRUCTURE) — restates
/root/reference/pkg/src/tileblas/oracle.py:46-111 (numpy / scipy)."""

from __future__ import annotations

import numpy as np
import scipy.linalg

from .tiled import sym_of, tri_of


def _op(a, t):
    return a.T if t else a


def _tri_update(c, full, uplo):
    # oracle.py:52-57
    out = c.copy()
    r, cc = np.triu_indices(c.shape[0]) if uplo == "upper" else np.tril_indices(c.shape[0])
    out[r, cc] = full[r, cc]
    return out


def dense_reference(kind, *, a, b=None, c=None, alpha=1.0, beta=0.0, trans_a=False,
                    trans_b=False, uplo="upper", side="left", diag="non-unit"):
    # oracle.py:95-111
    if kind == "gemm":        # oracle.py:46-48
        return alpha * (_op(a, trans_a) @ _op(b, trans_b)) + beta * c
    if kind == "syrk":        # oracle.py:60-63
        aa = _op(a, trans_a)
        return _tri_update(c, alpha * (aa @ aa.T) + beta * c, uplo)
    if kind == "syr2k":       # oracle.py:66-70
        aa, bb = _op(a, trans_a), _op(b, trans_a)
        return _tri_update(c, alpha * (aa @ bb.T + bb @ aa.T) + beta * c, uplo)
    if kind == "symm":        # oracle.py:73-76
        s = sym_of(a, uplo)
        return alpha * (s @ b if side == "left" else b @ s) + beta * c
    if kind == "trmm":        # oracle.py:79-82 (in place on c)
        m, _ = tri_of(a, uplo, diag, trans_a)
        return alpha * (m @ c if side == "left" else c @ m)
    if kind == "trsm":        # oracle.py:85-92
        m, eff_upper = tri_of(a, uplo, diag, trans_a)
        rhs = alpha * c
        if side == "left":
            return scipy.linalg.solve_triangular(m, rhs, lower=not eff_upper,
                                                 unit_diagonal=(diag == "unit"))
        return scipy.linalg.solve_triangular(m.T, rhs.T, lower=eff_upper,
                                             unit_diagonal=(diag == "unit")).T
    raise ValueError(kind)
