"""numpy restatement of the reference tiled runtime's numerics (TEST INFRASTRUCTURE).

Every function cites the reference code it restates (paths relative to
``/root/reference/pkg/src/tileblas``).  Inputs/outputs are plain 2-d float64
arrays; ``run_tiled`` mutates ``c`` in place exactly as ``run_call`` does
(``scheduler.py:665-669`` — output written into the caller's storage).

The tiled order matters for floating point: each output tile is computed by the
same step sequence as the reference planner (beta once at step 0, k ascending,
``routines.py:1-22``), so the oracle's rounding follows the reference's.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg


class OracleSingular(Exception):
    """Exact zero on a non-unit diagonal (kernels.py:105-109)."""


# --------------------------------------------------------------------------
# tile kernels (kernels.py)
# --------------------------------------------------------------------------

def _op(a, trans):
    return a.T if trans else a


def _accumulate(c, update, beta):
    # kernels.py:39-46: beta == 0 overwrites without reading c
    if beta == 0.0:
        c[:, :] = update
    elif beta == 1.0:
        c += update
    else:
        c *= beta
        c += update


def gemm_update(c, a, b, alpha, beta, ta=False, tb=False):
    # kernels.py:49-58
    _accumulate(c, alpha * (_op(a, ta) @ _op(b, tb)), beta)


def _tri_mask(n, uplo):
    return np.triu(np.ones((n, n), bool)) if uplo == "upper" else np.tril(np.ones((n, n), bool))


def syrk_update(c, a, alpha, beta, uplo, ta=False):
    # kernels.py:67-84: only the stored triangle is read/written
    aa = _op(a, ta)
    m = _tri_mask(c.shape[0], uplo)
    full = alpha * (aa @ aa.T)
    c[m] = full[m] if beta == 0.0 else beta * c[m] + full[m]


def syr2k_update(c, a, b, alpha, beta, uplo, ta=False, tb=False):
    # kernels.py:87-102
    aa, bb = _op(a, ta), _op(b, tb)
    m = _tri_mask(c.shape[0], uplo)
    full = alpha * (aa @ bb.T + bb @ aa.T)
    c[m] = full[m] if beta == 0.0 else beta * c[m] + full[m]


def tri_of(a, uplo, diag, ta):
    # kernels.py:164-170 (_masked_triangle)
    e = _op(a, ta)
    eff_upper = (uplo == "upper") != ta
    m = np.triu(e) if eff_upper else np.tril(e)
    if diag == "unit":
        m = m.copy()
        np.fill_diagonal(m, 1.0)
    return m, eff_upper


def sym_of(a, uplo):
    # kernels.py:188-195 (_symmetrized): unstored half never read
    if uplo == "upper":
        return np.triu(a) + np.triu(a, 1).T
    return np.tril(a) + np.tril(a, -1).T


def trsm_solve(b, a, alpha, uplo, diag, side="left", ta=False):
    # kernels.py:112-161: in-place substitution, alpha applied once, singular iff an
    # exact zero on a non-unit diagonal; unit diagonal never read.
    m, eff_upper = tri_of(a, uplo, diag, ta)
    if diag != "unit" and np.any(np.diagonal(m) == 0.0):
        raise OracleSingular("zero on a non-unit triangular diagonal")
    rhs = alpha * b if alpha != 1.0 else b
    if side == "left":
        x = scipy.linalg.solve_triangular(m, rhs, lower=not eff_upper,
                                          unit_diagonal=(diag == "unit"),
                                          check_finite=False)
    else:
        x = scipy.linalg.solve_triangular(m.T, rhs.T, lower=eff_upper,
                                          unit_diagonal=(diag == "unit"),
                                          check_finite=False).T
    b[:, :] = x


def trmm_diag(c, a, b, alpha, beta, uplo, diag, side="left", ta=False):
    # kernels.py:173-185
    m, _ = tri_of(a, uplo, diag, ta)
    _accumulate(c, alpha * (m @ b if side == "left" else b @ m), beta)


def symm_diag(c, a, b, alpha, beta, uplo, side="left"):
    # kernels.py:198-211
    s = sym_of(a, uplo)
    _accumulate(c, alpha * (s @ b if side == "left" else b @ s), beta)


def step_flops(kind, h, w, d):
    # kernels.py:214-231
    if kind in ("gemm", "symm_diag"):
        return 2 * h * w * d
    if kind == "syrk":
        return h * (h + 1) * d
    if kind == "syr2k":
        return 2 * h * (h + 1) * d
    other = w if d == h else h
    return d * d * other


# --------------------------------------------------------------------------
# tiled execution (routines.py planners + run_plan_on_host)
# --------------------------------------------------------------------------

def _ceil(a, b):
    return -(-a // b)


class _Tiles:
    """Tile views of a 2-d array at tile size t (tiling.py:135-167)."""

    def __init__(self, arr, t):
        self.arr, self.t = arr, t
        self.rows = _ceil(arr.shape[0], t)
        self.cols = _ceil(arr.shape[1], t)

    def phys(self, i, j):
        t = self.t
        return self.arr[i * t:(i + 1) * t, j * t:(j + 1) * t]

    def logical(self, i, j, trans):
        """(view of the physical tile, transposed flag) for logical tile (i,j) of op(X)."""
        return (self.phys(j, i), True) if trans else (self.phys(i, j), False)


def morton(i, j):
    # routines.py:123-132
    key, bit = 0, 0
    while i or j:
        key |= ((j & 1) << (2 * bit)) | ((i & 1) << (2 * bit + 1))
        i >>= 1
        j >>= 1
        bit += 1
    return key


def _tasks_gemm(A, B, C, p):
    # routines.py:227-236
    kt = A.rows if p["trans_a"] else A.cols
    for i in range(C.rows):
        for j in range(C.cols):
            steps = []
            for k in range(kt):
                a, ta = A.logical(i, k, p["trans_a"])
                b, tb = B.logical(k, j, p["trans_b"])
                steps.append(("gemm", a, ta, b, tb))
            yield (i, j), steps


def _tasks_rank(A, B, C, p, two):
    # routines.py:239-276 (syrk / syr2k)
    kt = A.rows if p["trans_a"] else A.cols
    ta = p["trans_a"]
    for i in range(C.rows):
        js = range(i, C.cols) if p["uplo"] == "upper" else range(0, i + 1)
        for j in js:
            steps = []
            for k in range(kt):
                a, fa = A.logical(i, k, ta)
                if i == j:
                    if two:
                        b, fb = B.logical(i, k, ta)
                        steps.append(("syr2k", a, fa, b, fb))
                    else:
                        steps.append(("syrk", a, fa, None, None))
                else:
                    if two:
                        b, fb = B.logical(i, k, ta)
                        bj, fbj = B.logical(j, k, ta)
                        aj, faj = A.logical(j, k, ta)
                        steps.append(("gemm", a, fa, bj, not fbj))
                        steps.append(("gemm", b, fb, aj, not faj))
                    else:
                        aj, faj = A.logical(j, k, ta)
                        steps.append(("gemm", a, fa, aj, not faj))
            yield (i, j), steps


def _sym_part(A, uplo, r, c):
    # routines.py:279-284
    stored = (c > r) if uplo == "upper" else (c < r)
    if stored:
        return A.phys(r, c), False
    return A.phys(c, r), True


def _tasks_symm(A, B, C, p):
    # routines.py:287-313
    for i in range(C.rows):
        for j in range(C.cols):
            steps = []
            for k in range(A.rows):
                if p["side"] == "left":
                    b = B.phys(k, j)
                    if k == i:
                        steps.append(("symm_diag", A.phys(i, i), False, b, False))
                    else:
                        a, fa = _sym_part(A, p["uplo"], i, k)
                        steps.append(("gemm", a, fa, b, False))
                else:
                    a = B.phys(i, k)
                    if k == j:
                        steps.append(("symm_diag", A.phys(j, j), False, a, False))
                    else:
                        s, fs = _sym_part(A, p["uplo"], k, j)
                        steps.append(("gemm", a, False, s, fs))
            yield (i, j), steps


def _eff_upper(p):
    return (p["uplo"] == "upper") != p["trans_a"]


def _tasks_trmm(A, S, C, p):
    # routines.py:320-347 (S = snapshot of the input, routines.py:393-400)
    for i in range(C.rows):
        for j in range(C.cols):
            if p["side"] == "left":
                ks = range(i, A.rows) if _eff_upper(p) else range(0, i + 1)
                dk = i
            else:
                ks = range(0, j + 1) if _eff_upper(p) else range(j, A.rows)
                dk = j
            steps = []
            for k in ks:
                if k == dk:
                    steps.append(("trmm_diag", A.phys(dk, dk), False, S.phys(i, j), False))
                elif p["side"] == "left":
                    a, fa = A.logical(i, k, p["trans_a"])
                    steps.append(("gemm", a, fa, S.phys(k, j), False))
                else:
                    b, fb = A.logical(k, j, p["trans_a"])
                    steps.append(("gemm", S.phys(i, k), False, b, fb))
            yield (i, j), steps


def _trsm_ks(p, i, j, nt):
    # routines.py:350-356
    if p["side"] == "left":
        return range(i + 1, nt) if _eff_upper(p) else range(0, i)
    return range(0, j) if _eff_upper(p) else range(j + 1, nt)


def _trsm_order(C, A, p):
    """Dependency order (routines.py:426-437): a topological order of the DAG."""
    order = []
    if p["side"] == "left":
        rows = range(C.rows - 1, -1, -1) if _eff_upper(p) else range(C.rows)
        for i in rows:
            for j in range(C.cols):
                order.append((i, j))
    else:
        cols = range(C.cols) if _eff_upper(p) else range(C.cols - 1, -1, -1)
        for j in cols:
            for i in range(C.rows):
                order.append((i, j))
    return order


def run_tiled(kind, a, c, b=None, *, tile_size, alpha=1.0, beta=0.0, trans_a=False,
              trans_b=False, uplo="upper", side="left", diag="non-unit"):
    """Execute one routine call tile by tile (routines.py:482-511); c is updated in place.

    Returns the plan's algorithmic flop count (routines.py:439-440)."""
    p = dict(trans_a=trans_a, trans_b=trans_b, uplo=uplo, side=side, diag=diag)
    t = tile_size
    A, C = _Tiles(a, t), _Tiles(c, t)
    B = _Tiles(b, t) if b is not None else None
    flops = 0
    if kind == "trsm":
        nt = A.rows
        for (i, j) in _trsm_order(C, A, p):
            ct = C.phys(i, j)
            first = True
            for k in _trsm_ks(p, i, j, nt):
                beta0 = alpha if first else 1.0
                first = False
                if side == "left":
                    av, fa = A.logical(i, k, trans_a)
                    gemm_update(ct, av, C.phys(k, j), -1.0, beta0, fa, False)
                    flops += 2 * ct.shape[0] * ct.shape[1] * av.shape[0 if fa else 1]
                else:
                    bv, fb = A.logical(k, j, trans_a)
                    xv = C.phys(i, k)
                    gemm_update(ct, xv, bv, -1.0, beta0, False, fb)
                    flops += 2 * ct.shape[0] * ct.shape[1] * xv.shape[1]
            dk = i if side == "left" else j
            dt = A.phys(dk, dk)
            trsm_solve(ct, dt, alpha if first else 1.0, uplo, diag, side, trans_a)
            flops += step_flops("trsm", ct.shape[0], ct.shape[1], dt.shape[0])
        return flops

    if kind == "trmm":
        S = _Tiles(c.copy(), t)
        gen = _tasks_trmm(A, S, C, p)
    elif kind == "gemm":
        gen = _tasks_gemm(A, B, C, p)
    elif kind == "syrk":
        gen = _tasks_rank(A, None, C, p, two=False)
    elif kind == "syr2k":
        gen = _tasks_rank(A, B, C, p, two=True)
    elif kind == "symm":
        gen = _tasks_symm(A, B, C, p)
    else:
        raise ValueError(kind)
    for (i, j), steps in gen:
        ct = C.phys(i, j)
        h, w = ct.shape
        for s_idx, (sk, av, fa, bv, fb) in enumerate(steps):
            if kind == "trmm":
                bt = 0.0 if s_idx == 0 else 1.0    # routines.py:330-332
            else:
                bt = beta if s_idx == 0 else 1.0   # routines.py:211-215
            if sk == "gemm":
                gemm_update(ct, av, bv, alpha, bt, fa, fb)
                flops += 2 * h * w * (av.shape[0] if fa else av.shape[1])
            elif sk == "syrk":
                syrk_update(ct, av, alpha, bt, uplo, fa)
                flops += step_flops("syrk", h, w, av.shape[0] if fa else av.shape[1])
            elif sk == "syr2k":
                syr2k_update(ct, av, bv, alpha, bt, uplo, fa, fb)
                flops += step_flops("syr2k", h, w, av.shape[0] if fa else av.shape[1])
            elif sk == "symm_diag":
                symm_diag(ct, av, bv, alpha, bt, uplo, side)
                flops += 2 * h * w * av.shape[0]
            elif sk == "trmm_diag":
                trmm_diag(ct, av, bv, alpha, bt, uplo, diag, side, trans_a)
                flops += step_flops("trmm", h, w, av.shape[0])
    return flops


def run_tiles_subset(kind, a, c, b=None, *, tile_size, tiles, alpha=1.0, beta=0.0,
                     trans_a=False, trans_b=False):
    """Sampled-tile oracle for GEMM (SURVEY §8c mode 2): compute only the listed output
    tiles (execute_task_on_host, routines.py:482-492) and return them as a dict
    {(i, j): tile}; ``c`` is not modified."""
    assert kind == "gemm"
    t = tile_size
    A, B, C = _Tiles(a, t), _Tiles(b, t), _Tiles(c, t)
    kt = A.rows if trans_a else A.cols
    out = {}
    for (i, j) in tiles:
        ct = C.phys(i, j).copy()
        for k in range(kt):
            av, fa = A.logical(i, k, trans_a)
            bv, fb = B.logical(k, j, trans_b)
            gemm_update(ct, av, bv, alpha, beta if k == 0 else 1.0, fa, fb)
        out[(i, j)] = ct
    return out
