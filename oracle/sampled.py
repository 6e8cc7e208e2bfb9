"""Sampled-block oracle for full-size parity (TEST INFRASTRUCTURE; SURVEY.md §8c mode 2).

At the BASELINE shapes (16384-32768) the whole tiled oracle takes minutes of CPU, so the
check recomputes only a seeded sample of output *blocks* with the reference's step
sequence (``execute_task_on_host``, /root/reference/pkg/src/tileblas/routines.py:482-492)
and holds each to the north-star bound restricted to the rows/columns that block reads:

* gemm / syrk / syr2k / symm: a block is one output tile (i, j); its steps read row panel
  i of op(A) (or sym(A)) and column panel j of op(B) and nothing else;
* trmm / trsm: a block is one tile *column* j (side left) or tile *row* i (side right) of
  the in-place operand: with the triangle fixed, column j of X depends only on column j
  of B (left), so each block is a complete, independent sub-problem (routines.py:320-356,
  426-437 — the dependency edges never cross columns).

Per-block bound (BASELINE.json north_star, restricted):
  ||C_blk - C_ref,blk||_F / (|alpha| ||opA_rows||_F ||opB_cols||_F k eps + |beta| ||C0_blk||_F eps) <= 10
and for TRSM the residual bound on the block,
  ||E X_blk - alpha B0_blk||_F / ((||E||_F ||X_blk||_F m + |alpha| ||B0_blk||_F) eps) <= 10.
"""

from __future__ import annotations

import numpy as np

from . import tiled


def _ceil(a, b):
    return -(-a // b)


def sample_blocks(kind, m, n, tile, count, seed=0, side="left", uplo="lower"):
    """A seeded sample of output blocks: (i, j) tiles, or ('col', j) / ('row', i) strips.
    Always includes the first and last tile (edge tiles), then random ones."""
    mt, nt = _ceil(m, tile), _ceil(n, tile)
    rng = np.random.default_rng(seed)
    if kind in ("trmm", "trsm"):
        if side == "left":
            cand = [("col", j) for j in range(nt)]
        else:
            cand = [("row", i) for i in range(mt)]
    else:
        if kind in ("syrk", "syr2k"):
            cand = [(i, j) for i in range(mt) for j in range(nt)
                    if (j <= i if uplo == "lower" else j >= i)]
        else:
            cand = [(i, j) for i in range(mt) for j in range(nt)]
    pick = list(dict.fromkeys([cand[0], cand[-1]]))[:max(1, count)]
    rest = [c for c in cand if c not in pick]
    if count > len(pick) and rest:
        idx = rng.choice(len(rest), size=min(count - len(pick), len(rest)), replace=False)
        pick += [rest[int(x)] for x in sorted(idx)]
    return pick


def _rows(blk, tile, m):
    if blk[0] == "col":
        return slice(0, m)
    if blk[0] == "row":
        return slice(blk[1] * tile, min(m, (blk[1] + 1) * tile))
    return slice(blk[0] * tile, min(m, (blk[0] + 1) * tile))


def _cols(blk, tile, n):
    if blk[0] == "row":
        return slice(0, n)
    if blk[0] == "col":
        return slice(blk[1] * tile, min(n, (blk[1] + 1) * tile))
    return slice(blk[1] * tile, min(n, (blk[1] + 1) * tile))


def block_views(c, blocks, tile):
    """{block: view of c} (c is the caller's 2-d output)."""
    m, n = c.shape
    return {b: c[_rows(b, tile, m), _cols(b, tile, n)] for b in blocks}


def snapshot_blocks(c, blocks, tile):
    """Copies of the blocks' current values (the C0 / B0 of the next call)."""
    return {b: v.copy() for b, v in block_views(c, blocks, tile).items()}


# ---- operator panels (materialised rows of op(A), sym(A), op(tri(A))) -----------------

def _op_rows(a, trans, r):
    return a[:, r].T if trans else a[r, :]


def tri_rows(a, uplo, diag, trans, r):
    """Rows r of E = op(tri(A)) (kernels.py:164-170), materialised."""
    e = _op_rows(a, trans, r)
    eff_upper = (uplo == "upper") != trans
    x = np.triu(e, k=r.start) if eff_upper else np.tril(e, k=r.start)
    if diag == "unit":
        x = x.copy()
        idx = np.arange(r.start, r.stop)
        x[idx - r.start, idx] = 1.0
    return x


def sym_rows(a, uplo, r):
    """Rows r of sym(A) (kernels.py:188-195), unstored half never read."""
    if uplo == "lower":
        return np.tril(a[r, :], k=r.start) + np.tril(a[:, r], k=-r.start - 1).T
    return np.triu(a[r, :], k=r.start) + np.triu(a[:, r], k=-r.start + 1).T


def tri_full(a, uplo, diag, trans):
    return tri_rows(a, uplo, diag, trans, slice(0, a.shape[0]))


# ---- reference blocks -----------------------------------------------------------------

def reference_blocks(kind, a, b, c0, *, tile, blocks, alpha, beta, trans_a=False,
                     trans_b=False, uplo="upper", side="left", diag="non-unit"):
    """{block: reference result} by the reference's step sequence (oracle/tiled.py).
    ``c0`` = {block: pre-call values} (``snapshot_blocks``); ``a``/``b`` full operands."""
    out = {}
    if kind in ("trmm", "trsm"):
        for blk in blocks:
            x = c0[blk].copy()
            tiled.run_tiled(kind, a, x, None, tile_size=tile, alpha=alpha, beta=beta,
                            trans_a=trans_a, uplo=uplo, side=side, diag=diag)
            out[blk] = x
        return out
    t = tile
    A = tiled._Tiles(a, t)
    B = tiled._Tiles(b, t) if b is not None else None
    p = dict(trans_a=trans_a, trans_b=trans_b, uplo=uplo, side=side, diag=diag)
    # the planners' step lists for just the wanted tiles: build a C grid of the right
    # shape whose tiles are the c0 copies
    want = set(blocks)
    if kind == "gemm":
        m = a.shape[1] if trans_a else a.shape[0]
        n = b.shape[0] if trans_b else b.shape[1]
    elif kind in ("syrk", "syr2k"):
        m = n = a.shape[1] if trans_a else a.shape[0]
    else:   # symm
        q = a.shape[0]
        m, n = (q, b.shape[1]) if side == "left" else (b.shape[0], q)
    grid = _Grid(m, n, t)
    if kind == "gemm":
        gen = tiled._tasks_gemm(A, B, grid, p)
    elif kind == "syrk":
        gen = tiled._tasks_rank(A, None, grid, p, two=False)
    elif kind == "syr2k":
        gen = tiled._tasks_rank(A, B, grid, p, two=True)
    elif kind == "symm":
        gen = tiled._tasks_symm(A, B, grid, p)
    else:
        raise ValueError(kind)
    for (i, j), steps in gen:
        if (i, j) not in want:
            continue
        ct = c0[(i, j)].copy()
        for s_idx, (sk, av, fa, bv, fb) in enumerate(steps):
            bt = beta if s_idx == 0 else 1.0          # routines.py:211-215
            if sk == "gemm":
                tiled.gemm_update(ct, av, bv, alpha, bt, fa, fb)
            elif sk == "syrk":
                tiled.syrk_update(ct, av, alpha, bt, uplo, fa)
            elif sk == "syr2k":
                tiled.syr2k_update(ct, av, bv, alpha, bt, uplo, fa, fb)
            elif sk == "symm_diag":
                tiled.symm_diag(ct, av, bv, alpha, bt, uplo, side)
        out[(i, j)] = ct
    return out


class _Grid:
    """Stands in for the output tile grid in the planners (only .rows/.cols are read)."""

    def __init__(self, m, n, t):
        self.rows, self.cols = _ceil(m, t), _ceil(n, t)


def compute_block(kind, a, b, c0_block, blk, *, tile, alpha, beta, trans_a=False, trans_b=False,
                  uplo="upper", side="left", diag="non-unit"):
    """One block's reference result, nothing else (the CPU-baseline timer's unit of work);
    GEMM works on the tile's own panels, widened to float64 panel by panel."""
    if kind == "gemm":
        m = a.shape[1] if trans_a else a.shape[0]
        n = b.shape[0] if trans_b else b.shape[1]
        r, c = _rows(blk, tile, m), _cols(blk, tile, n)
        a_sub = np.asarray(a[:, r] if trans_a else a[r, :], np.float64)
        b_sub = np.asarray(b[c, :] if trans_b else b[:, c], np.float64)
        return reference_blocks("gemm", a_sub, b_sub, {(0, 0): np.asarray(c0_block, np.float64)},
                                tile=tile, blocks=[(0, 0)], alpha=alpha, beta=beta,
                                trans_a=trans_a, trans_b=trans_b)[(0, 0)]
    return reference_blocks(kind, a, b, {blk: c0_block}, tile=tile, blocks=[blk], alpha=alpha,
                            beta=beta, trans_a=trans_a, trans_b=trans_b, uplo=uplo, side=side,
                            diag=diag)[blk]


# ---- per-block bound ------------------------------------------------------------------

def block_ratio(kind, blk, got, ref, c0, *, a, b, tile, alpha, beta, eps, trans_a=False,
                trans_b=False, uplo="upper", side="left", diag="non-unit", tri=None):
    """North-star ratio for one block (module docstring).  ``tri`` = materialised
    op(tri(A)) for trmm/trsm (computed once by the caller)."""
    num = float(np.linalg.norm(np.asarray(got, np.float64) - np.asarray(ref, np.float64)))
    c0n = float(np.linalg.norm(c0))
    t = tile
    if kind in ("trmm", "trsm"):
        en = float(np.linalg.norm(tri))
        k = tri.shape[0]
        den = abs(alpha) * en * c0n * k * eps
        return num / den if den else (0.0 if num == 0.0 else float("inf"))
    if kind == "gemm":
        m = a.shape[1] if trans_a else a.shape[0]
        n = b.shape[0] if trans_b else b.shape[1]
        k = a.shape[0] if trans_a else a.shape[1]
        r, c = _rows(blk, t, m), _cols(blk, t, n)
        an = float(np.linalg.norm(_op_rows(a, trans_a, r)))
        bn = float(np.linalg.norm(b[c, :] if trans_b else b[:, c]))
        scale = an * bn
    elif kind in ("syrk", "syr2k"):
        n = a.shape[1] if trans_a else a.shape[0]
        k = a.shape[0] if trans_a else a.shape[1]
        r, c = _rows(blk, t, n), _cols(blk, t, n)
        ar = float(np.linalg.norm(_op_rows(a, trans_a, r)))
        ac = float(np.linalg.norm(_op_rows(a, trans_a, c)))
        if kind == "syrk":
            scale = ar * ac
        else:
            br = float(np.linalg.norm(_op_rows(b, trans_a, r)))
            bc = float(np.linalg.norm(_op_rows(b, trans_a, c)))
            scale = ar * bc + br * ac
    else:   # symm
        q = a.shape[0]
        m, n = (q, b.shape[1]) if side == "left" else (b.shape[0], q)
        r, c = _rows(blk, t, m), _cols(blk, t, n)
        k = q
        if side == "left":
            scale = float(np.linalg.norm(sym_rows(a, uplo, r))) * float(np.linalg.norm(b[:, c]))
        else:
            scale = float(np.linalg.norm(b[r, :])) * float(np.linalg.norm(sym_rows(a, uplo, c)))
    den = abs(alpha) * scale * k * eps + abs(beta) * c0n * eps
    return num / den if den else (0.0 if num == 0.0 else float("inf"))


def trsm_block_residual(tri, x, b0, alpha, side, eps):
    """Residual bound on one strip (columns for side left, rows for side right)."""
    r = tri @ x - alpha * b0 if side == "left" else x @ tri - alpha * b0
    m = tri.shape[0]
    den = (np.linalg.norm(tri) * np.linalg.norm(x) * m + abs(alpha) * np.linalg.norm(b0)) * eps
    return float(np.linalg.norm(r) / den) if den else 0.0


def check_blocks(kind, got_c, c0_blocks, *, a, b, tile, alpha, beta, eps, trans_a=False,
                 trans_b=False, uplo="upper", side="left", diag="non-unit"):
    """Recompute the sampled blocks and return (max ratio, per-block ratios dict); for
    TRSM the per-block value is max(forward ratio, residual ratio)."""
    blocks = list(c0_blocks)
    f64 = lambda x: None if x is None else np.asarray(x, np.float64)   # noqa: E731
    views = block_views(got_c, blocks, tile)
    ratios = {}
    if kind == "gemm":
        # tile by tile on its own panels (row panel of op(A), column panel of op(B)): the
        # k tiling is the full problem's, and float32 operands are widened panel by panel
        m, n = got_c.shape
        for blk in blocks:
            r, c = _rows(blk, tile, m), _cols(blk, tile, n)
            a_sub = f64(a[:, r] if trans_a else a[r, :])
            b_sub = f64(b[c, :] if trans_b else b[:, c])
            c0t = f64(c0_blocks[blk])
            ref = reference_blocks("gemm", a_sub, b_sub, {(0, 0): c0t}, tile=tile,
                                   blocks=[(0, 0)], alpha=alpha, beta=beta, trans_a=trans_a,
                                   trans_b=trans_b)[(0, 0)]
            ratios[blk] = block_ratio("gemm", (0, 0), f64(views[blk]), ref, c0t, a=a_sub,
                                      b=b_sub, tile=max(tile, m, n), alpha=alpha, beta=beta,
                                      eps=eps, trans_a=trans_a, trans_b=trans_b)
        return max(ratios.values()), ratios
    a64, b64 = f64(a), f64(b)
    c0 = {k: f64(v) for k, v in c0_blocks.items()}
    ref = reference_blocks(kind, a64, b64, c0, tile=tile, blocks=blocks, alpha=alpha,
                           beta=beta, trans_a=trans_a, trans_b=trans_b, uplo=uplo, side=side,
                           diag=diag)
    tri = None
    if kind in ("trmm", "trsm"):
        tri = tri_full(a64, uplo, diag, trans_a)
    for blk in blocks:
        g = f64(views[blk])
        r = block_ratio(kind, blk, g, ref[blk], c0[blk], a=a64, b=b64, tile=tile, alpha=alpha,
                        beta=beta, eps=eps, trans_a=trans_a, trans_b=trans_b, uplo=uplo,
                        side=side, diag=diag, tri=tri)
        if kind == "trsm":
            r = max(r, trsm_block_residual(tri, g, c0[blk], alpha, side, eps))
        ratios[blk] = r
    return max(ratios.values()), ratios


# ---- RoutineCall-level helpers (duck-typed: .kind, .a/.b/.c tiled operands, flags) --------

def _dense(tm):
    return None if tm is None else tm.matrix.as_2d()


def call_blocks(call, count, seed=0):
    """A seeded sample of the call's output blocks (see ``sample_blocks``)."""
    c = _dense(call.c)
    return sample_blocks(call.kind, c.shape[0], c.shape[1], call.c.tile_size, count, seed,
                         side=call.side, uplo=call.uplo)


def call_snapshot(call, blocks):
    """The blocks' pre-call values, taken just before the call that is checked."""
    return snapshot_blocks(_dense(call.c), blocks, call.c.tile_size)


def call_check(call, c0_blocks, eps=None):
    """(max ratio, {block: ratio}) of the call's output against the sampled oracle; eps =
    the arithmetic type's epsilon (float32 for SGEMM, float64 otherwise)."""
    c = _dense(call.c)
    if eps is None:
        eps = float(np.finfo(c.dtype).eps)
    return check_blocks(call.kind, c, c0_blocks, a=_dense(call.a), b=_dense(call.b),
                        tile=call.c.tile_size, alpha=call.alpha, beta=call.beta, eps=eps,
                        trans_a=call.trans_a, trans_b=call.trans_b, uplo=call.uplo,
                        side=call.side, diag=call.diag)
