"""The sampled-block oracle (oracle/sampled.py) against the full tiled oracle: the blocks it
recomputes must equal the corresponding blocks of a full run (same step sequences), and
its per-block north-star ratios must pass an exact answer and flag a perturbed one."""

import numpy as np
import pytest

from oracle import sampled, tiled
from paper_1510_05041_b200.operands import build_call

EPS = np.finfo(np.float64).eps

CASES = [
    ("gemm", dict(beta=1.0)),
    ("gemm", dict(trans_a=True, trans_b=True, alpha=0.5, beta=-1.0)),
    ("gemm", dict(trans_b=True, beta=0.0)),
    ("syrk", dict(uplo="lower", beta=1.0)),
    ("syrk", dict(uplo="upper", trans_a=True, beta=0.5, alpha=-1.0)),
    ("syr2k", dict(uplo="lower", beta=1.0)),
    ("syr2k", dict(uplo="upper", trans_a=True, beta=0.0)),
    ("symm", dict(uplo="lower", side="left", beta=1.0)),
    ("symm", dict(uplo="upper", side="right", beta=0.5)),
    ("trmm", dict(uplo="lower", side="left")),
    ("trmm", dict(uplo="upper", side="right", trans_a=True, diag="unit", alpha=0.7)),
    ("trsm", dict(uplo="lower", side="left")),
    ("trsm", dict(uplo="upper", side="left", trans_a=True, alpha=2.0)),
    ("trsm", dict(uplo="lower", side="right", diag="unit")),
    ("trsm", dict(uplo="upper", side="right", trans_a=True)),
]


def _setup(kind, kw, m=70, n=58, k=45, t=16):
    call = build_call(kind, m=m, n=m if kind in ("syrk", "syr2k") else n, k=k, tile_size=t,
                      seed=5, trsm_scaled=True, **kw)
    a = call.a.matrix.as_2d().copy()
    b = call.b.matrix.as_2d().copy() if call.b is not None else None
    c0 = call.c.matrix.as_2d().copy()
    p = dict(kw)
    alpha, beta = p.pop("alpha", 1.0), p.pop("beta", 0.0)
    full = c0.copy()
    tiled.run_tiled(kind, a, full, b, tile_size=t, alpha=alpha, beta=beta, **p)
    return a, b, c0, full, alpha, beta, p, t


@pytest.mark.parametrize("kind,kw", CASES)
def test_sampled_blocks_equal_full_run(kind, kw):
    a, b, c0, full, alpha, beta, p, t = _setup(kind, kw)
    m, n = c0.shape
    blocks = sampled.sample_blocks(kind, m, n, t, 6, seed=1, side=p.get("side", "left"),
                                   uplo=p.get("uplo", "upper"))
    assert len(blocks) >= 2
    c0b = sampled.snapshot_blocks(c0, blocks, t)
    ref = sampled.reference_blocks(kind, a, b, c0b, tile=t, blocks=blocks, alpha=alpha,
                                   beta=beta, **p)
    views = sampled.block_views(full, blocks, t)
    for blk in blocks:
        np.testing.assert_allclose(ref[blk], views[blk], rtol=1e-13, atol=1e-14)
    r, per = sampled.check_blocks(kind, full, c0b, a=a, b=b, tile=t, alpha=alpha, beta=beta,
                                  eps=EPS, **p)
    assert r <= 1.0, per
    # a perturbation of one element by 1e-6 of the block scale must be flagged
    bad = full.copy()
    bv = sampled.block_views(bad, [blocks[-1]], t)[blocks[-1]]
    bv[0, 0] += 1e-6 * max(1.0, float(np.abs(bv).max()))
    r2, _ = sampled.check_blocks(kind, bad, c0b, a=a, b=b, tile=t, alpha=alpha, beta=beta,
                                 eps=EPS, **p)
    assert r2 > 10.0


def test_block_bound_matches_global_bound_on_one_tile():
    """A 1x1 tile grid: the block bound is the global north-star bound."""
    from oracle import tolerance
    a, b, c0, full, alpha, beta, p, t = _setup("gemm", dict(beta=1.0), m=16, n=16, k=16, t=16)
    got = full + 1e-13
    c0b = sampled.snapshot_blocks(c0, [(0, 0)], t)
    r, _ = sampled.check_blocks("gemm", got, c0b, a=a, b=b, tile=t, alpha=1.0, beta=1.0, eps=EPS)
    g = tolerance.routine_ratio("gemm", got, full, a=a, b=b, c0=c0, alpha=1.0, beta=1.0, k=16,
                                eps=EPS)
    assert r == pytest.approx(g, rel=1e-6)


def test_sym_and_tri_rows_materialise_operators():
    rng = np.random.default_rng(0)
    a = rng.random((37, 37))
    for uplo in ("lower", "upper"):
        s = tiled.sym_of(a, uplo)
        np.testing.assert_array_equal(sampled.sym_rows(a, uplo, slice(10, 25)), s[10:25])
        for trans in (False, True):
            for diag in ("unit", "non-unit"):
                e, _ = tiled.tri_of(a, uplo, diag, trans)
                np.testing.assert_array_equal(sampled.tri_rows(a, uplo, diag, trans, slice(8, 30)),
                                              e[8:30])


@pytest.mark.parametrize("kind,kw", CASES[:4] + CASES[9:12])
def test_compute_block_equals_reference_blocks(kind, kw):
    a, b, c0, full, alpha, beta, p, t = _setup(kind, kw)
    m, n = c0.shape
    blocks = sampled.sample_blocks(kind, m, n, t, 3, seed=2, side=p.get("side", "left"),
                                   uplo=p.get("uplo", "upper"))
    views = sampled.block_views(full, blocks, t)
    for blk in blocks:
        c0b = sampled.snapshot_blocks(c0, [blk], t)[blk]
        got = sampled.compute_block(kind, a, b, c0b, blk, tile=t, alpha=alpha, beta=beta, **p)
        np.testing.assert_allclose(got, views[blk], rtol=1e-13, atol=1e-14)
