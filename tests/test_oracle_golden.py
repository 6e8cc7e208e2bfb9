"""Pin the oracle (oracle/) against fixtures produced by the reference itself."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_variants
from oracle import dense, tiled, tolerance

CASES = load_variants()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_tiled_oracle_matches_reference_run_call(case):
    p = dict(case["params"])
    c = case["c"].copy()
    flops = tiled.run_tiled(case["kind"], case["a"], c, case["b"],
                            tile_size=case["shape"]["tile_size"], **p)
    # same step sequence as the reference planner -> same rounding up to BLAS order
    np.testing.assert_allclose(c, case["out"], rtol=1e-13, atol=1e-13)
    assert flops == case["plan"]["total_flops"]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_dense_oracle_matches_reference_run_call(case):
    p = dict(case["params"])
    ref = dense.dense_reference(case["kind"], a=case["a"], b=case["b"], c=case["c"], **p)
    np.testing.assert_allclose(ref, case["out"], rtol=1e-10, atol=1e-10)


def _cfg1_operands():
    from paper_1510_05041_b200.operands import build_call
    return build_call("gemm", m=2048, n=2048, k=2048, tile_size=512, seed=0,
                      alpha=1.0, beta=1.0)


def test_cfg1_oracle_against_reference_checksums():
    g = np.load(os.path.join(GOLDEN, "cfg1.npz"))
    call = _cfg1_operands()
    a, b, c = (x.matrix.as_2d() for x in (call.a, call.b, call.c))
    # same seeded operands as the reference build_call (operands.py:26-74)
    assert call.a.matrix.leading_dim == int(g["lda"])
    assert call.c.matrix.leading_dim == int(g["ldc"])
    np.testing.assert_array_equal(a.copy().sum(axis=0), g["a_colsum"])
    c0 = c.copy()
    out = c.copy()
    tiled.run_tiled("gemm", a, out, b, tile_size=512, alpha=1.0, beta=1.0)
    np.testing.assert_allclose(out[:64, :64], g["block"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(out[-64:, 1000:1064], g["block2"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(out.sum(axis=0), g["colsum"], rtol=1e-9, atol=1e-9)
    r = tolerance.gemm_ratio(out, dense.dense_reference("gemm", a=a, b=b, c=c0, alpha=1.0, beta=1.0),
                             a_norm=np.linalg.norm(a), b_norm=np.linalg.norm(b), k=2048,
                             alpha=1.0, beta=1.0, c0_norm=np.linalg.norm(c0),
                             eps=np.finfo(np.float64).eps)
    assert r <= tolerance.BOUND


def test_trsm_singular_raises():
    a = np.eye(4)
    a[2, 2] = 0.0
    with pytest.raises(tiled.OracleSingular):
        tiled.run_tiled("trsm", a, np.ones((4, 3)), tile_size=2, uplo="lower")


def test_sampled_tiles_match_full_run():
    rng = np.random.default_rng(3)
    a, b, c = (rng.random((40, 40)) for _ in range(3))
    full = c.copy()
    tiled.run_tiled("gemm", a, full, b, tile_size=16, alpha=0.5, beta=2.0)
    sub = tiled.run_tiles_subset("gemm", a, c, b, tile_size=16, tiles=[(0, 1), (2, 2)],
                                 alpha=0.5, beta=2.0)
    np.testing.assert_allclose(sub[(0, 1)], full[0:16, 16:32], rtol=1e-14)
    np.testing.assert_allclose(sub[(2, 2)], full[32:40, 32:40], rtol=1e-14)
