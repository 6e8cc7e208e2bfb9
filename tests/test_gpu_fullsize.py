"""Parity at the BASELINE shapes (north_star: "every config passes the reference tolerance
check"), on the GPU, at full size.

Each test builds the config's seeded host operands exactly as ``bench.py`` does, runs the
public ``run_call`` on them (host-resident operands, H2D tile loads, D2H write-back), and
holds a seeded sample of output blocks to the north-star bound restricted to the rows and
columns each block reads (oracle/sampled.py): >= 16 tiles for GEMM-type routines, tile
columns (complete independent sub-problems) for TRSM/TRMM, plus the TRSM residual bound.
SGEMM (TF32 tensor cores) is held to the bound with the float32 epsilon."""

import os
import sys

import numpy as np
import pytest

from oracle import sampled, tolerance

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

pytestmark = pytest.mark.gpu

FULL = [("cfg2", 16), ("cfg3_syrk", 16), ("cfg3_syr2k", 16), ("cfg4_trsm", 4),
        ("cfg4_trmm", 4), ("cfg5_sgemm", 8), ("dgemm32768", 16)]


@pytest.mark.parametrize("name,count", FULL, ids=[f[0] for f in FULL])
def test_baseline_config_full_size(name, count):
    from paper_1510_05041_b200 import run_call
    cfg = bench.CONFIGS[name]
    call = bench.make_operands(cfg, seed=0)
    blocks = sampled.call_blocks(call, count, seed=1)
    c0 = sampled.call_snapshot(call, blocks)
    res = run_call(call)
    assert sum(res.tasks_by_device.values()) == len(res.plan.tasks)
    worst, per = sampled.call_check(call, c0)
    print(f"{name}: max ratio {worst:.3g} over {len(per)} blocks")
    assert worst <= tolerance.BOUND, per
    n_tiles = sum(1 for b in per if b[0] not in ("col", "row"))
    n_strips = len(per) - n_tiles
    assert n_tiles >= 8 or n_strips >= 4


def test_repeated_calls_stay_in_bound():
    """The bench times repeated calls on the same buffers (beta = 1 accumulates): the
    check of the last call uses the blocks' values just before it."""
    from paper_1510_05041_b200 import run_call
    cfg = dict(bench.CONFIGS["cfg2"], m=8192, n=8192, k=8192)
    call = bench.make_operands(cfg, seed=3)
    blocks = sampled.call_blocks(call, 8, seed=2)
    for _ in range(2):
        run_call(call)
    c0 = sampled.call_snapshot(call, blocks)
    run_call(call)
    worst, per = sampled.call_check(call, c0)
    assert worst <= tolerance.BOUND, per


def test_sgemm_block_check_sees_fp32_eps():
    from paper_1510_05041_b200 import run_call
    cfg = dict(bench.CONFIGS["cfg5_sgemm"], m=4096, n=4096, k=4096, tile=1024)
    call = bench.make_operands(cfg, seed=4)
    assert call.c.matrix.storage.dtype == np.float32
    blocks = sampled.call_blocks(call, 8, seed=3)
    c0 = sampled.call_snapshot(call, blocks)
    run_call(call)
    worst, per = sampled.call_check(call, c0)
    assert worst <= tolerance.BOUND, per
    # the same output held to the float64 epsilon is far outside the bound (TF32 inputs)
    worst64, _ = sampled.call_check(call, c0, eps=float(np.finfo(np.float64).eps))
    assert worst64 > tolerance.BOUND
