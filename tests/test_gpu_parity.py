"""Parity of the B200 path against the reference (golden fixtures) and the oracle.

Tolerance (BASELINE.json north_star): ||C - C_ref||_F / (|alpha| ||A||_F ||B||_F k eps +
|beta| ||C0||_F eps) <= 10, eps = finfo(float64).eps; TRSM also by its residual."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_variants
from oracle import dense, tiled, tolerance
from paper_1510_05041_b200 import (InvalidArgumentError, RoutineCall, RunOptions,
                                   SingularMatrixError, build_call, dgemm, dsymm, dsyr2k, dsyrk,
                                   dtrmm, dtrsm, run_call)
from paper_1510_05041_b200.devices import DeviceDesc, Topology
from paper_1510_05041_b200.tiling import MatrixDesc, make_tiled

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps
CASES = load_variants()


def _ratio(kind, out, ref, a, b, c0, alpha, beta, k):
    return tolerance.routine_ratio(kind, out, ref, a=a, b=b, c0=c0, alpha=alpha, beta=beta,
                                   k=k, eps=EPS)


def _call(case):
    t = case["shape"]["tile_size"]

    def tm(mid, arr):
        return make_tiled(MatrixDesc.from_array(mid, arr, pad=case["pad"]), t)
    return RoutineCall(kind=case["kind"], a=tm("A", case["a"]),
                       b=None if case["b"] is None else tm("B", case["b"]),
                       c=tm("C", case["c"]), **case["params"])


def test_native_library_loaded():
    import paper_1510_05041_b200._native as N
    N.require_gpu()
    N.load()
    maps = open("/proc/self/maps").read()
    assert "libblasx_cuda.so" in maps


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_variants_match_reference_outputs(case):
    call = _call(case)
    a0 = call.a.matrix.storage.copy()
    res = run_call(call, options=RunOptions(chunk_steps=2))
    out = call.c.matrix.as_2d()
    np.testing.assert_allclose(out, case["out"], rtol=1e-11, atol=1e-12)
    assert np.array_equal(call.a.matrix.storage, a0)
    assert sum(res.tasks_by_device.values()) == len(res.plan.tasks)


def test_cfg1_against_reference_checksums_and_oracle():
    """BASELINE configs[0]: DGEMM 2048^3 NN, T=512, alpha=beta=1, seed 0."""
    g = np.load(os.path.join(GOLDEN, "cfg1.npz"))
    call = build_call("gemm", m=2048, n=2048, k=2048, tile_size=512, seed=0, alpha=1.0, beta=1.0)
    a, b = call.a.matrix.as_2d().copy(), call.b.matrix.as_2d().copy()
    c0 = call.c.matrix.as_2d().copy()
    run_call(call)
    out = call.c.matrix.as_2d()
    ref = c0.copy()
    tiled.run_tiled("gemm", a, ref, b, tile_size=512, alpha=1.0, beta=1.0)
    r = _ratio("gemm", out, ref, a, b, c0, 1.0, 1.0, 2048)
    assert r <= tolerance.BOUND, r
    np.testing.assert_allclose(out[:64, :64], g["block"], rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(out[-64:, 1000:1064], g["block2"], rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(np.ascontiguousarray(out).sum(axis=0), g["colsum"], rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("kind,kw", [
    ("gemm", dict(trans_a=True, beta=0.0)),
    ("gemm", dict(trans_b=True, beta=-0.5, alpha=0.3)),
    ("gemm", dict(trans_a=True, trans_b=True, beta=1.0)),
    ("syrk", dict(uplo="lower", beta=1.0)),
    ("syrk", dict(uplo="upper", trans_a=True, beta=0.0, alpha=-1.0)),
    ("syr2k", dict(uplo="lower", beta=1.0)),
    ("syr2k", dict(uplo="upper", trans_a=True, beta=0.5)),
    ("symm", dict(uplo="lower", side="left", beta=1.0)),
    ("symm", dict(uplo="upper", side="right", beta=0.0)),
    ("trmm", dict(uplo="lower", side="left")),
    ("trmm", dict(uplo="upper", side="right", trans_a=True, diag="unit", alpha=0.7)),
    ("trsm", dict(uplo="lower", side="left")),
    ("trsm", dict(uplo="upper", side="left", trans_a=True, alpha=2.0)),
    ("trsm", dict(uplo="lower", side="right", diag="unit")),
    ("trsm", dict(uplo="upper", side="right", trans_a=True)),
])
def test_routines_medium_against_oracle(kind, kw):
    n, k, t = 1300, 900, 512      # edge tiles in every dimension
    call = build_call(kind, m=n, n=n, k=k, tile_size=t, seed=7, trsm_scaled=True, **kw)
    a = call.a.matrix.as_2d().copy()
    b = call.b.matrix.as_2d().copy() if call.b is not None else None
    c0 = call.c.matrix.as_2d().copy()
    run_call(call)
    out = call.c.matrix.as_2d()
    p = dict(kw)
    alpha, beta = p.pop("alpha", 1.0), p.pop("beta", 0.0)
    ref = c0.copy()
    tiled.run_tiled(kind, a, ref, b, tile_size=t, alpha=alpha, beta=beta, **p)
    kk = k if kind in ("gemm", "syrk", "syr2k") else n
    r = _ratio(kind, out, ref, a, b, c0, alpha, beta, kk)
    assert r <= tolerance.BOUND, r
    if kind == "trsm":
        m, _ = tiled.tri_of(a, p.get("uplo", "upper"), p.get("diag", "non-unit"),
                            p.get("trans_a", False))
        rr = tolerance.trsm_residual_ratio(m, out, c0, alpha, p.get("side", "left"), EPS)
        assert rr <= tolerance.BOUND, rr
    if kind in ("syrk", "syr2k"):
        mask = np.triu(np.ones((n, n), bool), 1) if p["uplo"] == "lower" else np.tril(np.ones((n, n), bool), -1)
        assert np.array_equal(out[mask], c0[mask])     # unstored triangle untouched


def test_beta_zero_never_reads_c():
    call = build_call("gemm", m=700, n=600, k=500, tile_size=256, seed=3, beta=0.0)
    call.c.matrix.storage[:] = np.nan
    a, b = call.a.matrix.as_2d(), call.b.matrix.as_2d()
    run_call(call)
    out = call.c.matrix.as_2d()
    assert np.isfinite(out).all()
    np.testing.assert_allclose(out, a @ b, rtol=1e-12, atol=1e-12)


def test_unstored_triangle_never_read_symm_trmm():
    rng = np.random.default_rng(5)
    n = 600
    a = rng.random((n, n))
    poisoned = a.copy()
    poisoned[np.triu_indices(n, 1)] = np.nan            # lower is stored
    bm = rng.random((n, 300))
    for kind in ("symm", "trmm"):
        c = np.asfortranarray(rng.random((n, 300)))
        if kind == "symm":
            res_c = c.copy(order="F")
            dsymm("L", "L", n, 300, 1.0, np.asfortranarray(poisoned), n, np.asfortranarray(bm), n,
                  0.0, res_c, n, tile_size=256)
            s = np.tril(a) + np.tril(a, -1).T
            np.testing.assert_allclose(res_c, s @ bm, rtol=1e-11, atol=1e-11)
        else:
            x = np.asfortranarray(bm.copy())
            dtrmm("L", "L", "N", "U", n, 300, 1.0, np.asfortranarray(poisoned), n, x, n, tile_size=256)
            m = np.tril(a, -1) + np.eye(n)
            np.testing.assert_allclose(x, m @ bm, rtol=1e-11, atol=1e-11)


def test_trsm_singular_raises():
    rng = np.random.default_rng(1)
    a = np.asfortranarray(rng.random((512, 512)) + 2 * np.eye(512))
    a[300, 300] = 0.0
    b = np.asfortranarray(rng.random((512, 64)))
    with pytest.raises(SingularMatrixError):
        dtrsm("L", "L", "N", "N", 512, 64, 1.0, a, 512, b, 512, tile_size=256)


def test_trsm_unit_diag_ignores_zero_diagonal():
    rng = np.random.default_rng(2)
    n = 300
    a = rng.random((n, n)) / n
    np.fill_diagonal(a, 0.0)
    b = rng.random((n, 40))
    x = np.asfortranarray(b.copy())
    dtrsm("L", "L", "N", "U", n, 40, 1.0, np.asfortranarray(a), n, x, n, tile_size=128)
    m = np.tril(a, -1) + np.eye(n)
    np.testing.assert_allclose(m @ x, b, rtol=1e-11, atol=1e-11)


def test_cblas_dgemm_fortran_arrays_and_leading_dims():
    rng = np.random.default_rng(3)
    m, n, k, lda = 333, 222, 111, 340
    abuf = rng.random(lda * k)
    b = np.asfortranarray(rng.random((k, n)))
    c = np.asfortranarray(rng.random((m, n)))
    a2 = abuf.reshape(k, lda).T[:m, :]
    ref = 2.0 * a2 @ b + 0.5 * c
    dgemm("N", "N", m, n, k, 2.0, abuf, lda, b, k, 0.5, c, m, tile_size=128)
    np.testing.assert_allclose(c, ref, rtol=1e-12, atol=1e-12)
    with pytest.raises(InvalidArgumentError):
        dgemm("X", "N", m, n, k, 1.0, abuf, lda, b, k, 0.0, c, m)


def test_small_arena_eviction_on_gpu():
    call = build_call("gemm", m=1024, n=1024, k=2048, tile_size=256, seed=8, beta=1.0)
    a, b = call.a.matrix.as_2d().copy(), call.b.matrix.as_2d().copy()
    c0 = call.c.matrix.as_2d().copy()
    tile = 256 * 256 * 8
    res = run_call(call, Topology([DeviceDesc(0, arena_capacity=40 * tile)]),
                   RunOptions(chunk_steps=2))
    ref = c0.copy()
    tiled.run_tiled("gemm", a, ref, b, tile_size=256, alpha=1.0, beta=1.0)
    assert _ratio("gemm", call.c.matrix.as_2d(), ref, a, b, c0, 1.0, 1.0, 2048) <= 10
    assert res.metrics.host_fetches > 16 + 32       # evictions forced refetches


def test_capacity_deadlock_on_gpu_then_recovers():
    """Failure path on hardware: an arena one tile above the 12-tile floor cannot hold the
    C / C0 buffers of 8 in-flight tasks -> CapacityDeadlockError after the pressure sync
    (cache.py:232-250, scheduler.py:636-643); the engine stays usable and the next call
    (one task in flight) is correct."""
    from paper_1510_05041_b200 import CapacityDeadlockError
    tile = 256 * 256 * 8
    call = build_call("gemm", m=2048, n=2048, k=2048, tile_size=256, seed=12, beta=1.0)
    with pytest.raises(CapacityDeadlockError):
        run_call(call, Topology([DeviceDesc(0, arena_capacity=13 * tile)]),
                 RunOptions(n_streams=4, tasks_per_stream=2))
    call = build_call("gemm", m=2048, n=2048, k=2048, tile_size=256, seed=12, beta=1.0)
    a, b = call.a.matrix.as_2d().copy(), call.b.matrix.as_2d().copy()
    c0 = call.c.matrix.as_2d().copy()
    run_call(call, Topology([DeviceDesc(0, arena_capacity=13 * tile)]),
             RunOptions(n_streams=1, tasks_per_stream=1))
    ref = c0.copy()
    tiled.run_tiled("gemm", a, ref, b, tile_size=256, alpha=1.0, beta=1.0)
    assert _ratio("gemm", call.c.matrix.as_2d(), ref, a, b, c0, 1.0, 1.0, 2048) <= tolerance.BOUND


def test_concurrent_mode_and_trace():
    call = build_call("syr2k", m=1100, n=1100, k=700, tile_size=256, seed=9, beta=1.0, uplo="lower")
    a, b = call.a.matrix.as_2d().copy(), call.b.matrix.as_2d().copy()
    c0 = call.c.matrix.as_2d().copy()
    res = run_call(call, options=RunOptions(execution="concurrent", record_trace=True))
    ref = c0.copy()
    tiled.run_tiled("syr2k", a, ref, b, tile_size=256, alpha=1.0, beta=1.0, uplo="lower")
    assert _ratio("syr2k", call.c.matrix.as_2d(), ref, a, b, c0, 1.0, 1.0, 700) <= 10
    assert any(e.event == "KERNEL" for e in res.trace)
    ks = [e for e in res.trace if e.event == "KERNEL"]
    assert all(e.time_end >= e.time_start for e in ks)


@pytest.mark.parametrize("variant,mn3d,shape", [(1, 1, (1500, 1300, 1100)), (0, 1, (1500, 1300, 1100)),
                                                (1, 1, (1536, 1280, 1024)), (0, 1, (1536, 1280, 1024)),
                                                (1, 0, (1536, 1280, 1024)), (2, 1, (1500, 1300, 1100)),
                                                (2, 1, (4608, 4352, 1024)), (3, 1, (1500, 1300, 1100)),
                                                (3, 0, (1536, 1280, 1024)), (3, 1, (4608, 4352, 1024))])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
def test_sgemm_tcgen05_against_fp64_oracle(ta, tb, variant, mn3d, shape):
    """SGEMM has no reference path (tiling.py:57-60 is float64 only): compare with the
    float64 tiled oracle on the same float32-representable inputs, eps = 2^-23.  Both
    kernels (1-SM 128x256, 2-SM cta_group::2 256x256), MN-major operands by 3-d or 2-d TMA
    boxes, ragged (1500x1300x1100) and 32-aligned shapes."""
    from paper_1510_05041_b200 import _native
    lib = _native.load()
    lib.bx_set_sgemm_variant(variant)
    lib.bx_set_sgemm_mn3d(mn3d)
    try:
        _sgemm_case(ta, tb, *shape)
    finally:
        lib.bx_set_sgemm_variant(3)
        lib.bx_set_sgemm_mn3d(1)


def _sgemm_case(ta, tb, m, n, k):
    call = build_call("gemm", m=m, n=n, k=k, tile_size=512, seed=11, alpha=1.0, beta=0.5,
                      trans_a=ta, trans_b=tb, dtype=np.float32)
    a = call.a.matrix.as_2d().astype(np.float64)
    b = call.b.matrix.as_2d().astype(np.float64)
    c0 = call.c.matrix.as_2d().astype(np.float64)
    run_call(call)
    out = call.c.matrix.as_2d().astype(np.float64)
    ref = c0.copy()
    tiled.run_tiled("gemm", a, ref, b, tile_size=512, alpha=1.0, beta=0.5, trans_a=ta, trans_b=tb)
    r = tolerance.gemm_ratio(out, ref, a_norm=np.linalg.norm(a), b_norm=np.linalg.norm(b), k=k,
                             alpha=1.0, beta=0.5, c0_norm=np.linalg.norm(c0),
                             eps=float(np.finfo(np.float32).eps))
    assert r <= tolerance.BOUND, r


def test_cblas_sgemm():
    """The cblas-style sgemm at a short reduction (k = 100: auto 3xTF32) meets the north-
    star bound with the float32 epsilon."""
    from paper_1510_05041_b200 import sgemm
    rng = np.random.default_rng(4)
    m, n, k = 700, 600, 100
    a = np.asfortranarray(rng.random((m, k), dtype=np.float32))
    b = np.asfortranarray(rng.random((k, n), dtype=np.float32))
    c = np.asfortranarray(np.zeros((m, n), dtype=np.float32))
    sgemm("N", "N", m, n, k, 1.0, a, m, b, k, 0.0, c, m, tile_size=256)
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    r = tolerance.gemm_ratio(c, a64 @ b64, a_norm=np.linalg.norm(a64), b_norm=np.linalg.norm(b64),
                             k=k, alpha=1.0, beta=0.0, c0_norm=0.0,
                             eps=float(np.finfo(np.float32).eps))
    assert r <= tolerance.BOUND, r


VIRTUAL = [100, 101, 102]   # logical devices sharing GPU 0 (own streams, events, arenas)


def _virtual_topo(n=3, arena=0):
    return Topology([DeviceDesc(VIRTUAL[i], cuda_ordinal=0, peer_group="nvlink",
                                arena_capacity=arena) for i in range(n)])


@pytest.mark.parametrize("kind,kw", [
    ("gemm", dict(beta=1.0)),
    ("gemm", dict(trans_a=True, beta=0.0)),
    ("syr2k", dict(uplo="lower", beta=1.0)),
    ("trsm", dict(uplo="lower", side="left")),
    ("trmm", dict(uplo="upper", side="right", trans_a=True)),
])
@pytest.mark.parametrize("execution", ["deterministic", "concurrent"])
def test_multi_device_runtime_on_one_gpu(kind, kw, execution):
    """The multi-GPU path (L2 peer copies, directory, stealing, per-device engines) on three
    logical devices backed by one B200."""
    n, k, t = 1536, 1024, 256
    call = build_call(kind, m=n, n=n, k=k, tile_size=t, seed=21, trsm_scaled=True, **kw)
    a = call.a.matrix.as_2d().copy()
    b = call.b.matrix.as_2d().copy() if call.b is not None else None
    c0 = call.c.matrix.as_2d().copy()
    # small per-device claims (no start-up batch, 1 task per stream, 2-slot stations) so a
    # per-device thread that starts first cannot drain a 36-task call before the others run
    res = run_call(call, _virtual_topo(), RunOptions(execution=execution, ramp_tasks=0,
                                                    tasks_per_stream=1, rs_capacity=2))
    p = dict(kw)
    alpha, beta = p.pop("alpha", 1.0), p.pop("beta", 0.0)
    ref = c0.copy()
    tiled.run_tiled(kind, a, ref, b, tile_size=t, alpha=alpha, beta=beta, **p)
    kk = k if kind in ("gemm", "syrk", "syr2k") else n
    assert _ratio(kind, call.c.matrix.as_2d(), ref, a, b, c0, alpha, beta, kk) <= tolerance.BOUND
    m = res.metrics
    assert sum(res.tasks_by_device.values()) == len(res.plan.tasks)
    assert m.total_d2d_bytes() == sum(d.d2d_out_bytes for d in m.devices.values())
    if kind == "gemm" and execution == "deterministic":
        # one driver thread round-robins the devices: all take tasks and share tiles over L2
        assert m.l2_hits > 0 and len([v for v in res.tasks_by_device.values() if v]) > 1


def test_multi_device_concurrent_threads_share_tiles():
    """One host thread per logical device (execution="concurrent") on a call long enough
    that every thread joins before the queue drains: tasks spread over the devices and
    tiles move between them as L2 peer copies."""
    n, t = 4096, 256
    call = build_call("gemm", m=n, n=n, k=1024, tile_size=t, seed=23, beta=1.0)
    a, b = call.a.matrix.as_2d().copy(), call.b.matrix.as_2d().copy()
    c0 = call.c.matrix.as_2d().copy()
    res = run_call(call, _virtual_topo(), RunOptions(execution="concurrent", ramp_tasks=0,
                                                    tasks_per_stream=1, rs_capacity=2))
    ref = c0.copy()
    tiled.run_tiled("gemm", a, ref, b, tile_size=t, alpha=1.0, beta=1.0)
    assert _ratio("gemm", call.c.matrix.as_2d(), ref, a, b, c0, 1.0, 1.0, 1024) <= tolerance.BOUND
    m = res.metrics
    assert sum(res.tasks_by_device.values()) == len(res.plan.tasks)
    assert m.l2_hits > 0 and len([v for v in res.tasks_by_device.values() if v]) > 1


def test_multi_device_small_arenas_evict_on_one_gpu():
    call = build_call("gemm", m=1024, n=1024, k=2048, tile_size=256, seed=22, beta=1.0)
    a, b = call.a.matrix.as_2d().copy(), call.b.matrix.as_2d().copy()
    c0 = call.c.matrix.as_2d().copy()
    tile = 256 * 256 * 8
    res = run_call(call, _virtual_topo(2, arena=40 * tile), RunOptions(chunk_steps=2))
    ref = c0.copy()
    tiled.run_tiled("gemm", a, ref, b, tile_size=256, alpha=1.0, beta=1.0)
    assert _ratio("gemm", call.c.matrix.as_2d(), ref, a, b, c0, 1.0, 1.0, 2048) <= 10


def _random_cases(n_cases=120, seed=2026):
    import routine_cases as G
    return G.random_cases(n_cases, seed)


@pytest.mark.parametrize("case", _random_cases(), ids=lambda c: f"r{c[0]}_{c[1]}")
def test_randomized_routines_against_oracle(case):
    """Seeded random shapes (ragged, 1..639), tile sizes, flags, scalars and runtime options
    for every routine, against the tiled oracle with the north-star bound (and the TRSM
    residual bound) — the GPU counterpart of the reference's randomized acceptance sweep
    (tests/test_acceptance.py:595-619)."""
    _, kind, m, n, k, t, kw, opts = case
    call = build_call(kind, m=m, n=n, k=k, tile_size=t, seed=m * 7 + n, trsm_scaled=True, **kw)
    a = call.a.matrix.as_2d().copy()
    b = call.b.matrix.as_2d().copy() if call.b is not None else None
    c0 = call.c.matrix.as_2d().copy()
    res = run_call(call, options=RunOptions(**opts))
    assert sum(res.tasks_by_device.values()) == len(res.plan.tasks)
    out = call.c.matrix.as_2d()
    p = dict(kw)
    alpha, beta = p.pop("alpha", 1.0), p.pop("beta", 0.0)
    ref = c0.copy()
    tiled.run_tiled(kind, a, ref, b, tile_size=t, alpha=alpha, beta=beta, **p)
    side = p.get("side", "left")
    kk = k if kind in ("gemm", "syrk", "syr2k") else (m if side == "left" else n)
    assert _ratio(kind, out, ref, a, b, c0, alpha, beta, kk) <= tolerance.BOUND
    if kind == "trsm":
        tri, _ = tiled.tri_of(a, p.get("uplo", "upper"), p.get("diag", "non-unit"),
                              p.get("trans_a", False))
        assert tolerance.trsm_residual_ratio(tri, out, c0, alpha, side, EPS) <= tolerance.BOUND


def _sgemm_ratio(call, t, alpha, beta, ta, tb, k, opts):
    a = call.a.matrix.as_2d().astype(np.float64)
    b = call.b.matrix.as_2d().astype(np.float64)
    c0 = call.c.matrix.as_2d().astype(np.float64)
    run_call(call, options=opts)
    ref = c0.copy()
    tiled.run_tiled("gemm", a, ref, b, tile_size=t, alpha=alpha, beta=beta, trans_a=ta, trans_b=tb)
    return tolerance.gemm_ratio(call.c.matrix.as_2d().astype(np.float64), ref,
                                a_norm=np.linalg.norm(a), b_norm=np.linalg.norm(b), k=k,
                                alpha=alpha, beta=beta, c0_norm=np.linalg.norm(c0),
                                eps=float(np.finfo(np.float32).eps))


@pytest.mark.parametrize("i", range(24))
def test_randomized_sgemm_against_fp64_oracle(i):
    """Random ragged SGEMM calls with the default (auto) precision vs the float64 oracle,
    held to the north-star bound with the float32 epsilon (2^-23) at every k: calls whose
    reduction is shorter than SGEMM_TF32_MIN_K run 3xTF32, longer ones plain TF32."""
    rng = np.random.default_rng(500 + i)
    m, n = (int(x) for x in rng.integers(1, 900, size=2))
    k = int(rng.integers(1, 1400))
    ta, tb = bool(rng.integers(2)), bool(rng.integers(2))
    t = int(rng.choice([128, 256, 512]))
    alpha, beta = float(rng.choice([1.0, -0.5])), float(rng.choice([0.0, 1.0]))
    call = build_call("gemm", m=m, n=n, k=k, tile_size=t, seed=i, alpha=alpha, beta=beta,
                      trans_a=ta, trans_b=tb, dtype=np.float32)
    r = _sgemm_ratio(call, t, alpha, beta, ta, tb, k,
                     RunOptions(chunk_steps=int(rng.choice([1, 16]))))
    assert r <= tolerance.BOUND, (r, k)


@pytest.mark.parametrize("i", range(8))
def test_plain_tf32_meets_fp32_bound_from_crossover(i):
    """The crossover itself: plain TF32 (forced) at reduction depths just above
    SGEMM_TF32_MIN_K already meets the float32-epsilon bound."""
    from paper_1510_05041_b200.scheduler import SGEMM_TF32_MIN_K
    rng = np.random.default_rng(700 + i)
    m, n = int(rng.integers(64, 900)), int(rng.integers(64, 900))
    k = int(rng.integers(SGEMM_TF32_MIN_K, SGEMM_TF32_MIN_K + 128))
    ta, tb = bool(rng.integers(2)), bool(rng.integers(2))
    call = build_call("gemm", m=m, n=n, k=k, tile_size=256, seed=40 + i, alpha=1.0, beta=1.0,
                      trans_a=ta, trans_b=tb, dtype=np.float32)
    r = _sgemm_ratio(call, 256, 1.0, 1.0, ta, tb, k, RunOptions(sgemm_precise=False))
    assert r <= tolerance.BOUND / 2, (r, k)


@pytest.mark.parametrize("i", range(6))
def test_sgemm_precise_mode_meets_fp32_bound_at_small_k(i):
    """3xTF32 mode (bx_set_sgemm_precise): the hi/lo split products restore the north-star
    bound with the fp32 epsilon even at small k, where plain TF32 exceeds it."""
    from paper_1510_05041_b200 import _native
    lib = _native.load()
    rng = np.random.default_rng(900 + i)
    m, n, k = int(rng.integers(100, 900)), int(rng.integers(100, 900)), int(rng.integers(8, 120))
    ta, tb = bool(rng.integers(2)), bool(rng.integers(2))
    call = build_call("gemm", m=m, n=n, k=k, tile_size=256, seed=i, alpha=1.0, beta=1.0,
                      trans_a=ta, trans_b=tb, dtype=np.float32)
    a = call.a.matrix.as_2d().astype(np.float64)
    b = call.b.matrix.as_2d().astype(np.float64)
    c0 = call.c.matrix.as_2d().astype(np.float64)
    try:
        run_call(call, options=RunOptions(sgemm_precise=True))
    finally:
        lib.bx_set_sgemm_precise(0)
    ref = c0.copy()
    tiled.run_tiled("gemm", a, ref, b, tile_size=256, alpha=1.0, beta=1.0, trans_a=ta, trans_b=tb)
    r = tolerance.gemm_ratio(call.c.matrix.as_2d().astype(np.float64), ref, a_norm=np.linalg.norm(a),
                             b_norm=np.linalg.norm(b), k=k, alpha=1.0, beta=1.0,
                             c0_norm=np.linalg.norm(c0), eps=float(np.finfo(np.float32).eps))
    assert r <= tolerance.BOUND, (r, m, n, k)



@pytest.mark.parametrize("kind,kw,opts", [
    ("trsm", dict(uplo="lower", side="left"), dict(trsm_split_chain=True)),
    ("trsm", dict(uplo="upper", side="right", trans_a=True), dict(trsm_split_chain=True)),
    ("trsm", dict(uplo="lower", side="left"), dict(release_on_issue=True)),
    ("trsm", dict(uplo="lower", side="left"), dict(release_on_issue=True, trsm_inverse_min=0)),
    ("trmm", dict(uplo="lower", side="left"), dict(split_km=True)),
    ("trmm", dict(uplo="upper", side="right", trans_a=True), dict(split_km=True, chunk_steps=2)),
    ("gemm", dict(beta=1.0), dict(ramp_tasks=0)),
    ("gemm", dict(beta=1.0), dict(ramp_tasks=8, ramp_chunk_steps=1)),
    ("gemm", dict(beta=1.0), dict(prefetch=0)),
    ("syr2k", dict(uplo="lower", beta=1.0), dict(prefetch=0)),
    ("syrk", dict(uplo="upper", trans_a=True, beta=0.5), dict(prefetch=1)),
    ("symm", dict(uplo="lower", side="left", beta=1.0), dict(prefetch=1)),
])
def test_launch_shape_options_on_hardware(kind, kw, opts):
    """The launch-shape knobs (chain split, KM split, substitution path with the reference's
    release rule, start-up batch on/off) on the real kernels: same north-star bound."""
    n, k, t = 1300, 1100, 256
    call = build_call(kind, m=n, n=n, k=k, tile_size=t, seed=11, trsm_scaled=True, **kw)
    a = call.a.matrix.as_2d().copy()
    b = call.b.matrix.as_2d().copy() if call.b is not None else None
    c0 = call.c.matrix.as_2d().copy()
    run_call(call, options=RunOptions(**opts))
    out = call.c.matrix.as_2d()
    p = dict(kw)
    alpha, beta = p.pop("alpha", 1.0), p.pop("beta", 0.0)
    ref = c0.copy()
    tiled.run_tiled(kind, a, ref, b, tile_size=t, alpha=alpha, beta=beta, **p)
    r = _ratio(kind, out, ref, a, b, c0, alpha, beta, k if kind == "gemm" else n)
    assert r <= tolerance.BOUND, r
