"""Host runtime (planner -> scheduler -> cache -> engine) on the fake engine: numerics
against the reference's own outputs, byte accounting, stealing, eviction, errors."""

import numpy as np
import pytest

from conftest import load_variants
from fake_engine import FakeEngine
from paper_1510_05041_b200.devices import DeviceDesc, Topology
from paper_1510_05041_b200.errors import (CapacityDeadlockError, ConfigError,
                                          SingularMatrixError)
from paper_1510_05041_b200.operands import build_call
from paper_1510_05041_b200.routines import RoutineCall, generate_tasks
from paper_1510_05041_b200.scheduler import RunOptions, run_call
from paper_1510_05041_b200.tiling import MatrixDesc, make_tiled

CASES = load_variants()


def topo(n, arena=8 << 20):
    return Topology([DeviceDesc(i, arena_capacity=arena, peer_group="g") for i in range(n)])


def call_of(case):
    t = case["shape"]["tile_size"]

    def tiled(mid, arr):
        return make_tiled(MatrixDesc.from_array(mid, arr, pad=case["pad"]), t)
    return RoutineCall(kind=case["kind"], a=tiled("A", case["a"]),
                       b=None if case["b"] is None else tiled("B", case["b"]),
                       c=tiled("C", case["c"]), **case["params"])


@pytest.mark.parametrize("ndev", [1, 3])
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_variants_match_reference(case, ndev):
    call = call_of(case)
    a0 = call.a.matrix.storage.copy()
    eng = FakeEngine(ndev, seed=hash(case["name"]) % 1000)
    res = run_call(call, topo(ndev), RunOptions(chunk_steps=2), engine=eng)
    np.testing.assert_allclose(call.c.matrix.as_2d(), case["out"], rtol=1e-12, atol=1e-12)
    assert np.array_equal(call.a.matrix.storage, a0)          # inputs never written
    assert sum(res.tasks_by_device.values()) == len(res.plan.tasks)
    m = res.metrics
    assert m.total_d2h_bytes() == sum(t.out_ref.height * t.out_ref.width * 8 for t in res.plan.tasks)
    d_in = sum(d.d2d_in_bytes for d in m.devices.values())
    d_out = sum(d.d2d_out_bytes for d in m.devices.values())
    assert d_in == d_out


@pytest.mark.parametrize("execution", ["deterministic", "concurrent"])
def test_two_devices_split_and_l2(execution):
    call = build_call("gemm", m=64, n=64, k=64, tile_size=8, seed=1, beta=0.5)
    ref = call.c.matrix.as_2d().copy()
    a, b = call.a.matrix.as_2d().copy(), call.b.matrix.as_2d().copy()
    res = run_call(call, topo(2), RunOptions(execution=execution), engine=FakeEngine(2, seed=3))
    np.testing.assert_allclose(call.c.matrix.as_2d(), a @ b + 0.5 * ref, rtol=1e-12, atol=1e-12)
    assert all(v > 0 for v in res.tasks_by_device.values())
    m = res.metrics
    # L2 converts host traffic into peer traffic: with L2 off, H2D grows by exactly the
    # bytes moved peer-to-peer
    call2 = build_call("gemm", m=64, n=64, k=64, tile_size=8, seed=1, beta=0.5)
    res2 = run_call(call2, topo(2), RunOptions(execution=execution, l2_enabled=False),
                    engine=FakeEngine(2, seed=3))
    assert res2.metrics.total_d2d_bytes() == 0
    if execution == "deterministic":
        assert m.l2_hits > 0
        assert m.total_d2d_bytes() == m.l2_hits * 8 * 8 * 8


def test_l1_disabled_fetches_every_input():
    call = build_call("gemm", m=32, n=32, k=32, tile_size=8, seed=2)
    res = run_call(call, topo(1), RunOptions(l1_enabled=False), engine=FakeEngine(1))
    plan = res.plan
    n_refs = sum(len(s.input_refs()) for t in plan.tasks for s in t.steps)
    assert res.metrics.host_fetches == n_refs
    assert res.metrics.l1_hits == 0


def test_l1_hits_on_shared_panels():
    call = build_call("gemm", m=32, n=32, k=32, tile_size=8, seed=2)
    res = run_call(call, topo(1), RunOptions(), engine=FakeEngine(1))
    assert res.metrics.host_fetches == 32     # 16 A + 16 B tiles, each fetched once
    assert res.metrics.l1_hits == 16 * 4 * 2 - 32


def test_small_arena_evicts_and_stays_correct():
    call = build_call("gemm", m=48, n=48, k=48, tile_size=8, seed=4, beta=1.0)
    c0 = call.c.matrix.as_2d().copy()
    a, b = call.a.matrix.as_2d().copy(), call.b.matrix.as_2d().copy()
    tile = 8 * 8 * 8
    opts = RunOptions(chunk_steps=1)
    res = run_call(call, Topology([DeviceDesc(0, arena_capacity=14 * 512 * 4)]), opts,
                   engine=FakeEngine(1, seed=9))
    np.testing.assert_allclose(call.c.matrix.as_2d(), a @ b + c0, rtol=1e-12, atol=1e-12)
    assert res.metrics.host_fetches > 72        # evictions forced re-fetches
    assert tile == 512


def test_arena_floor_enforced():
    call = build_call("gemm", m=16, n=16, k=16, tile_size=8, seed=1)
    with pytest.raises(ConfigError):
        run_call(call, Topology([DeviceDesc(0, arena_capacity=1024)]), RunOptions(),
                 engine=FakeEngine(1))


def test_capacity_deadlock_when_concurrent_tasks_cannot_fit():
    """An arena one tile above the reference's 12-tile floor cannot hold 8 in-flight tasks'
    C (and deferred C0) buffers: after the pressure sync the allocation still fails ->
    CapacityDeadlockError (cache.py:232-250); with one task in flight the same arena works."""
    call = build_call("gemm", m=64, n=64, k=64, tile_size=8, seed=1, beta=1.0)
    with pytest.raises(CapacityDeadlockError):
        run_call(call, Topology([DeviceDesc(0, arena_capacity=13 * 512)]),
                 RunOptions(n_streams=4, tasks_per_stream=2), engine=FakeEngine(1))
    call = build_call("gemm", m=64, n=64, k=64, tile_size=8, seed=1, beta=1.0)
    a, b, c0 = (x.matrix.as_2d().copy() for x in (call.a, call.b, call.c))
    run_call(call, Topology([DeviceDesc(0, arena_capacity=13 * 512)]),
             RunOptions(n_streams=1, tasks_per_stream=1), engine=FakeEngine(1))
    np.testing.assert_allclose(call.c.matrix.as_2d(), a @ b + c0, rtol=1e-12, atol=1e-12)


def test_trsm_singular_raises():
    rng = np.random.default_rng(0)
    a = rng.random((16, 16)) + np.eye(16)
    a[5, 5] = 0.0
    call = RoutineCall("trsm", a=make_tiled(MatrixDesc.from_array("A", a), 8),
                       c=make_tiled(MatrixDesc.from_array("C", rng.random((16, 4))), 8),
                       uplo="lower")
    with pytest.raises(SingularMatrixError):
        run_call(call, topo(1), RunOptions(), engine=FakeEngine(1))


def test_trace_accounts_for_bytes_and_flops():
    call = build_call("syrk", m=24, n=24, k=16, tile_size=8, seed=5, beta=1.0, uplo="lower")
    res = run_call(call, topo(2), RunOptions(record_trace=True), engine=FakeEngine(2))
    kinds = {e.event for e in res.trace}
    assert {"H2D", "D2H", "KERNEL"} <= kinds
    h2d = sum(e.bytes_or_flops for e in res.trace if e.event == "H2D")
    assert h2d == res.metrics.total_h2d_bytes()


def test_stealing_feeds_idle_device():
    from paper_1510_05041_b200 import scheduler as S
    call = build_call("gemm", m=16, n=16, k=16, tile_size=8, seed=1)
    plan = generate_tasks(call)
    rs0 = S.ReservationStation(0, 8)
    for t in plan.tasks[:3]:
        rs0.put(S._SlotEntry(t))

    class W:
        def __init__(self, d, rs, rt):
            self.device_id, self.rs, self.runtime = d, rs, rt

    class RT:
        queue = S.TaskQueue()
    rt = RT()
    w0, w1 = W(0, rs0, rt), W(1, S.ReservationStation(1, 8), rt)
    rt.workers = [w0, w1]
    got = S.steal_for(w1)
    assert got is not None and rs0.pending_count() == 2
    rt.queue.put((0, 0.0))
    assert S.steal_for(w1) is None                # queue not empty -> no theft
    rt.queue.get()
    assert S.steal_for(w1) is not None and S.steal_for(w1) is None   # victim keeps its last


def test_sgemm_plan_runs_in_fp32():
    call = build_call("gemm", m=40, n=24, k=36, tile_size=16, seed=6, beta=0.5,
                      dtype=np.float32, trans_b=True)
    a = call.a.matrix.as_2d().astype(np.float64)
    b = call.b.matrix.as_2d().astype(np.float64)
    c0 = call.c.matrix.as_2d().astype(np.float64)
    run_call(call, topo(2), RunOptions(), engine=FakeEngine(2))
    np.testing.assert_allclose(call.c.matrix.as_2d(), a @ b.T + 0.5 * c0, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("kind", ["gemm", "trsm", "trmm", "syr2k"])
def test_resident_mode_multi_device(kind):
    """arena_capacity=0 lets the runtime size the arena for the whole working set
    (resident mode: permanent pins, no per-task ALRU bookkeeping)."""
    call = build_call(kind, m=48, n=40, k=32, tile_size=8, seed=12, beta=0.5, uplo="lower",
                      trsm_scaled=True)
    a = call.a.matrix.as_2d().copy()
    b = call.b.matrix.as_2d().copy() if call.b is not None else None
    c0 = call.c.matrix.as_2d().copy()
    topo = Topology([DeviceDesc(i, arena_capacity=0, peer_group="g") for i in range(3)])
    res = run_call(call, topo, RunOptions(), engine=FakeEngine(3, seed=5, arena_bytes=1 << 26))
    from oracle import tiled
    ref = c0.copy()
    tiled.run_tiled(kind, a, ref, b, tile_size=8, alpha=1.0, beta=0.0 if kind in ("trsm", "trmm") else 0.5,
                    uplo="lower")
    np.testing.assert_allclose(call.c.matrix.as_2d(), ref, rtol=1e-11, atol=1e-11)
    m = res.metrics
    assert m.total_d2d_bytes() == sum(d.d2d_out_bytes for d in m.devices.values())
    if kind == "gemm":
        assert m.l2_hits > 0


@pytest.mark.parametrize("defer", [False, True])
@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] in ("gemm", "syrk", "syr2k", "symm")],
                         ids=lambda c: c["name"])
def test_deferred_c_move_in_matches_reference(case, defer):
    """beta*C0 applied by a final axpy launch (first GEMM at beta=0) vs the C tile moved in
    before the first launch: both match the reference output; diagonal rank-k tasks
    (triangle epilogue) keep the move-in, so the unstored triangle is written back intact."""
    from paper_1510_05041_b200.program import AxpyOp, compile_task
    call = call_of(case)
    eng = FakeEngine(2, seed=5)
    res = run_call(call, topo(2), RunOptions(chunk_steps=2, defer_c_move_in=defer,
                                             ramp_tasks=3, ramp_chunk_steps=1), engine=eng)
    np.testing.assert_allclose(call.c.matrix.as_2d(), case["out"], rtol=1e-12, atol=1e-12)
    for t in res.plan.tasks:
        prog = compile_task(t, res.plan.call, 2, 0, defer)
        has_axpy = any(type(o) is AxpyOp for o in prog.ops)
        if not defer or not t.needs_c_move_in:
            assert not has_axpy
        elif any(getattr(o, "tri", 0) for o in prog.ops):
            assert not has_axpy               # triangle epilogue: C moved in first
        else:
            assert has_axpy and prog.ops[-1] == AxpyOp(res.plan.call.beta)


@pytest.mark.parametrize("weight", [1, 100])
def test_trsm_critical_path_priority(weight):
    """Eq. 3 plus a critical-path term for the TRSM DAG.  Same numerics; the
    chain length below a left/lower task (i, j) is (tiles - 1 - i)."""
    from paper_1510_05041_b200.scheduler import critical_path
    call = build_call("trsm", m=96, n=64, k=96, tile_size=24, seed=5, uplo="lower",
                      trsm_scaled=True)
    x0 = call.c.matrix.as_2d().copy()
    a = call.a.matrix.as_2d()
    res = run_call(call, topo(2), RunOptions(critical_path_weight=weight), engine=FakeEngine(2, seed=9))
    x = call.c.matrix.as_2d()
    np.testing.assert_allclose(np.tril(a) @ x, x0, rtol=1e-10, atol=1e-10)
    for t in res.plan.tasks:
        assert critical_path(t, res.plan) == 4 - 1 - t.out_ref.i


def _fake_random_cases():
    import routine_cases as G
    return G.random_cases(24, seed=77)


@pytest.mark.parametrize("case", _fake_random_cases(), ids=lambda c: f"r{c[0]}_{c[1]}")
def test_randomized_routines_fake_engine(case):
    """The GPU randomized sweep's case generator on the fake engine (2 devices, randomised
    stream interleaving): runtime options x routines x ragged shapes vs the oracle."""
    from oracle import tiled as OT
    from oracle import tolerance as TOL
    _, kind, m, n, k, t, kw, opts = case
    call = build_call(kind, m=m, n=n, k=k, tile_size=t, seed=m * 7 + n, trsm_scaled=True, **kw)
    a = call.a.matrix.as_2d().copy()
    b = call.b.matrix.as_2d().copy() if call.b is not None else None
    c0 = call.c.matrix.as_2d().copy()
    res = run_call(call, topo(2, arena=64 << 20), RunOptions(**opts), engine=FakeEngine(2, seed=m))
    assert sum(res.tasks_by_device.values()) == len(res.plan.tasks)
    p = dict(kw)
    alpha, beta = p.pop("alpha", 1.0), p.pop("beta", 0.0)
    ref = c0.copy()
    OT.run_tiled(kind, a, ref, b, tile_size=t, alpha=alpha, beta=beta, **p)
    np.testing.assert_allclose(call.c.matrix.as_2d(), ref, rtol=1e-10,
                               atol=1e-10 * max(1.0, float(np.max(np.abs(ref)))))


@pytest.mark.parametrize("ndev", [1, 2])
@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "trsm"], ids=lambda c: c["name"])
def test_trsm_inverse_path_matches_reference(case, ndev):
    """The inverse-based diagonal step (X = alpha inv(E) B, inv(E) computed once per
    diagonal tile) forced on every tile order, resident arenas: same results as the
    reference's substitution (every side / uplo / trans / diag variant)."""
    call = call_of(case)
    topo_r = Topology([DeviceDesc(i, peer_group="g") for i in range(ndev)])
    eng = FakeEngine(ndev, seed=len(case["name"]), arena_bytes=1 << 24)
    res = run_call(call, topo_r, RunOptions(chunk_steps=2, trsm_inverse_min=1), engine=eng)
    np.testing.assert_allclose(call.c.matrix.as_2d(), case["out"], rtol=1e-10, atol=1e-10)
    assert sum(res.tasks_by_device.values()) == len(res.plan.tasks)


def test_trsm_inverse_computed_once_per_diagonal_tile():
    call = build_call("trsm", m=64, n=96, k=64, tile_size=16, seed=3, uplo="lower",
                      trsm_scaled=True)
    eng = FakeEngine(1, seed=1, arena_bytes=1 << 24)
    calls = []
    orig = eng.trsm_inverse

    def spy(*a, **kw):
        calls.append(a[7] if len(a) > 7 else None)
        return orig(*a, **kw)
    eng.trsm_inverse = spy
    a = call.a.matrix.as_2d().copy()
    c0 = call.c.matrix.as_2d().copy()
    run_call(call, Topology([DeviceDesc(0)]), RunOptions(trsm_inverse_min=1), engine=eng)
    assert len(calls) == 4                     # 4 diagonal tiles, 6 tile columns each
    from oracle import tiled
    ref = c0.copy()
    tiled.run_tiled("trsm", a, ref, None, tile_size=16, alpha=1.0, uplo="lower")
    np.testing.assert_allclose(call.c.matrix.as_2d(), ref, rtol=1e-11, atol=1e-11)


def test_trsm_inverse_path_raises_singular():
    call = build_call("trsm", m=48, n=32, k=48, tile_size=16, seed=2, uplo="lower",
                      trsm_scaled=True)
    call.a.matrix.as_2d()[20, 20] = 0.0
    with pytest.raises(SingularMatrixError):
        run_call(call, Topology([DeviceDesc(0)]), RunOptions(trsm_inverse_min=1),
                 engine=FakeEngine(1, seed=1, arena_bytes=1 << 24))


@pytest.mark.parametrize("release", [True, False])
@pytest.mark.parametrize("ndev", [1, 3])
@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "trsm"], ids=lambda c: c["name"])
def test_trsm_release_on_issue_matches_reference(case, ndev, release, monkeypatch):
    """Release-on-issue (resident arenas): a solved tile is cached and its dependents
    released when its solve is enqueued, their launches (or peers' P2P copies) waiting on
    the solve's event on the device.  The randomised stream order of the fake engine
    exposes a missing wait as wrong numbers; both settings give the reference's output."""
    from paper_1510_05041_b200 import scheduler as S
    released = []
    orig = S._Runtime.release_dependents

    def spy(self, task, at_time=0.0):
        released.append(task.task_id)
        return orig(self, task, at_time)
    monkeypatch.setattr(S._Runtime, "release_dependents", spy)
    call = call_of(case)
    topo_r = Topology([DeviceDesc(i, peer_group="g") for i in range(ndev)])
    eng = FakeEngine(ndev, seed=len(case["name"]) + ndev, arena_bytes=1 << 24)
    res = run_call(call, topo_r, RunOptions(chunk_steps=2, release_on_issue=release,
                                            trsm_inverse_min=1 if ndev == 1 else 0), engine=eng)
    np.testing.assert_allclose(call.c.matrix.as_2d(), case["out"], rtol=1e-10, atol=1e-10)
    assert sum(res.tasks_by_device.values()) == len(res.plan.tasks)
    with_deps = [t.task_id for t in res.plan.tasks if t.dependents]
    assert sorted(released) == (sorted(with_deps) if release else [])


def test_trsm_release_on_issue_singular_still_raises():
    """A zero diagonal is still reported (at the producer's retirement) when dependents
    were released at issue."""
    a = np.tril(np.random.default_rng(0).uniform(-1, 1, (32, 32))) + 4 * np.eye(32)
    a[5, 5] = 0.0
    b = np.random.default_rng(1).uniform(-1, 1, (32, 16))
    call = RoutineCall("trsm", a=make_tiled(MatrixDesc.from_array("A", a), 8),
                       b=None, c=make_tiled(MatrixDesc.from_array("C", b), 8), uplo="lower")
    with pytest.raises(SingularMatrixError):
        run_call(call, Topology([DeviceDesc(0)]), RunOptions(chunk_steps=2, trsm_inverse_min=0,
                                                             release_on_issue=True),
                 engine=FakeEngine(1, seed=2, arena_bytes=1 << 24))


@pytest.mark.parametrize("split", ["l2_off", "two_groups"])
def test_trsm_release_on_issue_off_without_shared_l2(split, monkeypatch):
    """Dependents on another GPU would read a solved tile from the host before its
    write-back: with L2 off or GPUs in separate peer groups release-on-issue stays off
    (and the results stay exact)."""
    from paper_1510_05041_b200 import scheduler as S
    released = []
    monkeypatch.setattr(S._Runtime, "release_dependents",
                        lambda self, task, at_time=0.0: released.append(task.task_id))
    call = build_call("trsm", m=64, n=96, k=64, tile_size=16, seed=9, uplo="lower",
                      trsm_scaled=True)
    a = call.a.matrix.as_2d().copy()
    c0 = call.c.matrix.as_2d().copy()
    groups = ["g", "g", "g"] if split == "l2_off" else ["g", "h", "h"]
    topo_r = Topology([DeviceDesc(i, peer_group=g) for i, g in enumerate(groups)])
    run_call(call, topo_r, RunOptions(chunk_steps=2, l2_enabled=split != "l2_off",
                                      release_on_issue=True),
             engine=FakeEngine(3, seed=4, arena_bytes=1 << 24))
    assert released == []
    from oracle import tiled
    ref = c0.copy()
    tiled.run_tiled("trsm", a, ref, None, tile_size=16, alpha=1.0, uplo="lower")
    np.testing.assert_allclose(call.c.matrix.as_2d(), ref, rtol=1e-11, atol=1e-11)


def _spy_ic(eng):
    calls = {"gemm": 0, "resolve": 0}
    for name in ("gemm", "resolve"):
        orig = getattr(eng, "ic_" + name)

        def spy(*a, _o=orig, _n=name, **kw):
            calls[_n] += 1
            return _o(*a, **kw)
        setattr(eng, "ic_" + name, spy)
    return calls


@pytest.mark.parametrize("execution", ["deterministic", "concurrent"])
@pytest.mark.parametrize("groups", [("g",), ("g", "g", "g"), ("g", "h", "h"), ("g", "g", "g", "g")])
@pytest.mark.parametrize("kind,kw", [("gemm", dict(trans_b=True)), ("syrk", {}),
                                     ("syr2k", dict(uplo="upper", trans_a=True)),
                                     ("symm", dict(side="right", uplo="upper"))])
def test_resident_issue_engine_matches_oracle(kind, kw, groups, execution):
    """The resident issue engine (bx_ic_*: tile ids in, translation + copies + launch in
    one engine call) on resident arenas: every routine it serves, 1-4 GPUs, split peer
    groups, both driver modes, random stream order — exact against the oracle, and every
    input tile crosses the host link once per peer group."""
    from oracle import tiled as OT
    ndev = len(groups)
    call = build_call(kind, m=112, n=96, k=80 if kind != "symm" else 112, tile_size=16, seed=ndev,
                      alpha=0.75, beta=0.5, **kw)
    a = call.a.matrix.as_2d().copy()
    b = call.b.matrix.as_2d().copy() if call.b is not None else None
    c0 = call.c.matrix.as_2d().copy()
    eng = FakeEngine(ndev, seed=11 + ndev, arena_bytes=1 << 24)
    calls = _spy_ic(eng)
    topo_r = Topology([DeviceDesc(i, peer_group=g) for i, g in enumerate(groups)])
    res = run_call(call, topo_r, RunOptions(chunk_steps=2, execution=execution), engine=eng)
    assert calls["gemm"] > 0
    p = dict(kw)
    ref = c0.copy()
    OT.run_tiled(kind, a, ref, b, tile_size=16, alpha=0.75, beta=0.5, **p)
    np.testing.assert_allclose(call.c.matrix.as_2d(), ref, rtol=1e-12, atol=1e-12)
    m = res.metrics
    n_inputs = len({k for t in res.plan.tasks for k in __import__(
        "paper_1510_05041_b200.scheduler", fromlist=["task_keys"]).task_keys(t)})
    # each tile crosses the host link at most once per peer group (exactly once with one)
    assert m.host_fetches <= n_inputs * len(set(groups))
    if len(set(groups)) == 1:
        assert m.host_fetches == n_inputs
    assert m.total_d2d_bytes() == sum(d.d2d_out_bytes for d in m.devices.values())


def test_resident_issue_engine_off_paths():
    """Not used where it does not apply: an explicit (evicting) arena, tracing, TRSM/TRMM,
    BX_IC=0 — those take the Python translation path, with the same results."""
    for opts, kind, arena in ((RunOptions(chunk_steps=2), "gemm", 8 << 20),
                              (RunOptions(chunk_steps=2, record_trace=True), "gemm", 0),
                              (RunOptions(chunk_steps=2), "trsm", 0),
                              (RunOptions(chunk_steps=2), "trmm", 0)):
        call = build_call(kind, m=64, n=48, k=64, tile_size=16, seed=1, trsm_scaled=True)
        eng = FakeEngine(2, seed=3, arena_bytes=1 << 24)
        calls = _spy_ic(eng)
        topo_r = Topology([DeviceDesc(i, peer_group="g", arena_capacity=arena)
                           for i in range(2)])
        run_call(call, topo_r, opts, engine=eng)
        assert calls == {"gemm": 0, "resolve": 0}, (kind, opts)


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "trsm"], ids=lambda c: c["name"])
def test_trsm_split_chain_matches_reference(case, split):
    """RunOptions.trsm_split_chain: the update step that reads the chain predecessor's
    solved tile runs as its own launch (program.compile_task) — same results on every
    side / uplo / trans / diag variant, with and without release-on-issue."""
    from paper_1510_05041_b200.program import GemmOp, TrsmOp, compile_task
    call = call_of(case)
    eng = FakeEngine(2, seed=len(case["name"]) + 3, arena_bytes=1 << 24)
    topo_r = Topology([DeviceDesc(i, peer_group="g") for i in range(2)])
    res = run_call(call, topo_r, RunOptions(chunk_steps=4, trsm_split_chain=split), engine=eng)
    np.testing.assert_allclose(call.c.matrix.as_2d(), case["out"], rtol=1e-10, atol=1e-10)
    pc = res.plan.call
    for t in res.plan.tasks:
        prog = compile_task(t, pc, 4, 0, False, split)
        gemms = [o for o in prog.ops if type(o) is GemmOp]
        assert type(prog.ops[-1]) is TrsmOp
        n_upd = len(t.steps) - 1
        assert sum(len(g.subs) for g in gemms) == n_upd          # every update step, once
        toward = n_upd >= 2 and abs(t.steps[-2].k - t.steps[-1].k) == 1
        if split and toward:
            assert len(gemms[-1].subs) == 1 and gemms[-1].subs[0][0] == t.steps[-2].a.key()
            assert len(gemms) == -(-(n_upd - 1) // 4) + 1
        else:
            assert len(gemms) == -(-n_upd // 4)


def test_trsm_split_chain_cfg4_shape():
    """cfg4 (left / lower / notrans): task (i, j) updates k = 0..i-1 then solves; with the
    split its last launch is the k = i-1 step alone."""
    from paper_1510_05041_b200.program import GemmOp, compile_task
    call = build_call("trsm", m=64, n=32, k=64, tile_size=8, seed=1, uplo="lower", trsm_scaled=True)
    from paper_1510_05041_b200.routines import generate_tasks
    plan = generate_tasks(call)
    for t in plan.tasks:
        i = t.out_ref.i
        prog = compile_task(t, call, 16, 0, False, True)
        gemms = [o for o in prog.ops if type(o) is GemmOp]
        if i >= 2:
            assert [len(g.subs) for g in gemms] == [i - 1, 1]
        elif i == 1:
            assert [len(g.subs) for g in gemms] == [1]
        else:
            assert gemms == []


@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "trmm"], ids=lambda c: c["name"])
def test_split_km_trmm_matches_reference(case):
    """RunOptions.split_km: TRMM diagonal (triangular-operand) steps run as launches of
    their own; plain steps never share a launch with them; same results."""
    from paper_1510_05041_b200.program import KM_NONE, GemmOp, compile_task
    call = call_of(case)
    eng = FakeEngine(2, seed=len(case["name"]) + 11, arena_bytes=1 << 24)
    topo_r = Topology([DeviceDesc(i, peer_group="g") for i in range(2)])
    res = run_call(call, topo_r, RunOptions(chunk_steps=4, split_km=True), engine=eng)
    np.testing.assert_allclose(call.c.matrix.as_2d(), case["out"], rtol=1e-10, atol=1e-10)
    for t in res.plan.tasks:
        prog = compile_task(t, res.plan.call, 4, 0, False, False, True)
        for g in (o for o in prog.ops if type(o) is GemmOp):
            kms = {km != KM_NONE for _, _, _, km in g.subs}
            assert len(kms) == 1


@pytest.mark.parametrize("kind", ["gemm", "syrk", "syr2k", "symm"])
@pytest.mark.parametrize("prefetch", [-1, 0, 1])
def test_small_call_prefetch(kind, prefetch, monkeypatch):
    """RunOptions.prefetch: a small call on one GPU (resident issue engine) loads every
    input tile at the start in first-use order; results, H2D bytes (each tile once) and
    the task count are those of the unprefetched call."""
    call = build_call(kind, m=96, n=80, k=72, tile_size=24, seed=4, beta=1.0, uplo="lower")
    c0 = call.c.matrix.as_2d().copy()
    eng = FakeEngine(1, seed=17, arena_bytes=1 << 24)
    import paper_1510_05041_b200.scheduler as S
    calls, inside = [], [False]
    orig, real_prefetch = eng.ic_resolve, S._ic_prefetch

    def spy(table, d, tids):
        if inside[0]:
            calls.append(list(tids))
        return orig(table, d, tids)

    def prefetch_spy(*a):
        inside[0] = True
        try:
            real_prefetch(*a)
        finally:
            inside[0] = False
    eng.ic_resolve = spy
    monkeypatch.setattr(S, "_ic_prefetch", prefetch_spy)
    topo1 = Topology([DeviceDesc(0)])
    res = run_call(call, topo1, RunOptions(prefetch=prefetch), engine=eng)
    out = call.c.matrix.as_2d().copy()
    call.c.matrix.as_2d()[:] = c0
    ref = run_call(call, topo1, RunOptions(prefetch=0), engine=FakeEngine(1, seed=3, arena_bytes=1 << 24))
    np.testing.assert_allclose(out, call.c.matrix.as_2d(), rtol=1e-13, atol=1e-13)
    assert res.metrics.total_h2d_bytes() == ref.metrics.total_h2d_bytes()
    assert res.metrics.host_fetches == ref.metrics.host_fetches
    n_inputs = len(res.plan.tasks[0]._bx_icgeom)
    if prefetch != 0:                   # 1 and auto (this call has < 64 tasks)
        assert calls and sorted(t for c in calls for t in c) == list(range(n_inputs))
    else:
        assert not calls


def test_prefetch_only_on_one_gpu_and_small_calls():
    from paper_1510_05041_b200.scheduler import LINK_BOUND_CALL_TASKS
    call = build_call("gemm", m=96, n=80, k=72, tile_size=24, seed=4, beta=1.0)
    eng = FakeEngine(2, seed=1, arena_bytes=1 << 24)
    seen = []
    orig = eng.ic_resolve
    eng.ic_resolve = lambda *a: (seen.append(a), orig(*a))[1]
    run_call(call, Topology([DeviceDesc(i, peer_group="g") for i in range(2)]),
             RunOptions(prefetch=1), engine=eng)
    assert not seen                                # two GPUs: no prefetch

    big = build_call("gemm", m=12 * 24, n=12 * 24, k=48, tile_size=24, seed=2, beta=0.0)
    eng1 = FakeEngine(1, seed=1, arena_bytes=1 << 24)
    seen1 = []
    orig1 = eng1.ic_resolve
    eng1.ic_resolve = lambda *a: (seen1.append(a), orig1(*a))[1]
    res = run_call(big, Topology([DeviceDesc(0)]), RunOptions(), engine=eng1)
    assert len(res.plan.tasks) > LINK_BOUND_CALL_TASKS and not seen1   # auto: large call, none


@pytest.mark.parametrize("kind", ["gemm", "syrk", "syr2k", "symm", "trmm"])
def test_rampdown_batch_matches_reference(kind):
    """RunOptions.rampdown_tasks: the last tasks start together in extra slots with short
    launches; same results, every task once."""
    call = build_call(kind, m=192, n=192, k=96, tile_size=24, seed=8, beta=1.0 if kind != "trmm" else 0.0,
                      uplo="lower", trsm_scaled=True)
    a = call.a.matrix.as_2d().copy()
    b = call.b.matrix.as_2d().copy() if call.b is not None else None
    c0 = call.c.matrix.as_2d().copy()
    eng = FakeEngine(1, seed=21, arena_bytes=1 << 26)
    res = run_call(call, Topology([DeviceDesc(0)]),
                   RunOptions(rampdown_tasks=12, ramp_chunk_steps=1, prefetch=0), engine=eng)
    assert sum(res.tasks_by_device.values()) == len(res.plan.tasks)
    from oracle import tiled as OT
    ref = c0.copy()
    OT.run_tiled(kind, a, ref, b, tile_size=24, alpha=1.0, beta=1.0 if kind != "trmm" else 0.0,
                 uplo="lower")
    np.testing.assert_allclose(call.c.matrix.as_2d(), ref, rtol=1e-11, atol=1e-11)


@pytest.mark.parametrize("kind", ["gemm", "syrk", "syr2k", "symm"])
def test_prefetch_window_large_call(kind):
    """RunOptions.prefetch_window_mb on a large one-GPU call (> LINK_BOUND_CALL_TASKS tasks):
    first-use loads kept ahead of the tasks; results and host bytes as without it."""
    from paper_1510_05041_b200.scheduler import LINK_BOUND_CALL_TASKS
    call = build_call(kind, m=12 * 16, n=12 * 16, k=64, tile_size=16, seed=3, beta=1.0, uplo="lower")
    c0 = call.c.matrix.as_2d().copy()
    topo1 = Topology([DeviceDesc(0)])
    res = run_call(call, topo1, RunOptions(prefetch_window_mb=1), engine=FakeEngine(1, seed=5, arena_bytes=1 << 24))
    out = call.c.matrix.as_2d().copy()
    call.c.matrix.as_2d()[:] = c0
    ref = run_call(call, topo1, RunOptions(), engine=FakeEngine(1, seed=6, arena_bytes=1 << 24))
    assert len(res.plan.tasks) > LINK_BOUND_CALL_TASKS or kind in ("syrk", "syr2k")
    np.testing.assert_allclose(out, call.c.matrix.as_2d(), rtol=1e-12, atol=1e-12)
    assert res.metrics.total_h2d_bytes() == ref.metrics.total_h2d_bytes()
