"""Runtime safety on the fake engine: the TRMM snapshot may alias the live operand only
when no snapshot tile can be re-fetched from the host after its owner's write-back, calls
from several threads are serialised, and a call never mixes resident and evicting arenas.

TRMM reads its in-place operand through a snapshot taken at plan time
(/root/reference/pkg/src/tileblas/routines.py:393-400); every configuration below would
read an already-updated tile if the runtime aliased the snapshot."""

import threading

import numpy as np
import pytest

import spmd_cases as SC
from fake_engine import FakeEngine
from oracle import tiled
from paper_1510_05041_b200 import spmd
from paper_1510_05041_b200.devices import DeviceDesc, Topology
from paper_1510_05041_b200.operands import build_call
from paper_1510_05041_b200.scheduler import RunOptions, run_call


def _trmm(uplo, seed=3):
    call = build_call("trmm", m=128, n=64, k=128, tile_size=8, seed=seed, uplo=uplo,
                      trsm_scaled=True)
    a = call.a.matrix.as_2d().copy()
    c0 = call.c.matrix.as_2d().copy()
    ref = c0.copy()
    tiled.run_tiled("trmm", a, ref, None, tile_size=8, alpha=1.0, beta=0.0, uplo=uplo)
    return call, ref


TILE = 8 * 8 * 8
CONFIGS = {
    # 2 GPUs in one group, L2 off: each GPU fetches snapshot tiles from the host itself
    "two_gpus_l2_off": (lambda: Topology([DeviceDesc(i, peer_group="g") for i in range(2)]),
                        dict(l2_enabled=False), 2),
    # 3 GPUs in 3 peer groups: no L2 between them
    "split_peer_groups": (lambda: Topology([DeviceDesc(i, peer_group=f"g{i}") for i in range(3)]),
                          {}, 3),
    # L1 off: every reference is a fresh host fetch
    "l1_off": (lambda: Topology([DeviceDesc(i, peer_group="g") for i in range(2)]),
               dict(l1_enabled=False), 2),
    # one GPU with an evicting arena that holds the whole snapshot (128 tiles) but not the
    # working set: an evicted snapshot tile is re-fetched from the host
    "evicting_arena": (lambda: Topology([DeviceDesc(0, arena_capacity=180 * TILE)]), {}, 1),
    # mixed residency: one bounded arena, one auto-sized
    "mixed_residency": (lambda: Topology([DeviceDesc(0, arena_capacity=180 * TILE, peer_group="g"),
                                          DeviceDesc(1, peer_group="g")]), {}, 2),
}


@pytest.mark.parametrize("uplo", ["lower", "upper"])
@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_trmm_snapshot_never_reads_updated_tiles(name, uplo):
    topo_fn, opts, ndev = CONFIGS[name]
    for seed in range(3):
        call, ref = _trmm(uplo, seed)
        run_call(call, topo_fn(), RunOptions(chunk_steps=2, n_streams=2, **opts),
                 engine=FakeEngine(ndev, seed=11 + seed, arena_bytes=1 << 24))
        np.testing.assert_allclose(call.c.matrix.as_2d(), ref, rtol=1e-12, atol=1e-12)


def test_trmm_alias_kept_when_safe():
    """All-resident, one peer group, L2 on: the snapshot stays an alias (no host copy)."""
    from paper_1510_05041_b200 import scheduler as S
    from paper_1510_05041_b200.routines import generate_tasks
    call, ref = _trmm("lower")
    plan = generate_tasks(call, snapshot="alias")
    S.run_plan(plan, Topology([DeviceDesc(i, peer_group="g") for i in range(2)]),
               RunOptions(chunk_steps=2), engine=FakeEngine(2, seed=4, arena_bytes=1 << 24))
    assert plan.snapshot_alias is not None
    np.testing.assert_allclose(call.c.matrix.as_2d(), ref, rtol=1e-12, atol=1e-12)


def test_concurrent_callers_are_serialised():
    """Two threads each running DGEMMs through one engine: every call carves its tiles out
    of the same arena, so unserialised calls would overwrite each other's tiles."""
    import sys
    eng = FakeEngine(1, seed=2, arena_bytes=1 << 24)
    topo = Topology([DeviceDesc(0)])
    errs = []
    old = sys.getswitchinterval()
    sys.setswitchinterval(1e-6)       # interleave the callers as much as the GIL allows

    def worker(seed):
        try:
            for r in range(3):
                call = build_call("gemm", m=96, n=96, k=96, tile_size=16, seed=seed * 10 + r,
                                  beta=1.0)
                a, b = call.a.matrix.as_2d().copy(), call.b.matrix.as_2d().copy()
                c0 = call.c.matrix.as_2d().copy()
                run_call(call, topo, RunOptions(), engine=eng)
                errs.append(float(np.max(np.abs(call.c.matrix.as_2d() - (a @ b + c0)))))
        except BaseException as exc:     # surfaced below
            errs.append(exc)

    ts = [threading.Thread(target=worker, args=(s,)) for s in (1, 2, 3)]
    try:
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    finally:
        sys.setswitchinterval(old)
    assert len(errs) == 9
    assert all(isinstance(e, float) and e < 1e-12 for e in errs), errs


def test_spmd_trmm_without_l2_copies_snapshot():
    outs = spmd.launch(2, SC.run_case, "trmm", 192, 192, 64, 5, True, dict(l2_enabled=False),
                       None, timeout=600)
    errs = [o.get("error") for o in outs]
    assert errs == [None, None], errs
    assert outs[0]["max_err"] <= 1e-11 * max(1.0, outs[0]["scale"]), outs[0]
