"""Rank entry points for the one-process-per-GPU tests (run in spawned processes by
``spmd.launch``; module-level so the children can import them)."""

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (HERE, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)

import numpy as np  # noqa: E402


def _reference(call):
    """Oracle result for rank 0 (the tiled restatement of the reference's numerics)."""
    from oracle import tiled
    a = call.a.matrix.as_2d().copy()
    c = call.c.matrix.as_2d().copy()
    b = call.b.matrix.as_2d().copy() if call.b is not None else None
    tiled.run_tiled(call.kind, a, c, b, tile_size=call.c.tile_size, alpha=call.alpha,
                    beta=call.beta, trans_a=call.trans_a, trans_b=call.trans_b, uplo=call.uplo,
                    side=call.side, diag=call.diag)
    return c


def run_case(kind, n, k, tile, seed, fake, options=None, extra=None):
    """Every rank: share the operands, run the call with execution="spmd", rank 0 checks
    the result against the oracle.  Returns per-rank facts for the parent to assert on."""
    from paper_1510_05041_b200 import RunOptions, build_call, run_call, spmd
    sess = spmd.init()
    call = None
    ref = None
    kw = dict(extra or {})
    if sess.rank == 0:
        call = build_call(kind, m=n, n=n, k=k, tile_size=tile, seed=seed, alpha=kw.pop("alpha", 1.0),
                          beta=kw.pop("beta", 1.0 if kind in ("gemm", "syrk", "syr2k", "symm") else 0.0),
                          uplo=kw.pop("uplo", "lower"), trsm_scaled=True, **kw)
        ref = _reference(call)
    call = sess.share_call(call)
    eng = None
    if fake:
        from fake_spmd import SpmdFakeEngine
        eng = SpmdFakeEngine(sess.rank, sess.job, seed=sess.rank + 7)
    opts = RunOptions(execution="spmd", **(options or {}))
    out = {}
    try:
        res = run_call(call, options=opts, engine=eng)
        if sess.rank == 0:
            got = call.c.matrix.as_2d()
            out["max_err"] = float(np.max(np.abs(got - ref)))
            out["scale"] = float(np.max(np.abs(ref)))
        m = res.metrics
        out.update(tasks=dict(res.tasks_by_device), h2d=m.total_h2d_bytes(),
                   d2d=m.total_d2d_bytes(), d2d_out=sum(d.d2d_out_bytes for d in m.devices.values()),
                   l2=m.l2_hits, host=m.host_fetches, n_tasks=len(res.plan.tasks))
        # a second call on the same session reuses arenas / IPC mappings
        if kind == "gemm":
            res2 = run_call(call, options=opts, engine=eng)
            out["second_tasks"] = sum(res2.tasks_by_device.values())
    except Exception as exc:   # reported as data so the parent can assert on the type
        out["error"] = type(exc).__name__
    finally:
        if eng is not None:
            eng.cleanup()
    return out


def run_singular(n, tile, fake):
    from paper_1510_05041_b200 import RunOptions, build_call, run_call, spmd
    sess = spmd.init()
    call = None
    if sess.rank == 0:
        call = build_call("trsm", m=n, n=n, k=n, tile_size=tile, seed=3, trsm_scaled=True)
        a = call.a.matrix.as_2d()
        a[n - 3, n - 3] = 0.0             # singular: the last diagonal tile's solve fails
    call = sess.share_call(call)
    eng = None
    if fake:
        from fake_spmd import SpmdFakeEngine
        eng = SpmdFakeEngine(sess.rank, sess.job)
    try:
        run_call(call, options=RunOptions(execution="spmd"), engine=eng)
        return "no error"
    except Exception as exc:
        return type(exc).__name__
    finally:
        if eng is not None:
            eng.cleanup()


def check_shared_required(fake):
    from paper_1510_05041_b200 import RunOptions, build_call, run_call, spmd
    spmd.init()
    call = build_call("gemm", m=64, n=64, k=64, tile_size=32, seed=0)
    eng = None
    if fake:
        from fake_spmd import SpmdFakeEngine
        eng = SpmdFakeEngine(0, "x")
    try:
        run_call(call, options=RunOptions(execution="spmd"), engine=eng)
        return "no error"
    except Exception as exc:
        return type(exc).__name__


def run_steal_stress(n, tile, calls, rs_capacity):
    """Every rank: several calls of one session with small stations (heavy stealing);
    returns per call (tasks executed by this rank, tasks in the plan, rank 0's max error)."""
    from paper_1510_05041_b200 import RunOptions, build_call, run_call, spmd
    from fake_spmd import SpmdFakeEngine
    sess = spmd.init()
    call = ref = None
    if sess.rank == 0:
        call = build_call("gemm", m=n, n=n, k=n // 2, tile_size=tile, seed=3, alpha=1.0, beta=1.0)
    call = sess.share_call(call)
    eng = SpmdFakeEngine(sess.rank, sess.job, seed=sess.rank * 31 + 1)
    out = []
    try:
        for _ in range(calls):
            if sess.rank == 0:
                ref = _reference(call)
            sess.barrier("reference taken")
            res = run_call(call, options=RunOptions(execution="spmd", rs_capacity=rs_capacity),
                           engine=eng)
            err = None
            if sess.rank == 0:
                err = float(np.max(np.abs(call.c.matrix.as_2d() - ref)) / max(1.0, np.max(np.abs(ref))))
            out.append((res.tasks_by_device[sess.rank], len(res.plan.tasks), err))
            sess.barrier("call checked")
    finally:
        eng.cleanup()
    return out


def run_size_sequence(sizes, tile, fake):
    """Every rank: one session, calls of alternating sizes (the pooled call files are reused
    by alternate calls and grown when a larger call comes); rank 0 checks each result.
    Returns, per call, (tasks this rank ran, tasks in the plan, rank 0's max error)."""
    from paper_1510_05041_b200 import RunOptions, build_call, run_call, spmd
    sess = spmd.init()
    eng = None
    if fake:
        from fake_spmd import SpmdFakeEngine
        eng = SpmdFakeEngine(sess.rank, sess.job, seed=sess.rank * 13 + 5)
    out = []
    try:
        for i, n in enumerate(sizes):
            call = ref = None
            if sess.rank == 0:
                call = build_call("gemm", m=n, n=n, k=n // 2, tile_size=tile, seed=i, alpha=1.0,
                                  beta=1.0)
                ref = _reference(call)
            call = sess.share_call(call)
            res = run_call(call, options=RunOptions(execution="spmd"), engine=eng)
            err = float(np.max(np.abs(call.c.matrix.as_2d() - ref))) if sess.rank == 0 else 0.0
            out.append((res.tasks_by_device[sess.rank], len(res.plan.tasks), err))
        return out
    finally:
        if eng is not None:
            eng.cleanup()
