"""Generate golden fixtures by running the REFERENCE implementation (tileblas) itself.

Run in the build container only (needs /root/reference, read-only):
    python tests/golden/make_golden.py
Writes tests/golden/*.npz / *.json.  The GPU box never runs this; tests there read
the committed fixtures.

Fixtures
--------
variants.npz   every parameter variant the reference suite sweeps
               (/root/reference/pkg/tests/conftest.py:62-82) at edge-tile shapes,
               inputs and the reference ``run_call`` output (1 and 2 simulated devices).
plans.json     the reference planner's TaskPlan for the same calls
               (task coords, step kinds, tile keys, transposes, alpha/beta, flops,
               needs_c_move_in, TRSM dependency edges).
plan_stats.json task/step/flop/edge counts of the BASELINE configs (planner only).
cfg1.npz       cfg1 (DGEMM 2048^3 NN, T=512, alpha=beta=1, seed 0): checksums of the
               reference run_call output (column/row sums, norm, a sampled block).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import tileblas  # noqa: E402
from tileblas import (DeviceDesc, RoutineCall, RunOptions, Topology,  # noqa: E402
                      build_call, generate_tasks, run_call)
from tileblas.tiling import MatrixDesc, make_tiled  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# /root/reference/pkg/tests/conftest.py:62-82
VARIANTS = [
    ("gemm", dict(trans_a=False, trans_b=False, alpha=1.0, beta=0.0)),
    ("gemm", dict(trans_a=True, trans_b=False, alpha=-0.7, beta=1.0)),
    ("gemm", dict(trans_a=False, trans_b=True, alpha=2.0, beta=0.3)),
    ("gemm", dict(trans_a=True, trans_b=True, alpha=1.1, beta=-0.4)),
    ("syrk", dict(uplo="upper", trans_a=False, alpha=1.0, beta=0.5)),
    ("syrk", dict(uplo="lower", trans_a=True, alpha=-1.2, beta=0.0)),
    ("syr2k", dict(uplo="upper", trans_a=True, alpha=0.9, beta=1.0)),
    ("syr2k", dict(uplo="lower", trans_a=False, alpha=1.0, beta=-0.2)),
    ("syr2k", dict(uplo="upper", trans_a=False, alpha=1.0, beta=0.0)),
    ("symm", dict(uplo="upper", side="left", alpha=1.3, beta=0.6)),
    ("symm", dict(uplo="lower", side="right", alpha=-1.0, beta=0.0)),
    ("trmm", dict(uplo="upper", side="left", trans_a=False, diag="non-unit", alpha=1.0)),
    ("trmm", dict(uplo="lower", side="left", trans_a=True, diag="unit", alpha=-0.8)),
    ("trmm", dict(uplo="upper", side="right", trans_a=True, diag="non-unit", alpha=0.5)),
    ("trmm", dict(uplo="lower", side="right", trans_a=False, diag="unit", alpha=1.0)),
    ("trsm", dict(uplo="upper", side="left", trans_a=False, diag="non-unit", alpha=1.0)),
    ("trsm", dict(uplo="lower", side="left", trans_a=True, diag="unit", alpha=-0.9)),
    ("trsm", dict(uplo="upper", side="right", trans_a=True, diag="unit", alpha=1.5)),
    ("trsm", dict(uplo="lower", side="right", trans_a=False, diag="non-unit", alpha=1.0)),
]

# edge-tile shapes: m, n, k not multiples of the tile size
SHAPES = [dict(m=13, n=11, k=10, tile_size=4), dict(m=9, n=9, k=9, tile_size=3)]


def rand(rng, r, c):
    return rng.random((r, c)) * 2.0 - 1.0


def make_arrays(rng, kind, m, n, k, p):
    side = p.get("side", "left")
    q = m if side == "left" else n
    ta, tb = p.get("trans_a", False), p.get("trans_b", False)
    if kind == "gemm":
        a = rand(rng, *((k, m) if ta else (m, k)))
        b = rand(rng, *((n, k) if tb else (k, n)))
        c = rand(rng, m, n)
    elif kind in ("syrk", "syr2k"):
        a = rand(rng, *((k, n) if ta else (n, k)))
        b = rand(rng, *a.shape) if kind == "syr2k" else None
        c = rand(rng, n, n)
    elif kind == "symm":
        a, b, c = rand(rng, q, q), rand(rng, m, n), rand(rng, m, n)
    else:
        a = rand(rng, q, q)
        if kind == "trsm":
            d = np.diagonal(a).copy()
            np.fill_diagonal(a, np.sign(d + (d == 0)) * (1.0 + np.abs(d)))
        b, c = None, rand(rng, m, n)
    return a, b, c


def make_call(kind, a, b, c, tile_size, pad, p):
    def tiled(mid, arr):
        return make_tiled(MatrixDesc.from_array(mid, arr, pad=pad), tile_size)
    return RoutineCall(kind=kind, a=tiled("A", a), b=None if b is None else tiled("B", b),
                       c=tiled("C", c), **p)


def plan_to_json(plan):
    out = []
    for t in plan.tasks:
        out.append(dict(
            task_id=t.task_id, i=t.i, j=t.j, needs_c_move_in=t.needs_c_move_in,
            deps_remaining=t.deps_remaining, dependents=list(t.dependents), flops=t.flops,
            out=[t.out_ref.matrix_id, t.out_ref.i, t.out_ref.j, t.out_ref.height, t.out_ref.width],
            steps=[dict(k=s.k, kind=s.kind,
                        a=[s.a.matrix_id, s.a.i, s.a.j, s.a.height, s.a.width, s.a.transposed],
                        b=None if s.b is None else [s.b.matrix_id, s.b.i, s.b.j, s.b.height,
                                                    s.b.width, s.b.transposed],
                        alpha=s.alpha, beta=s.beta, flops=s.flops) for s in t.steps]))
    return dict(tasks=out, total_flops=plan.total_flops)


def main():
    rng = np.random.default_rng(20151016)
    arrays, plans = {}, {}
    for si, shape in enumerate(SHAPES):
        for vi, (kind, p) in enumerate(VARIANTS):
            name = f"s{si}_v{vi:02d}_{kind}"
            a, b, c = make_arrays(rng, kind, shape["m"], shape["n"], shape["k"], p)
            pad = 2 if vi % 2 else 0
            outs = []
            for ndev in (1, 2):
                call = make_call(kind, a, b, c.copy(), shape["tile_size"], pad, p)
                topo = Topology([DeviceDesc(d, peer_group="g" if ndev > 1 else None)
                                 for d in range(ndev)])
                run_call(call, topo, RunOptions())
                outs.append(call.c.matrix.as_2d().copy())
            assert np.array_equal(outs[0], outs[1]) or np.allclose(outs[0], outs[1], rtol=1e-13)
            arrays[name + "__a"] = a
            if b is not None:
                arrays[name + "__b"] = b
            arrays[name + "__c"] = c
            arrays[name + "__out"] = outs[0]
            call = make_call(kind, a, b, c.copy(), shape["tile_size"], pad, p)
            plans[name] = dict(kind=kind, params=p, shape=shape, pad=pad,
                               plan=plan_to_json(generate_tasks(call)))
    np.savez_compressed(os.path.join(HERE, "variants.npz"), **arrays)
    with open(os.path.join(HERE, "plans.json"), "w") as f:
        json.dump(plans, f, indent=0, sort_keys=True)

    # planner statistics at the BASELINE configs (no numerics: tiny storage + stride 0
    # is not allowed by MatrixDesc, so build real but small-dtype-irrelevant descs lazily)
    stats = {}
    cfgs = [("cfg1_gemm", "gemm", dict(m=2048, n=2048, k=2048, tile_size=512, beta=1.0)),
            ("cfg2_gemm", "gemm", dict(m=16384, n=16384, k=16384, tile_size=1024, beta=1.0)),
            ("cfg3_syrk", "syrk", dict(m=16384, n=16384, k=8192, tile_size=1024, beta=1.0, uplo="lower")),
            ("cfg3_syr2k", "syr2k", dict(m=16384, n=16384, k=8192, tile_size=1024, beta=1.0, uplo="lower")),
            ("cfg4_trsm", "trsm", dict(m=16384, n=16384, k=16384, tile_size=1024, uplo="lower")),
            ("cfg4_trmm", "trmm", dict(m=16384, n=16384, k=16384, tile_size=1024, uplo="lower"))]
    for name, kind, kw in cfgs:
        m, n, k, t = kw.pop("m"), kw.pop("n"), kw.pop("k"), kw.pop("tile_size")

        def tm(mid, r, c):
            # one-column-stride trick keeps memory tiny: storage only needs ld*cols elements,
            # so use a shared zero buffer large enough (planner never reads values)
            return make_tiled(MatrixDesc(mid, r, c, r, _zeros(r * c)), t)
        q = m
        if kind == "gemm":
            call = RoutineCall(kind, a=tm("A", m, k), b=tm("B", k, n), c=tm("C", m, n), **kw)
        elif kind == "syrk":
            call = RoutineCall(kind, a=tm("A", n, k), c=tm("C", n, n), **kw)
        elif kind == "syr2k":
            call = RoutineCall(kind, a=tm("A", n, k), b=tm("B", n, k), c=tm("C", n, n), **kw)
        else:
            call = RoutineCall(kind, a=tm("A", q, q), c=tm("C", m, n), **kw)
        plan = generate_tasks(call)
        kinds = {}
        for tsk in plan.tasks:
            for s in tsk.steps:
                kinds[s.kind] = kinds.get(s.kind, 0) + 1
        stats[name] = dict(tasks=len(plan.tasks), steps=sum(len(x.steps) for x in plan.tasks),
                           total_flops=plan.total_flops, step_kinds=kinds,
                           dep_edges=sum(len(x.dependents) for x in plan.tasks),
                           initially_ready=len(plan.initially_ready()),
                           c_move_in=sum(1 for x in plan.tasks if x.needs_c_move_in))
    with open(os.path.join(HERE, "plan_stats.json"), "w") as f:
        json.dump(stats, f, indent=1, sort_keys=True)

    # cfg1 through the reference runtime (BASELINE configs[0]); operands from build_call
    call = build_call("gemm", m=2048, n=2048, k=2048, tile_size=512, seed=0, alpha=1.0, beta=1.0)
    descs = {x: getattr(call, x).matrix for x in ("a", "b", "c")}
    a0 = descs["a"].as_2d().copy()
    lds = {x: descs[x].leading_dim for x in descs}
    run_call(call, Topology([DeviceDesc(0, arena_capacity=4 << 30)]))
    out = call.c.matrix.as_2d()
    np.savez_compressed(
        os.path.join(HERE, "cfg1.npz"),
        colsum=out.sum(axis=0), rowsum=out.sum(axis=1), fro=np.linalg.norm(out),
        block=out[:64, :64].copy(), block2=out[-64:, 1000:1064].copy(),
        a_colsum=a0.sum(axis=0), lda=lds["a"], ldb=lds["b"], ldc=lds["c"])
    print("wrote fixtures to", HERE)


_ZBUF = {}


def _zeros(n):
    buf = _ZBUF.get("z")
    if buf is None or buf.size < n:
        buf = np.zeros(n)
        _ZBUF["z"] = buf
    return buf[:n]


if __name__ == "__main__":
    main()
