"""Planner parity: our task DAG equals the reference planner's on every variant
(golden plans.json produced by /root/reference tileblas.generate_tasks)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_variants
from paper_1510_05041_b200.errors import InvalidArgumentError
from paper_1510_05041_b200.routines import (RoutineCall, degree_of_parallelism,
                                            gemm_flop_fraction, generate_tasks, morton_key,
                                            step_flops)
from paper_1510_05041_b200.tiling import MatrixDesc, make_tiled

CASES = load_variants()


def make_call(case):
    t = case["shape"]["tile_size"]

    def tiled(mid, arr):
        return make_tiled(MatrixDesc.from_array(mid, arr, pad=case["pad"]), t)
    return RoutineCall(kind=case["kind"], a=tiled("A", case["a"]),
                       b=None if case["b"] is None else tiled("B", case["b"]),
                       c=tiled("C", case["c"]), **case["params"])


def ref_tuple(r):
    return None if r is None else [r.matrix_id, r.i, r.j, r.height, r.width, r.transposed]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_plan_matches_reference(case):
    plan = generate_tasks(make_call(case))
    gold = case["plan"]
    assert plan.total_flops == gold["total_flops"]
    assert len(plan.tasks) == len(gold["tasks"])
    for t, g in zip(plan.tasks, gold["tasks"]):
        assert (t.task_id, t.i, t.j) == (g["task_id"], g["i"], g["j"])
        assert t.needs_c_move_in == g["needs_c_move_in"]
        assert t.deps_remaining == g["deps_remaining"]
        assert list(t.dependents) == g["dependents"]
        assert t.flops == g["flops"]
        assert [t.out_ref.matrix_id, t.out_ref.i, t.out_ref.j, t.out_ref.height,
                t.out_ref.width] == g["out"]
        assert len(t.steps) == len(g["steps"])
        for s, gs in zip(t.steps, g["steps"]):
            assert (s.k, s.kind, s.alpha, s.beta, s.flops) == (
                gs["k"], gs["kind"], gs["alpha"], gs["beta"], gs["flops"])
            assert ref_tuple(s.a) == gs["a"]
            assert ref_tuple(s.b) == gs["b"]


def test_baseline_config_plan_stats():
    with open(os.path.join(GOLDEN, "plan_stats.json")) as f:
        stats = json.load(f)
    zb = np.zeros(16384 * 16384)

    def tm(mid, r, c, t):
        return make_tiled(MatrixDesc(mid, r, c, r, zb[:r * c]), t)
    calls = {
        "cfg1_gemm": RoutineCall("gemm", a=tm("A", 2048, 2048, 512), b=tm("B", 2048, 2048, 512),
                                 c=tm("C", 2048, 2048, 512), beta=1.0),
        "cfg3_syr2k": RoutineCall("syr2k", a=tm("A", 16384, 8192, 1024), b=tm("B", 16384, 8192, 1024),
                                  c=tm("C", 16384, 16384, 1024), beta=1.0, uplo="lower"),
        "cfg4_trsm": RoutineCall("trsm", a=tm("A", 16384, 16384, 1024), c=tm("C", 16384, 16384, 1024),
                                 uplo="lower"),
    }
    for name, call in calls.items():
        plan = generate_tasks(call)
        s = stats[name]
        assert len(plan.tasks) == s["tasks"]
        assert sum(len(t.steps) for t in plan.tasks) == s["steps"]
        assert plan.total_flops == s["total_flops"]
        assert sum(len(t.dependents) for t in plan.tasks) == s["dep_edges"]
        assert len(plan.initially_ready()) == s["initially_ready"]


def test_degree_of_parallelism_brute_force():
    rng = np.random.default_rng(11)
    for _ in range(100):
        r, c, t = (int(x) for x in rng.integers(1, 200, 3))
        assert degree_of_parallelism(r, c, t) == sum(1 for _ in range(0, r, t) for _ in range(0, c, t))
    with pytest.raises(InvalidArgumentError):
        degree_of_parallelism(0, 3, 1)


def test_morton_first_quad():
    order = sorted([(i, j) for i in range(4) for j in range(4)], key=lambda p: morton_key(*p))
    assert order[:4] == [(0, 0), (0, 1), (1, 0), (1, 1)]
    assert set(order[4:8]) == {(0, 2), (0, 3), (1, 2), (1, 3)}


def test_step_flops_literals():
    assert step_flops("gemm_update", 2, 3, 4) == 48
    assert step_flops("syrk_update", 4, 4, 2) == 40
    assert step_flops("syr2k_update", 4, 4, 2) == 80
    assert step_flops("trsm_solve", 4, 2, 4) == 32
    assert step_flops("trmm_diag", 4, 2, 4) == 32
    with pytest.raises(InvalidArgumentError):
        step_flops("nope", 1, 1, 1)


def test_validation_errors(rng):
    def tm(mid, r, c):
        return make_tiled(MatrixDesc.from_array(mid, rng.random((r, c))), 4)
    with pytest.raises(InvalidArgumentError):
        generate_tasks(RoutineCall("gemm", a=tm("A", 4, 5), b=tm("B", 4, 4), c=tm("C", 4, 4)))
    with pytest.raises(InvalidArgumentError):
        generate_tasks(RoutineCall("syrk", a=tm("A", 4, 4), c=tm("C", 4, 4), trans_b=True))
    with pytest.raises(InvalidArgumentError):
        generate_tasks(RoutineCall("nope", a=tm("A", 4, 4), c=tm("C", 4, 4)))
    a = tm("A", 4, 4)
    with pytest.raises(InvalidArgumentError):
        generate_tasks(RoutineCall("gemm", a=a, b=a, c=tm("C", 4, 4)))


def test_gemm_flop_fraction_trend():
    zb = np.zeros(64 * 64)
    fr = []
    for n in (16, 32, 64):
        t = make_tiled(MatrixDesc("A", n, n, n, zb[:n * n]), 4)
        c = make_tiled(MatrixDesc("C", n, n, n, zb[:n * n].copy()), 4)
        fr.append(gemm_flop_fraction(generate_tasks(RoutineCall("syrk", a=t, c=c))))
    assert fr == sorted(fr) and fr[-1] > 0.9
