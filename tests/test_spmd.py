"""One process per GPU (paper_1510_05041_b200/spmd.py): the shared task queue, stations
with cross-process stealing, first-holder directory with IPC peer copies gated by arrival
flags, cross-rank TRSM dependencies, and error propagation.

CPU: every rank is a spawned process on the fake engine with /dev/shm arenas (each rank
checks nothing itself; rank 0 compares the shared output with the oracle).  GPU: the same
cases with the real engine, several ranks sharing GPU 0 (IPC + stream memory operations on
hardware)."""

import os
import pytest

import spmd_cases as SC
from paper_1510_05041_b200 import spmd

CASES = [
    ("gemm", 192, 160, 64, {}),
    ("gemm", 200, 130, 64, dict(trans_a=True, trans_b=True, alpha=0.5, beta=-1.0)),
    ("syrk", 192, 96, 64, {}),
    ("syr2k", 160, 96, 64, dict(uplo="upper")),
    ("symm", 160, 160, 64, dict(side="right")),
    ("trmm", 192, 192, 64, {}),
    ("trsm", 192, 192, 64, {}),
    ("trsm", 160, 160, 64, dict(side="right", uplo="upper", trans_a=True)),
]


def _check(outs, world):
    errs = [o.get("error") for o in outs]
    assert errs == [None] * world, errs
    o0 = outs[0]
    assert o0["max_err"] <= 1e-11 * max(1.0, o0["scale"]), o0
    for o in outs:
        # every rank returns the same gathered metrics
        assert o["tasks"] == o0["tasks"] and o["h2d"] == o0["h2d"]
        assert sum(o["tasks"].values()) == o["n_tasks"]      # every task exactly once
        assert o["d2d"] == o["d2d_out"]                     # peer bytes in == out


@pytest.mark.parametrize("kind,n,k,tile,extra", CASES)
def test_spmd_routines_fake_two_ranks(kind, n, k, tile, extra):
    outs = spmd.launch(2, SC.run_case, kind, n, k, tile, 1, True, None, extra, timeout=600)
    _check(outs, 2)


def test_spmd_gemm_three_ranks_host_bytes_once():
    outs = spmd.launch(3, SC.run_case, "gemm", 256, 256, 64, 2, True, timeout=600)
    _check(outs, 3)
    o = outs[0]
    # first-holder policy: each input tile crosses the host link once (A + B + C move-in)
    assert o["h2d"] == (256 * 256 * 3) * 8, outs
    assert o["host"] == 2 * 16, outs
    assert o["second_tasks"] == o["n_tasks"], outs


def test_spmd_trsm_three_ranks_small_station():
    outs = spmd.launch(3, SC.run_case, "trsm", 256, 256, 64, 4, True, dict(rs_capacity=2),
                       timeout=600)
    _check(outs, 3)


def test_spmd_singular_aborts_every_rank():
    outs = spmd.launch(2, SC.run_singular, 160, 64, True, timeout=600)
    assert outs == ["SingularMatrixError", "SingularMatrixError"]


def test_spmd_needs_shared_operands():
    outs = spmd.launch(1, SC.check_shared_required, True, timeout=300)
    assert outs == ["InvalidArgumentError"]


@pytest.mark.gpu
@pytest.mark.parametrize("kind,n,k,tile,extra", [
    ("gemm", 1536, 1280, 512, {}),
    ("syr2k", 1280, 768, 512, {}),
    ("trmm", 1536, 1536, 512, {}),
    ("trsm", 1536, 1536, 512, {}),
])
def test_spmd_gpu_ranks_share_one_b200(kind, n, k, tile, extra):
    outs = spmd.launch(2, SC.run_case, kind, n, k, tile, 5, False, None, extra, timeout=900,
                       devices=[0, 0])
    _check(outs, 2)


@pytest.mark.gpu
def test_spmd_gpu_singular_aborts_both_ranks():
    """Failure path on hardware: a zero on the triangle's diagonal, 2 ranks on one B200 —
    the rank whose solve sees it aborts the call and both ranks raise."""
    outs = spmd.launch(2, SC.run_singular, 1536, 512, False, timeout=900, devices=[0, 0])
    assert outs == ["SingularMatrixError", "SingularMatrixError"]


@pytest.mark.gpu
def test_spmd_gpu_three_ranks_trsm():
    outs = spmd.launch(3, SC.run_case, "trsm", 2048, 2048, 512, 6, False, timeout=900,
                       devices=[0, 0, 0])
    _check(outs, 3)


def test_spmd_station_stealing_stress():
    """Four ranks with 2-slot stations over three calls: owners pop and thieves steal the
    same slots concurrently; every task runs exactly once (a slot read twice used to turn a
    concurrently emptied slot into a claim of task -1, i.e. a duplicate of the last task)."""
    outs = spmd.launch(6, SC.run_steal_stress, 256, 16, 3, 2, timeout=600)
    for c in range(3):
        assert sum(o[c][0] for o in outs) == outs[0][c][1], [o[c] for o in outs]
        assert outs[0][c][2] <= 1e-11, outs[0][c]


def test_spmd_pooled_call_files_reuse_and_growth():
    """Calls alternate between two pooled node-shared call files: small, large (grows one
    file), small, large, larger (grows the other) — every call still runs every task once
    and matches the reference."""
    sizes = [64, 256, 64, 256, 320, 64]
    outs = spmd.launch(2, SC.run_size_sequence, sizes, 32, True, timeout=600)
    for c in range(len(sizes)):
        assert sum(o[c][0] for o in outs) == outs[0][c][1], [o[c] for o in outs]
        assert outs[0][c][2] <= 1e-11 * 64, outs[0][c]


def test_call_file_pool_growth_is_collective():
    """Session.call_file: alternate calls use two files; a file is replaced (unregistered,
    unlinked by rank 0) only when a call needs more bytes, and the replacement at least
    doubles it."""

    class Eng:
        def __init__(self):
            self.mapped, self.unmapped = [], []

        def register_mapped(self, a):
            self.mapped.append(a.nbytes)
            return 1 << 40

        def unregister_host(self, a):
            self.unmapped.append(a.nbytes)

    sess = spmd.Session.__new__(spmd.Session)
    sess.rank, sess.job, sess._blocks = 0, f"t{os.getpid()}", [None, None]
    eng = Eng()
    try:
        f1, _ = sess.call_file(eng, 1, 5000)
        f2, _ = sess.call_file(eng, 2, 5000)
        assert f1 is not f2 and eng.mapped == [5000, 5000]
        assert sess.call_file(eng, 3, 4000)[0] is f1          # reused: big enough
        f5, _ = sess.call_file(eng, 5, 6000)                    # parity 1 grows
        assert f5 is not f1 and f5.nbytes >= 10000 and eng.unmapped == [5000]
        assert not os.path.exists(f1.path)
        assert sess.call_file(eng, 4, 5000)[0] is f2
    finally:
        for b in sess._blocks:
            if b is not None:
                b[0].unlink()


def test_torchrun_job_name_is_launch_unique(monkeypatch):
    """torchrun without an rdzv id exports TORCHELASTIC_RUN_ID=none: the session name then
    carries the port and the agent's pid (every rank's parent), so two launches on one port
    never share session files."""
    for k in ("BX_SPMD_JOB",):
        monkeypatch.delenv(k, raising=False)
    monkeypatch.setenv("TORCHELASTIC_RUN_ID", "none")
    monkeypatch.setenv("MASTER_PORT", "29577")
    monkeypatch.setenv("RANK", "0")
    monkeypatch.setenv("WORLD_SIZE", "1")
    monkeypatch.setenv("LOCAL_RANK", "0")
    monkeypatch.setattr(spmd, "_SESSION", None)
    sess = spmd.init()
    try:
        assert sess.job == f"p29577_{os.getppid()}"
    finally:
        spmd.shutdown()


def test_spmd_trsm_release_on_issue_fake():
    """Release-on-issue across ranks (the producer's compute stream sets the solved tile's
    flag; peers wait on it on the GPU) — opt-in since round 2."""
    outs = spmd.launch(2, SC.run_case, "trsm", 192, 192, 64, 1, True, dict(release_on_issue=True),
                       timeout=600)
    _check(outs, 2)


@pytest.mark.gpu
def test_spmd_gpu_trsm_release_on_issue():
    outs = spmd.launch(2, SC.run_case, "trsm", 1536, 1536, 512, 7, False, dict(release_on_issue=True),
                       timeout=900, devices=[0, 0])
    _check(outs, 2)


@pytest.mark.parametrize("kind,n,k,tile,extra", CASES)
def test_spmd_owner_prefetch_fake_three_ranks(kind, n, k, tile, extra):
    """RunOptions.owner_prefetch: input tiles dealt round-robin to the ranks and loaded at
    the call's start; every routine family still matches the oracle, every input tile
    crosses a host link once, every task runs once."""
    outs = spmd.launch(3, SC.run_case, kind, n, k, tile, 2, True, dict(owner_prefetch=True), extra,
                       timeout=600)
    _check(outs, 3)


def test_spmd_owner_prefetch_balances_host_links():
    """With owner prefetch the input (A/B) host bytes split evenly over the ranks' links."""
    import balance_case as BC
    outs = spmd.launch(4, BC.input_bytes_by_rank, 256, 32, timeout=600)
    per = outs[0]
    assert sum(per.values()) == 2 * 256 * 256 * 8          # A and B, each tile once
    assert max(per.values()) <= 1.25 * (sum(per.values()) / len(per)), per


@pytest.mark.gpu
@pytest.mark.parametrize("kind,n,k,tile,extra", [
    ("gemm", 1536, 1280, 512, {}),
    ("syr2k", 1280, 768, 512, {}),
    ("trmm", 1536, 1536, 512, {}),
    ("trsm", 1536, 1536, 512, {}),
])
def test_spmd_gpu_owner_prefetch(kind, n, k, tile, extra):
    outs = spmd.launch(2, SC.run_case, kind, n, k, tile, 5, False, dict(owner_prefetch=True), extra,
                       timeout=900, devices=[0, 0])
    _check(outs, 2)
