"""CLI (reference cli.py formats and exit codes)."""

import json

import pytest

from paper_1510_05041_b200 import cli


def test_parser_defaults_match_reference():
    a = cli.build_parser().parse_args([])
    assert (a.routine, a.n, a.tile_size, a.alpha, a.beta, a.mode, a.execution) == (
        "gemm", 256, 1024, 1.0, 0.0, "verify", "det")


def test_invalid_arguments_exit_5():
    assert cli.main(["--tile-size", "0"]) == cli.EXIT_INVALID
    assert cli.main(["--n", "0"]) == cli.EXIT_INVALID


def test_dense_expected_matches_oracle(rng):
    import numpy as np
    from oracle import dense
    from paper_1510_05041_b200.operands import build_call, dense_snapshot
    for kind, kw in [("gemm", dict(trans_a=True, beta=0.5)), ("syr2k", dict(uplo="lower", beta=0.3)),
                     ("symm", dict(side="right", beta=1.0)), ("trmm", dict(trans_a=True, diag="unit")),
                     ("trsm", dict(side="right", uplo="lower"))]:
        call = build_call(kind, m=12, n=10 if kind not in ("syrk", "syr2k") else 12, k=7,
                          tile_size=4, seed=3, **kw)
        snap = dense_snapshot(call)
        got = cli._dense_expected(call, snap)
        ref = dense.dense_reference(kind, a=snap["a"], b=snap.get("b"), c=snap["c"],
                                    alpha=call.alpha, beta=call.beta, trans_a=call.trans_a,
                                    trans_b=call.trans_b, uplo=call.uplo, side=call.side,
                                    diag=call.diag)
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("routine,extra", [("gemm", []), ("trsm", ["--uplo", "lower", "--scaled-triangle"]),
                                           ("syr2k", ["--uplo", "lower", "--beta", "0.5"])])
def test_cli_verify_on_gpu(routine, extra, tmp_path):
    out = tmp_path / "m.json"
    tr = tmp_path / "t.csv"
    rc = cli.main(["--routine", routine, "--n", "600", "--tile-size", "256", "--metrics-out", str(out),
                   "--trace-out", str(tr)] + extra)
    assert rc == cli.EXIT_OK
    m = json.loads(out.read_text())
    assert set(m) == {"cache", "devices", "makespan_seconds"}
    assert tr.read_text().splitlines()[0] == cli.TRACE_HEADER


@pytest.mark.gpu
def test_cli_singular_exit_6():
    # the reference generator pushes the diagonal away from zero; unit=False with a
    # zero diagonal cannot be produced through the CLI, so check the code path via trsm
    # on a tiny singular call through the API instead
    import numpy as np
    from paper_1510_05041_b200 import SingularMatrixError, dtrsm
    a = np.asfortranarray(np.eye(64))
    a[10, 10] = 0.0
    b = np.asfortranarray(np.ones((64, 8)))
    with pytest.raises(SingularMatrixError):
        dtrsm("L", "L", "N", "N", 64, 8, 1.0, a, 64, b, 64, tile_size=32)
