"""Seeded random routine cases shared by the GPU parity sweep and its fake-engine twin."""

import numpy as np


def random_cases(n_cases=40, seed=2026):
    rng = np.random.default_rng(seed)
    kinds = ["gemm", "syrk", "syr2k", "symm", "trmm", "trsm"]
    out = []
    for i in range(n_cases):
        kind = kinds[i % len(kinds)]
        m, n, k = (int(x) for x in rng.integers(1, 640, size=3))
        kw = dict(alpha=float(rng.choice([1.0, -0.5, 2.0])), uplo=str(rng.choice(["lower", "upper"])))
        if kind in ("gemm", "syrk", "syr2k", "symm"):
            kw["beta"] = float(rng.choice([0.0, 1.0, 0.25]))
        if kind == "gemm":
            kw.update(trans_a=bool(rng.integers(2)), trans_b=bool(rng.integers(2)))
        if kind in ("syrk", "syr2k"):
            kw["trans_a"] = bool(rng.integers(2))
            m = n
        if kind in ("symm", "trmm", "trsm"):
            kw["side"] = str(rng.choice(["left", "right"]))
        if kind in ("trmm", "trsm"):
            kw.update(trans_a=bool(rng.integers(2)), diag=str(rng.choice(["unit", "non-unit"])))
        opts = dict(chunk_steps=int(rng.choice([1, 2, 16])), n_streams=int(rng.choice([0, 2, 8])),
                    defer_c_move_in=bool(rng.integers(2)), ramp_tasks=int(rng.choice([-1, 0, 3])))
        out.append((i, kind, m, n, k, int(rng.choice([64, 96, 160, 256])), kw, opts))
    return out
