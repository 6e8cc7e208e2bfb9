"""Interleaved A/B of RunOptions sets on one host-resident call (device-event time per call,
sets alternated round by round so clock / thermal drift hits every set alike).
python tools/opts_ab.py kind n k tile rounds 'dict(...)' 'dict(...)' ...
(BX_IC=0 etc. apply to every set; BX_F32=1: SGEMM; prints min / median ms and TF/s per set)"""
import statistics
import sys

sys.path.insert(0, ".")
from paper_1510_05041_b200 import RunOptions, build_call, run_call  # noqa: E402
from paper_1510_05041_b200.engine import get_engine  # noqa: E402

kind, n, k, t, rounds = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
sets = [eval(x) for x in sys.argv[6:]] or [{}]
import os  # noqa: E402
import numpy as np  # noqa: E402
call = build_call(kind, m=n, n=n, k=k, tile_size=t, seed=0, alpha=1.0,
                  beta=1.0 if kind in ("gemm", "syrk", "syr2k", "symm") else 0.0, uplo="lower",
                  trsm_scaled=True, **({"dtype": np.float32} if os.environ.get("BX_F32") else {}))
eng = get_engine([0])
for x in [y for y in (call.a, call.b, call.c) if y is not None]:
    eng.register_host(x.matrix.storage)
flops = run_call(call).plan.total_flops
times = [[] for _ in sets]
for kw in sets:
    run_call(call, options=RunOptions(**kw))
for _ in range(rounds):
    for i, kw in enumerate(sets):
        opts = RunOptions(**kw)
        e0 = eng.record(0, 0, timing=True)
        run_call(call, options=opts)
        e1 = eng.record(0, 0, timing=True)
        eng.sync(e1)
        times[i].append(eng.elapsed_ms(e0, e1))
        eng.release(e0)
        eng.release(e1)
for kw, ts in zip(sets, times):
    print(f"{kind} {n} k={k} T={t} {kw}: min {min(ts):.1f} ms median {statistics.median(ts):.1f} ms "
          f"-> {flops / statistics.median(ts) / 1e9:.2f} TF/s (n={len(ts)})", flush=True)
