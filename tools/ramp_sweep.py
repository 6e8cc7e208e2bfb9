"""e2e time of one host-resident call under several RunOptions (start-up ramp tuning).
python tools/ramp_sweep.py [kind] [n] [k] [tile]   — prints one line per option set."""
import itertools
import os
import statistics
import sys

sys.path.insert(0, ".")
from paper_1510_05041_b200 import RunOptions, build_call, run_call  # noqa: E402
from paper_1510_05041_b200.engine import get_engine  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "gemm"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
k = int(sys.argv[3]) if len(sys.argv) > 3 else n
t = int(sys.argv[4]) if len(sys.argv) > 4 else 1024
call = build_call(kind, m=n, n=n, k=k, tile_size=t, seed=0, alpha=1.0,
                  beta=1.0 if kind in ("gemm", "syrk", "syr2k", "symm") else 0.0, uplo="lower",
                  trsm_scaled=True)
eng = get_engine([0], 8)
if os.environ.get("BX_TRSM_LEAF"):
    eng.lib.bx_set_trsm_leaf(int(os.environ["BX_TRSM_LEAF"]))
if os.environ.get("BX_TRSM_RHS"):
    eng.lib.bx_set_trsm_rhs(int(os.environ["BX_TRSM_RHS"]))
for x in [y for y in (call.a, call.b, call.c) if y is not None]:
    eng.register_host(x.matrix.storage)

grid = os.environ.get("BX_SWEEP", "default")
if grid == "default":
    sets = [dict()]
    for st, tps, rt, rc, fc in itertools.product((4, 8), (2, 3), (0, 8, 16, 32), (2, 4), (4,)):
        if rt == 0 and rc != 4:
            continue
        sets.append(dict(n_streams=st, tasks_per_stream=tps, ramp_tasks=rt, ramp_chunk_steps=rc,
                         first_chunk_steps=fc))
else:
    sets = [eval(x) for x in grid.split(";")]

res = run_call(call, options=RunOptions())
flops = res.plan.total_flops
for kw in sets:
    opts = RunOptions(**kw)
    run_call(call, options=opts)
    ts = []
    for _ in range(3):
        e0 = eng.record(0, 0, timing=True)
        run_call(call, options=opts)
        e1 = eng.record(0, 0, timing=True)
        eng.sync(e1)
        ts.append(eng.elapsed_ms(e0, e1))
        eng.release(e0)
        eng.release(e1)
    ms = statistics.median(ts)
    print(f"{kind} {n} {kw}: {ms:.1f} ms  {flops / ms / 1e9:.2f} TF/s  (min {min(ts):.1f})", flush=True)
