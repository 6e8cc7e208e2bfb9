"""Timeline analysis of one host-resident call (record_trace=True): where does e2e time go?
python tools/trace_e2e.py [n] [tile] [chunk] [tasks_per_stream] [first_chunk]
(BX_KIND=gemm|syrk|syr2k|trsm|trmm, BX_K=depth, BX_F32=1 for SGEMM; chunk 0 = auto)"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np

from paper_1510_05041_b200 import RunOptions, build_call, run_call
from paper_1510_05041_b200.engine import get_engine

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
t = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 0   # 0 = auto
tps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
fc = int(sys.argv[5]) if len(sys.argv) > 5 else 0
import os
kind = os.environ.get("BX_KIND", "gemm")
call = build_call(kind, m=n, n=n, k=int(os.environ.get("BX_K", n)), tile_size=t, seed=0, alpha=1.0,
                  beta=1.0 if kind in ("gemm", "syrk", "syr2k", "symm") else 0.0, uplo="lower",
                  trsm_scaled=True, **({"dtype": np.float32} if os.environ.get("BX_F32") else {}))
eng = get_engine([0])
for x in [y for y in (call.a, call.b, call.c) if y is not None]:
    eng.register_host(x.matrix.storage)
kw = dict(chunk_steps=chunk, tasks_per_stream=tps, first_chunk_steps=fc)
run_call(call, options=RunOptions(**kw))
t0 = time.perf_counter()
res = run_call(call, options=RunOptions(**kw))
wall = time.perf_counter() - t0
res2 = run_call(call, options=RunOptions(record_trace=True, **kw))
tr = res2.trace
m = res.metrics
print("phases", {k: round(v * 1e3, 2) for k, v in res.metrics.phases.items()})
print(f"untraced: wall {wall*1e3:.1f} ms makespan {m.makespan_seconds*1e3:.1f} ms "
      f"-> {res.plan.total_flops / m.makespan_seconds / 1e12:.2f} TF/s")
print(f"traced makespan {res2.metrics.makespan_seconds*1e3:.1f} ms")
ks = sorted((e.time_start, e.time_end) for e in tr if e.event == "KERNEL")
hs = sorted((e.time_start, e.time_end) for e in tr if e.event == "H2D")
ds = sorted((e.time_start, e.time_end) for e in tr if e.event == "D2H")


def union(iv):
    tot, cs, ce = 0.0, None, None
    for s, e in iv:
        if cs is None or s > ce:
            if cs is not None:
                tot += ce - cs
            cs, ce = s, e
        else:
            ce = max(ce, e)
    if cs is not None:
        tot += ce - cs
    return tot


print(f"first kernel start {ks[0][0]*1e3:.2f} ms, last kernel end {ks[-1][1]*1e3:.2f} ms, "
      f"last D2H end {ds[-1][1]*1e3:.2f} ms")
print(f"kernel-busy union {union(ks)*1e3:.1f} ms; H2D busy {union(hs)*1e3:.1f} ms; D2H busy {union(ds)*1e3:.1f} ms")
print(f"kernel launches {len(ks)}; sum of kernel durations {sum(e-s for s,e in ks)*1e3:.1f} ms")
# concurrency histogram of kernels over time
pts = sorted([(s, 1) for s, e in ks] + [(e, -1) for s, e in ks])
cur, last, hist = 0, pts[0][0], {}
for x, d in pts:
    hist[cur] = hist.get(cur, 0) + (x - last)
    cur += d
    last = x
print("kernel concurrency (streams busy -> ms):", {k: round(v * 1e3, 1) for k, v in sorted(hist.items())})
gaps = []
for (s0, e0), (s1, e1) in zip(ks, ks[1:]):
    pass
# per-task issue timing not traced; print H2D progress vs kernels at quartiles
for frac in (0.1, 0.25, 0.5, 0.75, 1.0):
    tq = ks[-1][1] * frac
    hb = sum(1 for s, e in hs if e <= tq)
    kb = sum(1 for s, e in ks if e <= tq)
    print(f"t={tq*1e3:7.1f} ms  H2D done {hb}/{len(hs)}  kernels done {kb}/{len(ks)}")
# utilisation over time: fraction of 1 ms bins where >= 3 kernels run
import math
end = ks[-1][1]
bins = int(math.ceil(end * 1e3))
occ = [0.0] * bins
for s0, e0 in ks:
    b0, b1 = int(s0 * 1e3), int(e0 * 1e3)
    for b in range(b0, min(b1 + 1, bins)):
        lo, hi = max(s0, b / 1e3), min(e0, (b + 1) / 1e3)
        if hi > lo:
            occ[b] += (hi - lo) * 1e3
print("kernel-streams busy per 5 ms window:", [round(sum(occ[i:i + 5]) / 5, 1) for i in range(0, bins, 5)])
h2d_bins = [0.0] * bins
for s0, e0 in hs:
    for b in range(int(s0 * 1e3), min(int(e0 * 1e3) + 1, bins)):
        lo, hi = max(s0, b / 1e3), min(e0, (b + 1) / 1e3)
        if hi > lo:
            h2d_bins[b] += (hi - lo) * 1e3
print("H2D busy fraction per 5 ms window:", [round(sum(h2d_bins[i:i + 5]) / 5, 2) for i in range(0, bins, 5)])
