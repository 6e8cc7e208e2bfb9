#!/bin/bash
# round 2: why 8 logical devices on one B200 run DGEMM 16384^3 slower than 1 device
cd "$(dirname "$0")/.."
O=gpurun_out/aa; mkdir -p $O
timeout 600 python tools/logical_e2e.py 16384 1024 1 8 > $O/logical.txt 2>&1
for o in "dict(n_streams=8)" "dict(ramp_tasks=0)" "dict(n_streams=2)" "dict(n_streams=8, ramp_tasks=0)" "dict(execution='concurrent')"; do
  BX_OPTS="$o" timeout 600 python tools/logical_e2e.py 16384 1024 8 >> $O/logical.txt 2>&1
done
BX_KIND=gemm timeout 600 python - >> $O/trace8.txt 2>&1 <<'PY'
import sys; sys.path.insert(0, ".")
from paper_1510_05041_b200 import RunOptions, build_call, run_call
from paper_1510_05041_b200.devices import DeviceDesc, Topology
from paper_1510_05041_b200.engine import get_engine
call = build_call("gemm", m=16384, n=16384, k=16384, tile_size=1024, seed=0, alpha=1.0, beta=1.0)
eng = get_engine([0])
for x in (call.a, call.b, call.c): eng.register_host(x.matrix.storage)
topo = Topology([DeviceDesc(100 + i, cuda_ordinal=0, peer_group="g") for i in range(8)])
run_call(call, topo, RunOptions())
res = run_call(call, topo, RunOptions(record_trace=True))
tr = res.trace
ks = sorted((e.time_start, e.time_end) for e in tr if e.event == "KERNEL")
ds = sorted((e.time_start, e.time_end) for e in tr if e.event in ("D2D", "P2P"))
hs = sorted((e.time_start, e.time_end) for e in tr if e.event == "H2D")
end = max(e.time_end for e in tr)
print("makespan", res.metrics.makespan_seconds * 1e3, "events", len(tr), "kernels", len(ks), "d2d", len(ds), "h2d", len(hs))
import math
bins = int(math.ceil(end * 1e3 / 5))
def occ(iv):
    o = [0.0] * bins
    for s, e in iv:
        for b in range(int(s * 200), min(int(e * 200) + 1, bins)):
            lo, hi = max(s, b / 200), min(e, (b + 1) / 200)
            if hi > lo: o[b] += (hi - lo) * 200
    return [round(x, 1) for x in o]
print("kernels busy per 5 ms:", occ(ks))
print("d2d busy per 5 ms:", occ(ds))
print("h2d busy per 5 ms:", occ(hs))
print("event kinds:", sorted({e.event for e in tr}))
PY
echo done > $O/status.txt
