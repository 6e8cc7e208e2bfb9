import sys, time, cProfile, pstats
sys.path.insert(0, ".")
import numpy as np
from paper_1510_05041_b200 import RunOptions, build_call, run_call
from paper_1510_05041_b200.engine import get_engine
n, t = int(sys.argv[1]), int(sys.argv[2])
call = build_call("gemm", m=n, n=n, k=n, tile_size=t, seed=0, alpha=1.0, beta=1.0, dtype=np.float32)
eng = get_engine([0])
for x in (call.a, call.b, call.c): eng.register_host(x.matrix.storage)
run_call(call)
t0 = time.perf_counter(); r = run_call(call); w = time.perf_counter() - t0
print(f"wall {w*1e3:.1f} ms, {len(r.plan.tasks)} tasks, {w/len(r.plan.tasks)*1e6:.0f} us/task, phases", {k: round(v*1e3,1) for k,v in r.metrics.phases.items()})
cProfile.run("run_call(call)", "/tmp/ps")
pstats.Stats("/tmp/ps").sort_stats("tottime").print_stats(22)
