"""Per-task host cost of the runtime with the REAL engine wrappers (ctypes marshalling
included) over a no-op stub of the C ABI (tools/stub_abi.c): what the Python side costs
per task before any CUDA driver time.  python tools/host_cost.py [n] [tile] [ndev] [--prof]"""
import os
import subprocess
import sys
import time

sys.path.insert(0, ".")
stub = "/tmp/libbx_stub.so"
subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-w", "-o", stub, "tools/stub_abi.c"], check=True)
from paper_1510_05041_b200 import _native
_native.load(stub)
from paper_1510_05041_b200 import RunOptions, build_call, run_call
from paper_1510_05041_b200.devices import DeviceDesc, Topology

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
t = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
nd = int(sys.argv[3]) if len(sys.argv) > 3 else 8
call = build_call("gemm", m=n, n=n, k=n, tile_size=t, seed=0, alpha=1.0, beta=1.0) if n <= 16384 else None
if call is None:
    import numpy as np
    from paper_1510_05041_b200 import RoutineCall
    from paper_1510_05041_b200.tiling import MatrixDesc, make_tiled
    buf = np.zeros(n * n)
    call = RoutineCall("gemm", a=make_tiled(MatrixDesc("A", n, n, n, buf), t),
                       b=make_tiled(MatrixDesc("B", n, n, n, buf), t),
                       c=make_tiled(MatrixDesc("C", n, n, n, buf), t), beta=1.0)
topo = Topology([DeviceDesc(i, peer_group="g") for i in range(nd)])
run_call(call, topo, RunOptions())
best = 1e9
for _ in range(5):
    t0 = time.perf_counter()
    r = run_call(call, topo, RunOptions())
    best = min(best, time.perf_counter() - t0)
print(f"n={n} T={t} ndev={nd}: {len(r.plan.tasks)} tasks, {best*1e3:.1f} ms = "
      f"{best/len(r.plan.tasks)*1e6:.0f} us/task -> {len(r.plan.tasks)/best:.0f} tasks/s; "
      f"phases { {k: round(v*1e3, 1) for k, v in r.metrics.phases.items()} }")
if "--prof" in sys.argv:
    import cProfile
    import pstats
    cProfile.run("run_call(call, topo, RunOptions())", "/tmp/hostcost")
    pstats.Stats("/tmp/hostcost").sort_stats("tottime").print_stats(25)
