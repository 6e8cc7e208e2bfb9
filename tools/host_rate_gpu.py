"""Host issue rate on hardware: a call with tiny GPU work per task (SGEMM 16384^3 at T=512:
1024 tasks of ~14 us of tensor time each) is host-bound, so wall time / tasks is the
runtime's real per-task host cost (ctypes, driver calls, event polling, bookkeeping) — on
1..8 logical devices sharing GPU 0, one driver thread (execution="deterministic").

  python tools/host_rate_gpu.py [T] [ndev,...] [mode,...]
BX_PKG_ROOT=<dir> imports the runtime from another tree (before/after comparisons)."""
import os
import sys
import time

sys.path.insert(0, os.environ.get("BX_PKG_ROOT", "."))
import numpy as np  # noqa: E402

from paper_1510_05041_b200 import RoutineCall, RunOptions, run_call  # noqa: E402
from paper_1510_05041_b200.devices import DeviceDesc, Topology  # noqa: E402
from paper_1510_05041_b200.engine import get_engine  # noqa: E402
from paper_1510_05041_b200.tiling import MatrixDesc, make_tiled  # noqa: E402

n = 16384
t = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ndevs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8").split(",")]
modes = (sys.argv[3] if len(sys.argv) > 3 else "deterministic").split(",")
rng = np.random.default_rng(0)
bufs = {m: (rng.random(n * n, dtype=np.float32) * 2 - 1) for m in "ABC"}
eng = get_engine([0])
for b in bufs.values():
    eng.register_host(b)
call = RoutineCall("gemm", a=make_tiled(MatrixDesc("A", n, n, n, bufs["A"]), t),
                   b=make_tiled(MatrixDesc("B", n, n, n, bufs["B"]), t),
                   c=make_tiled(MatrixDesc("C", n, n, n, bufs["C"]), t), alpha=1.0, beta=1.0)
print(f"package: {os.path.abspath(os.environ.get('BX_PKG_ROOT', '.'))}", flush=True)
for ndev in ndevs:
    topo = Topology([DeviceDesc(200 + i, cuda_ordinal=0, peer_group="g") for i in range(ndev)])
    for mode in modes:
        opts = RunOptions(execution=mode, sgemm_precise=False)
        run_call(call, topo, opts)
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            r = run_call(call, topo, opts)
            best = min(best, time.perf_counter() - t0)
        m = r.metrics
        nt = len(r.plan.tasks)
        print(f"ndev={ndev} {mode:13s}: {best*1e3:7.1f} ms  {nt/best:7.0f} tasks/s  "
              f"{best/nt*1e6:6.1f} us/task  H2D {m.total_h2d_bytes()/1e9:.2f} GB "
              f"P2P {m.total_d2d_bytes()/1e9:.2f} GB tasks/dev {sorted(r.tasks_by_device.values())}",
              flush=True)
if os.environ.get("BX_PROF"):
    import cProfile
    import pstats
    ndev = ndevs[-1]
    topo = Topology([DeviceDesc(200 + i, cuda_ordinal=0, peer_group="g") for i in range(ndev)])
    opts = RunOptions(execution=modes[0], sgemm_precise=False)
    cProfile.run("run_call(call, topo, opts)", "/tmp/host_rate.prof")
    st = pstats.Stats("/tmp/host_rate.prof")
    st.sort_stats("tottime").print_stats(30)
