"""Host issue rate on hardware: SGEMM 16384^3 at T=512 (1024 tasks, tiny GPU work per task,
host-bound) on 1..8 logical devices sharing GPU 0, deterministic vs concurrent driver."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np

from paper_1510_05041_b200 import RoutineCall, RunOptions, run_call
from paper_1510_05041_b200.devices import DeviceDesc, Topology
from paper_1510_05041_b200.engine import get_engine
from paper_1510_05041_b200.tiling import MatrixDesc, make_tiled

n, t = 16384, int(sys.argv[1]) if len(sys.argv) > 1 else 512
rng = np.random.default_rng(0)
bufs = {m: (rng.random(n * n, dtype=np.float32) * 2 - 1) for m in "ABC"}
eng = get_engine([0])
for b in bufs.values():
    eng.register_host(b)
call = RoutineCall("gemm", a=make_tiled(MatrixDesc("A", n, n, n, bufs["A"]), t),
                   b=make_tiled(MatrixDesc("B", n, n, n, bufs["B"]), t),
                   c=make_tiled(MatrixDesc("C", n, n, n, bufs["C"]), t), alpha=1.0, beta=1.0)
for ndev in (1, 2, 4, 8):
    topo = Topology([DeviceDesc(200 + i, cuda_ordinal=0, peer_group="g") for i in range(ndev)])
    for mode in ("deterministic", "concurrent"):
        opts = RunOptions(execution=mode)
        run_call(call, topo, opts)
        best = 1e9
        for _ in range(2):
            t0 = time.perf_counter()
            r = run_call(call, topo, opts)
            best = min(best, time.perf_counter() - t0)
        m = r.metrics
        print(f"ndev={ndev} {mode:13s}: {best*1e3:7.1f} ms  {len(r.plan.tasks)/best:7.0f} tasks/s  "
              f"H2D {m.total_h2d_bytes()/1e9:.2f} GB P2P {m.total_d2d_bytes()/1e9:.2f} GB "
              f"tasks/dev {sorted(r.tasks_by_device.values())}", flush=True)
