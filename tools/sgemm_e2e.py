"""Host-resident SGEMM e2e through run_call at several tile sizes (cfg5-style sweep, 1 GPU).
python tools/sgemm_e2e.py N tiles..."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np

from paper_1510_05041_b200 import RoutineCall, RunOptions, run_call
from paper_1510_05041_b200.engine import get_engine
from paper_1510_05041_b200.tiling import MatrixDesc, make_tiled

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
tiles = [int(x) for x in sys.argv[2:]] or [1024]
rng = np.random.default_rng(0)
eng = get_engine([0])
bufs = {}
for mid in ("A", "B", "C"):
    arr = rng.random(n * n, dtype=np.float32)
    arr *= 2
    arr -= 1
    bufs[mid] = arr
    eng.register_host(arr)
for t in tiles:
    def tm(mid):
        return make_tiled(MatrixDesc(mid, n, n, n, bufs[mid]), t)
    call = RoutineCall("gemm", a=tm("A"), b=tm("B"), c=tm("C"), alpha=1.0, beta=1.0)
    res = run_call(call)
    times = []
    for _ in range(2):
        t0 = time.perf_counter()
        res = run_call(call)
        times.append(time.perf_counter() - t0)
    m = res.metrics
    dt = min(times)
    print(f"SGEMM {n}^3 T={t}: {dt*1e3:.1f} ms {2*n**3/dt/1e12:.1f} TF/s  H2D {m.total_h2d_bytes()/1e9:.2f} GB "
          f"P2P {m.total_d2d_bytes()/1e9:.2f} GB D2H {m.total_d2h_bytes()/1e9:.2f} GB "
          f"(link floor {m.total_h2d_bytes()/53e9*1e3:.0f} ms)  phases {({k: round(v*1e3,1) for k, v in m.phases.items()})}")
