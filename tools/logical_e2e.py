"""Host-resident DGEMM through run_call on N logical devices sharing GPU 0 (DeviceDesc.cuda_ordinal):
exercises the 8-device scheduler / L2 peer path with the real engine and reports host drive time
vs GPU time.  python tools/logical_e2e.py [n] [tile] [ndev...]   (BX_OPTS='dict(...)': RunOptions)"""
import os
import sys
import time

sys.path.insert(0, ".")
from paper_1510_05041_b200 import RunOptions, build_call, run_call
from paper_1510_05041_b200.devices import DeviceDesc, Topology
from paper_1510_05041_b200.engine import get_engine

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
t = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
ndevs = [int(x) for x in sys.argv[3:]] or [1, 2, 4, 8]
call = build_call("gemm", m=n, n=n, k=n, tile_size=t, seed=0, alpha=1.0, beta=1.0)
eng = get_engine([0])
for x in (call.a, call.b, call.c):
    eng.register_host(x.matrix.storage)
for nd in ndevs:
    topo = Topology([DeviceDesc(100 + i, cuda_ordinal=0, peer_group="g") for i in range(nd)])
    kw = eval(os.environ.get("BX_OPTS", "dict()"))
    run_call(call, topo, RunOptions(**kw))
    best = None
    for _ in range(2):
        t0 = time.perf_counter()
        r = run_call(call, topo, RunOptions(**kw))
        w = time.perf_counter() - t0
        if best is None or w < best[0]:
            best = (w, r)
    w, r = best
    m = r.metrics
    print(f"{kw} n={n} T={t} ndev={nd}: wall {w*1e3:.0f} ms -> {r.plan.total_flops/w/1e12:.2f} TF/s; "
          f"phases { {k: round(v*1e3, 1) for k, v in m.phases.items()} }; H2D {m.total_h2d_bytes()/1e9:.2f} GB "
          f"P2P {m.total_d2d_bytes()/1e9:.2f} GB l2 {m.l2_hits} tasks/dev {sorted(r.tasks_by_device.values())}",
          flush=True)
