"""Fixed per-call cost of the one-process-per-GPU runtime: a tiny call (few tasks, ~no GPU
work) repeated, per-rank phases (plan / setup / drive / finalize) and wall, vs the same call
in one process.  python tools/spmd_overhead.py [ranks] [calls]   (ranks share GPU 0)"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rank_main(calls, n=512, t=256):
    import numpy as np
    from paper_1510_05041_b200 import RunOptions, build_call, run_call, spmd
    sess = spmd.current()
    call = build_call("gemm", m=n, n=n, k=n, tile_size=t, seed=0, beta=1.0) if sess.rank == 0 else None
    call = sess.share_call(call)
    from paper_1510_05041_b200.engine import get_engine
    eng = get_engine([sess.rank], 4, [sess.device])
    for t in (call.a, call.b, call.c):
        eng.register_host(t.matrix.storage)   # page-locking outside the timed calls, as bench.py
    opts = RunOptions(execution="spmd")
    for _ in range(3):
        run_call(call, options=opts)
    if os.environ.get("BX_PROF"):
        import cProfile
        cProfile.runctx("for _ in range(int(os.environ.get('BX_PROF_CALLS', '20'))): run_call(call, options=opts)", globals(), locals(),
                        f"{os.environ['BX_PROF']}.{sess.rank}")
    ph, wall = {}, []
    for _ in range(calls):
        sess.barrier("t")
        t0 = time.perf_counter()
        r = run_call(call, options=opts)
        wall.append((time.perf_counter() - t0) * 1e3)
        for k, v in r.metrics.phases.items():
            ph.setdefault(k, []).append(v * 1e3)
    return {"rank": sess.rank, "wall_ms": statistics.median(wall),
            **{k: round(statistics.median(v), 3) for k, v in ph.items()}}


if __name__ == "__main__":
    ranks = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    calls = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 512
    t = int(sys.argv[4]) if len(sys.argv) > 4 else 256
    from paper_1510_05041_b200 import RunOptions, build_call, run_call, spmd
    call = build_call("gemm", m=n, n=n, k=n, tile_size=t, seed=0, beta=1.0)
    from paper_1510_05041_b200 import pin_host
    for t in (call.a, call.b, call.c):
        pin_host(t.matrix.storage)
    for _ in range(3):
        run_call(call)
    ph, wall = {}, []
    for _ in range(calls):
        t0 = time.perf_counter()
        r = run_call(call)
        wall.append((time.perf_counter() - t0) * 1e3)
        for k, v in r.metrics.phases.items():
            ph.setdefault(k, []).append(v * 1e3)
    print("single process:", {"wall_ms": round(statistics.median(wall), 3),
                               **{k: round(statistics.median(v), 3) for k, v in ph.items()}}, flush=True)
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import spmd_overhead as me
    for out in spmd.launch(ranks, me.rank_main, calls, n, t, devices=[0] * ranks):
        print(f"spmd {ranks} ranks:", out, flush=True)
