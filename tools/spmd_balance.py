"""Per-rank host-link bytes of the one-process-per-GPU runtime (first-holder policy) on the
CPU fake engine: how evenly does the H2D traffic spread over W ranks' host links?
python tools/spmd_balance.py [ranks] [n] [tile] ['dict(...)' RunOptions]   (CPU only; fake engine)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def rank_main(n, t, opts):
    from paper_1510_05041_b200 import RunOptions, build_call, run_call, spmd
    from fake_spmd import SpmdFakeEngine
    sess = spmd.current()
    call = build_call("gemm", m=n, n=n, k=n, tile_size=t, seed=1, beta=1.0) if sess.rank == 0 else None
    call = sess.share_call(call)
    eng = SpmdFakeEngine(sess.rank, sess.job, seed=sess.rank * 7 + 1)
    try:
        res = run_call(call, options=RunOptions(execution="spmd", **opts), engine=eng)
        m = res.metrics
        return {q: (m.devices[q].tasks, m.devices[q].h2d_bytes, m.devices[q].d2d_in_bytes)
                for q in sorted(m.devices)}
    finally:
        eng.cleanup()


if __name__ == "__main__":
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    t = int(sys.argv[3]) if len(sys.argv) > 3 else 32
    opts = eval(sys.argv[4]) if len(sys.argv) > 4 else {}
    from paper_1510_05041_b200 import spmd
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import spmd_balance as me
    out = spmd.launch(W, me.rank_main, n, t, opts, devices=list(range(W)))[0]
    h = [v[1] for v in out.values()]
    print(f"W={W} n={n} T={t} {opts}: per rank (tasks, H2D bytes, peer-in bytes): {out}")
    print(f"H2D max/mean = {max(h) / (sum(h) / len(h)):.2f}")
