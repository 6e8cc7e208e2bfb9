"""The one-process-per-GPU runtime with a single rank on one B200 vs the single-process
runtime on the same call: the per-GPU efficiency of the path the multi-GPU bench uses
(no peers, so no scaling effects).  python tools/spmd_one_rank.py [kind] [n] [k] [tile] [rounds]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rank_main(kind, n, k, t, rounds):
    from paper_1510_05041_b200 import RunOptions, build_call, run_call, spmd
    from paper_1510_05041_b200.engine import get_engine
    sess = spmd.current()
    call = build_call(kind, m=n, n=n, k=k, tile_size=t, seed=0, alpha=1.0,
                      beta=1.0 if kind in ("gemm", "syrk", "syr2k", "symm") else 0.0, uplo="lower",
                      trsm_scaled=True)
    call = sess.share_call(call)
    eng = get_engine([sess.rank], 4, [sess.device])
    for x in [y for y in (call.a, call.b, call.c) if y is not None]:
        eng.register_host(x.matrix.storage)
    opts = RunOptions(execution="spmd")
    res = run_call(call, options=opts)
    ts = []
    for _ in range(rounds):
        sess.barrier("t")
        e0 = eng.record(0, 0, timing=True)
        run_call(call, options=opts)
        e1 = eng.record(0, 0, timing=True)
        eng.sync(e1)
        ts.append(eng.elapsed_ms(e0, e1))
    ms = statistics.median(ts)
    return f"spmd 1 rank {kind} {n} k={k} T={t}: median {ms:.1f} ms {res.plan.total_flops / ms / 1e9:.2f} TF/s"


if __name__ == "__main__":
    kind = sys.argv[1] if len(sys.argv) > 1 else "gemm"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
    k = int(sys.argv[3]) if len(sys.argv) > 3 else n
    t = int(sys.argv[4]) if len(sys.argv) > 4 else 1024
    rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 5
    from paper_1510_05041_b200 import spmd
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import spmd_one_rank as me
    print(spmd.launch(1, me.rank_main, kind, n, k, t, rounds, devices=[0])[0], flush=True)
