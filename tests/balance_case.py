"""spmd rank entry for test_spmd_owner_prefetch_balances_host_links (spawned ranks import it)."""


def input_bytes_by_rank(n, tile):
    """Every rank: GEMM n^3 (beta = 0: no C move-in, so all host bytes are A/B input tiles)
    with owner prefetch on the fake engine; returns {rank: host bytes} gathered by rank 0."""
    from paper_1510_05041_b200 import RunOptions, build_call, run_call, spmd
    from fake_spmd import SpmdFakeEngine
    sess = spmd.init()
    call = build_call("gemm", m=n, n=n, k=n, tile_size=tile, seed=2, beta=0.0) if sess.rank == 0 else None
    call = sess.share_call(call)
    eng = SpmdFakeEngine(sess.rank, sess.job, seed=sess.rank + 3)
    try:
        res = run_call(call, options=RunOptions(execution="spmd", owner_prefetch=True), engine=eng)
        return {q: res.metrics.devices[q].h2d_bytes for q in sorted(res.metrics.devices)}
    finally:
        eng.cleanup()
