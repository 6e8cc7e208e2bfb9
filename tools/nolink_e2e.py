"""Diagnostic: the host-resident call with the host link removed (H2D / D2H replaced by
stream events, so tiles are garbage but the task schedule, kernels and stream waits are
unchanged).  Separates the link-bound start-up from the task-kernel schedule's own
efficiency.  python tools/nolink_e2e.py [n] [options-dict]"""
import statistics
import sys

sys.path.insert(0, ".")
from paper_1510_05041_b200 import RunOptions, build_call, run_call  # noqa: E402
from paper_1510_05041_b200.engine import CudaEngine, get_engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
sets = [eval(x) for x in sys.argv[2:]] or [{}]
import os
BETA = float(os.environ.get("BX_BETA", "1.0"))
KIND = os.environ.get("BX_KIND", "gemm")
call = build_call(KIND, m=n, n=n, k=int(os.environ.get("BX_K", n)), tile_size=1024, seed=0,
                  alpha=1.0, beta=BETA if KIND in ("gemm", "syrk", "syr2k", "symm") else 0.0,
                  uplo="lower", trsm_scaled=True)
eng = get_engine([0], 8)
for x in [y for y in (call.a, call.b, call.c) if y is not None]:
    eng.register_host(x.matrix.storage)


def timed(opts):
    run_call(call, options=opts)
    ts = []
    for _ in range(3):
        e0 = eng.record(0, 0, timing=True)
        res = run_call(call, options=opts)
        e1 = eng.record(0, 0, timing=True)
        eng.sync(e1)
        ts.append(eng.elapsed_ms(e0, e1))
        eng.release(e0)
        eng.release(e1)
    return statistics.median(ts), res.plan.total_flops


real_h2d, real_d2h = CudaEngine.h2d, CudaEngine.d2h
for kw in sets:
    opts = RunOptions(**kw)
    CudaEngine.h2d, CudaEngine.d2h = real_h2d, real_d2h
    ms, fl = timed(opts)
    CudaEngine.h2d = lambda self, slot, *a, waits=(), **k: (
        [self.stream_wait(slot, -1, w) for w in (a[7] if len(a) > 7 else waits)],
        self.record(slot, -1))[1]
    CudaEngine.d2h = lambda self, slot, *a, waits=(), **k: (
        [self.stream_wait(slot, -2, w) for w in (a[7] if len(a) > 7 else waits)],
        self.record(slot, -2))[1]
    ms2, _ = timed(opts)
    extra = ""
    if KIND == "trsm":
        real_trsm = CudaEngine.trsm
        CudaEngine.trsm = lambda self, slot, stream, *a, **k: (
            [self.stream_wait(slot, stream, w) for w in (a[-1] if a else ())],
            self.record(slot, stream))[1]
        ms3, _ = timed(opts)
        CudaEngine.h2d, CudaEngine.d2h = real_h2d, real_d2h
        ms4, _ = timed(opts)
        CudaEngine.trsm = real_trsm
        extra = f"; no link + no solve {ms3:.1f} ms; no solve (link on) {ms4:.1f} ms"
    print(f"{kw}: with link {ms:.1f} ms ({fl / ms / 1e9:.2f} TF/s); no link {ms2:.1f} ms "
          f"({fl / ms2 / 1e9:.2f} TF/s){extra}", flush=True)
CudaEngine.h2d, CudaEngine.d2h = real_h2d, real_d2h
