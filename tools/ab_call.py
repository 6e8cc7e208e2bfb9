"""A/B of two builds of libblasx_cuda.so on one host-resident routine call (run the script
once per build, alternating): python tools/ab_call.py LIB.so kind n k tile reps
-> median device-event ms of `reps` calls after one warm-up (the current runtime, the given
kernels library)."""
import statistics
import sys

sys.path.insert(0, ".")
from paper_1510_05041_b200 import _native  # noqa: E402

lib_path, kind, n, k, t, reps = sys.argv[1], sys.argv[2], *(int(x) for x in sys.argv[3:7])
_native.load(lib_path)
from paper_1510_05041_b200 import RunOptions, build_call, run_call  # noqa: E402
from paper_1510_05041_b200.engine import get_engine  # noqa: E402

call = build_call(kind, m=n, n=n, k=k, tile_size=t, seed=0, alpha=1.0,
                  beta=1.0 if kind in ("gemm", "syrk", "syr2k", "symm") else 0.0, uplo="lower",
                  trsm_scaled=True)
eng = get_engine([0])
for x in [y for y in (call.a, call.b, call.c) if y is not None]:
    eng.register_host(x.matrix.storage)
res = run_call(call)
ts = []
for _ in range(reps):
    e0 = eng.record(0, 0, timing=True)
    run_call(call)
    e1 = eng.record(0, 0, timing=True)
    eng.sync(e1)
    ts.append(eng.elapsed_ms(e0, e1))
    eng.release(e0)
    eng.release(e1)
ms = statistics.median(ts)
print(f"{lib_path.split('/')[-1]} {kind} {n} k={k} T={t}: median {ms:.2f} ms "
      f"{res.plan.total_flops / ms / 1e9:.2f} TF/s (min {min(ts):.2f})", flush=True)
