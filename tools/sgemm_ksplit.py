"""SGEMM 32768^3 device-resident: one launch over the whole K vs K split into chained
launches (beta = 1 after the first: C read + written once per chunk, A/B panels of each
chunk small enough to stay in L2), per raster group; alternating rounds, device events.
python tools/sgemm_ksplit.py [n] [rounds] [splits,...] [groups,...]   (BX_ONCE=1: one of each, for ncu)"""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, ".")
from paper_1510_05041_b200 import _native as N  # noqa: E402
from paper_1510_05041_b200.engine import get_engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 4
splits = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "1,2,4").split(",")]
groups = [int(x) for x in (sys.argv[4] if len(sys.argv) > 4 else "4").split(",")]
eng = get_engine([0])
lib = eng.lib
ptrs = []
for i in range(3):
    p = C.c_uint64()
    N.check(lib.bx_dev_alloc(0, n * n * 4, C.byref(p)))
    N.check(lib.bx_dev_fill_uniform_f32(0, p.value, n * n, 11 + i, 0))
    ptrs.append(p.value)
a, b, c = ptrs


def run(split, group):
    N.check(lib.bx_set_sgemm_debug(group << 8))
    kc = n // split
    for s in range(split):
        N.check(lib.bx_sgemm_device(0, 0, 0, 0, n, n, kc, 1.0, a + 4 * s * kc * n, n,
                                    b + 4 * s * kc, n, 0.0 if s == 0 else 1.0, c, n))


sets = [(s, g) for s in splits for g in groups]
if os.environ.get("BX_ONCE") == "1":
    for s, g in sets:
        run(s, g)
        eng.device_sync(0)
    sys.exit(0)
for s, g in sets:
    run(s, g)
eng.device_sync(0)
times = {k: [] for k in sets}
for _ in range(rounds):
    for s, g in sets:
        e0 = eng.record(0, 0, timing=True)
        run(s, g)
        e1 = eng.record(0, 0, timing=True)
        eng.sync(e1)
        times[(s, g)].append(eng.elapsed_ms(e0, e1))
        eng.release(e0)
        eng.release(e1)
N.check(lib.bx_set_sgemm_debug(0))
for (s, g), ts in times.items():
    ms = statistics.median(ts)
    print(f"n={n} K split {s} group {g}: median {ms:.2f} ms = {2 * n ** 3 / ms / 1e9:.1f} TF/s (min {min(ts):.2f})", flush=True)
