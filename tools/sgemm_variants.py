"""Device-resident SGEMM (tcgen05 kind::tf32) rate per operand major-ness and kernel variant.
python tools/sgemm_variants.py [n]"""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, ".")
from paper_1510_05041_b200 import _native as N  # noqa: E402
from paper_1510_05041_b200.engine import get_engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
eng = get_engine([0])
lib = eng.lib
ptrs = []
for i in range(3):
    p = C.c_uint64()
    N.check(lib.bx_dev_alloc(0, n * n * 4, C.byref(p)))
    N.check(lib.bx_dev_fill_uniform_f32(0, p.value, n * n, 11 + i, 0))
    ptrs.append(p.value)
a, b, c = ptrs
M, NN, K = (int(x) for x in os.environ.get("BX_MNK", f"{n},{n},{n}").split(","))
variants = [int(x) for x in sys.argv[2:]] or [0, 1]
dbgs = [int(x) for x in os.environ.get("BX_SGEMM_DEBUG", "0").split(",")]
layouts = [tuple(int(c) for c in x) for x in os.environ.get("BX_LAYOUTS", "00,10,01,11").split(",")]
reps = int(os.environ.get("BX_REPS", "1"))
for var, dbg in [(v, d) for _ in range(reps) for v in variants for d in dbgs]:
    N.check(lib.bx_set_sgemm_variant(var))
    N.check(lib.bx_set_sgemm_debug(dbg))
    for ta, tb in layouts:
        ts = []
        for i in range(5):
            e0 = eng.record(0, 0, timing=True)
            N.check(lib.bx_sgemm_device(0, 0, ta, tb, M, NN, K, 1.0, a, M if not ta else K, b,
                                        K if not tb else NN, 0.0, c, M))
            e1 = eng.record(0, 0, timing=True)
            eng.sync(e1)
            if i:
                ts.append(eng.elapsed_ms(e0, e1))
            eng.release(e0)
            eng.release(e1)
        ms = statistics.median(ts)
        print(f"variant {var} dbg {dbg} ta={ta} tb={tb} {M}x{NN}x{K}: {ms:.3f} ms  "
              f"{2 * M * NN * K / ms / 1e9:.1f} TF/s", flush=True)
