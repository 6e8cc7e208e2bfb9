"""Device-resident DGEMM rate per operand layout (NN, TN, NT, TT) on the FP64 task GEMM.
python tools/dgemm_layouts.py [n] [reps]"""
import ctypes as C
import statistics
import sys

sys.path.insert(0, ".")
from paper_1510_05041_b200 import _native as N  # noqa: E402
from paper_1510_05041_b200.engine import get_engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
eng = get_engine([0])
lib = eng.lib
ptrs = []
for i in range(3):
    p = C.c_uint64()
    N.check(lib.bx_dev_alloc(0, n * n * 8, C.byref(p)))
    N.check(lib.bx_dev_fill_uniform(0, p.value, n * n, 11 + i, 0))
    ptrs.append(p.value)
a, b, c = ptrs
for ta, tb in ((0, 0), (1, 0), (0, 1), (1, 1)):
    N.check(lib.bx_dgemm_device(0, 0, ta, tb, n, n, n, 1.0, a, n, b, n, 1.0, c, n))
    eng.device_sync(0)
    ts = []
    for _ in range(reps):
        e0 = eng.record(0, 0, timing=True)
        N.check(lib.bx_dgemm_device(0, 0, ta, tb, n, n, n, 1.0, a, n, b, n, 1.0, c, n))
        e1 = eng.record(0, 0, timing=True)
        eng.sync(e1)
        ts.append(eng.elapsed_ms(e0, e1))
        eng.release(e0)
        eng.release(e1)
    ms = statistics.median(ts)
    print(f"{'NT'[ta]}{'NT'[tb]} n={n}: {ms:.2f} ms {2 * n ** 3 / ms / 1e9:.2f} TF/s", flush=True)
