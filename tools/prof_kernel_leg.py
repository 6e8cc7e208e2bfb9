"""The bench's kernel leg (one device-resident launch of the dominant kernel on uniform
operands, bench.py kernel_leg) for ncu: python tools/prof_kernel_leg.py m n k [f32] [reps]"""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_1510_05041_b200 import _native as N  # noqa: E402
from paper_1510_05041_b200.engine import get_engine  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4])
f32 = len(sys.argv) > 4 and sys.argv[4] == "f32"
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
eng = get_engine([0])
lib = eng.lib
esz = 4 if f32 else 8
ptrs = []
for i, nel in enumerate((m * k, k * n, m * n)):
    p = C.c_uint64()
    N.check(lib.bx_dev_alloc(0, nel * esz, C.byref(p)))
    fill = lib.bx_dev_fill_uniform_f32 if f32 else lib.bx_dev_fill_uniform
    N.check(fill(0, p.value, nel, 11 + i, 0))
    ptrs.append(p.value)
a, b, c = ptrs
for _ in range(reps):
    if f32:
        N.check(lib.bx_sgemm_device(0, 0, 0, 0, m, n, k, 1.0, a, m, b, k, 0.0, c, m))
    else:
        N.check(lib.bx_dgemm_device(0, 0, 0, 0, m, n, k, 1.0, a, m, b, k, 1.0, c, m))
eng.device_sync(0)
print("done")
