"""One device-resident DGEMM launch for ncu (python tools/prof_gemm.py N [ta tb])."""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_1510_05041_b200 import _native as N
from paper_1510_05041_b200.engine import get_engine

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
ta = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tb = int(sys.argv[3]) if len(sys.argv) > 3 else 0
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
eng = get_engine([0])
lib = eng.lib
ptrs = []
for i in range(3):
    p = C.c_uint64()
    N.check(lib.bx_dev_alloc(0, n * n * 8, C.byref(p)))
    N.check(lib.bx_dev_fill_uniform(0, p.value, n * n, 11 + i, 0))
    ptrs.append(p.value)
for _ in range(reps):
    N.check(lib.bx_dgemm_device(0, 0, ta, tb, n, n, n, 1.0, ptrs[0], n, ptrs[1], n, 1.0, ptrs[2], n))
eng.device_sync(0)
print("done")
