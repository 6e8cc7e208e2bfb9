"""A/B of two builds of libblasx_cuda.so on the device-resident DGEMM (same box):
python tools/ab_dgemm.py LIB.so N reps -> ms per launch (host clock around `reps` launches
after one warm-up, device-synchronised).  Plain ctypes, so older builds load too."""
import ctypes as C
import sys
import time

lib_path, n, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
lib = C.CDLL(lib_path)
u64, i, d = C.c_uint64, C.c_int, C.c_double
lib.bx_dev_alloc.argtypes = [i, u64, C.POINTER(u64)]
lib.bx_dev_fill_uniform.argtypes = [i, u64, u64, u64, i]
lib.bx_dgemm_device.argtypes = [i, i, i, i, i, i, i, d, u64, i, u64, i, d, u64, i]


def ok(rc):
    assert rc == 0, rc


ok(lib.bx_init(1, (i * 1)(0), (u64 * 1)(0), 1))
ptrs = []
for s in range(3):
    p = u64()
    ok(lib.bx_dev_alloc(0, n * n * 8, C.byref(p)))
    ok(lib.bx_dev_fill_uniform(0, p.value, n * n, 11 + s, 0))
    ptrs.append(p.value)
ok(lib.bx_dgemm_device(0, 0, 0, 0, n, n, n, 1.0, ptrs[0], n, ptrs[1], n, 1.0, ptrs[2], n))
ok(lib.bx_device_sync(0))
t0 = time.perf_counter()
for _ in range(reps):
    ok(lib.bx_dgemm_device(0, 0, 0, 0, n, n, n, 1.0, ptrs[0], n, ptrs[1], n, 1.0, ptrs[2], n))
ok(lib.bx_device_sync(0))
dt = (time.perf_counter() - t0) / reps
print(f"{lib_path}: n={n} {dt * 1e3:.2f} ms {2 * n ** 3 / dt / 1e12:.2f} TF/s", flush=True)
