"""Stand-alone GPU check of the tile kernels through the C ABI (dev tool; the real parity
suite is tests/test_gpu_*.py).  Usage: python tools/kernel_check.py [--perf]"""
import ctypes as C
import sys
import time

import numpy as np
import scipy.linalg

sys.path.insert(0, ".")
from paper_1510_05041_b200 import _native as N

lib = N.load()
N.check(lib.bx_init(1, N.int_array([0]), N.u64_array([4 << 30]), 4), "init")
base = C.c_uint64()
lib.bx_arena_base(0, C.byref(base))
_next = [0]


def alloc(h, w):
    ld = (h + 7) // 8 * 8
    off = _next[0]
    _next[0] += (ld * w * 8 + 255) // 256 * 256
    return off, ld


def put(arr):
    arr = np.asfortranarray(arr, dtype=np.float64)
    h, w = arr.shape
    off, ld = alloc(h, w)
    ev = C.c_int(-1)
    N.check(lib.bx_h2d_tile(0, off, ld, arr.ctypes.data, h, h, w, 8, 0, None, C.byref(ev)), "h2d")
    N.check(lib.bx_event_sync(ev.value))
    lib.bx_event_release(ev.value)
    return off, ld


def get(off, ld, h, w):
    out = np.empty((h, w), order="F")
    ev = C.c_int(-1)
    N.check(lib.bx_d2h_tile(0, off, ld, out.ctypes.data, h, h, w, 8, 0, None, C.byref(ev)), "d2h")
    N.check(lib.bx_event_sync(ev.value))
    lib.bx_event_release(ev.value)
    return out


def gemm(ta, tb, tri, alpha, beta, A_list, B_list, c_arr):
    h, w = c_arr.shape
    offs_a, lda, offs_b, ldb, dep = [], [], [], [], []
    for a, b in zip(A_list, B_list):
        oa, la = put(a)
        ob, lb = put(b)
        offs_a.append(oa); lda.append(la); offs_b.append(ob); ldb.append(lb)
        dep.append(a.shape[0] if ta else a.shape[1])
    oc, lc = put(c_arr)
    ev = C.c_int(-1)
    N.check(lib.bx_gemm_task(0, 0, ta, tb, tri, h, w, len(A_list), N.u64_array(offs_a), N.int_array(lda),
                             N.u64_array(offs_b), N.int_array(ldb), N.int_array(dep), alpha, beta, oc, lc,
                             0, None, C.byref(ev)), "gemm")
    N.check(lib.bx_event_sync(ev.value))
    return get(oc, lc, h, w)


variants = [0]
for a in sys.argv:
    if a.startswith("--variants="):
        variants = [int(x) for x in a.split("=")[1].split(",")]
rng = np.random.default_rng(1)
fails = 0
for var in variants:
  lib.bx_set_gemm_variant(var)
  for (h, w, d, ns) in [(13, 11, 10, 1), (200, 130, 77, 3), (257, 255, 33, 5)]:
    for ta in (0, 1):
        for tb in (0, 1):
            _next[0] = 0
            As = [rng.random((d, h) if ta else (h, d)) * 2 - 1 for _ in range(ns)]
            Bs = [rng.random((w, d) if tb else (d, w)) * 2 - 1 for _ in range(ns)]
            c = rng.random((h, w)) * 2 - 1
            ref = sum((a.T if ta else a) @ (b.T if tb else b) for a, b in zip(As, Bs)) * 1.7 - 0.3 * c
            out = gemm(ta, tb, 0, 1.7, -0.3, As, Bs, c)
            err = np.abs(out - ref).max() / max(1.0, np.abs(ref).max())
            if not err < 1e-13:
                fails += 1
                print("FAIL variant", var, h, w, d, ns, ta, tb, err)
lib.bx_set_gemm_variant(variants[0])
for (h, w, d, ns) in [(13, 11, 10, 1), (128, 128, 16, 1), (200, 130, 77, 3), (1024, 1024, 1024, 2), (257, 255, 33, 5)]:
    for ta in (0, 1):
        for tb in (0, 1):
            for beta in (0.0, 1.0, -0.3):
                _next[0] = 0
                As = [rng.random((d, h) if ta else (h, d)) * 2 - 1 for _ in range(ns)]
                Bs = [rng.random((w, d) if tb else (d, w)) * 2 - 1 for _ in range(ns)]
                c = rng.random((h, w)) * 2 - 1
                if beta == 0.0:
                    c[:] = np.nan
                ref = sum((a.T if ta else a) @ (b.T if tb else b) for a, b in zip(As, Bs)) * 1.7
                if beta != 0.0:
                    ref = ref + beta * c
                out = gemm(ta, tb, 0, 1.7, beta, As, Bs, c)
                err = np.abs(out - ref).max() / max(1.0, np.abs(ref).max())
                ok = err < 1e-13 and np.isfinite(out).all()
                fails += not ok
                if not ok:
                    print("FAIL gemm", h, w, d, ns, ta, tb, beta, err)
# triangle epilogue
for tri in (1, 2):
    _next[0] = 0
    n, d = 300, 50
    a = rng.random((n, d)); c = rng.random((n, n))
    out = gemm(0, 1, tri, 1.0, 0.5, [a], [a], c)
    full = a @ a.T + 0.5 * c
    m = np.tril(np.ones((n, n), bool)) if tri == 1 else np.triu(np.ones((n, n), bool))
    ok = np.allclose(out[m], full[m], rtol=1e-13) and np.array_equal(out[~m], c[~m])
    fails += not ok
    print("tri", tri, "ok" if ok else "FAIL")

# trsm
for n, other in [(37, 29), (256, 100), (1024, 1024), (1500, 64)]:
    for side in ("left", "right"):
        for uplo in ("upper", "lower"):
            for trans in (0, 1):
                for unit in (0, 1):
                    _next[0] = 0
                    a = (rng.random((n, n)) * 2 - 1) / n
                    np.fill_diagonal(a, 1.0 + rng.random(n))
                    b = rng.random((n, other) if side == "left" else (other, n)) * 2 - 1
                    alpha = 0.75
                    e = a.T if trans else a
                    eff_upper = (uplo == "upper") != bool(trans)
                    m = np.triu(e) if eff_upper else np.tril(e)
                    if unit:
                        m = m.copy(); np.fill_diagonal(m, 1.0)
                    if side == "left":
                        ref = scipy.linalg.solve_triangular(m, alpha * b, lower=not eff_upper)
                    else:
                        ref = scipy.linalg.solve_triangular(m.T, alpha * b.T, lower=eff_upper).T
                    oa, la = put(a)
                    ob, lb = put(b)
                    ev = C.c_int(-1)
                    N.check(lib.bx_trsm_tile(0, 0, side == "right", uplo == "upper", trans, unit, b.shape[0],
                                             b.shape[1], alpha, oa, la, ob, lb, 0, None, C.byref(ev)), "trsm")
                    N.check(lib.bx_event_sync(ev.value))
                    out = get(ob, lb, *b.shape)
                    err = np.linalg.norm(out - ref) / np.linalg.norm(ref)
                    ok = err < 1e-12
                    fails += not ok
                    if not ok:
                        print("FAIL trsm", n, other, side, uplo, trans, unit, err)
print("kernel_check fails:", fails)

for var in (variants if "--perf" in sys.argv else []):
    lib.bx_set_gemm_variant(var)
    print("== variant", var)
    for n in (8192, 16384):
        ptrs = []
        for _ in range(3):
            p = C.c_uint64()
            N.check(lib.bx_dev_alloc(0, n * n * 8, C.byref(p)))
            N.check(lib.bx_dev_fill_uniform(0, p.value, n * n, 7, 0))
            ptrs.append(p.value)
        N.check(lib.bx_dgemm_device(0, 0, 0, 0, n, n, n, 1.0, ptrs[0], n, ptrs[1], n, 1.0, ptrs[2], n))
        e0, e1 = C.c_int(), C.c_int()
        best = 1e9
        for rep in range(3):
            lib.bx_event_record(0, 0, 1, C.byref(e0))
            N.check(lib.bx_dgemm_device(0, 0, 0, 0, n, n, n, 1.0, ptrs[0], n, ptrs[1], n, 1.0, ptrs[2], n))
            lib.bx_event_record(0, 0, 1, C.byref(e1))
            lib.bx_event_sync(e1.value)
            ms = C.c_float()
            lib.bx_event_elapsed(e0.value, e1.value, C.byref(ms))
            best = min(best, ms.value)
        print(f"dgemm_device NN n={n}: {best:.3f} ms  {2*n**3/best/1e9:.2f} TF/s")
        for tt in [(0, 1), (1, 0), (1, 1)]:
            N.check(lib.bx_dgemm_device(0, 0, tt[0], tt[1], n, n, n, 1.0, ptrs[0], n, ptrs[1], n, 1.0, ptrs[2], n))
            lib.bx_event_record(0, 0, 1, C.byref(e0))
            N.check(lib.bx_dgemm_device(0, 0, tt[0], tt[1], n, n, n, 1.0, ptrs[0], n, ptrs[1], n, 1.0, ptrs[2], n))
            lib.bx_event_record(0, 0, 1, C.byref(e1))
            lib.bx_event_sync(e1.value)
            lib.bx_event_elapsed(e0.value, e1.value, C.byref(ms))
            print(f"   trans {tt}: {ms.value:.3f} ms {2*n**3/ms.value/1e9:.2f} TF/s")
        for p in ptrs:
            lib.bx_dev_free(0, p)

if "--trsm-perf" in sys.argv:
    for leaf in (32, 64, 128):
        lib.bx_set_trsm_leaf(leaf)
        print("leaf", leaf)
        for n, other in [(1024, 1024), (2048, 2048)]:
            for side in ("left", "right"):
                _next[0] = 0
                a = (rng.random((n, n)) * 2 - 1) / n
                np.fill_diagonal(a, 1.5)
                b = rng.random((n, other) if side == "left" else (other, n)) * 2 - 1
                oa, la = put(a)
                ob, lb = put(b)
                e0, e1, ev = C.c_int(), C.c_int(), C.c_int()
                args = (0, 0, side == "right", 0, 0, 0, b.shape[0], b.shape[1], 1.0, oa, la, ob, lb, 0, None, C.byref(ev))
                N.check(lib.bx_trsm_tile(*args))
                lib.bx_event_sync(ev.value)
                best = 1e9
                for _ in range(3):
                    lib.bx_event_record(0, 0, 1, C.byref(e0))
                    N.check(lib.bx_trsm_tile(*args))
                    lib.bx_event_record(0, 0, 1, C.byref(e1))
                    lib.bx_event_sync(e1.value)
                    ms = C.c_float()
                    lib.bx_event_elapsed(e0.value, e1.value, C.byref(ms))
                    best = min(best, ms.value)
                fl = n * n * other
                print(f"trsm {side} n={n} rhs={other}: {best*1e3:.1f} us  {fl/best/1e9:.2f} TF/s")

if "--small-gemm" in sys.argv:
    for var in variants:
        lib.bx_set_gemm_variant(var)
        for (m, n, k) in [(64, 1024, 64), (128, 1024, 128), (512, 1024, 512), (1024, 1024, 1024), (64, 64, 64)]:
            ptrs = []
            for nel in (m * k, k * n, m * n):
                p = C.c_uint64()
                N.check(lib.bx_dev_alloc(0, nel * 8, C.byref(p)))
                N.check(lib.bx_dev_fill_uniform(0, p.value, nel, 3, 0))
                ptrs.append(p.value)
            e0, e1 = C.c_int(), C.c_int()
            N.check(lib.bx_dgemm_device(0, 0, 0, 0, m, n, k, 1.0, ptrs[0], m, ptrs[1], k, 1.0, ptrs[2], m))
            lib.bx_device_sync(0)
            lib.bx_event_record(0, 0, 1, C.byref(e0))
            for _ in range(20):
                N.check(lib.bx_dgemm_device(0, 0, 0, 0, m, n, k, 1.0, ptrs[0], m, ptrs[1], k, 1.0, ptrs[2], m))
            lib.bx_event_record(0, 0, 1, C.byref(e1))
            lib.bx_event_sync(e1.value)
            ms = C.c_float()
            lib.bx_event_elapsed(e0.value, e1.value, C.byref(ms))
            print(f"variant {var} gemm {m}x{n}x{k}: {ms.value / 20 * 1e3:.1f} us per launch")
            for p in ptrs:
                lib.bx_dev_free(0, p)

if "--launch-overhead" in sys.argv:
    import time as _t
    p = C.c_uint64()
    N.check(lib.bx_dev_alloc(0, 1 << 20, C.byref(p)))
    ptrs = []
    for nel in (64 * 64, 64 * 64, 64 * 64):
        q = C.c_uint64()
        N.check(lib.bx_dev_alloc(0, nel * 8, C.byref(q)))
        ptrs.append(q.value)
    e0, e1 = C.c_int(), C.c_int()
    for label, fn in [("fill n=1", lambda: lib.bx_dev_fill_uniform(0, p.value, 1, 1, 0)),
                      ("gemm 64^3", lambda: lib.bx_dgemm_device(0, 0, 0, 0, 64, 64, 64, 1.0, ptrs[0], 64, ptrs[1], 64, 1.0, ptrs[2], 64))]:
        fn(); lib.bx_device_sync(0)
        t0 = _t.perf_counter()
        lib.bx_event_record(0, 0, 1, C.byref(e0))
        for _ in range(50):
            fn()
        lib.bx_event_record(0, 0, 1, C.byref(e1))
        t1 = _t.perf_counter()
        lib.bx_event_sync(e1.value)
        ms = C.c_float()
        lib.bx_event_elapsed(e0.value, e1.value, C.byref(ms))
        print(f"{label}: host {(t1 - t0) / 50 * 1e6:.1f} us/call, gpu {ms.value / 50 * 1e3:.1f} us/launch")

for _a in sys.argv:
    if _a.startswith("--sgemm-variant="):
        N.check(lib.bx_set_sgemm_variant(int(_a.split("=")[1])))

if "--sgemm-only-perf" in sys.argv:
    for n in (16384,):
        ptrs = []
        for _ in range(3):
            p = C.c_uint64()
            N.check(lib.bx_dev_alloc(0, n * n * 4, C.byref(p)))
            N.check(lib.bx_dev_fill_uniform_f32(0, p.value, n * n, 5, 0))
            ptrs.append(p.value)
        for _ in range(2):
            N.check(lib.bx_sgemm_device(0, 0, 0, 0, n, n, n, 1.0, ptrs[0], n, ptrs[1], n, 0.0, ptrs[2], n))
        lib.bx_device_sync(0)

if "--sgemm" in sys.argv:
    def put32(arr):
        arr = np.asfortranarray(arr, dtype=np.float32)
        h, w = arr.shape
        ld = (h + 7) // 8 * 8
        off = _next[0]
        _next[0] += (ld * w * 4 + 1023) // 1024 * 1024
        ev = C.c_int(-1)
        N.check(lib.bx_h2d_tile(0, off, ld, arr.ctypes.data, h, h, w, 4, 0, None, C.byref(ev)), "h2d32")
        N.check(lib.bx_event_sync(ev.value))
        return off, ld

    def get32(off, ld, h, w):
        out = np.empty((h, w), order="F", dtype=np.float32)
        ev = C.c_int(-1)
        N.check(lib.bx_d2h_tile(0, off, ld, out.ctypes.data, h, h, w, 4, 0, None, C.byref(ev)), "d2h32")
        N.check(lib.bx_event_sync(ev.value))
        return out

    sf = 0
    for (h, w, d, ns) in [(128, 256, 32, 1), (300, 500, 100, 1), (1024, 1024, 1024, 2), (77, 33, 45, 3)]:
        for ta in (0, 1):
            for tb in (0, 1):
                for beta in (0.0, 0.5):
                    _next[0] = 0
                    As = [(rng.random((d, h) if ta else (h, d)) * 2 - 1).astype(np.float32) for _ in range(ns)]
                    Bs = [(rng.random((w, d) if tb else (d, w)) * 2 - 1).astype(np.float32) for _ in range(ns)]
                    c = (rng.random((h, w)) * 2 - 1).astype(np.float32)
                    ref = sum((a.T if ta else a).astype(np.float64) @ (b.T if tb else b).astype(np.float64)
                              for a, b in zip(As, Bs)) * 1.25 + beta * c.astype(np.float64)
                    ao, al, bo, bl, dep = [], [], [], [], []
                    for a, b in zip(As, Bs):
                        o, l = put32(a); ao.append(o); al.append(l)
                        o, l = put32(b); bo.append(o); bl.append(l)
                        dep.append(d)
                    oc, lc = put32(c)
                    ev = C.c_int(-1)
                    N.check(lib.bx_sgemm_task(0, 0, ta, tb, h, w, ns, N.u64_array(ao), N.int_array(al), N.u64_array(bo),
                                              N.int_array(bl), N.int_array(dep), 1.25, beta, oc, lc, 0, None, C.byref(ev)), "sgemm")
                    N.check(lib.bx_event_sync(ev.value))
                    out = get32(oc, lc, h, w).astype(np.float64)
                    err = np.linalg.norm(out - ref) / np.linalg.norm(ref)
                    ok = err < 2e-3 and np.isfinite(out).all()
                    sf += not ok
                    if not ok:
                        print("FAIL sgemm", h, w, d, ns, ta, tb, beta, err, np.abs(out - ref).max())
    print("sgemm fails:", sf)
    if "--perf" in sys.argv or "--sgemm-perf" in sys.argv:
        for n in (8192, 16384, 32768):
            ptrs = []
            for _ in range(3):
                p = C.c_uint64()
                N.check(lib.bx_dev_alloc(0, n * n * 4, C.byref(p)))
                N.check(lib.bx_dev_fill_uniform_f32(0, p.value, n * n, 9, 0))
                ptrs.append(p.value)
            for tt in [(0, 0), (0, 1), (1, 0), (1, 1)]:
                N.check(lib.bx_sgemm_device(0, 0, tt[0], tt[1], n, n, n, 1.0, ptrs[0], n, ptrs[1], n, 0.0, ptrs[2], n))
                e0, e1 = C.c_int(), C.c_int()
                lib.bx_event_record(0, 0, 1, C.byref(e0))
                N.check(lib.bx_sgemm_device(0, 0, tt[0], tt[1], n, n, n, 1.0, ptrs[0], n, ptrs[1], n, 0.0, ptrs[2], n))
                lib.bx_event_record(0, 0, 1, C.byref(e1))
                lib.bx_event_sync(e1.value)
                ms = C.c_float()
                lib.bx_event_elapsed(e0.value, e1.value, C.byref(ms))
                print(f"sgemm_device n={n} trans {tt}: {ms.value:.3f} ms {2*n**3/ms.value/1e9:.1f} TF/s")
            for p in ptrs:
                lib.bx_dev_free(0, p)
