"""The inverse-based TRSM diagonal step through the C ABI, for ncu: inv(E) of one n x n
lower triangle (bx_trsm_inverse: identity + recursive substitution) and X = inv(E) B with
n right-hand sides (bx_trsm_apply: FP64 task GEMM with the triangular-operand k-range).
python tools/prof_trsm_inv.py [n] [reps]"""
import sys

sys.path.insert(0, ".")
import numpy as np

from paper_1510_05041_b200.engine import get_engine

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
eng = get_engine([0])
eng.ensure_arenas({0: 4 * n * n * 8 + (16 << 20)})
rng = np.random.default_rng(0)
a = np.asfortranarray(np.tril(rng.random((n, n)) * 2 - 1) / n)
np.fill_diagonal(a, 1.5)
b = np.asfortranarray(rng.random((n, n)))


class D:  # minimal desc for engine.h2d / d2h
    def __init__(self, arr):
        self.arr = arr
        self.leading_dim = arr.shape[0]
        self.itemsize = 8

    def element_address(self, r, c):
        return self.arr.ctypes.data + (r + c * self.leading_dim) * 8


A, B, INV, X = 0, n * n * 8, 2 * n * n * 8, 3 * n * n * 8
for arr in (a, b):
    eng.register_host(arr)
eng.sync(eng.h2d(0, A, n, D(a), 0, 0, n, n))
eng.sync(eng.h2d(0, B, n, D(b), 0, 0, n, n))
for _ in range(reps):
    ev = eng.trsm_inverse(0, 0, False, False, False, n, A, n, INV, n)
    ev = eng.trsm_apply(0, 0, False, False, n, n, 1.0, INV, n, B, n, X, n, waits=(ev,))
    eng.sync(ev)
x = np.zeros((n, n), order="F")
eng.sync(eng.d2h(0, X, n, D(x), 0, 0, n, n))
res = np.linalg.norm(a @ x - b) / (np.linalg.norm(a) * np.linalg.norm(x) * n * np.finfo(float).eps)
print(f"n={n}: residual ratio {res:.3e}")
