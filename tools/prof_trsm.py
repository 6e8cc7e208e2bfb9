"""One TRSM tile solve (n x n triangle, n RHS) through the C ABI, for ncu launch lists."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np

from paper_1510_05041_b200 import _native as N
from paper_1510_05041_b200.engine import get_engine

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
leaf = int(sys.argv[2]) if len(sys.argv) > 2 else 128
eng = get_engine([0])
lib = eng.lib
eng.ensure_arenas({0: 64 << 20})
lib.bx_set_trsm_leaf(leaf)
rng = np.random.default_rng(0)
a = np.asfortranarray((rng.random((n, n)) * 2 - 1) / n)
np.fill_diagonal(a, 1.5)
b = np.asfortranarray(rng.random((n, n)))


class D:  # minimal desc for engine.h2d
    def __init__(self, arr):
        self.arr = arr
        self.leading_dim = arr.shape[0]
        self.itemsize = 8

    def element_address(self, r, c):
        return self.arr.ctypes.data + (r + c * self.leading_dim) * 8


ea = eng.h2d(0, 0, n, D(a), 0, 0, n, n)
eb = eng.h2d(0, n * n * 8, n, D(b), 0, 0, n, n)
eng.sync(eb)
for _ in range(3):
    ev = eng.trsm(0, 0, False, False, False, False, n, n, 1.0, 0, n, n * n * 8, n)
    eng.sync(ev)
print("done")
