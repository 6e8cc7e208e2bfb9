"""One SYRK diagonal-tile launch (triangle epilogue, C_lower += A A^T over k-steps) through
the engine, for ncu: python tools/prof_syrk.py [T] [ksteps]"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_1510_05041_b200.engine import get_engine  # noqa: E402

t = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ks = int(sys.argv[2]) if len(sys.argv) > 2 else 8
eng = get_engine([0])
eng.ensure_arenas({0: (ks + 2) * t * t * 8 + (64 << 20)})
rng = np.random.default_rng(0)


class D:
    def __init__(self, arr):
        self.arr, self.leading_dim, self.itemsize = arr, arr.shape[0], 8

    def element_address(self, r, c):
        return self.arr.ctypes.data + (r + c * self.leading_dim) * 8


tiles = [np.asfortranarray(rng.random((t, t)) * 2 - 1) for _ in range(ks)]
offs = [i * t * t * 8 for i in range(ks)]
for o, a in zip(offs, tiles):
    eng.sync(eng.h2d(0, o, t, D(a), 0, 0, t, t))
c_off = ks * t * t * 8
eng.sync(eng.h2d(0, c_off, t, D(np.asfortranarray(rng.random((t, t)))), 0, 0, t, t))
steps = [(o, t, o, t, t) for o in offs]
for _ in range(3):
    ev = eng.gemm(0, 0, False, True, 1, t, t, steps, 1.0, 1.0, c_off, t)
    eng.sync(ev)
print("done")
