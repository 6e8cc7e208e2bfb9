"""Time one diagonal solve (n-triangle, n RHS) in isolation per leaf order, on one stream.
python tools/trsm_solve_time.py [n]"""
import statistics
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_1510_05041_b200.engine import get_engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
eng = get_engine([0])
eng.ensure_arenas({0: 64 << 20})
rng = np.random.default_rng(0)
a = np.asfortranarray((rng.random((n, n)) * 2 - 1) / n)
np.fill_diagonal(a, 1.5)
b = np.asfortranarray(rng.random((n, n)))


class D:
    def __init__(self, arr):
        self.arr, self.leading_dim, self.itemsize = arr, arr.shape[0], 8

    def element_address(self, r, c):
        return self.arr.ctypes.data + (r + c * self.leading_dim) * 8


eng.sync(eng.h2d(0, 0, n, D(a), 0, 0, n, n))
import itertools  # noqa: E402
import os  # noqa: E402
rhs_list = [int(x) for x in os.environ.get("BX_RHS", "16").split(",")]
for leaf, nr in itertools.product([int(x) for x in (sys.argv[2:] or ["32", "64", "128", "256", "512"])], rhs_list):
    eng.lib.bx_set_trsm_leaf(leaf)
    eng.lib.bx_set_trsm_rhs(nr)
    ts = []
    for i in range(12):
        eng.sync(eng.h2d(0, n * n * 8, n, D(b), 0, 0, n, n))
        e0 = eng.record(0, 0, timing=True)
        ev = eng.trsm(0, 0, False, False, False, False, n, n, 1.0, 0, n, n * n * 8, n)
        e1 = eng.record(0, 0, timing=True)
        eng.sync(e1)
        if i >= 2:
            ts.append(eng.elapsed_ms(e0, e1))
        for e in (e0, e1, ev):
            eng.release(e)
    ms = statistics.median(ts)
    print(f"n={n} leaf={leaf} rhs={nr}: {ms * 1e3:.1f} us  ({n ** 3 / ms / 1e9:.2f} TF/s)", flush=True)
