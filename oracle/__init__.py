"""CPU oracle for the tiled level-3 BLAS hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything from this package, and only as the
checker (or as the timed CPU baseline), never as the product path.  The product
(`paper_1510_05041_b200`) never imports it and has no CPU fallback.

Contents
--------
``tiled``     numpy restatement of the reference's tiled runtime numerics: the tile
              kernels (``/root/reference/pkg/src/tileblas/kernels.py``) and the
              per-output-tile step sequences of the planner
              (``/root/reference/pkg/src/tileblas/routines.py:227-380``) executed in
              dependency order (``routines.py:482-511``).
``dense``     whole-matrix references (``/root/reference/pkg/src/tileblas/oracle.py``).
``tolerance`` the north-star normwise bounds (BASELINE.json ``north_star``).

Pinning: ``tests/test_oracle_golden.py`` checks ``tiled`` and ``dense`` against
golden vectors produced by running the reference itself
(``tests/golden/make_golden.py`` imports ``/root/reference/pkg/src`` in the build
container; the ``.npz`` fixtures it writes are committed).
"""
