"""Python half of the legacy BLAS ABI (``libblasx.so``, ``include/blasx_cblas.h``).

``csrc/blasx_cblas.c`` turns every ``cblas_*`` / Fortran ``*_`` call into one call of a
function below with plain integers (CBLAS enum values; Fortran flag characters are mapped to
the same enums in C), raw host addresses and sizes.  Here the arguments are checked the way
reference BLAS checks them (xerbla numbering), CblasRowMajor is rewritten
as the equivalent column-major call, and the column-major call runs through the cblas-style
adapter (``blas.py``) — i.e. through ``RoutineCall`` + ``run_call``, the reference's own API
(/root/reference/pkg/src/tileblas/routines.py:49-67, scheduler.py:665-669).

Every function returns the status ``blasx_last_status()`` reports (include/blasx_cblas.h):
0 ok, ``-i`` illegal parameter i, 5/6/7 runtime errors.  Exceptions never cross into C.

The only host arithmetic here is BLAS's quick-return scaling (``k == 0`` or ``alpha == 0``:
C <- beta C, B <- 0), which reference BLAS also performs without a product.
"""

from __future__ import annotations

import ctypes
import os
import sys

import numpy as np

from . import blas
from .errors import (ArenaOutOfMemoryError, CapacityDeadlockError, InvalidArgumentError,
                     SingularMatrixError)

ROW, COL = 101, 102
NOTRANS, TRANS, CONJTRANS = 111, 112, 113
UPPER, LOWER = 121, 122
NONUNIT, UNIT = 131, 132
LEFT, RIGHT = 141, 142

_tile = [0]


def set_tile(t: int) -> int:
    _tile[0] = int(t) if int(t) > 0 else 0
    return 0


def get_tile() -> int:
    if _tile[0] <= 0:
        _tile[0] = int(os.environ.get("BLASX_TILE", blas.DEFAULT_TILE))
    return _tile[0]


def _xerbla(api: int, name: str, pos: int) -> int:
    """pos = Fortran parameter position; the cblas entry points number Order as 1."""
    info = pos + 1 if api else pos
    label = f"cblas_{name.lower()}" if api else name.upper()
    sys.stderr.write(f" ** On entry to {label} parameter number {info} had an illegal value\n")
    sys.stderr.flush()
    return -info


def _view(addr: int, rows: int, cols: int, ld: int, dtype):
    """1-d numpy view over a column-major (rows x cols, ld) host buffer."""
    n = 0 if rows == 0 or cols == 0 else ld * (cols - 1) + rows
    if n == 0:
        return np.zeros(0, dtype)
    ct = ctypes.c_double if dtype == np.float64 else ctypes.c_float
    return np.ctypeslib.as_array((ct * n).from_address(addr))


def _mat2d(v, rows, cols, ld):
    """(rows x cols) column-major window of a 1-d view (for quick-return scaling)."""
    return np.lib.stride_tricks.as_strided(v, shape=(rows, cols),
                                           strides=(v.itemsize, v.itemsize * ld))


def _flip_uplo(u):
    return LOWER if u == UPPER else UPPER


def _flip_side(s):
    return RIGHT if s == LEFT else LEFT


def _flip_trans(t):
    return NOTRANS if t in (TRANS, CONJTRANS) else TRANS


def _tchar(t):
    return "N" if t == NOTRANS else "T"


def _run(fn):
    try:
        fn()
        return 0
    except SingularMatrixError as e:
        sys.stderr.write(f"blasx: {e}\n")
        return 6
    except (ArenaOutOfMemoryError, CapacityDeadlockError) as e:
        sys.stderr.write(f"blasx: {e}\n")
        return 7
    except InvalidArgumentError as e:
        sys.stderr.write(f"blasx: {e}\n")
        return 5


def _ld_ok(ld, rows, cols, order):
    """Leading-dimension check in the caller's layout."""
    need = rows if order == COL else cols
    return ld >= max(1, need)


# ----------------------------------------------------------------------------- GEMM

def gemm(api, order, ta, tb, m, n, k, alpha, pa, lda, pb, ldb, beta, pc, ldc, esz):
    name = "SGEMM" if esz == 4 else "DGEMM"
    dtype = np.float32 if esz == 4 else np.float64
    if api and order not in (ROW, COL):
        return _xerbla(api, name, 0)
    if ta not in (NOTRANS, TRANS, CONJTRANS):
        return _xerbla(api, name, 1)
    if tb not in (NOTRANS, TRANS, CONJTRANS):
        return _xerbla(api, name, 2)
    if m < 0:
        return _xerbla(api, name, 3)
    if n < 0:
        return _xerbla(api, name, 4)
    if k < 0:
        return _xerbla(api, name, 5)
    ar, ac = (k, m) if ta != NOTRANS else (m, k)
    br, bc = (n, k) if tb != NOTRANS else (k, n)
    if not _ld_ok(lda, ar, ac, order):
        return _xerbla(api, name, 8)
    if not _ld_ok(ldb, br, bc, order):
        return _xerbla(api, name, 10)
    if not _ld_ok(ldc, m, n, order):
        return _xerbla(api, name, 13)
    if order == ROW:      # C^T = op(B)^T op(A)^T : a column-major gemm with swapped operands
        ta, tb, m, n, pa, lda, pb, ldb = tb, ta, n, m, pb, ldb, pa, lda
        ar, ac = (k, m) if ta != NOTRANS else (m, k)
        br, bc = (n, k) if tb != NOTRANS else (k, n)
    if m == 0 or n == 0 or ((alpha == 0.0 or k == 0) and beta == 1.0):
        return 0
    c = _view(pc, m, n, ldc, dtype)
    if alpha == 0.0 or k == 0:
        w = _mat2d(c, m, n, ldc)
        if beta == 0.0:
            w[...] = 0
        else:
            w *= dtype(beta)
        return 0
    a = _view(pa, ar, ac, lda, dtype)
    b = _view(pb, br, bc, ldb, dtype)
    return _run(lambda: blas.dgemm(_tchar(ta), _tchar(tb), m, n, k, alpha, a, lda, b, ldb, beta,
                                   c, ldc, tile_size=get_tile(), dtype=dtype))


# ----------------------------------------------------------------------------- SYRK / SYR2K

def _rank_k(kind, api, order, uplo, trans, n, k, alpha, pa, lda, pb, ldb, beta, pc, ldc):
    name = "DSYRK" if kind == "syrk" else "DSYR2K"
    two = kind == "syr2k"
    if api and order not in (ROW, COL):
        return _xerbla(api, name, 0)
    if uplo not in (UPPER, LOWER):
        return _xerbla(api, name, 1)
    if trans not in (NOTRANS, TRANS, CONJTRANS):
        return _xerbla(api, name, 2)
    if n < 0:
        return _xerbla(api, name, 3)
    if k < 0:
        return _xerbla(api, name, 4)
    ar, ac = (k, n) if trans != NOTRANS else (n, k)
    if not _ld_ok(lda, ar, ac, order):
        return _xerbla(api, name, 7)
    if two and not _ld_ok(ldb, ar, ac, order):
        return _xerbla(api, name, 9)
    if not _ld_ok(ldc, n, n, order):
        return _xerbla(api, name, 12 if two else 10)
    if order == ROW:      # row-major storage = transposed column-major: flip uplo and trans
        uplo, trans = _flip_uplo(uplo), _flip_trans(trans)
        ar, ac = ac, ar
    if n == 0 or ((alpha == 0.0 or k == 0) and beta == 1.0):
        return 0
    c = _view(pc, n, n, ldc, np.float64)
    if alpha == 0.0 or k == 0:
        w = _mat2d(c, n, n, ldc)
        mask = np.tril(np.ones((n, n), bool)) if uplo == LOWER else np.triu(np.ones((n, n), bool))
        w[mask] = 0.0 if beta == 0.0 else w[mask] * beta
        return 0
    a = _view(pa, ar, ac, lda, np.float64)
    u = "L" if uplo == LOWER else "U"
    if two:
        b = _view(pb, ar, ac, ldb, np.float64)
        return _run(lambda: blas.dsyr2k(u, _tchar(trans), n, k, alpha, a, lda, b, ldb, beta, c,
                                        ldc, tile_size=get_tile()))
    return _run(lambda: blas.dsyrk(u, _tchar(trans), n, k, alpha, a, lda, beta, c, ldc,
                                   tile_size=get_tile()))


def syrk(api, order, uplo, trans, n, k, alpha, pa, lda, beta, pc, ldc):
    return _rank_k("syrk", api, order, uplo, trans, n, k, alpha, pa, lda, 0, 1, beta, pc, ldc)


def syr2k(api, order, uplo, trans, n, k, alpha, pa, lda, pb, ldb, beta, pc, ldc):
    return _rank_k("syr2k", api, order, uplo, trans, n, k, alpha, pa, lda, pb, ldb, beta, pc, ldc)


# ----------------------------------------------------------------------------- SYMM

def symm(api, order, side, uplo, m, n, alpha, pa, lda, pb, ldb, beta, pc, ldc):
    name = "DSYMM"
    if api and order not in (ROW, COL):
        return _xerbla(api, name, 0)
    if side not in (LEFT, RIGHT):
        return _xerbla(api, name, 1)
    if uplo not in (UPPER, LOWER):
        return _xerbla(api, name, 2)
    if m < 0:
        return _xerbla(api, name, 3)
    if n < 0:
        return _xerbla(api, name, 4)
    q = m if side == LEFT else n
    if not _ld_ok(lda, q, q, order):
        return _xerbla(api, name, 7)
    if not _ld_ok(ldb, m, n, order):
        return _xerbla(api, name, 9)
    if not _ld_ok(ldc, m, n, order):
        return _xerbla(api, name, 12)
    if order == ROW:      # C^T = B^T sym(A)^T: the other side, the other triangle
        side, uplo, m, n = _flip_side(side), _flip_uplo(uplo), n, m
    if m == 0 or n == 0 or (alpha == 0.0 and beta == 1.0):
        return 0
    c = _view(pc, m, n, ldc, np.float64)
    if alpha == 0.0:
        w = _mat2d(c, m, n, ldc)
        if beta == 0.0:
            w[...] = 0.0
        else:
            w *= beta
        return 0
    a = _view(pa, q, q, lda, np.float64)
    b = _view(pb, m, n, ldb, np.float64)
    return _run(lambda: blas.dsymm("L" if side == LEFT else "R", "L" if uplo == LOWER else "U",
                                   m, n, alpha, a, lda, b, ldb, beta, c, ldc,
                                   tile_size=get_tile()))


# ----------------------------------------------------------------------------- TRMM / TRSM

def _tri(kind, api, order, side, uplo, ta, diag, m, n, alpha, pa, lda, pb, ldb):
    name = "DTRMM" if kind == "trmm" else "DTRSM"
    if api and order not in (ROW, COL):
        return _xerbla(api, name, 0)
    if side not in (LEFT, RIGHT):
        return _xerbla(api, name, 1)
    if uplo not in (UPPER, LOWER):
        return _xerbla(api, name, 2)
    if ta not in (NOTRANS, TRANS, CONJTRANS):
        return _xerbla(api, name, 3)
    if diag not in (NONUNIT, UNIT):
        return _xerbla(api, name, 4)
    if m < 0:
        return _xerbla(api, name, 5)
    if n < 0:
        return _xerbla(api, name, 6)
    q = m if side == LEFT else n
    if not _ld_ok(lda, q, q, order):
        return _xerbla(api, name, 9)
    if not _ld_ok(ldb, m, n, order):
        return _xerbla(api, name, 11)
    if order == ROW:
        side, uplo, m, n = _flip_side(side), _flip_uplo(uplo), n, m
    if m == 0 or n == 0:
        return 0
    b = _view(pb, m, n, ldb, np.float64)
    if alpha == 0.0:
        _mat2d(b, m, n, ldb)[...] = 0.0
        return 0
    a = _view(pa, q, q, lda, np.float64)
    fn = blas.dtrmm if kind == "trmm" else blas.dtrsm
    return _run(lambda: fn("L" if side == LEFT else "R", "L" if uplo == LOWER else "U",
                           _tchar(ta), "U" if diag == UNIT else "N", m, n, alpha, a, lda, b, ldb,
                           tile_size=get_tile()))


def trmm(api, order, side, uplo, ta, diag, m, n, alpha, pa, lda, pb, ldb):
    return _tri("trmm", api, order, side, uplo, ta, diag, m, n, alpha, pa, lda, pb, ldb)


def trsm(api, order, side, uplo, ta, diag, m, n, alpha, pa, lda, pb, ldb):
    return _tri("trsm", api, order, side, uplo, ta, diag, m, n, alpha, pa, lda, pb, ldb)
