"""cblas-style level-3 entry points over host-resident column-major operands.

A thin adapter over ``RoutineCall`` / ``run_call`` (the reference's API,
/root/reference/pkg/src/tileblas/routines.py:49-67, scheduler.py:665-669): it builds
zero-copy ``MatrixDesc`` views over the caller's buffers (leading dimension = lda) and
runs the tiled multi-GPU runtime; the output is written in place into the caller's
buffer.  Buffers are 1-d numpy arrays (column-major storage, BLAS style) or
Fortran-ordered 2-d arrays.  Flags accept BLAS characters ('N'/'T'/'C', 'U'/'L',
'L'/'R', 'N'/'U') or the reference's words.
"""

from __future__ import annotations

from typing import Optional

import numpy as np

from .errors import InvalidArgumentError
from .routines import RoutineCall
from .scheduler import RunOptions, RunResult, run_call
from .tiling import MatrixDesc, make_tiled

DEFAULT_TILE = 1024


def _trans(x) -> bool:
    if isinstance(x, bool):
        return x
    s = str(x).strip().lower()
    if s in ("n", "notrans", "no", "none"):
        return False
    if s in ("t", "c", "trans", "conjtrans", "transpose"):
        return True
    raise InvalidArgumentError(f"bad transpose flag {x!r}")


def _uplo(x) -> str:
    s = str(x).strip().lower()
    if s in ("u", "upper"):
        return "upper"
    if s in ("l", "lower"):
        return "lower"
    raise InvalidArgumentError(f"bad uplo {x!r}")


def _side(x) -> str:
    s = str(x).strip().lower()
    if s in ("l", "left"):
        return "left"
    if s in ("r", "right"):
        return "right"
    raise InvalidArgumentError(f"bad side {x!r}")


def _diag(x) -> str:
    s = str(x).strip().lower()
    if s in ("n", "non-unit", "nonunit"):
        return "non-unit"
    if s in ("u", "unit"):
        return "unit"
    raise InvalidArgumentError(f"bad diag {x!r}")


def _storage(buf, ld, dtype):
    arr = np.asarray(buf)
    if arr.dtype != dtype:
        raise InvalidArgumentError(f"expected a {np.dtype(dtype).name} buffer, got {arr.dtype}")
    if arr.ndim == 1:
        return arr, ld
    if arr.ndim == 2 and arr.flags.f_contiguous:
        ld_arr = arr.shape[0]
        if ld is not None and ld != ld_arr:
            raise InvalidArgumentError(f"leading dimension {ld} != rows of the 2-d array {ld_arr}")
        return arr.reshape(-1, order="F"), ld_arr
    raise InvalidArgumentError("operands must be 1-d column-major buffers or Fortran-ordered 2-d arrays")


def _tm(mid, buf, rows, cols, ld, tile, dtype):
    st, ld = _storage(buf, ld, dtype)
    if ld is None:
        ld = rows
    return make_tiled(MatrixDesc(mid, rows, cols, ld, st), tile)


def _run(call, tile_size, topology, options) -> RunResult:
    return run_call(call, topology, options)


def dgemm(transa, transb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, *,
          tile_size: int = DEFAULT_TILE, topology=None, options: Optional[RunOptions] = None,
          dtype=np.float64) -> RunResult:
    """C <- alpha op(A) op(B) + beta C   (C is m x n, op(A) m x k, op(B) k x n)."""
    ta, tb = _trans(transa), _trans(transb)
    a = _tm("A", A, k if ta else m, m if ta else k, lda, tile_size, dtype)
    b = _tm("B", B, n if tb else k, k if tb else n, ldb, tile_size, dtype)
    c = _tm("C", C, m, n, ldc, tile_size, dtype)
    return _run(RoutineCall("gemm", a=a, b=b, c=c, alpha=alpha, beta=beta, trans_a=ta,
                            trans_b=tb), tile_size, topology, options)


def sgemm(transa, transb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, **kw) -> RunResult:
    """Single precision GEMM (float32 host buffers; tcgen05 TF32 tile kernel)."""
    return dgemm(transa, transb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc,
                 dtype=np.float32, **kw)


def dsyrk(uplo, trans, n, k, alpha, A, lda, beta, C, ldc, *, tile_size: int = DEFAULT_TILE,
          topology=None, options=None) -> RunResult:
    """stored triangle of C <- alpha op(A) op(A)^T + beta C   (C n x n, op(A) n x k)."""
    t = _trans(trans)
    a = _tm("A", A, k if t else n, n if t else k, lda, tile_size, np.float64)
    c = _tm("C", C, n, n, ldc, tile_size, np.float64)
    return _run(RoutineCall("syrk", a=a, c=c, alpha=alpha, beta=beta, trans_a=t, uplo=_uplo(uplo)),
                tile_size, topology, options)


def dsyr2k(uplo, trans, n, k, alpha, A, lda, B, ldb, beta, C, ldc, *,
           tile_size: int = DEFAULT_TILE, topology=None, options=None) -> RunResult:
    """stored triangle of C <- alpha (op(A) op(B)^T + op(B) op(A)^T) + beta C."""
    t = _trans(trans)
    r, c_ = (k, n) if t else (n, k)
    a = _tm("A", A, r, c_, lda, tile_size, np.float64)
    b = _tm("B", B, r, c_, ldb, tile_size, np.float64)
    c = _tm("C", C, n, n, ldc, tile_size, np.float64)
    return _run(RoutineCall("syr2k", a=a, b=b, c=c, alpha=alpha, beta=beta, trans_a=t,
                            uplo=_uplo(uplo)), tile_size, topology, options)


def dsymm(side, uplo, m, n, alpha, A, lda, B, ldb, beta, C, ldc, *,
          tile_size: int = DEFAULT_TILE, topology=None, options=None) -> RunResult:
    """C <- alpha sym(A) B + beta C (left) or alpha B sym(A) + beta C (right)."""
    s = _side(side)
    q = m if s == "left" else n
    a = _tm("A", A, q, q, lda, tile_size, np.float64)
    b = _tm("B", B, m, n, ldb, tile_size, np.float64)
    c = _tm("C", C, m, n, ldc, tile_size, np.float64)
    return _run(RoutineCall("symm", a=a, b=b, c=c, alpha=alpha, beta=beta, side=s,
                            uplo=_uplo(uplo)), tile_size, topology, options)


def _tri(kind, side, uplo, transa, diag, m, n, alpha, A, lda, B, ldb, tile_size, topology,
         options):
    s = _side(side)
    q = m if s == "left" else n
    a = _tm("A", A, q, q, lda, tile_size, np.float64)
    b = _tm("C", B, m, n, ldb, tile_size, np.float64)
    return _run(RoutineCall(kind, a=a, c=b, alpha=alpha, side=s, uplo=_uplo(uplo),
                            trans_a=_trans(transa), diag=_diag(diag)), tile_size, topology, options)


def dtrmm(side, uplo, transa, diag, m, n, alpha, A, lda, B, ldb, *,
          tile_size: int = DEFAULT_TILE, topology=None, options=None) -> RunResult:
    """B <- alpha op(tri(A)) B (left) or alpha B op(tri(A)) (right), in place."""
    return _tri("trmm", side, uplo, transa, diag, m, n, alpha, A, lda, B, ldb, tile_size,
                topology, options)


def dtrsm(side, uplo, transa, diag, m, n, alpha, A, lda, B, ldb, *,
          tile_size: int = DEFAULT_TILE, topology=None, options=None) -> RunResult:
    """Solve op(tri(A)) X = alpha B (left) or X op(tri(A)) = alpha B (right); X over B."""
    return _tri("trsm", side, uplo, transa, diag, m, n, alpha, A, lda, B, ldb, tile_size,
                topology, options)


def pin_host(array) -> None:
    """Page-lock a host buffer for the lifetime of the process (or until ``unpin_host``):
    calls then skip per-call registration, as the paper times.
    The caller must not free a pinned buffer before unpinning it."""
    from .engine import get_engine
    from .devices import discover_topology
    topo = discover_topology()
    get_engine([d.device_id for d in topo.devices]).register_host(np.asarray(array))


def unpin_host(array) -> None:
    from .engine import get_engine
    from .devices import discover_topology
    topo = discover_topology()
    get_engine([d.device_id for d in topo.devices]).unregister_host(np.asarray(array))
