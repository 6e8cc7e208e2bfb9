"""ctypes binding of libblasx_cuda.so (include/blasx_cuda.h).

The product path has no CPU fallback: importing the engine on a machine where the
library or a GPU is missing raises ``NativeUnavailable`` instead of degrading."""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import (ArenaOutOfMemoryError, InvalidArgumentError, SingularMatrixError,
                     TileBlasError)

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libblasx_cuda.so")
_lock = threading.Lock()
_lib = None

BX_OK, BX_EINVAL, BX_ESINGULAR, BX_ENOMEM, BX_ECUDA = 0, 5, 6, 7, -1
LANE_H2D, LANE_D2H, LANE_P2P = -1, -2, -3


class NativeUnavailable(TileBlasError):
    """libblasx_cuda.so could not be loaded or no CUDA device is visible."""


class CudaError(TileBlasError):
    """A CUDA runtime call inside the engine failed."""


_i, _u64, _i64, _d, _p = C.c_int, C.c_uint64, C.c_int64, C.c_double, C.c_void_p
_pi, _pu64, _pf = C.POINTER(C.c_int), C.POINTER(C.c_uint64), C.POINTER(C.c_float)

_SIGS = {
    "bx_version": [],
    "bx_device_count": [_pi],
    "bx_device_info": [_i, C.c_char_p, _i, _pi, _pu64, _pu64],
    "bx_mem_info": [_i, _pu64, _pu64],
    "bx_init": [_i, _pi, _pu64, _i],
    "bx_shutdown": [],
    "bx_arena_base": [_i, _pu64],
    "bx_peer_enabled": [_i, _i, _pi],
    "bx_host_register": [_p, _u64],
    "bx_host_unregister": [_p],
    "bx_host_is_registered": [_p, _pi],
    "bx_h2d_tile": [_i, _u64, _i, _p, _i64, _i, _i, _i, _i, _pi, _pi],
    "bx_d2h_tile": [_i, _u64, _i, _p, _i64, _i, _i, _i, _i, _pi, _pi],
    "bx_p2p_tile": [_i, _u64, _i, _u64, _u64, _i, _pi, _pi],
    "bx_copy_batch": [_i, _i, _p, _i, _pi, _pi, _pi],
    "bx_ic_create": [_i, _pi, _pi, _i, _p, _pu64, _pu64, _i, _pi],
    "bx_ic_destroy": [_i],
    "bx_ic_state": [_i, _p, _p, _p, _p],
    "bx_ic_resolve": [_i, _i, _i, _p, _p, _p, _pi, _pi, _i],
    "bx_ic_gemm": [_i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _p, _p, _i, _d, _d, _u64, _i, _i, _pi,
                   _pi],
    "bx_gemm_task": [_i, _i, _i, _i, _i, _i, _i, _i, _pu64, _pi, _pu64, _pi, _pi, _d, _d,
                     _u64, _i, _i, _pi, _pi],
    "bx_sgemm_task": [_i, _i, _i, _i, _i, _i, _i, _pu64, _pi, _pu64, _pi, _pi, C.c_float, C.c_float,
                      _u64, _i, _i, _pi, _pi],
    "bx_gemm_task_packed": [_i, _i, _i, _i, _i, _i, _i, _i, _i, _p, _d, _d, _u64, _i, _i, _pi, _pi],
    "bx_sgemm_device": [_i, _i, _i, _i, _i, _i, _i, C.c_float, _u64, _i, _u64, _i, C.c_float, _u64, _i],
    "bx_trsm_tile": [_i, _i, _i, _i, _i, _i, _i, _i, _d, _u64, _i, _u64, _i, _i, _pi, _pi],
    "bx_trsm_inverse": [_i, _i, _i, _i, _i, _i, _u64, _i, _u64, _i, _i, _pi, _pi],
    "bx_trsm_apply": [_i, _i, _i, _i, _i, _i, _d, _u64, _i, _u64, _i, _u64, _i, _i, _pi, _pi],
    "bx_materialize": [_i, _i, _i, _i, _i, _i, _i, _u64, _i, _u64, _i, _i, _pi, _pi],
    "bx_axpy_tile": [_i, _i, _i, _i, _i, _d, _u64, _i, _u64, _i, _i, _pi, _pi],
    "bx_singular_flag": [_i, _i, _pi],
    "bx_event_record": [_i, _i, _i, _pi],
    "bx_event_query": [_i],
    "bx_event_sync": [_i],
    "bx_event_wait_any": [_i, _pi, _pi, _i],
    "bx_event_elapsed": [_i, _i, _pf],
    "bx_event_release": [_i],
    "bx_event_release_many": [_i, _pi],
    "bx_stream_wait": [_i, _i, _i],
    "bx_device_sync": [_i],
    "bx_launch_count": [_pu64],
    "bx_dev_alloc": [_i, _u64, _pu64],
    "bx_dev_free": [_i, _u64],
    "bx_dev_fill_uniform": [_i, _u64, _u64, _u64, _i],
    "bx_dev_fill_uniform_f32": [_i, _u64, _u64, _u64, _i],
    "bx_dev_copy_h2d": [_i, _u64, _p, _u64],
    "bx_dev_copy_d2h": [_i, _p, _u64, _u64],
    "bx_dgemm_device": [_i, _i, _i, _i, _i, _i, _i, _d, _u64, _i, _u64, _i, _d, _u64, _i],
    "bx_fp64_peak_probe": [_i, _i, C.POINTER(C.c_double)],
    "bx_set_gemm_variant": [_i],
    "bx_set_trsm_leaf": [_i],
    "bx_set_trsm_rhs": [_i],
    "bx_set_sgemm_debug": [_i],
    "bx_set_sgemm_mn3d": [_i],
    "bx_set_sgemm_precise": [_i],
    "bx_set_gemm_group": [_i],
    "bx_set_sgemm_variant": [_i],
    "bx_last_error": [C.c_char_p, _i],
    "bx_ipc_arena_handle": [_i, _p, _pu64],
    "bx_ipc_open": [_i, _p, _pu64],
    "bx_ipc_close": [_i, _u64],
    "bx_host_register_mapped": [_p, _u64, _pu64],
    "bx_copy_remote": [_i, _u64, _u64, _u64, _u64, C.c_uint32, _i, _pi, _pi],
    "bx_write_flag": [_i, _i, _u64, C.c_uint32, _i, _pi],
    "bx_atomic_add": [_p, C.c_int64, C.POINTER(C.c_int64)],
    "bx_atomic_cas": [_p, C.c_int64, C.c_int64, C.POINTER(C.c_int64)],
}


def exported_symbols():
    """Entry points include/blasx_cuda.h declares (checked by the CPU test-suite)."""
    return sorted(_SIGS)


def load(path: str = _LIB_PATH):
    """Load and type the library (no CUDA call is made)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: run `python -m paper_1510_05041_b200._build` "
                f"(or __graft_entry__.build()) first")
        try:
            lib = C.CDLL(path)
        except OSError as exc:
            raise NativeUnavailable(f"cannot load {path}: {exc}") from exc
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = C.c_int
        # kernel-variant knobs from the environment (tuning runs / variant test sweeps)
        for env, fn in (("BX_GEMM_VARIANT", "bx_set_gemm_variant"),
                        ("BX_SGEMM_VARIANT", "bx_set_sgemm_variant"),
                        ("BX_TRSM_LEAF", "bx_set_trsm_leaf"), ("BX_TRSM_RHS", "bx_set_trsm_rhs"),
                        ("BX_SGEMM_PRECISE", "bx_set_sgemm_precise"),
                        ("BX_GEMM_GROUP", "bx_set_gemm_group")):
            if os.environ.get(env):
                getattr(lib, fn)(int(os.environ[env]))
        _lib = lib
        return lib


def last_error() -> str:
    buf = C.create_string_buffer(512)
    load().bx_last_error(buf, 512)
    return buf.value.decode(errors="replace")


def check(rc: int, what: str = "") -> int:
    """Map a status code to the reference's exception taxonomy (errors.py:4-41)."""
    if rc == BX_OK:
        return rc
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == BX_EINVAL:
        raise InvalidArgumentError(msg)
    if rc == BX_ESINGULAR:
        raise SingularMatrixError(msg)
    if rc == BX_ENOMEM:
        raise ArenaOutOfMemoryError(msg)
    raise CudaError(msg)


def device_count() -> int:
    n = C.c_int(0)
    rc = load().bx_device_count(C.byref(n))
    if rc != BX_OK:
        return 0
    return n.value


def require_gpu() -> None:
    if device_count() < 1:
        raise NativeUnavailable("no CUDA device visible; this library has no CPU fallback")


def int_array(values):
    arr = (C.c_int * max(1, len(values)))(*values)
    return arr


def u64_array(values):
    return (C.c_uint64 * max(1, len(values)))(*values)
