"""The CUDA tile engine seen from the host runtime (a thin object over the C ABI).

One process-wide engine owns the per-GPU state created by ``bx_init`` (arena reservation,
4 compute streams + H2D / D2H / P2P copy streams, event pool).  The scheduler talks to it
through the methods below; tests substitute a fake with the same surface.  There is no
CPU implementation of any of these operations.
"""

from __future__ import annotations

import ctypes as C
from array import array
import threading

from . import _native as N

LANE_H2D, LANE_D2H, LANE_P2P = N.LANE_H2D, N.LANE_D2H, N.LANE_P2P


class CudaEngine:
    kind = "cuda"

    def __init__(self, cuda_ids, n_compute: int = 4, logical_ids=None):
        self.lib = N.load()
        N.require_gpu()
        self.cuda_ids = list(cuda_ids)
        # logical device ids (DeviceDesc.device_id) -> engine slot; normally the CUDA
        # ordinal itself, but several logical devices may share one GPU (multi-device
        # tests on a single B200: each slot has its own streams, events and arena)
        self.ids = list(logical_ids) if logical_ids is not None else list(cuda_ids)
        self.n_compute = n_compute
        self._arena = [0] * len(self.cuda_ids)
        self._lock = threading.Lock()
        N.check(self.lib.bx_init(len(self.cuda_ids), N.int_array(self.cuda_ids), None, n_compute),
                "bx_init")

    # ---- devices / memory -------------------------------------------------------------

    def slot(self, device_id: int) -> int:
        return self.ids.index(device_id)

    def extend(self, more, n_compute) -> None:
        """Add (logical id, cuda ordinal) pairs."""
        new = [(i, c) for i, c in more if i not in self.ids]
        ids = self.ids + [i for i, _ in new]
        cuda = self.cuda_ids + [c for _, c in new]
        n_compute = max(n_compute, self.n_compute)
        N.check(self.lib.bx_init(len(cuda), N.int_array(cuda), None, n_compute), "bx_init")
        self._arena += [0] * len(new)
        self.ids, self.cuda_ids, self.n_compute = ids, cuda, n_compute

    @property
    def ndev(self) -> int:
        return len(self.cuda_ids)

    def device_info(self, slot: int) -> dict:
        name = C.create_string_buffer(128)
        sms, tot, free = C.c_int(), C.c_uint64(), C.c_uint64()
        N.check(self.lib.bx_device_info(self.cuda_ids[slot], name, 128, C.byref(sms),
                                        C.byref(tot), C.byref(free)), "device_info")
        return dict(name=name.value.decode(), sms=sms.value, total_bytes=tot.value,
                    free_bytes=free.value)

    def free_bytes(self, slot: int) -> int:
        free, tot = C.c_uint64(), C.c_uint64()
        N.check(self.lib.bx_mem_info(slot, C.byref(free), C.byref(tot)), "mem info")
        return free.value

    def ensure_arenas(self, capacities: dict) -> None:
        """Grow-only per-device reservations (one cudaMalloc each); {slot: bytes}."""
        need = [max(int(capacities.get(i, 0)), cur) for i, cur in enumerate(self._arena)]
        if need == self._arena:
            return
        N.check(self.lib.bx_init(self.ndev, N.int_array(self.cuda_ids), N.u64_array(need),
                                 self.n_compute), "arena reservation")
        self._arena = need

    def arena_capacity(self, slot: int) -> int:
        return self._arena[slot]

    def register_host(self, array) -> bool:
        """Page-lock a host buffer; returns True if this call registered it (the caller
        then owns the matching ``unregister_host``)."""
        yes = C.c_int(0)
        self.lib.bx_host_is_registered(C.c_void_p(array.ctypes.data), C.byref(yes))
        if yes.value:
            return False
        N.check(self.lib.bx_host_register(C.c_void_p(array.ctypes.data), array.nbytes),
                "host register")
        return True

    def unregister_host(self, array) -> None:
        N.check(self.lib.bx_host_unregister(C.c_void_p(array.ctypes.data)), "host unregister")

    # ---- transfers ----------------------------------------------------------------------

    @staticmethod
    def _waits(waits):
        if not waits:
            return 0, None
        return len(waits), N.int_array(waits)

    def h2d(self, slot, dst_off, dst_ld, desc, r0, c0, h, w, waits=()) -> int:
        ev = C.c_int(-1)
        nw, wp = self._waits(waits)
        N.check(self.lib.bx_h2d_tile(slot, dst_off, dst_ld, C.c_void_p(desc.element_address(r0, c0)),
                                     desc.leading_dim, h, w, desc.itemsize, nw, wp, C.byref(ev)),
                "h2d tile")
        return ev.value

    def d2h(self, slot, src_off, src_ld, desc, r0, c0, h, w, waits=()) -> int:
        ev = C.c_int(-1)
        nw, wp = self._waits(waits)
        N.check(self.lib.bx_d2h_tile(slot, src_off, src_ld, C.c_void_p(desc.element_address(r0, c0)),
                                     desc.leading_dim, h, w, desc.itemsize, nw, wp, C.byref(ev)),
                "d2h tile")
        return ev.value

    def p2p(self, dst_slot, dst_off, src_slot, src_off, nbytes, waits=()) -> int:
        ev = C.c_int(-1)
        nw, wp = self._waits(waits)
        N.check(self.lib.bx_p2p_tile(dst_slot, dst_off, src_slot, src_off, nbytes, nw, wp,
                                     C.byref(ev)), "p2p tile")
        return ev.value

    def copy_batch(self, slot, rows, waits=()):
        """One launch group's tile fetches (``rows``: array('q'), 8 per copy, see
        include/blasx_cuda.h bx_copy_batch); returns (H2D lane event, P2P lane event),
        -1 for a lane the batch did not use."""
        eh, ep = C.c_int(-1), C.c_int(-1)
        nw, wp = self._waits(waits)
        N.check(self.lib.bx_copy_batch(slot, len(rows) // 8, rows.buffer_info()[0], nw, wp,
                                       C.byref(eh), C.byref(ep)), "copy batch")
        return eh.value, ep.value

    # ---- resident issue engine (one routine call) ------------------------------------------

    def ic_create(self, slots, groups, tiles, region_off, region_bytes, l2) -> "IcTable":
        """The call's tile table (``tiles``: array('q'), 6 per tile, see bx_ic_create)."""
        tid = C.c_int(-1)
        N.check(self.lib.bx_ic_create(len(slots), N.int_array(slots), N.int_array(groups),
                                      len(tiles) // 6, tiles.buffer_info()[0],
                                      N.u64_array(region_off), N.u64_array(region_bytes),
                                      int(l2), C.byref(tid)), "ic create")
        return IcTable(self, tid.value, len(slots), len(tiles) // 6)

    def ic_destroy(self, table) -> None:
        N.check(self.lib.bx_ic_destroy(table.id), "ic destroy")

    def ic_resolve(self, table, d, tids):
        """Offsets, device lds and pending arrival events of ``tids`` (array('i')) on GPU
        ``d`` of the table, fetching the missing ones."""
        n = len(tids)
        offs, lds = (C.c_int64 * max(1, n))(), (C.c_int32 * max(1, n))()
        cap = 2 * n + 2
        waits, nw = (C.c_int * cap)(), C.c_int(0)
        N.check(self.lib.bx_ic_resolve(table.id, d, n, tids.buffer_info()[0], offs, lds,
                                       C.byref(nw), waits, cap), "ic resolve")
        return list(offs[:n]), list(lds[:n]), list(waits[:nw.value])

    def ic_gemm(self, table, d, stream, f32, ta, tb, tri, h, w, steps, raw, alpha, beta, c_off,
                ldc, waits=(), event=True) -> int:
        """One task GEMM launch over tile ids (``steps``: array('i'), 4 per step; ``raw``:
        array('q') of (offset, ld) for negative ids, or None)."""
        ev = C.c_int(-1)
        nw, wp = self._waits(waits)
        N.check(self.lib.bx_ic_gemm(table.id, d, stream, int(f32), int(ta), int(tb), tri, h, w,
                                    len(steps) // 4, steps.buffer_info()[0],
                                    raw.buffer_info()[0] if raw else None,
                                    len(raw) // 2 if raw else 0, float(alpha), float(beta), c_off,
                                    ldc, nw, wp, C.byref(ev) if event else None),
                "ic gemm")
        return ev.value

    # ---- one process per GPU (spmd.py) ---------------------------------------------------

    def ipc_export(self, slot):
        """(64-byte IPC handle of the arena, arena bytes)."""
        h = C.create_string_buffer(64)
        n = C.c_uint64()
        N.check(self.lib.bx_ipc_arena_handle(slot, h, C.byref(n)), "ipc handle")
        return h.raw, n.value

    def ipc_open(self, slot, handle: bytes) -> int:
        base = C.c_uint64()
        N.check(self.lib.bx_ipc_open(slot, C.create_string_buffer(handle, 64), C.byref(base)),
                "ipc open")
        return base.value

    def ipc_close(self, slot, base) -> None:
        N.check(self.lib.bx_ipc_close(slot, base), "ipc close")

    def register_mapped(self, array) -> int:
        """Page-lock + map a host buffer (device-written flags); returns its device address."""
        d = C.c_uint64()
        N.check(self.lib.bx_host_register_mapped(C.c_void_p(array.ctypes.data), array.nbytes,
                                                 C.byref(d)), "register mapped")
        return d.value

    def copy_remote(self, slot, dst_off, src_ptr, nbytes, flag_dptr=0, flag_min=0, waits=()) -> int:
        ev = C.c_int(-1)
        nw, wp = self._waits(waits)
        N.check(self.lib.bx_copy_remote(slot, dst_off, src_ptr, nbytes, flag_dptr, flag_min, nw, wp,
                                        C.byref(ev)), "copy remote")
        return ev.value

    def write_flag(self, slot, lane, flag_dptr, value, waits=()) -> None:
        nw, wp = self._waits(waits)
        N.check(self.lib.bx_write_flag(slot, lane, flag_dptr, value, nw, wp), "write flag")

    # ---- kernels ------------------------------------------------------------------------

    def gemm(self, slot, stream, ta, tb, tri, h, w, steps, alpha, beta, c_off, ldc, waits=(),
             f32=False, event=True) -> int:
        """One task GEMM launch; ``f32`` selects the tcgen05 TF32 kernel (SGEMM).  ``steps``
        = [(a_off, lda, b_off, ldb, depth, kmode), ...], marshalled as one packed int64
        array (kmode: triangular operand, program.KM_*)."""
        n = len(steps)
        if f32 and tri:
            raise ValueError("the fp32 task GEMM has no triangle mode")
        flat = array("q", [v for st in steps for v in st])
        ev = C.c_int(-1)
        if waits:
            nw, wp = len(waits), (C.c_int * len(waits))(*waits)
        else:
            nw, wp = 0, None
        N.check(self.lib.bx_gemm_task_packed(slot, stream, int(f32), int(ta), int(tb), tri, h, w, n,
                                             flat.buffer_info()[0], float(alpha), float(beta), c_off,
                                             ldc, nw, wp, C.byref(ev) if event else None),
                "sgemm task" if f32 else "gemm task")
        return ev.value

    def trsm(self, slot, stream, right, upper, trans, unit, h, w, alpha, a_off, lda, b_off, ldb,
             waits=()) -> int:
        ev = C.c_int(-1)
        nw, wp = self._waits(waits)
        N.check(self.lib.bx_trsm_tile(slot, stream, int(right), int(upper), int(trans), int(unit),
                                      h, w, float(alpha), a_off, lda, b_off, ldb, nw, wp,
                                      C.byref(ev)), "trsm tile")
        return ev.value

    def trsm_inverse(self, slot, stream, upper, trans, unit, n, a_off, lda, inv_off, ldi,
                     waits=()) -> int:
        ev = C.c_int(-1)
        nw, wp = self._waits(waits)
        N.check(self.lib.bx_trsm_inverse(slot, stream, int(upper), int(trans), int(unit), n, a_off,
                                         lda, inv_off, ldi, nw, wp, C.byref(ev)), "trsm inverse")
        return ev.value

    def trsm_apply(self, slot, stream, right, eff_upper, h, w, alpha, inv_off, ldi, b_off, ldb,
                   x_off, ldx, waits=()) -> int:
        ev = C.c_int(-1)
        nw, wp = self._waits(waits)
        N.check(self.lib.bx_trsm_apply(slot, stream, int(right), int(eff_upper), h, w, float(alpha),
                                       inv_off, ldi, b_off, ldb, x_off, ldx, nw, wp, C.byref(ev)),
                "trsm apply")
        return ev.value

    def materialize(self, slot, stream, mode_sym, upper, trans, unit, n, a_off, lda, dst_off, ldd,
                    waits=(), event=True) -> int:
        ev = C.c_int(-1)
        nw, wp = self._waits(waits)
        N.check(self.lib.bx_materialize(slot, stream, int(mode_sym), int(upper), int(trans),
                                        int(unit), n, a_off, lda, dst_off, ldd, nw, wp,
                                        C.byref(ev) if event else None), "materialize")
        return ev.value

    def axpy(self, slot, stream, esz, h, w, beta, src_off, src_ld, dst_off, dst_ld,
             waits=()) -> int:
        ev = C.c_int(-1)
        nw, wp = self._waits(waits)
        N.check(self.lib.bx_axpy_tile(slot, stream, esz, h, w, float(beta), src_off, src_ld,
                                      dst_off, dst_ld, nw, wp, C.byref(ev)), "axpy tile")
        return ev.value

    def singular(self, slot, reset=True) -> bool:
        f = C.c_int(0)
        N.check(self.lib.bx_singular_flag(slot, int(reset), C.byref(f)))
        return bool(f.value)

    # ---- events -------------------------------------------------------------------------

    def record(self, slot, lane, timing=False) -> int:
        ev = C.c_int(-1)
        N.check(self.lib.bx_event_record(slot, lane, int(timing), C.byref(ev)), "event record")
        return ev.value

    def done(self, ev) -> bool:
        rc = self.lib.bx_event_query(ev)
        if rc < 0 or rc > 1:
            N.check(rc, "event query")
        return rc == 0

    def wait_any(self, evs, spin_us=-1) -> int:
        idx = C.c_int(-1)
        N.check(self.lib.bx_event_wait_any(len(evs), N.int_array(evs), C.byref(idx), spin_us),
                "wait_any")
        return idx.value

    def sync(self, ev) -> None:
        N.check(self.lib.bx_event_sync(ev), "event sync")

    def elapsed_ms(self, ev0, ev1) -> float:
        ms = C.c_float(0.0)
        N.check(self.lib.bx_event_elapsed(ev0, ev1, C.byref(ms)), "event elapsed")
        return ms.value

    def release(self, ev) -> None:
        if ev is not None and ev >= 0:
            N.check(self.lib.bx_event_release(ev), "event release")

    def release_many(self, evs) -> None:
        """Return several events to the pool in one call (a task's events at retirement)."""
        ids = [e for e in evs if e is not None and e >= 0]
        if ids:
            N.check(self.lib.bx_event_release_many(len(ids), N.int_array(ids)), "event release")

    def stream_wait(self, slot, lane, ev) -> None:
        N.check(self.lib.bx_stream_wait(slot, lane, ev), "stream wait")

    def device_sync(self, slot) -> None:
        N.check(self.lib.bx_device_sync(slot), "device sync")

    def launches(self) -> int:
        n = C.c_uint64(0)
        self.lib.bx_launch_count(C.byref(n))
        return n.value


class IcTable:
    """A call's resident tile table in the engine, with numpy views of its state arrays
    (offsets, pending arrival events, holder masks, per-GPU counters) for Eq. 3 and the
    metrics."""

    def __init__(self, eng, tid, ndev, ntiles):
        import numpy as np
        self.id, self.ndev, self.ntiles = tid, ndev, ntiles
        ptrs = [C.c_void_p() for _ in range(4)]
        N.check(eng.lib.bx_ic_state(tid, *[C.byref(p) for p in ptrs]), "ic state")
        n = max(1, ndev * ntiles)

        def view(p, ctype, count):
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(ctype)), shape=(count,))
        self.off = view(ptrs[0], C.c_int64, n)[:ndev * ntiles].reshape(ndev, ntiles)
        self.ev = view(ptrs[1], C.c_int32, n)[:ndev * ntiles].reshape(ndev, ntiles)
        self.holders = view(ptrs[2], C.c_uint32, max(1, ntiles))[:ntiles]
        self.metrics = view(ptrs[3], C.c_int64, ndev * 8).reshape(ndev, 8)


_ENGINE = None
_ELOCK = threading.Lock()


def get_engine(device_ids, n_compute=4, cuda_ordinals=None) -> CudaEngine:
    """The process-wide engine, extended to cover ``device_ids`` (logical ids; their CUDA
    ordinals default to the ids themselves).  Use ``engine.slot(device_id)``."""
    global _ENGINE
    device_ids = list(device_ids)
    cuda = list(cuda_ordinals) if cuda_ordinals is not None else list(device_ids)
    with _ELOCK:
        if _ENGINE is None:
            _ENGINE = CudaEngine(cuda, n_compute, logical_ids=device_ids)
            return _ENGINE
        for i, c in zip(device_ids, cuda):
            if i in _ENGINE.ids and _ENGINE.cuda_ids[_ENGINE.ids.index(i)] != c:
                raise ValueError(f"logical device {i} is already bound to another GPU")
        missing = [(i, c) for i, c in zip(device_ids, cuda) if i not in _ENGINE.ids]
        if missing or n_compute > _ENGINE.n_compute:
            _ENGINE.extend(missing, n_compute)
        return _ENGINE
