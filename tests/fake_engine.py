"""Fake device engine for the GPU-less CPU suite (TEST DOUBLE, never shipped).

Same surface as ``paper_1510_05041_b200.engine.CudaEngine``.  Operations are queued per
(device, lane) with their wait events and executed by a randomised in-order-per-stream
simulator, so a missing event dependency in the runtime shows up as wrong numbers.
Numerics come from the oracle (tests may import it)."""

from __future__ import annotations

import functools
import random
import threading

import numpy as np

from oracle import tiled as O

LANES = (-1, -2, -3)


def _locked(fn):
    @functools.wraps(fn)
    def wrap(self, *a, **kw):
        with self._lock:
            return fn(self, *a, **kw)
    return wrap


class FakeEngine:
    """Thread-safe (the runtime's concurrent mode drives it from one thread per GPU)."""
    kind = "fake"

    def __init__(self, n_devices=1, seed=0, n_compute=4, arena_bytes=64 << 20):
        self.cuda_ids = list(range(n_devices))
        self.n_compute = n_compute
        self.rng = random.Random(seed)
        self.arenas = {}
        self.default_arena = arena_bytes
        self._arena_cap = [0] * n_devices
        self.queues = {}         # (slot, lane) -> list of ops
        self.ev_done = {}        # ev -> bool
        self._next_ev = 0
        self.n_launches = 0
        self.registered = 0
        self.flag = [False] * n_devices
        self.ops_log = []
        self.released = set()
        self._lock = threading.RLock()
        for name in ("ensure_arenas", "register_host", "unregister_host", "h2d", "d2h", "p2p",
                     "copy_batch", "ic_create", "ic_resolve", "ic_gemm", "ic_destroy", "gemm", "trsm", "trsm_inverse", "trsm_apply", "materialize", "singular", "record", "done", "wait_any",
                     "sync", "stream_wait", "device_sync"):
            setattr(self, name, _locked(getattr(type(self), name)).__get__(self))

    # ---- devices ----
    def slot(self, cuda_id):
        return self.cuda_ids.index(cuda_id)

    @property
    def ndev(self):
        return len(self.cuda_ids)

    def device_info(self, slot):
        return dict(name="fake", sms=148, total_bytes=1 << 34, free_bytes=self.default_arena)

    def free_bytes(self, slot):
        return self.default_arena + (2 << 30)

    def ensure_arenas(self, caps):
        for slot, c in caps.items():
            if c > self._arena_cap[slot]:
                self._arena_cap[slot] = c
                self.arenas[slot] = np.zeros((c + 7) // 8, dtype=np.float64)

    def arena_capacity(self, slot):
        return self._arena_cap[slot]

    def register_host(self, array):
        self.registered += 1
        return True

    def unregister_host(self, array):
        self.registered -= 1

    # ---- event / queue machinery ----
    def _new_ev(self):
        ev = self._next_ev
        self._next_ev += 1
        self.ev_done[ev] = False
        return ev

    def _enqueue(self, slot, lane, fn, waits, cond=None):
        """``cond``: extra readiness predicate (a flag another process raises)."""
        ev = self._new_ev()
        for w in waits:
            assert w in self.ev_done, f"wait on unknown event {w}"
            assert w not in self.released, f"wait on released event {w}"
        self.queues.setdefault((slot, lane), []).append((list(waits), fn, ev, cond))
        return ev

    def _step(self) -> bool:
        """Execute the head op of one random runnable stream."""
        ready = [k for k, q in self.queues.items()
                 if q and all(self.ev_done[w] for w in q[0][0]) and (q[0][3] is None or q[0][3]())]
        if not ready:
            return False
        k = self.rng.choice(sorted(ready))
        waits, fn, ev, _ = self.queues[k].pop(0)
        fn()
        self.ev_done[ev] = True
        return True

    def _remote_blocked(self) -> bool:
        return any(q and q[0][3] is not None for q in self.queues.values())

    def _run_until(self, pred, limit=10_000_000, timeout=120.0):
        import time as _t
        t0 = _t.perf_counter()
        for _ in range(limit):
            if pred():
                return
            if not self._step():
                if self._remote_blocked() and _t.perf_counter() - t0 < timeout:
                    _t.sleep(1e-4)          # another process will raise the flag
                    continue
                assert pred(), "fake GPU deadlock: pending ops wait on events that never fire"
                return

    # ---- memory views ----
    def _view(self, slot, off, ld, h, w):
        a = self.arenas[slot]
        assert off % 8 == 0
        base = off // 8
        assert base + ld * w <= a.size, "access outside arena"
        return a[base:base + ld * w].reshape(w, ld).T[:h, :]

    def _view32(self, slot, off, ld, h, w):
        a = self.arenas[slot].view(np.float32)
        assert off % 4 == 0
        base = off // 4
        assert base + ld * w <= a.size, "access outside arena"
        return a[base:base + ld * w].reshape(w, ld).T[:h, :]

    def _viewT(self, slot, off, ld, h, w, esz):
        return self._view32(slot, off, ld, h, w) if esz == 4 else self._view(slot, off, ld, h, w)

    # ---- transfers ----
    def h2d(self, slot, dst_off, dst_ld, desc, r0, c0, h, w, waits=()):
        def fn():
            self._viewT(slot, dst_off, dst_ld, h, w, desc.itemsize)[:, :] = desc.as_2d()[r0:r0 + h, c0:c0 + w]
        return self._enqueue(slot, -1, fn, waits)

    def d2h(self, slot, src_off, src_ld, desc, r0, c0, h, w, waits=()):
        def fn():
            desc.as_2d()[r0:r0 + h, c0:c0 + w] = self._viewT(slot, src_off, src_ld, h, w, desc.itemsize)
        return self._enqueue(slot, -2, fn, waits)

    def p2p(self, dst_slot, dst_off, src_slot, src_off, nbytes, waits=()):
        def fn():
            s = self.arenas[src_slot][src_off // 8:(src_off + nbytes) // 8]
            self.arenas[dst_slot][dst_off // 8:(dst_off + nbytes) // 8] = s
        return self._enqueue(dst_slot, -3, fn, waits)

    def copy_batch(self, slot, rows, waits=()):
        """bx_copy_batch: each row a 2-d H2D copy from a raw host address or a peer copy;
        one event per lane used, recorded after the batch."""
        import ctypes
        used = {}
        for i in range(len(rows) // 8):
            kind, dst_off, dst_ld, src, srcx, hb, w, wait = rows[8 * i:8 * i + 8]
            eb, kind = kind >> 8, kind & 0xFF
            wt = list(waits) + ([wait] if wait >= 0 else [])
            if kind == 0:
                h = hb
                dt = np.float64 if eb == 8 else np.float32
                nbytes = (srcx * (w - 1) + h) * eb

                def fn(src=src, srcx=srcx, h=h, w=w, dst_off=dst_off, dst_ld=dst_ld, eb=eb, dt=dt,
                       nbytes=nbytes):
                    raw = np.frombuffer((ctypes.c_char * nbytes).from_address(src), dtype=dt)
                    full = np.lib.stride_tricks.as_strided(raw, shape=(h, w),
                                                           strides=(eb, srcx * eb))
                    self._viewT(slot, dst_off, dst_ld, h, w, eb)[:, :] = full
                used[-1] = self._enqueue(slot, -1, fn, wt)
            else:
                def fn(src=src, srcx=srcx, hb=hb, dst_off=dst_off):
                    s = self.arenas[src][srcx // 8:(srcx + hb) // 8]
                    self.arenas[slot][dst_off // 8:(dst_off + hb) // 8] = s
                used[-3] = self._enqueue(slot, -3, fn, wt)
        eh = self.record(slot, -1) if -1 in used else -1
        ep = self.record(slot, -3) if -3 in used else -1
        return eh, ep

    # ---- resident issue engine (bx_ic_*) ----
    def ic_create(self, slots, groups, tiles, region_off, region_bytes, l2):
        return _FakeIcTable(slots, groups, tiles, region_off, region_bytes, l2)

    def ic_destroy(self, table):
        assert not table.destroyed, "ic table destroyed twice"
        table.destroyed = True

    def _ic_resolve(self, table, d, tids, waits):
        """bx_ic_resolve semantics: missing tiles are copied from the lowest-id holder of
        d's peer group (waiting on its arrival event) or from the host, one arrival event
        per copy lane for the batch; pending arrival events of present tiles are waited."""
        import ctypes
        assert not table.destroyed
        slot = table.slots[d]
        new = {-1: [], -3: []}
        seen = set()
        for t in tids:
            t = int(t)
            if t in seen:
                continue
            seen.add(t)
            if table.off[d, t] >= 0:
                e = int(table.ev[d, t])
                if e >= 0:
                    if self.ev_done[e]:
                        table.ev[d, t] = -1
                    elif e not in waits:
                        waits.append(e)
                continue
            host, hld, h, w, esz, ld = table.tiles[t]
            nbytes = ld * w * esz
            o = -(-table.cur[d] // 256) * 256
            if o + nbytes > table.end[d]:
                from paper_1510_05041_b200.errors import ArenaOutOfMemoryError
                raise ArenaOutOfMemoryError("ic: resident region exhausted")
            table.cur[d] = o + nbytes
            table.off[d, t] = o
            src = -1
            if table.l2:
                for e in range(table.ndev):
                    if e != d and (int(table.holders[t]) >> e) & 1 and table.groups[e] == table.groups[d]:
                        src = e
                        break
            payload = h * w * esz
            if src >= 0:
                so, sslot = int(table.off[src, t]), table.slots[src]
                se = int(table.ev[src, t])

                def fn(so=so, sslot=sslot, o=o, nbytes=nbytes):
                    self.arenas[slot][o // 8:(o + nbytes) // 8] = self.arenas[sslot][so // 8:(so + nbytes) // 8]
                self._enqueue(slot, -3, fn, [se] if se >= 0 else [])
                new[-3].append(t)
                table.metrics[d, 1] += payload
                table.metrics[d, 3] += 1
                table.metrics[src, 4] += payload
            else:
                dt = np.float64 if esz == 8 else np.float32
                hbytes = (hld * (w - 1) + h) * esz

                def fn(host=host, hld=hld, h=h, w=w, o=o, ld=ld, esz=esz, dt=dt, hbytes=hbytes):
                    raw = np.frombuffer((ctypes.c_char * hbytes).from_address(host), dtype=dt)
                    full = np.lib.stride_tricks.as_strided(raw, shape=(h, w), strides=(esz, hld * esz))
                    self._viewT(slot, o, ld, h, w, esz)[:, :] = full
                self._enqueue(slot, -1, fn, [])
                new[-1].append(t)
                table.metrics[d, 0] += payload
                table.metrics[d, 2] += 1
            table.holders[t] = int(table.holders[t]) | (1 << d)
        for lane, lst in new.items():
            if lst:
                e = self.record(slot, lane)
                for t in lst:
                    table.ev[d, t] = e
                waits.append(e)

    def ic_resolve(self, table, d, tids):
        waits = []
        self._ic_resolve(table, d, tids, waits)
        table.metrics[d, 5] += len(tids)
        return ([int(table.off[d, t]) for t in tids], [table.tiles[t][5] for t in tids], waits)

    def ic_gemm(self, table, d, stream, f32, ta, tb, tri, h, w, steps, raw, alpha, beta, c_off,
                ldc, waits=(), event=True):
        tids = [v for i in range(len(steps) // 4) for v in steps[4 * i:4 * i + 2] if v >= 0]
        wts = list(waits)
        self._ic_resolve(table, d, tids, wts)
        table.metrics[d, 5] += len(tids)
        rows = []
        for i in range(len(steps) // 4):
            a, b, dep, km = steps[4 * i:4 * i + 4]
            ops = []
            for v in (a, b):
                if v >= 0:
                    ops += [int(table.off[d, v]), table.tiles[v][5]]
                else:
                    ops += [raw[2 * (-v - 1)], raw[2 * (-v - 1) + 1]]
            rows.append((ops[0], ops[1], ops[2], ops[3], dep, km))
        return self.gemm(table.slots[d], stream, ta, tb, tri, h, w, rows, alpha, beta, c_off, ldc,
                         wts, f32=f32, event=event)

    # ---- kernels ----
    def gemm(self, slot, stream, ta, tb, tri, h, w, steps, alpha, beta, c_off, ldc, waits=(),
             f32=False, event=True):
        self.n_launches += 1
        view = self._view32 if f32 else self._view

        def fn():
            c = view(slot, c_off, ldc, h, w)
            acc = np.zeros((h, w))
            for (ao, lda, bo, ldb, d, km) in steps:
                a = view(slot, ao, lda, d if ta else h, h if ta else d)
                b = view(slot, bo, ldb, w if tb else d, d if tb else w)
                oa, ob = (a.T if ta else a), (b.T if tb else b)
                # a triangular-operand step: the half the kernel skips must be zero
                if km == 1:
                    assert not np.triu(oa, 1).any(), "KM_A_LOWER on a non-lower operand"
                elif km == 2:
                    assert not np.tril(oa, -1).any(), "KM_A_UPPER on a non-upper operand"
                elif km == 3:
                    assert not np.tril(ob, -1).any(), "KM_B_UPPER on a non-upper operand"
                elif km == 4:
                    assert not np.triu(ob, 1).any(), "KM_B_LOWER on a non-lower operand"
                acc += oa @ ob
            new = alpha * acc if beta == 0.0 else alpha * acc + beta * c
            if tri:
                m = np.tril(np.ones((h, w), bool)) if tri == 1 else np.triu(np.ones((h, w), bool))
                c[m] = new[m]
            else:
                c[:, :] = new
        ev = self._enqueue(slot, stream, fn, waits)
        return ev if event else -1

    def trsm(self, slot, stream, right, upper, trans, unit, h, w, alpha, a_off, lda, b_off, ldb,
             waits=()):
        self.n_launches += 1
        n = w if right else h

        def fn():
            a = self._view(slot, a_off, lda, n, n)
            b = self._view(slot, b_off, ldb, h, w)
            try:
                O.trsm_solve(b, a.copy(), alpha, "upper" if upper else "lower",
                             "unit" if unit else "non-unit", "right" if right else "left",
                             bool(trans))
            except O.OracleSingular:
                self.flag[slot] = True
        return self._enqueue(slot, stream, fn, waits)

    def trsm_inverse(self, slot, stream, upper, trans, unit, n, a_off, lda, inv_off, ldi, waits=()):
        self.n_launches += 1

        def fn():
            a = self._view(slot, a_off, lda, n, n).copy()
            z = np.eye(n)
            try:
                O.trsm_solve(z, a, 1.0, "upper" if upper else "lower",
                             "unit" if unit else "non-unit", "left", bool(trans))
            except O.OracleSingular:
                self.flag[slot] = True
                z[:] = np.nan
            self._view(slot, inv_off, ldi, n, n)[:, :] = z
        return self._enqueue(slot, stream, fn, waits)

    def trsm_apply(self, slot, stream, right, eff_upper, h, w, alpha, inv_off, ldi, b_off, ldb,
                   x_off, ldx, waits=()):
        self.n_launches += 1
        n = w if right else h
        assert x_off != b_off

        def fn():
            z = self._view(slot, inv_off, ldi, n, n)
            b = self._view(slot, b_off, ldb, h, w)
            self._view(slot, x_off, ldx, h, w)[:, :] = alpha * (b @ z if right else z @ b)
        return self._enqueue(slot, stream, fn, waits)

    def axpy(self, slot, stream, esz, h, w, beta, src_off, src_ld, dst_off, dst_ld, waits=()):
        self.n_launches += 1
        view = self._view32 if esz == 4 else self._view

        def fn():
            view(slot, dst_off, dst_ld, h, w)[:, :] += beta * view(slot, src_off, src_ld, h, w)
        return self._enqueue(slot, stream, fn, waits)

    def materialize(self, slot, stream, mode_sym, upper, trans, unit, n, a_off, lda, dst_off, ldd,
                    waits=(), event=True):
        self.n_launches += 1

        def fn():
            a = self._view(slot, a_off, lda, n, n).copy()
            uplo = "upper" if upper else "lower"
            if mode_sym:
                m = O.sym_of(a, uplo)
            else:
                m, _ = O.tri_of(a, uplo, "unit" if unit else "non-unit", bool(trans))
            self._view(slot, dst_off, ldd, n, n)[:, :] = m
        ev = self._enqueue(slot, stream, fn, waits)
        return ev if event else -1

    def singular(self, slot, reset=True):
        f = self.flag[slot]
        if reset:
            self.flag[slot] = False
        return f

    # ---- events ----
    def record(self, slot, lane, timing=False):
        return self._enqueue(slot, lane, lambda: None, ())

    def done(self, ev):
        assert ev not in self.released, f"query of released event {ev}"
        # make progress a random amount, then answer
        for _ in range(self.rng.randint(0, 3)):
            if not self._step():
                break
        return self.ev_done[ev]

    def wait_any(self, evs, spin_us=-1):
        if spin_us is not None and spin_us >= 0 and self._remote_blocked():
            self._step()
        else:
            self._run_until(lambda: any(self.ev_done[e] for e in evs))
        for i, e in enumerate(evs):
            if self.ev_done[e]:
                return i
        return -1

    def sync(self, ev):
        self._run_until(lambda: self.ev_done[ev])

    def elapsed_ms(self, e0, e1):
        return 1.0

    def release(self, ev):
        # the real pool recycles ids: a double release hands one event to two owners, and a
        # released id may already name someone else's event
        if ev is not None and ev >= 0:
            assert ev not in self.released, f"event {ev} released twice"
            self.released.add(ev)

    def release_many(self, evs):
        for ev in evs:
            self.release(ev)

    def stream_wait(self, slot, lane, ev):
        self._enqueue(slot, lane, lambda: None, (ev,))

    def device_sync(self, slot):
        self._run_until(lambda: all(not q for (s, _), q in self.queues.items() if s == slot))

    def launches(self):
        return self.n_launches


class _FakeIcTable:
    """engine.IcTable stand-in: the same numpy state arrays, kept in Python."""

    def __init__(self, slots, groups, tiles, region_off, region_bytes, l2):
        n = len(tiles) // 6
        self.ndev, self.ntiles = len(slots), n
        self.slots, self.groups, self.l2 = list(slots), list(groups), bool(l2)
        self.tiles = [tuple(int(v) for v in tiles[6 * t:6 * t + 6]) for t in range(n)]
        self.off = np.full((self.ndev, n), -1, dtype=np.int64)
        self.ev = np.full((self.ndev, n), -1, dtype=np.int64)
        self.holders = np.zeros(n, dtype=np.int64)
        self.metrics = np.zeros((self.ndev, 8), dtype=np.int64)
        self.cur = list(region_off)
        self.end = [o + b for o, b in zip(region_off, region_bytes)]
        self.destroyed = False
