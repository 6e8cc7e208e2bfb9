"""One process per GPU: the runtime's host side split across ranks (SPMD execution).

The reference runs the whole scheduler in one process (one thread per device,
/root/reference/pkg/src/tileblas/scheduler.py:597-663).  With Python as the host language
that process becomes the 8-GPU bottleneck (~330 µs of issue work per task
when one interpreter feeds 8 GPUs).  Here every GPU gets its own process — launched by
``torchrun`` / any launcher that sets RANK, WORLD_SIZE, LOCAL_RANK, or by ``launch()`` —
and each rank runs the same planner and the same per-GPU worker (``scheduler._GpuWorker``)
on its own GPU, with the state the reference keeps in shared Python objects moved into
node-shared memory (``/dev/shm``) and updated with host atomics (``bx_atomic_*``):

* **TaskQueue** (scheduler.py:55-77): a shared FIFO of ready task ids (atomic head/tail),
  filled in Morton order; TRSM dependents are appended when their last producer completes
  (release after the producer's write-back, scheduler.py:488-505).
* **ReservationStation + stealing** (scheduler.py:106-153, 542-558): each rank's station is
  a row of shared slots.  The owner pops its highest Eq. 3 priority entry (ties: lowest id)
  with a CAS; a rank with an empty station and an empty queue steals the lowest-priority
  entry of the fullest station holding >= 2 entries, also with a CAS.
* **CoherenceDirectory** (cache.py:52-130): per tile, the *first holder* (claimed with a
  CAS) and every rank's arena offset.  The first holder fetches the tile from host memory
  (each tile crosses the host link once, as the reference's policy); every other rank
  copies it from the first holder's arena over NVLink (``copy_from_peer``, cache.py:312-322).
  Peer arenas are reached through CUDA IPC; the copy waits *on the GPU* for the holder's
  arrival flag (a 32-bit flag in node-shared pinned memory written by the holder's H2D
  stream, ``cuStreamWaitValue32`` / ``cuStreamWriteValue32``), so no host round trip
  sits between a holder's H2D and its peers' copies.
* Metrics, errors (an exception on any rank aborts every rank), and barriers live in the
  same shared block.

SPMD calls always use resident arenas (each rank's arena holds every tile it may touch; no
ALRU eviction across processes) and need the host operands in node-shared memory
(``Session.shared_array`` / ``share_call``) so every rank reads and writes the same bytes.
All ranks call ``run_call(call, options=RunOptions(execution="spmd"))`` with the same call.
"""

from __future__ import annotations

import ctypes as C
import json
import mmap
import os
import time
from typing import Optional

import numpy as np

from .devices import DeviceDesc, DeviceMetrics, Metrics, Topology
from .errors import (CapacityDeadlockError, ConfigError, InvalidArgumentError,
                     SingularMatrixError, TileBlasError)

SHM_DIR = "/dev/shm"
MAGIC = 0x42585350
RS_SLOTS = 16
MET_FIELDS = 16          # per-rank metric fields before the per-source d2d vector
BARRIER_TIMEOUT = float(os.environ.get("BX_SPMD_TIMEOUT", "900"))

_atomic_lib = None


def _alib():
    global _atomic_lib
    if _atomic_lib is None:
        from . import _native
        _atomic_lib = _native.load()
    return _atomic_lib


def atomic_add(arr: np.ndarray, i: int, v: int) -> int:
    old = C.c_int64()
    _alib().bx_atomic_add(C.c_void_p(arr.ctypes.data + 8 * i), v, C.byref(old))
    return old.value


def atomic_cas(arr: np.ndarray, i: int, expected: int, desired: int) -> int:
    old = C.c_int64()
    _alib().bx_atomic_cas(C.c_void_p(arr.ctypes.data + 8 * i), expected, desired, C.byref(old))
    return old.value


def _spin(pred, what, abort=None, timeout=BARRIER_TIMEOUT):
    """Wait for pred() with a short spin, then progressively longer sleeps."""
    t0 = time.perf_counter()
    n = 0
    while not pred():
        n += 1
        if abort is not None and abort():
            raise TileBlasError(f"spmd: another rank failed while waiting for {what}")
        if n > 200:
            time.sleep(min(1e-3, 1e-6 * (n - 200)))
            if time.perf_counter() - t0 > timeout:
                raise TileBlasError(f"spmd: timed out after {timeout:.0f}s waiting for {what}")


class ShmFile:
    """A named node-shared buffer (/dev/shm), mapped into this process."""

    def __init__(self, name: str, nbytes: int, create: bool, timeout: float = BARRIER_TIMEOUT):
        self.name = name
        self.path = os.path.join(SHM_DIR, name)
        nbytes = max(int(nbytes), 8)
        if create:
            tmp = self.path + f".tmp{os.getpid()}"
            fd = os.open(tmp, os.O_RDWR | os.O_CREAT | os.O_TRUNC, 0o600)
            os.ftruncate(fd, nbytes)
            os.rename(tmp, self.path)
        else:
            _spin(lambda: os.path.exists(self.path) and os.path.getsize(self.path) >= nbytes,
                  f"{self.path}", timeout=timeout)
            fd = os.open(self.path, os.O_RDWR)
        try:
            self.mm = mmap.mmap(fd, nbytes)
        finally:
            os.close(fd)
        self.buf = np.frombuffer(self.mm, dtype=np.uint8)
        self.nbytes = nbytes

    def view(self, offset: int, count: int, dtype) -> np.ndarray:
        dt = np.dtype(dtype)
        return self.buf[offset:offset + count * dt.itemsize].view(dt)

    def unlink(self) -> None:
        try:
            os.unlink(self.path)
        except FileNotFoundError:
            pass


class Session:
    """Rank membership, barriers and node-shared allocations of one SPMD job.

    Header (int64): 0 magic, 1 world, 2 call sequence, 3 barrier count, 4 barrier
    generation, 5 abort, 6 error code, 7 creation time (ns); then per rank: arena IPC handle
    (64 B) + arena bytes + arena generation, and a float64 scratch slot for reductions."""

    HDR = 16
    IPC_STRIDE = 80

    def __init__(self, rank: int, world: int, device: int, job: str):
        if not 0 <= rank < world:
            raise ConfigError(f"bad spmd rank {rank} of {world}")
        self.rank, self.world, self.device, self.job = rank, world, device, job
        self.t_start = time.time()
        nbytes = 8 * self.HDR + self.IPC_STRIDE * world + 8 * world
        name = f"bx_{job}_session"
        if rank == 0:
            f = ShmFile(name, nbytes, create=True)
            hdr = f.view(0, self.HDR, np.int64)
            hdr[1] = world
            hdr[7] = time.time_ns()
            hdr[0] = MAGIC
        else:
            def fresh():
                try:
                    if os.path.getsize(os.path.join(SHM_DIR, name)) < nbytes:
                        return False
                    g = ShmFile(name, nbytes, create=False)
                except (FileNotFoundError, ValueError):
                    return False
                h = g.view(0, self.HDR, np.int64)
                ok = h[0] == MAGIC and h[1] == world and h[7] >= (self.t_start - 600) * 1e9
                if ok:
                    self._f = g
                return ok
            _spin(fresh, f"rank 0 to create {name}")
            f = self._f
        self.f = f
        self.hdr = f.view(0, self.HDR, np.int64)
        self.ipc = f.view(8 * self.HDR, self.IPC_STRIDE * world, np.uint8).reshape(world, self.IPC_STRIDE)
        self.red = f.view(8 * self.HDR + self.IPC_STRIDE * world, world, np.float64)
        self._arrays = []            # (start, end) of this process's shared arrays
        self._shm = []
        self._peer = {}              # rank -> (arena gen, base)
        self._arena_gen = 0
        self._seq = 0                # calls made (every rank calls in the same order)
        self._nshare = 0             # share_call invocations
        self._blocks = [None, None]  # pooled call files, by call parity: (ShmFile, mapped dptr)
        self.barrier("session start")

    # ---- coordination ----------------------------------------------------------------

    def aborted(self) -> bool:
        return bool(self.hdr[5])

    def abort(self, code: int = -1) -> None:
        self.hdr[6] = code
        self.hdr[5] = 1

    def barrier(self, what: str = "barrier") -> None:
        """Every rank arrives (a failed rank still arrives: errors are reported after the
        barrier, so the count never goes out of step)."""
        hdr = self.hdr
        gen = int(hdr[4])
        if atomic_add(hdr, 3, 1) == self.world - 1:
            hdr[3] = 0
            atomic_add(hdr, 4, 1)
        else:
            _spin(lambda: int(hdr[4]) != gen, what)

    def allreduce_max(self, value: float) -> float:
        self.red[self.rank] = value
        self.barrier("allreduce")
        out = float(self.red.max())
        self.barrier("allreduce done")
        return out

    def allgather(self, value: float) -> np.ndarray:
        """Every rank's ``value`` (collective), as a float64 array indexed by rank."""
        self.red[self.rank] = value
        self.barrier("allgather")
        out = self.red.copy()
        self.barrier("allgather done")
        return out

    def next_call(self) -> int:
        """All ranks advance the call sequence together (collective: every rank makes the
        same calls in the same order)."""
        self._seq += 1
        return self._seq

    def call_file(self, eng, seq: int, nbytes: int):
        """The pooled node-shared file for call ``seq`` (calls alternate between two, so a
        file is reused only after every rank has started the following call, i.e. finished
        reading this one), at least ``nbytes`` long, page-locked and mapped for the GPU.
        Returns (ShmFile, device address of its first byte).  Collective."""
        par = seq & 1
        have = self._blocks[par]
        if have is not None and have[0].nbytes >= nbytes:
            return have
        if have is not None:              # too small: last used two calls ago
            try:
                eng.unregister_host(have[0].buf)
            except Exception:
                pass
            if self.rank == 0:
                have[0].unlink()
        size = max(nbytes, 2 * have[0].nbytes if have is not None else 0)
        f = ShmFile(f"bx_{self.job}_callblk{par}_{seq}", size, create=self.rank == 0)
        self._blocks[par] = (f, eng.register_mapped(f.buf))
        return self._blocks[par]

    # ---- node-shared host memory -----------------------------------------------------

    def shared_array(self, name: str, n: int, dtype=np.float64) -> np.ndarray:
        """A 1-d array in node-shared memory, the same bytes in every rank (rank 0 creates
        it; collective: every rank must call it in the same order)."""
        dt = np.dtype(dtype)
        f = ShmFile(f"bx_{self.job}_arr_{name}", n * dt.itemsize, create=self.rank == 0)
        self.barrier(f"shared array {name}")
        arr = f.view(0, n, dt)
        self._shm.append(f)
        self._arrays.append((arr.ctypes.data, arr.ctypes.data + arr.nbytes))
        return arr

    def is_shared(self, arr: np.ndarray) -> bool:
        p = arr.ctypes.data
        return any(a <= p < b for a, b in self._arrays)

    def share_call(self, call=None):
        """Rank 0 passes a RoutineCall over private host arrays; every rank gets back the
        same call over node-shared copies of them (collective)."""
        from .routines import RoutineCall
        from .tiling import MatrixDesc, make_tiled
        meta = None
        if self.rank == 0:
            if call is None:
                raise InvalidArgumentError("share_call: rank 0 must pass the call")
            ops = {k: getattr(call, k) for k in ("a", "b", "c") if getattr(call, k) is not None}
            meta = dict(kind=call.kind, alpha=call.alpha, beta=call.beta, trans_a=call.trans_a,
                        trans_b=call.trans_b, uplo=call.uplo, side=call.side, diag=call.diag,
                        ops={k: dict(id=t.matrix.matrix_id, rows=t.matrix.rows, cols=t.matrix.cols,
                                     ld=t.matrix.leading_dim, base=t.matrix.base_offset,
                                     n=int(t.matrix.storage.size), dtype=t.matrix.storage.dtype.str,
                                     tile=t.tile_size)
                             for k, t in ops.items()})
            f = ShmFile(f"bx_{self.job}_callmeta", 1 << 16, create=True)
            raw = json.dumps(meta).encode()
            f.view(8, len(raw), np.uint8)[:] = np.frombuffer(raw, np.uint8)
            f.view(0, 1, np.int64)[0] = len(raw)
        self.barrier("share_call meta")
        if self.rank != 0:
            f = ShmFile(f"bx_{self.job}_callmeta", 1 << 16, create=False)
            n = int(f.view(0, 1, np.int64)[0])
            meta = json.loads(bytes(f.view(8, n, np.uint8)).decode())
        self._nshare += 1
        tiled = {}
        for k, d in meta["ops"].items():
            arr = self.shared_array(f"share{self._nshare}_{k}_{d['id']}", d["n"], np.dtype(d["dtype"]))
            if self.rank == 0:
                arr[:] = getattr(call, k).matrix.storage
            tiled[k] = make_tiled(MatrixDesc(d["id"], d["rows"], d["cols"], d["ld"], arr, d["base"]),
                                  d["tile"])
        self.barrier("share_call data")
        return RoutineCall(kind=meta["kind"], a=tiled["a"], b=tiled.get("b"), c=tiled["c"],
                           alpha=meta["alpha"], beta=meta["beta"], trans_a=meta["trans_a"],
                           trans_b=meta["trans_b"], uplo=meta["uplo"], side=meta["side"],
                           diag=meta["diag"])

    # ---- arenas ------------------------------------------------------------------------

    def publish_arena(self, eng, slot) -> None:
        handle, nbytes = eng.ipc_export(slot)
        row = self.ipc[self.rank]
        old = bytes(row[:64])
        size = row[64:72].view(np.int64)
        gen = row[72:80].view(np.int64)
        if old != handle or int(size[0]) != nbytes:
            row[:64] = np.frombuffer(handle, np.uint8)
            size[0] = nbytes
            gen[0] = int(gen[0]) + 1

    def peer_bases(self, eng, slot) -> list:
        """Device addresses of every rank's arena in this process (own slot: 0)."""
        out = []
        for r in range(self.world):
            if r == self.rank:
                out.append(0)
                continue
            row = self.ipc[r]
            gen = int(row[72:80].view(np.int64)[0])
            have = self._peer.get(r)
            if have is None or have[0] != gen:
                if have is not None:
                    eng.ipc_close(slot, have[1])
                self._peer[r] = (gen, eng.ipc_open(slot, bytes(row[:64])))
            out.append(self._peer[r][1])
        return out

    def close(self) -> None:
        for f in self._shm + [b[0] for b in self._blocks if b is not None]:
            if self.rank == 0:
                f.unlink()
        if self.rank == 0:
            self.f.unlink()


_SESSION: Optional[Session] = None


def init(rank: Optional[int] = None, world: Optional[int] = None, device: Optional[int] = None,
         job: Optional[str] = None) -> Session:
    """Join (or create) this process's SPMD session; defaults come from the launcher's
    environment (RANK, WORLD_SIZE, LOCAL_RANK, TORCHELASTIC_RUN_ID / MASTER_PORT)."""
    global _SESSION
    if _SESSION is not None:
        return _SESSION
    env = os.environ
    rank = int(env.get("RANK", 0)) if rank is None else rank
    world = int(env.get("WORLD_SIZE", 1)) if world is None else world
    device = int(env.get("LOCAL_RANK", rank)) if device is None else device
    if job is None:
        job = env.get("BX_SPMD_JOB") or env.get("TORCHELASTIC_RUN_ID")
        if not job or job == "none":
            # torchrun without an rdzv id: the ranks of one launch share the agent process
            # (their parent), so a rerun on the same port never joins a stale session file
            job = f"p{env.get('MASTER_PORT', '0')}_{os.getppid()}"
    job = "".join(ch if ch.isalnum() else "_" for ch in str(job))
    _SESSION = Session(rank, world, device, job)
    return _SESSION


def current() -> Session:
    if _SESSION is None:
        return init()
    return _SESSION


def shutdown() -> None:
    global _SESSION
    if _SESSION is not None:
        _SESSION.close()
        _SESSION = None


# ============================================================================ per-call block

class _CallBlock:
    """Shared state of one call.  int64 regions: header (0 queue head, 1 queue tail,
    2 tasks done), queue, dependency counters, station slots + published priorities, first
    holder per tile, arena offset per (tile, rank); float64 metrics per rank; uint32 arrival
    flags per (tile, rank) (page-aligned: mapped for the GPU's stream memory operations).

    The views lie over a pooled node-shared file (``Session.call_file``): a session keeps
    two, used by alternate calls, page-locked and mapped for the GPU once, so a call pays
    neither the file creation nor the registration (≈ 3 ms per call per rank)."""

    @staticmethod
    def layout(W: int, n_tasks: int, n_tiles: int):
        sizes = [("hdr", 8), ("queue", n_tasks), ("deps", n_tasks), ("rs", W * RS_SLOTS),
                 ("rsprio", W * RS_SLOTS), ("owner", n_tiles), ("offs", n_tiles * W),
                 ("met", W * (MET_FIELDS + W))]
        off = 0
        lay = {}
        for name, n in sizes:
            lay[name] = (off, n)
            off += 8 * n
        flags_off = (off + 4095) // 4096 * 4096
        total = flags_off + max(4096, (4 * n_tiles * W + 4095) // 4096 * 4096)
        return lay, flags_off, total

    def __init__(self, sess: Session, file: "ShmFile", n_tasks: int, n_tiles: int):
        W = sess.world
        self.W = W
        lay, self.flags_off, self.total = self.layout(W, n_tasks, n_tiles)
        self.file = file
        for name, (o, n) in lay.items():
            setattr(self, name, self.file.view(o, n, np.float64 if name == "met" else np.int64))
        self.flags = self.file.view(self.flags_off, n_tiles * W, np.uint32)
        self.rs2 = self.rs.reshape(W, RS_SLOTS)
        self.rsprio2 = self.rsprio.reshape(W, RS_SLOTS)
        self.met2 = self.met.reshape(W, MET_FIELDS + W)

    def clear(self) -> None:
        """Zero this call's regions (rank 0, before the block is published)."""
        self.file.buf[:self.total] = 0

    # ---- shared FIFO ----
    def push(self, task_id: int) -> None:
        pos = atomic_add(self.hdr, 1, 1)
        self.queue[pos] = task_id + 1

    def pop(self):
        hdr = self.hdr
        while True:
            h = int(hdr[0])
            if h >= int(hdr[1]):
                return None
            if atomic_cas(hdr, 0, h, h + 1) == h:
                q = self.queue
                _spin(lambda: q[h] != 0, "queue slot publication")
                return int(q[h]) - 1

    def queued(self) -> int:
        return int(self.hdr[1]) - int(self.hdr[0])


def _first_use_inputs(plan, tbase):
    """The plan's input tiles (every matrix but the output) as [(key, ref)] in the order the
    tasks first read them (task order, then step order).  Memoised on the (cached,
    immutable) tasks: an owner-prefetch call only slices it (≈ 1-5 ms of Python per call at
    the BASELINE shapes otherwise)."""
    hit = getattr(plan.tasks[0], "_bx_first_use", None) if plan.tasks else None
    if hit is not None:
        return hit
    from . import scheduler as S
    out_id = plan.call.c.matrix.matrix_id
    seen, order = set(), []
    for task in plan.tasks:
        for key, (ref, _m) in S.task_keys(task).items():
            if key in seen or key[0] == out_id or key[0] not in tbase:
                continue
            seen.add(key)
            order.append((key, ref))
    if plan.tasks:
        plan.tasks[0]._bx_first_use = order
    return order


def _tile_index(plan):
    """(matrix_id, i, j) -> dense tile index over every matrix of the plan."""
    base = {}
    n = 0
    t = plan.tile_size
    for mid in sorted(plan.matrices):
        m = plan.matrices[mid]
        gr, gc = -(-m.rows // t), -(-m.cols // t)
        base[mid] = (n, gc)
        n += gr * gc
    return base, n


# ============================================================================ runtime pieces

def _build_runtime_classes():
    """Subclasses of the single-process runtime (defined lazily: scheduler imports us)."""
    from . import scheduler as S
    from .cache import LruBlock, CoherenceDirectory

    class SpmdQueue:
        def __init__(self, blk):
            self.blk = blk

        def get(self):
            t = self.blk.pop()
            return None if t is None else (t, 0.0)

        def put(self, item):
            self.blk.push(item[0])

        def __len__(self):
            return self.blk.queued()

    class SpmdRuntime(S._Runtime):
        def __init__(self, plan, topology, options, engine, sess, blk):
            self.plan = plan
            self.topology = topology
            self.options = options
            self.engine = engine
            self.sess = sess
            self.blk = blk
            self.queue = SpmdQueue(blk)
            self.directory = CoherenceDirectory()      # this rank's own holdings only
            self.total = len(plan.tasks)
            self._lock = S.threading.Lock()
            self.trace = []
            self.device_metrics = {d.device_id: DeviceMetrics() for d in topology.devices}
            self.workers = []
            self.error = None
            self.d2d_from = [0] * sess.world
            self.worker = None
            self._released = set()

        def done(self) -> bool:
            return int(self.blk.hdr[2]) >= self.total

        def complete_task(self, task, at_time: float = 0.0) -> None:
            if task.task_id not in self._released:
                self.worker.publish_output(task)
                self._release(task)
            atomic_add(self.blk.hdr, 2, 1)

        def release_dependents(self, task, at_time: float = 0.0) -> None:
            """Release-on-issue across ranks: the producer published its solved tile with
            a flag its compute stream sets after the solve (SpmdWorker._retain_on_issue)."""
            self._released.add(task.task_id)
            self._release(task)

        def _release(self, task) -> None:
            blk = self.blk
            for dep in task.dependents:
                if atomic_add(blk.deps, dep, -1) == 1:
                    blk.push(dep)

        def add_d2d_out(self, src_rank, nbytes) -> None:
            self.d2d_from[src_rank] += nbytes

    class SpmdWorker(S._GpuWorker):
        def __init__(self, desc, runtime, sess, blk, tindex, peer_bases, flags_dptr):
            super().__init__(desc, runtime)
            self.sess = sess
            self.rank = sess.rank
            self.W = sess.world
            self.blk = blk
            self.tbase = tindex
            self.peer_bases = peer_bases
            self.flags_dptr = flags_dptr
            self.resident = True
            runtime.worker = self

        # ---- tile indices ----
        def _kidx(self, key) -> int:
            b, gc = self.tbase[key[0]]
            return b + key[1] * gc + key[2]

        def _task_index(self, task):
            kx = getattr(task, "_bx_kidx", None)
            if kx is None:
                keys = S.task_keys(task)
                kx = np.array([self._kidx(k) for k in keys], dtype=np.int64)
                task._bx_kidx = kx
                task._bx_kmult = np.array([m for _, m in keys.values()], dtype=np.int64)
                task._bx_klist = list(keys)
            return kx

        # ---- Eq. 3 on the shared directory ----
        def _priority(self, task) -> int:
            w = self.runtime.options.critical_path_weight
            p = self._eq3(task)
            return p + w * S.critical_path(task, self.plan) if w else p

        def _eq3(self, task) -> int:
            kx = self._task_index(task)
            blocks = self.cache._blocks
            local = np.fromiter((k in blocks for k in task._bx_klist), dtype=bool, count=len(kx))
            if not self.runtime.options.l2_enabled:
                return int(2 * (task._bx_kmult * local).sum())
            held = self.blk.owner[kx] != 0
            return int((task._bx_kmult * np.where(local, 2, held.astype(np.int64))).sum())

        # ---- reservation station in shared slots ----
        def _next_entry(self):
            blk, r = self.blk, self.rank
            row, prow = blk.rs2[r], blk.rsprio2[r]
            cap = min(self.runtime.options.rs_capacity, RS_SLOTS)
            for s in range(cap):
                if row[s] == 0:
                    t = blk.pop()
                    if t is None:
                        break
                    prow[s] = 0
                    row[s] = t + 1
            while True:
                # each slot is read ONCE: a thief may empty it between two reads, and a
                # second read of 0 would turn into a CAS(0 -> 0) that "claims" task -1
                live = [(s, v - 1) for s, v in ((s, int(row[s])) for s in range(cap)) if v > 0]
                if not live:
                    return self._steal()
                best = None
                for s, t in live:
                    p = self._priority(self.plan.tasks[t])
                    prow[s] = p
                    if best is None or (-p, t) < (-best[2], best[1]):
                        best = (s, t, p)
                s, t, _ = best
                if atomic_cas(blk.rs, r * RS_SLOTS + s, t + 1, 0) == t + 1:
                    return S._SlotEntry(self.plan.tasks[t])
                # stolen meanwhile: re-read the station

        def _steal(self):
            blk = self.blk
            if blk.queued() > 0:
                return None
            cap = min(self.runtime.options.rs_capacity, RS_SLOTS)
            counts = [(int(np.count_nonzero(blk.rs2[v, :cap])), v) for v in range(self.W) if v != self.rank]
            for n, v in sorted(counts, key=lambda x: (-x[0], x[1])):
                if n < 2:
                    break
                row, prow = blk.rs2[v], blk.rsprio2[v]
                live = []
                for s in range(cap):
                    val = int(row[s])            # read once (see _next_entry)
                    if val > 0:
                        live.append((int(prow[s]), val - 1, s))
                if len(live) < 2:
                    continue
                p, t, s = min(live)
                if atomic_cas(blk.rs, v * RS_SLOTS + s, t + 1, 0) == t + 1:
                    return S._SlotEntry(self.plan.tasks[t])
            return None

        # ---- L2 over IPC: first holder fetches from host, the rest copy from it ----
        def _fetch_many(self, misses):
            # per tile: each copy publishes its own arrival flag for the other ranks
            for key, ref in misses:
                self._fetch_resident(key, ref)

        def _fetch_resident(self, key, ref):
            h, w = ref.phys_height, ref.phys_width
            ld = S.device_ld(h)
            nbytes = ld * w * self.esz
            try:
                off = self.arena.alloc(nbytes)
            except S.ArenaOutOfMemoryError:
                raise CapacityDeadlockError(
                    f"rank {self.rank}: resident arena exhausted; spmd execution needs the "
                    f"working set to fit in HBM") from None
            blk = LruBlock(key, off, nbytes, ld, self.device_id)
            blk.reader = 1
            payload = h * w * self.esz
            idx = self._kidx(key)
            W, r = self.W, self.rank
            cb = self.blk
            cb.offs[idx * W + r] = off + 1
            holder = 0
            if self.runtime.options.l2_enabled:
                holder = atomic_cas(cb.owner, idx, 0, r + 1)
            if holder == 0:
                desc, r0, c0 = self._host_of(ref)
                blk.ready_ev = self._timed(S.LANE_H2D, lambda wt: self.eng.h2d(
                    self.slot, off, ld, desc, r0, c0, h, w, wt), (), "H2D", payload)
                self.eng.write_flag(self.slot, S.LANE_H2D, self.flags_dptr + 4 * (idx * W + r), 1)
                self.dm.h2d_bytes += payload
                self.host_fetches += 1
            else:
                src = holder - 1
                offs = cb.offs
                _spin(lambda: offs[idx * W + src] != 0, "a holder's arena offset",
                      abort=self.sess.aborted)
                src_ptr = self.peer_bases[src] + int(offs[idx * W + src]) - 1
                flag = self.flags_dptr + 4 * (idx * W + src)
                blk.ready_ev = self._timed(S.LANE_P2P, lambda wt: self.eng.copy_remote(
                    self.slot, off, src_ptr, nbytes, flag, 1, wt), (), "D2D", payload)
                self.dm.d2d_in_bytes += payload
                self.runtime.add_d2d_out(src, payload)
                self.l2_hits += 1
            self._pending_keys.add(key)
            with self.cache.lock:
                self.cache._blocks[key] = blk
            self.runtime.directory.add_holder(key, self.device_id)
            self._permanent.append(blk)
            return blk

        def owner_plan(self) -> None:
            """Balanced host traffic (RunOptions.owner_prefetch): the call's input tiles, in
            the order the tasks first read them (Morton task order, then step order), are
            dealt round-robin to the ranks.  Each rank loads its share over its own host link
            (``owner_step``), claiming each tile in the first-holder directory and raising
            its arrival flag after the copy; the other ranks' tasks copy it from the owner
            over NVLink, waiting on the flag on the GPU.  Every tile still crosses a host link
            once, and the W links carry 1/W of the input bytes each whatever order the dynamic
            schedule takes — without it the first rank to need a tile fetches it, which can
            load one link with several times the mean (tools/spmd_balance.py: max/mean 2.4
            at 8 ranks on the fake engine).  A tile some task needs before its owner got to
            it is fetched by that task's rank as before (the owner then skips it)."""
            W, r = self.W, self.rank
            self._owned, self._owned_next, self._owned_inflight = [], 0, []
            if W < 2 or not self.runtime.options.l2_enabled:
                return
            self._owned = _first_use_inputs(self.plan, self.tbase)[r::W]
            tile_bytes = S.device_ld(self.plan.tile_size) * self.plan.tile_size * self.esz
            self._owned_window = max(4, (self.runtime.options.owner_prefetch_mb << 20) // tile_bytes)

        def owner_step(self) -> bool:
            """Issue owner loads while fewer than the window are in flight on this rank's
            host link (so a task's own C tile never queues behind the whole share)."""
            if not self._owned or self._owned_next >= len(self._owned):
                return False
            live = [e for e in self._owned_inflight if not self.eng.done(e)]
            self._owned_inflight = live
            issued = False
            W, r = self.W, self.rank
            cb = self.blk
            while len(self._owned_inflight) < self._owned_window and self._owned_next < len(self._owned):
                key, ref = self._owned[self._owned_next]
                self._owned_next += 1
                if self.cache.contains(key):
                    continue
                idx = self._kidx(key)
                if atomic_cas(cb.owner, idx, 0, r + 1) != 0:
                    continue                     # a task got there first
                h, w = ref.phys_height, ref.phys_width
                ld = S.device_ld(h)
                nbytes = ld * w * self.esz
                try:
                    off = self.arena.alloc(nbytes)
                except S.ArenaOutOfMemoryError:
                    raise CapacityDeadlockError(
                        f"rank {r}: resident arena exhausted; spmd execution needs the "
                        f"working set to fit in HBM") from None
                blk = LruBlock(key, off, nbytes, ld, self.device_id)
                blk.reader = 1
                payload = h * w * self.esz
                cb.offs[idx * W + r] = off + 1
                desc, r0, c0 = self._host_of(ref)
                blk.ready_ev = self._timed(S.LANE_H2D, lambda wt: self.eng.h2d(
                    self.slot, off, ld, desc, r0, c0, h, w, wt), (), "H2D", payload)
                self.eng.write_flag(self.slot, S.LANE_H2D, self.flags_dptr + 4 * (idx * W + r), 1)
                self.dm.h2d_bytes += payload
                self.host_fetches += 1
                self._pending_keys.add(key)
                with self.cache.lock:
                    self.cache._blocks[key] = blk
                self.runtime.directory.add_holder(key, self.device_id)
                self._permanent.append(blk)
                self._owned_inflight.append(blk.ready_ev)
                issued = True
            return issued

        def _retain_on_issue(self, act) -> None:
            """Release-on-issue (one process per GPU): cache the solved tile locally (base
            class), publish its arena offset, and have this task's compute stream set the
            tile's arrival flag after the solve — other ranks' IPC copies wait for that flag
            on their GPU (cuStreamWaitValue32), exactly as for a holder's H2D — then
            release the dependents through the shared counters."""
            task = act.entry.task
            key = task.out_ref.key()
            if (act.last_ev is None or act.last_ev < 0 or self.cache.contains(key)
                    or key[0] not in self.tbase):
                return
            idx = self._kidx(key)
            W, r = self.W, self.rank
            cb = self.blk
            if self.runtime.options.l2_enabled:
                if atomic_cas(cb.owner, idx, 0, r + 1) != 0:
                    return                     # cannot happen: outputs are written once
                cb.offs[idx * W + r] = act.c_off + 1
                self.eng.write_flag(self.slot, act.stream, self.flags_dptr + 4 * (idx * W + r), 1)
            super()._retain_on_issue(act)

        def publish_output(self, task) -> None:
            """A retained solved TRSM tile (written back, M -> E) becomes a holder copy
            its dependents on other ranks can copy over NVLink."""
            if not self._retain:
                return
            key = task.out_ref.key()
            blk = self.cache._blocks.get(key)
            if blk is None or key[0] not in self.tbase:
                return
            idx = self._kidx(key)
            W, r = self.W, self.rank
            cb = self.blk
            cb.offs[idx * W + r] = blk.offset + 1
            if atomic_cas(cb.owner, idx, 0, r + 1) == 0:
                cb.flags[idx * W + r] = 1          # the D2H (and the solve) completed

    return SpmdRuntime, SpmdWorker


_CLASSES = None


def _classes():
    global _CLASSES
    if _CLASSES is None:
        _CLASSES = _build_runtime_classes()
    return _CLASSES


# ============================================================================ run_plan_spmd

def run_plan_spmd(plan, options, engine=None, session: Optional[Session] = None,
                  _t_plan: float = 0.0):
    """Execute ``plan`` with every rank of the session (collective; see module doc)."""
    from . import scheduler as S
    from .engine import get_engine
    sess = session or current()
    SpmdRuntime, SpmdWorker = _classes()
    t_setup0 = time.perf_counter()
    r, W = sess.rank, sess.world
    options = S.resolve_streams(plan, options, W)
    options = S.resolve_ramp(plan, options, W)
    if options.rs_capacity > RS_SLOTS:
        raise ConfigError(f"spmd execution supports rs_capacity <= {RS_SLOTS}")
    if not options.l1_enabled:
        raise ConfigError("spmd execution needs the L1 tile cache (l1_enabled=True)")
    for m in plan.matrices.values():
        if not sess.is_shared(m.storage):
            raise InvalidArgumentError(
                f"matrix {m.matrix_id!r}: spmd execution needs node-shared host operands "
                f"(spmd.Session.shared_array / share_call)")
    if engine is None:
        engine = get_engine([r], options.n_streams, [sess.device])
    slot = engine.slot(r)
    esz = plan.dtype.itemsize
    full = S._auto_arena_bytes(plan, options, None)
    want = max(full, options.arena_bytes)
    if want > engine.arena_capacity(slot):
        avail = engine.free_bytes(slot) + engine.arena_capacity(slot)
        if S._auto_arena_bytes(plan, options, avail) < full:
            raise CapacityDeadlockError(
                f"rank {r}: the call's working set ({full} bytes) does not fit in HBM; spmd "
                f"execution keeps every tile resident")
        engine.ensure_arenas({slot: want})
    if plan.dtype.itemsize == 4 and hasattr(engine, "lib"):
        engine.lib.bx_set_sgemm_precise(int(S.sgemm_precise_for(plan, options)))
    sess.publish_arena(engine, slot)
    seq = sess.next_call()
    snap_shm = None
    if plan.snapshot_alias is not None and not options.l2_enabled:
        # TRMM snapshot aliasing the live storage is safe only if each snapshot tile is
        # fetched from the host once, by its first holder, before the owning task writes it
        # back (the others copy it over L2).  Without L2 every rank fetches on its own:
        # take the reference's copy (routines.py:393-400), in node-shared memory.
        from .tiling import MatrixDesc
        snap = plan.matrices[plan.snapshot_alias]
        arr = sess.shared_array(f"{seq}_snapshot", int(snap.storage.size), snap.storage.dtype)
        if r == 0:
            arr[:] = snap.storage
        sess.barrier("snapshot copied")
        snap_shm = sess._shm[-1]
        plan.matrices[plan.snapshot_alias] = MatrixDesc(
            snap.matrix_id, snap.rows, snap.cols, snap.leading_dim, arr, snap.base_offset)
        plan.snapshot_alias = None
    pinned_here = [m.storage for m in plan.matrices.values() if engine.register_host(m.storage)]

    tbase, n_tiles = _tile_index(plan)
    n_tasks = len(plan.tasks)
    _lay, flags_off, total = _CallBlock.layout(W, n_tasks, n_tiles)
    cfile, base_dptr = sess.call_file(engine, seq, total)
    blk = _CallBlock(sess, cfile, n_tasks, n_tiles)
    if r == 0:
        blk.clear()
        tail = 0
        for t in plan.tasks:
            blk.deps[t.task_id] = t.deps_remaining
            if t.deps_remaining == 0:
                blk.queue[tail] = t.task_id + 1
                tail += 1
        blk.hdr[1] = tail
    sess.barrier("call block created")
    flags_dptr = base_dptr + flags_off
    bases = sess.peer_bases(engine, slot)
    topo = Topology([DeviceDesc(q, peer_group="spmd") for q in range(W)])
    rt = SpmdRuntime(plan, topo, options, engine, sess, blk)
    w = SpmdWorker(topo.devices[r], rt, sess, blk, tbase, bases, flags_dptr)
    # release-on-issue needs other ranks to read a solved tile over L2 (never from the host
    # before its write-back)
    w._early_release = (w._retain and options.l1_enabled and options.release_on_issue
                        and (W == 1 or options.l2_enabled))
    w.runtime_trace = []
    rt.workers = [w]
    sess.barrier("call start")
    w.epoch = engine.record(slot, 0, timing=True)
    t0 = time.perf_counter()
    t_setup = t0 - t_setup0
    err = None
    try:
        if options.owner_prefetch:
            w.owner_plan()
        _drive(rt, w, sess)
    except BaseException as exc:   # abort every rank; reported after the end barrier
        err = exc
        if not isinstance(exc, _PeerFailed):
            sess.abort(6 if isinstance(exc, SingularMatrixError) else -1)
        try:
            engine.device_sync(slot)
        except Exception:
            pass
    wall = time.perf_counter() - t0
    t_fin0 = time.perf_counter()
    row = blk.met2[r]
    if err is None:
        end = engine.record(slot, S.LANE_D2H, timing=True)
        engine.sync(end)
        span = engine.elapsed_ms(w.epoch, end) / 1e3 if w.tasks_done else 0.0
        engine.release(end)
        engine.device_sync(slot)
        dm = w.dm
        row[:9] = [dm.h2d_bytes, dm.d2h_bytes, dm.d2d_in_bytes, w.l1_hits, w.l2_hits,
                   w.host_fetches, w.tasks_done, dm.kernel_launches, span]
        row[9] = wall
        row[MET_FIELDS:MET_FIELDS + W] = rt.d2d_from
    engine.release(w.epoch)
    sess.barrier("call end")
    failed, code = sess.aborted(), int(sess.hdr[6])
    w.release_all()
    for p in pinned_here:
        try:
            engine.unregister_host(p)
        except Exception:
            pass
    metrics = None
    if not failed:
        # the block is reused two calls later, after every rank has passed the next call's
        # "call block created" barrier, i.e. after this read
        metrics = _gather_metrics(plan, blk, W, wall)
    else:
        sess.barrier("call results read")
        if r == 0:
            sess.hdr[5] = 0
            sess.hdr[6] = 0
        sess.barrier("call closed")
    if snap_shm is not None:
        try:
            engine.unregister_host(arr)
        except Exception:
            pass
        sess._shm.remove(snap_shm)
        sess._arrays.pop()
        if r == 0:
            snap_shm.unlink()
    if failed:
        if err is not None and not isinstance(err, _PeerFailed):
            raise err
        if code == 6:
            raise SingularMatrixError("zero on a non-unit triangular diagonal (on another rank)")
        raise TileBlasError("spmd: another rank failed")
    metrics.phases = {"plan_s": _t_plan, "setup_s": t_setup, "drive_s": wall,
                      "finalize_s": time.perf_counter() - t_fin0}
    tasks_by_device = {q: metrics.devices[q].tasks for q in range(W)}
    return S.RunResult(metrics, [], tasks_by_device, plan)


class _PeerFailed(TileBlasError):
    pass


def _gather_metrics(plan, blk, W, wall) -> Metrics:
    metrics = Metrics(total_flops=plan.total_flops)
    devs = {}
    span = 0.0
    for q in range(W):
        row = blk.met2[q]
        dm = DeviceMetrics(h2d_bytes=int(row[0]), d2h_bytes=int(row[1]), d2d_in_bytes=int(row[2]),
                           tasks=int(row[6]), kernel_launches=int(row[7]))
        dm.d2d_out_bytes = int(sum(blk.met2[c][MET_FIELDS + q] for c in range(W)))
        dm.other_seconds = float(row[8])
        devs[q] = dm
        metrics.l1_hits += int(row[3])
        metrics.l2_hits += int(row[4])
        metrics.host_fetches += int(row[5])
        span = max(span, float(row[8]))
    metrics.devices = devs
    metrics.makespan_seconds = span if span > 0 else wall
    metrics.wall_seconds = float(blk.met2[:, 9].max())
    return metrics


def _drive(rt, w, sess) -> None:
    eng = rt.engine
    owned = getattr(w, "_owned", None)
    if owned:
        w.owner_step()                    # the first window goes out before any task
    while not rt.done():
        if sess.aborted():
            raise _PeerFailed("spmd: another rank failed")
        progressed = w.poll()
        progressed |= w.fill()
        if owned:
            progressed |= w.owner_step()
        if rt.done():
            break
        if not progressed:
            evs = w.in_flight()
            if owned and w._owned_inflight and w._owned_next < len(owned):
                evs = list(evs) + w._owned_inflight[:1]
            if evs:
                eng.wait_any(evs, spin_us=200)
            else:
                time.sleep(20e-6)
    # drain our own write-backs (tasks counted done by other ranks may still be in flight here)
    while not w.idle():
        if not w.poll():
            evs = w.in_flight()
            if evs:
                eng.wait_any(evs, spin_us=200)


# ============================================================================ launcher

def _child(rank, world, device, job, fn, args, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(device),
                      BX_SPMD_JOB=job)
    if os.environ.get("BX_SPMD_STACKS"):
        # debugging aid: `kill -USR1 <pid>` dumps every thread's Python stack to a file
        import faulthandler
        import signal
        faulthandler.register(signal.SIGUSR1, file=open(f"/tmp/bx_stack_{os.getpid()}.txt", "w"),
                              all_threads=True)
    try:
        out = fn(*args)
        q.put((rank, "ok", out))
    except BaseException as exc:  # reported to the parent
        import traceback
        q.put((rank, "err", f"{type(exc).__name__}: {exc}\n{traceback.format_exc()}"))


def launch(world: int, fn, *args, job: Optional[str] = None, timeout: float = 1800.0,
           devices=None):
    """Run ``fn(*args)`` in ``world`` fresh processes (one per rank, spawn), return the list
    of their results by rank.  ``fn`` must be importable (module-level).  ``devices``: the
    CUDA ordinal of each rank (default: rank r drives GPU r; several ranks may share a GPU,
    which is how the multi-process path is exercised on a one-GPU box)."""
    import multiprocessing as mp
    job = job or f"l{os.getpid()}_{int(time.time() * 1e3) % 10**9}"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    devices = list(devices) if devices is not None else list(range(world))
    procs = [ctx.Process(target=_child, args=(r, world, devices[r], job, fn, args, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [None] * world
    errs = []
    try:
        import queue as _queue
        deadline = time.monotonic() + timeout
        pending = set(range(world))
        while pending:
            try:
                rank, status, val = q.get(timeout=1.0)
            except _queue.Empty:
                # a rank that died without reporting (import error, signal) would otherwise
                # leave the parent waiting for the full timeout
                dead = [r for r in pending if procs[r].exitcode is not None]
                if dead:
                    time.sleep(0.5)
                    while True:
                        try:
                            rank, status, val = q.get_nowait()
                        except _queue.Empty:
                            break
                        pending.discard(rank)
                        (errs.append((rank, val)) if status != "ok"
                         else out.__setitem__(rank, val))
                    for r in [r for r in pending if procs[r].exitcode is not None]:
                        errs.append((r, f"exited with code {procs[r].exitcode} without a result"))
                        pending.discard(r)
                    if errs:
                        break
                if time.monotonic() > deadline:
                    errs.extend((r, f"no result after {timeout:.0f} s") for r in sorted(pending))
                    break
                continue
            pending.discard(rank)
            if status == "ok":
                out[rank] = val
            else:
                errs.append((rank, val))
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
        for f in os.listdir(SHM_DIR):
            if f.startswith(f"bx_{job}_"):
                try:
                    os.unlink(os.path.join(SHM_DIR, f))
                except OSError:
                    pass
    if errs:
        raise RuntimeError("spmd rank failure(s):\n" + "\n".join(f"[rank {r}] {e}" for r, e in errs))
    return out
