"""BLASX runtime on real GPUs: demand-driven work sharing, per-GPU reservation stations
with locality priorities and work stealing, whole-task issue onto 4 CUDA streams per GPU,
a two-level tile cache, and event-driven completion.

Scheduling policy = the reference's (/root/reference/pkg/src/tileblas/scheduler.py):
  * ready tasks sit in one global FIFO (TaskQueue, scheduler.py:55-77);
  * each GPU keeps a reservation station of up to ``rs_capacity`` pending tasks, refilled
    from the FIFO; only a GPU whose queue pull and station both come up empty steals,
    taking the lowest-priority task of the station with the most pending tasks, and only
    from stations holding >= 2 (scheduler.py:297-318, 542-558, 140-149);
  * a task's priority counts +2 per input tile already in this GPU's L1 and +1 per tile
    held by a peer (Eq. 3, scheduler.py:341-354); the best pending task (ties -> lowest id)
    runs next;
  * up to 4 tasks run concurrently per GPU, one per compute stream (devices.py:36).

What is different on hardware (SURVEY.md §7 "hard parts" 3-4):
  * a task is issued *whole*: its tile translations (L1 hit / P2P copy from a peer / H2D
    copy from pinned host memory) and its kernels are enqueued in one pass, the kernels
    waiting on the copies' CUDA events; consecutive k-steps are fused into one kernel
    launch (``chunk_steps``) so C stays in registers across them;
  * C is written back with a D2H copy ordered after the last kernel; the task completes
    when that copy's event fires — only then are its reader pins released, its buffers
    freed and TRSM dependents enqueued (readiness tied to write-back);
  * pressure sync (every cached tile pinned) = flush + drain this GPU + release the pins of
    all launched work, then retry once (cache.py:232-250; scheduler.py:272-281).
"""

from __future__ import annotations

import os
import threading
import time
from array import array
from collections import deque
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .cache import HOST_FETCH, L2_HIT, CoherenceDirectory, DeviceTileCache, LruBlock
from .devices import (DeviceMetrics, Metrics, Topology, TraceEvent, discover_topology,
                      exposed_comm_time)
from .errors import (ArenaOutOfMemoryError, CapacityDeadlockError, ConfigError,
                     SingularMatrixError)
from .memory import Arena
from .routines import RoutineCall, Task, TaskPlan, generate_tasks
from .program import AxpyOp, GemmOp, MatOp, TrsmOp, compile_task, scratch_key
from .tiling import device_ld

WORKING_SET_TILES = 12   # reference floor (scheduler.py:49-52): 4 tasks x (C + 2 inputs)
SGEMM_TF32_MIN_K = 512   # auto SGEMM: plain TF32 from this reduction depth up
LANE_H2D, LANE_D2H, LANE_P2P = -1, -2, -3


class TaskQueue:
    """Global FIFO of ready task ids (append / popleft are atomic)."""

    def __init__(self):
        self._items = deque()

    def put(self, item) -> None:
        self._items.append(item)

    def get(self):
        try:
            return self._items.popleft()
        except IndexError:
            return None

    def __len__(self) -> int:
        return len(self._items)


@dataclass
class RunOptions:
    execution: str = "deterministic"   # one driver thread; "concurrent": one per GPU;
                                       # "spmd": one process per GPU (spmd.py)
    rs_capacity: int = 8
    l1_enabled: bool = True
    l2_enabled: bool = True
    record_trace: bool = False
    n_streams: int = 0                 # compute streams per GPU; 0 = auto (resolve_streams)
    chunk_steps: int = 0               # k-steps fused per kernel launch; 0 = auto
                                       # (resolve_streams: GEMM/SYMM/SYR2K 8, others 16)
    tasks_per_stream: int = 2          # tasks kept issued per compute stream (lookahead)
    first_chunk_steps: int = 0         # shorter first launch per task; 0 = off
    ramp_tasks: int = -1               # start-up batch: the first N tasks a GPU starts run
    ramp_chunk_steps: int = 4          # in extra slots with ramp_chunk_steps-long launches,
                                       # advancing k-major together while their panels
                                       # stream in (-1 = auto, 0 = off; resident mode only)
    defer_c_move_in: bool = True       # beta*C0 added by a final axpy launch, so a task's
                                       # GEMMs do not wait for its C tile (program.py)
    sgemm_precise: Optional[bool] = None   # float32 calls: True = 3xTF32 (fp32 accuracy,
                                       # 1/3 rate), False = TF32 inputs, None = auto (3xTF32
                                       # below SGEMM_TF32_MIN_K, sgemm_precise_for)
    critical_path_weight: int = 0      # TRSM: + weight x (longest chain of dependents) on
                                       # top of Eq. 3; 0 = the reference's Eq. 3
    retain_outputs: bool = True        # TRSM: keep written-back solved tiles cached (M->E)
    release_on_issue: bool = False     # TRSM (one process, resident arenas): a solved tile
                                       # is cached and its dependents released once its
                                       # solve is *enqueued*; their launches wait on the
                                       # solve's event on the GPU instead of the producer's
                                       # write-back + a host poll (the write-back still
                                       # completes the task).  Off: the reference's
                                       # release-after-write-back measured
                                       # as fast or faster (cfg4 134.7 vs 135.6 ms,
                                       # profiles/trsm_ab_r02.txt)
    trsm_split_chain: bool = False     # TRSM: the update step reading the chain
                                       # predecessor's solved tile gets its own launch, so
                                       # the task's other updates need not wait for that
                                       # solve (program.compile_task).  Measured slower on
                                       # cfg4: 139.1 vs 135.5 ms (profiles/trsm_ab_r02.txt)
    split_km: bool = False             # TRMM: the diagonal (triangular-operand) step gets
                                       # its own launch, so the plain steps skip the k-range
                                       # bookkeeping of the KM kernel instantiation.
                                       # Measured slower on cfg4 TRMM: 139.2 vs 136.7 ms
                                       # (profiles/trmm_syrk_ab_r02.txt)
    trsm_inverse_min: int = 128        # TRSM diagonal steps on tiles of at least this order
                                       # (resident arenas): X = alpha inv(E) B with inv(E)
                                       # computed once per diagonal tile; 0 = substitution
    prefetch_window_mb: int = 0        # large one-GPU calls: keep this much of first-use
                                       # tile loads in flight ahead of the tasks (0 = off)
    rampdown_tasks: int = 0            # wind-down batch: when at most this many tasks are
                                       # left to start, start them all at once with
                                       # ramp_chunk_steps-long launches (one GPU, resident
                                       # arenas, no TRSM DAG); 0 = off
    prefetch: int = -1                 # 1: load every input tile at the call's start in
                                       # first-use order (one GPU, resident issue engine);
                                       # -1 = auto (scheduler.small_call), 0 off
    owner_prefetch: bool = True        # one process per GPU (W >= 2, L2 on): deal the
                                       # input tiles round-robin in first-use order to the
                                       # ranks, each loads its share over its own host link,
                                       # at most owner_prefetch_mb ahead (spmd.py)
    owner_prefetch_mb: int = 64        # the per-rank window of owner loads in flight, so a
                                       # task's own C tile never queues behind all of them
    arena_bytes: int = 0               # per GPU; 0 = sized for the call


@dataclass
class RunResult:
    metrics: Metrics
    trace: list
    tasks_by_device: dict
    plan: TaskPlan


class _SlotEntry:
    __slots__ = ("task", "release_time", "priority", "pver")

    def __init__(self, task: Task, release_time: float = 0.0):
        self.task = task
        self.release_time = release_time
        self.priority = 0
        self.pver = -1          # directory version the priority was computed at


class ReservationStation:
    """Per-GPU buffer of upcoming tasks, open to theft (scheduler.py:106-153)."""

    def __init__(self, device_id: int, capacity: int):
        self.device_id = device_id
        self.capacity = capacity
        self.lock = threading.Lock()
        self._pending = []

    def pending_count(self) -> int:
        with self.lock:
            return len(self._pending)

    def room(self, in_flight: int = 0) -> int:
        with self.lock:
            return self.capacity - in_flight - len(self._pending)

    def put(self, entry) -> None:
        with self.lock:
            self._pending.append(entry)

    def pop_best(self):
        with self.lock:
            if not self._pending:
                return None
            best = min(self._pending, key=lambda e: (-e.priority, e.task.task_id))
            self._pending.remove(best)
            return best

    def steal_lowest(self):
        with self.lock:
            if len(self._pending) < 2:
                return None
            worst = min(self._pending, key=lambda e: (e.priority, e.task.task_id))
            self._pending.remove(worst)
            return worst

    def entries(self) -> list:
        with self.lock:
            return list(self._pending)


def steal_for(thief):
    """Victim = most pending (ties: lowest device id); it gives up its lowest-priority
    task; never robs a station with < 2 pending; only when the global queue is empty."""
    if len(thief.runtime.queue) > 0:
        return None
    victims = sorted((w for w in thief.runtime.workers if w.device_id != thief.device_id),
                     key=lambda w: (-w.rs.pending_count(), w.device_id))
    for v in victims:
        e = v.rs.steal_lowest()
        if e is not None:
            return e
    return None


class _Runtime:
    def __init__(self, plan: TaskPlan, topology: Topology, options: RunOptions, engine):
        self.plan = plan
        self.topology = topology
        self.options = options
        self.engine = engine
        self.queue = TaskQueue()
        self.directory = CoherenceDirectory()
        self.total = len(plan.tasks)
        self._done = 0
        self._deps = {t.task_id: t.deps_remaining for t in plan.tasks}
        self._released = set()   # tasks whose dependents were released at issue
        self._lock = threading.Lock()
        self.trace = []
        self.device_metrics = {d.device_id: DeviceMetrics() for d in topology.devices}
        self.workers = []
        self.error = None
        for t in plan.tasks:
            if t.deps_remaining == 0:
                self.queue.put((t.task_id, 0.0))

    def done(self) -> bool:
        with self._lock:
            return self._done >= self.total

    def complete_task(self, task: Task, at_time: float = 0.0) -> None:
        with self._lock:
            self._done += 1
            if task.task_id in self._released:
                return
            for dep in task.dependents:
                self._deps[dep] -= 1
                if self._deps[dep] == 0:
                    self.queue.put((dep, at_time))

    def release_dependents(self, task: Task, at_time: float = 0.0) -> None:
        """Release-on-issue (RunOptions.release_on_issue): the task's output is cached on
        its device with the solve's event as arrival event, so dependents may be issued
        now; ``complete_task`` then only counts the task."""
        with self._lock:
            self._released.add(task.task_id)
            for dep in task.dependents:
                self._deps[dep] -= 1
                if self._deps[dep] == 0:
                    self.queue.put((dep, at_time))

    def add_d2d_out(self, device_id, nbytes) -> None:
        with self._lock:
            self.device_metrics[device_id].d2d_out_bytes += nbytes

    def record(self, ev: TraceEvent) -> None:
        with self._lock:
            self.trace.append(ev)


class _Active:
    """A task in flight on one compute stream."""
    __slots__ = ("entry", "stream", "c_off", "c_ld", "scratch", "pins", "launched_pins",
                 "events", "last_ev", "done_ev", "pending_waits", "flops", "prog", "res",
                 "next_op", "lazy", "misses", "misses_epoch", "c_pending", "c0_off", "ramp",
                 "slot_index", "retained")

    def __init__(self, entry, stream, slot_index=-1):
        self.entry = entry
        self.stream = stream
        self.slot_index = slot_index
        self.c_off = -1
        self.c_ld = 0
        self.scratch = []        # arena offsets freed at retirement
        self.pins = []           # (cache, block) pinned for the not-yet-launched chunk
        self.launched_pins = []  # pins of launched chunks (releasable after a drain)
        self.events = []         # event ids owned by the task
        self.last_ev = None      # event after the last kernel
        self.done_ev = None      # write-back completion
        self.pending_waits = []  # waits to attach to the next launch (C move-in)
        self.flops = 0
        self.c_pending = False   # C move-in not yet enqueued
        self.c0_off = -1         # deferred C move-in buffer (program.defer_c)
        self.ramp = False        # part of the start-up batch (extra slot, short launches)
        self.retained = None     # output block cached at issue (release_on_issue)


class _GpuWorker:
    """One GPU: reservation station, L1 cache over its arena, 4 stream slots; also the
    ``fetch`` object of its cache's translate protocol."""

    def __init__(self, desc, runtime: _Runtime):
        self.desc = desc
        self.device_id = desc.device_id
        self.runtime = runtime
        self.eng = runtime.engine
        self.slot = self.eng.slot(desc.device_id)
        opts = runtime.options
        self.arena = Arena(self.eng.arena_capacity(self.slot))
        self.cache = DeviceTileCache(desc.device_id, self.arena, runtime.directory,
                                     peer_group=runtime.topology.peer_group_of(desc),
                                     l2_enabled=opts.l2_enabled, on_evict=self._on_evict)
        self.rs = ReservationStation(desc.device_id, opts.rs_capacity)
        self.dm = runtime.device_metrics[desc.device_id]
        # active slots: tasks_per_stream tasks may be queued on each compute stream, so the
        # next task's copies and kernels are already enqueued when the current one drains
        self.n_streams = opts.n_streams
        self.base_slots = opts.n_streams * opts.tasks_per_stream
        self.active = [None] * (self.base_slots + max(0, opts.ramp_tasks))
        self.l1_hits = self.l2_hits = self.host_fetches = 0
        self.tasks_done = 0
        self._cur: Optional[_Active] = None
        self.plan = runtime.plan
        self.esz = runtime.plan.dtype.itemsize
        self.f32 = self.esz == 4
        self.tile = runtime.plan.tile_size
        self.trace_on = opts.record_trace
        self.epoch = None
        self._snap_id = runtime.plan.snapshot_alias
        self._permanent = []
        self._retain = opts.retain_outputs and runtime.plan.call.kind == "trsm"
        self._early_release = False   # set by run_plan (single process, resident arenas)
        self.ic = None                # resident issue engine table (engine.IcTable), if used
        self.ic_d = -1                # this GPU's index in it
        self._ic_region = -1
        self._ic_group = 0            # bit mask of the GPUs in this GPU's peer group
        self._ic_refs = 0             # step references of the tasks issued (L1 hit count)
        self.resident = False   # set by run_plan when the arena holds the whole working set
        self._sync_epoch = 0
        self._task_misses = 0
        self.chunk_steps = opts.chunk_steps
        self._ramp_left = max(0, opts.ramp_tasks)
        self._pf = None               # windowed first-use prefetch (large one-GPU calls)
        self._pf_next, self._pf_events = 0, []
        # wind-down batch: one GPU, resident arenas, no DAG (set by run_plan)
        self._rampdown = 0
        grp = runtime.topology.peer_group_of(desc)
        self._group_peers = frozenset(d.device_id for d in runtime.topology.devices
                                      if d.device_id != desc.device_id
                                      and runtime.topology.peer_group_of(d) == grp)
        self._one_group = len(self._group_peers) == len(runtime.topology.devices) - 1
        self._pending_keys = set()   # resident blocks whose arrival event is not known done
        self._inv = {}               # diagonal tile key -> [offset, ld, event, landed]
        self._inv_events = []
        self._group_events = []      # arrival events shared by a batch of resident blocks
        self._wb_order = deque()     # issued tasks in write-back order (one in-order D2H lane)

    # ---- cache callbacks ------------------------------------------------------------

    def _on_evict(self, blk) -> None:
        if blk.ready_ev is not None:
            self.eng.release(blk.ready_ev)
            blk.ready_ev = None

    def _tile_geom(self, ref):
        h, w = ref.phys_height, ref.phys_width
        ld = device_ld(h)
        return h, w, ld, ld * w * self.esz

    def _host_of(self, ref):
        return self.plan.matrices[ref.matrix_id], ref.i * self.tile, ref.j * self.tile

    def _timed(self, lane, op, waits, kind, amount, k=-1):
        """Run ``op(waits)``; in trace mode bracket it with timing events."""
        if not self.trace_on:
            return op(waits)
        for w in waits:
            self.eng.stream_wait(self.slot, lane, w)
        e0 = self.eng.record(self.slot, lane, timing=True)
        ev = op(())
        e1 = self.eng.record(self.slot, lane, timing=True)
        task_id = self._cur.entry.task.task_id if self._cur is not None else -1
        self.runtime_trace.append((kind, lane, e0, e1, amount, task_id, k))
        return ev

    def copy_from_host(self, ref, blk) -> None:
        desc, r0, c0 = self._host_of(ref)
        h, w, ld, _ = self._tile_geom(ref)
        blk.ld = ld
        blk.ready_ev = self._timed(
            LANE_H2D, lambda wt: self.eng.h2d(self.slot, blk.offset, ld, desc, r0, c0, h, w, wt),
            (), "H2D", h * w * self.esz)
        self.dm.h2d_bytes += h * w * self.esz

    def copy_from_peer(self, src_cache, src_blk, ref, blk) -> bool:
        h, w, ld, nbytes = self._tile_geom(ref)
        blk.ld = ld
        waits = []
        if src_blk.ready_ev is not None and not src_blk.ready_done:
            if self.eng.done(src_blk.ready_ev):
                src_blk.ready_done = True
            else:
                waits.append(src_blk.ready_ev)
        src_slot = self.eng.slot(src_cache.device_id)
        blk.ready_ev = self._timed(
            LANE_P2P, lambda wt: self.eng.p2p(self.slot, blk.offset, src_slot, src_blk.offset,
                                              nbytes, wt), waits, "D2D", h * w * self.esz)
        self.dm.d2d_in_bytes += h * w * self.esz
        self.runtime.add_d2d_out(src_cache.device_id, h * w * self.esz)
        # the source stays pinned until the consumer task completes
        self._cur.pins.append((src_cache, src_blk))
        return True

    def pressure_sync(self) -> None:
        """Every cached block is pinned: drain the GPU, release the pins of all launched work
        and retire finished tasks, then let the caller retry (cache.py:232-250)."""
        cur = self._cur
        self._sync_epoch += 1
        self.eng.device_sync(self.slot)
        for act in [a for a in self.active if a is not None] + ([cur] if cur else []):
            for cache, blk in act.launched_pins:
                cache.unpin(blk)
            act.launched_pins = []
        self._retire_finished(block=False)
        if self.trace_on:
            t = self._now()
            self.runtime.record(TraceEvent(t, t, self.device_id, -1, "SYNC", 0, -1, -1))

    def _now(self) -> float:
        e = self.eng.record(self.slot, 0, timing=True)
        self.eng.sync(e)
        t = self.eng.elapsed_ms(self.epoch, e) / 1e3
        self.eng.release(e)
        return t

    # ---- scheduling -----------------------------------------------------------------

    def _refill(self) -> None:
        while self.rs.room(0) > 0:
            item = self.runtime.queue.get()
            if item is None:
                break
            self.rs.put(_SlotEntry(self.plan.tasks[item[0]], item[1]))
        if len(self.runtime.workers) > 1 and self.rs.pending_count() == 0:
            stolen = steal_for(self)
            if stolen is not None:
                self.rs.put(stolen)

    def _dir_version(self):
        """Changes whenever some GPU's cache gains a tile (Eq. 3 inputs changed)."""
        if self.ic is not None:
            met = self.ic.metrics
            return int(met[:, 2].sum() + met[:, 3].sum())
        return self.runtime.directory.version

    def _priority(self, task: Task) -> int:
        w = self.runtime.options.critical_path_weight
        if w:
            return self._eq3(task) + w * critical_path(task, self.plan)
        return self._eq3(task)

    def _eq3(self, task: Task) -> int:
        """Eq. 3: +2 per input-tile reference already in this GPU's L1, +1 per reference
        held by a peer of the same group (counted per step reference, scheduler.py:341-354)."""
        if self.ic is not None:
            tids, mult = ic_task_tiles(task)
            local = self.ic.off[self.ic_d, tids] >= 0
            if not self.runtime.options.l2_enabled:
                return int(2 * mult[local].sum())
            held = (self.ic.holders[tids] & self._ic_group) != 0
            return int((mult * np.where(local, 2, held)).sum())
        blocks = self.cache._blocks
        holders = self.runtime.directory._holders if self.runtime.options.l2_enabled else None
        group = self._group_peers
        keys = task_keys(task)
        if task._bx_single and self._one_group:
            # every tile referenced once and every GPU in one peer group (NVSwitch):
            # Eq. 3 = 2 |keys & L1| + |(keys & held anywhere) - L1|, in C-level set ops
            ks = task._bx_keyset
            local = ks & blocks.keys()
            if holders is None:
                return 2 * len(local)
            return 2 * len(local) + len((ks & holders.keys()) - local)
        p = 0
        for key, (_ref, mult) in keys.items():
            if key in blocks:
                p += 2 * mult
            elif holders is not None:
                held = holders.get(key)
                if held and not group.isdisjoint(held):
                    p += mult
        return p

    def _next_entry(self):
        self._refill()
        # Eq. 3 only changes when some cache gains or loses a tile: recompute an entry's
        # priority only if the directory changed since it was last computed
        ver = self._dir_version()
        for e in self.rs.entries():
            if e.pver != ver:
                e.priority = self._priority(e.task)
                e.pver = ver
        return self.rs.pop_best()

    def prefetch_step(self) -> bool:
        """Windowed first-use prefetch (RunOptions.prefetch_window_mb, one GPU, large
        calls): keep loading input tiles in the order the tasks first read them, in
        batches of 8 with one arrival event each, while less than the window is in flight
        on the H2D lane.  Tiles a task already fetched are L1 hits and skipped by C."""
        pf = self._pf
        if pf is None or self._pf_next >= len(pf[0]):
            return False
        order, window = pf
        self._pf_events = [e for e in self._pf_events if not self.eng.done(e)]
        issued = False
        while len(self._pf_events) * 8 < window and self._pf_next < len(order):
            batch = order[self._pf_next:self._pf_next + 8]
            self._pf_next += len(batch)
            _offs, _lds, waits = self.eng.ic_resolve(self.ic, self.ic_d, array("i", batch))
            self._pf_events.extend(waits[-1:])
            issued = True
        return issued

    def fill(self) -> bool:
        fresh = []
        if self._rampdown > 0:
            # wind-down batch (RunOptions.rampdown_tasks): once at most that many tasks are
            # left to start, start them all at once in extra slots with short launches
            # issued k-major, so the call ends on many tasks' last steps instead of a few
            # tasks' whole k-loops
            left = len(self.runtime.queue) + self.rs.pending_count()
            if 0 < left <= self._rampdown:
                self.active.extend([None] * left)
                self._ramp_left = left
                self._rampdown = 0
        # ramp tasks (start-up batch) use extra slots; the others are capped at base_slots
        normal = sum(1 for a in self.active if a is not None and not a.ramp)
        for s, act in enumerate(self.active):
            if act is not None:
                continue
            if self._ramp_left <= 0 and normal >= self.base_slots:
                break
            entry = self._next_entry()
            if entry is None:
                break
            act = self._begin(entry, s)
            normal += not act.ramp
            fresh.append(act)
        # one launch group per fresh task per round (k-major fetch order across them)
        pending = fresh
        while pending:
            pending = [a for a in pending if not self._advance(a)]
        return bool(fresh)

    # ---- issue ----------------------------------------------------------------------

    def _resolve_op(self, task, op, res):
        """Evicting (non-resident) mode: translate and pin only the tiles one launch needs,
        just before it is enqueued, so a task never needs more than one chunk of inputs in
        the arena at once (the reference holds one step's tiles, scheduler.py:426-461).
        If a pressure sync fires meanwhile (pins of launched work released), entries
        resolved for earlier launches are dropped and re-translated on demand."""
        keys = task_keys(task)
        if type(op) is GemmOp:
            want = [k for ak, bk, _, _ in op.subs for k in (ak, bk)]
        else:
            want = [op.key]
        cache = self.cache
        for _attempt in range(4):
            epoch = self._sync_epoch
            pinned_now = set()
            restart = False
            for key in want:
                if key in res or key[0] == "#scratch":
                    continue
                ref = keys[key][0]
                h, w, ld, nbytes = self._tile_geom(ref)
                blk, outcome = cache.translate(ref, self, nbytes=nbytes, ld=ld)
                if outcome == L2_HIT:
                    self.l2_hits += 1
                    self._task_misses += 1
                elif outcome == HOST_FETCH:
                    self.host_fetches += 1
                    self._task_misses += 1
                cache.pin(blk)
                self._cur.pins.append((cache, blk))
                pinned_now.add(key)
                wait = None
                if blk.ready_ev is not None and not blk.ready_done:
                    if self.eng.done(blk.ready_ev):
                        blk.ready_done = True
                    else:
                        wait = blk.ready_ev
                res[key] = (blk.offset, blk.ld, wait)
                if self._sync_epoch != epoch:
                    restart = True
                    break
            if not restart:
                return res
            # launched pins were released by the drain: keep only what is pinned now
            for k in list(res):
                if k not in pinned_now and k[0] != "#scratch":
                    del res[k]
        raise CapacityDeadlockError(
            f"device {self.device_id}: one launch's tiles cannot all fit in the arena at once; "
            f"enlarge the arena or shrink the tiles")

    def _resolve_resident(self, task, subset=None):
        """Resident mode: the arena was sized to hold every input tile of the call, so the
        ALRU can never evict.  Each block is pinned once, permanently, when it arrives, and
        a task's translation reduces to lookups (no per-task pins / recency updates).
        ``subset`` restricts the work to some of the task's tiles (one launch group)."""
        cache = self.cache
        blocks = cache._blocks
        keys = task_keys(task)
        ks = task._bx_keyset
        if subset is not None:
            ks = subset
            keys = {k: keys[k] for k in subset}
        pend = self._pending_keys
        if pend and not pend.isdisjoint(ks):
            # drop keys whose copies have landed
            eng = self.eng
            for k in list(pend & ks):
                b = blocks.get(k)
                if b is None or b.ready_done or eng.done(b.ready_ev):
                    if b is not None:
                        b.ready_done = True
                    pend.discard(k)
        if ks <= blocks.keys() and pend.isdisjoint(ks):
            # steady state: every tile resident and landed
            self.l1_hits += task._bx_refs if subset is None else sum(m for _, m in keys.values())
            return {k: (b.offset, b.ld, None) for k in ks for b in (blocks[k],)}
        out = {}
        eng = self.eng
        hits = 0
        misses = [(key, ref) for key, (ref, _m) in keys.items() if key not in blocks]
        if misses:
            self._fetch_many(misses)
            hits -= len(misses)
        for key, (ref, mult) in keys.items():
            blk = blocks[key]
            hits += mult
            wait = None
            ev = blk.ready_ev
            if ev is not None and not blk.ready_done:
                if eng.done(ev):
                    blk.ready_done = True
                else:
                    wait = ev
                    pend.add(key)
            out[key] = (blk.offset, blk.ld, wait)
        self.l1_hits += hits
        return out

    def _fetch_many(self, misses) -> None:
        """Resident-mode misses of one launch group, fetched with ONE engine call
        (``copy_batch``): per tile the same policy as ``_fetch_resident`` (L2 copy from the
        lowest-id peer holding the tile, else H2D from pinned host memory), but a single
        arrival event per copy lane for the whole batch (the lanes are in-order) instead
        of an engine call and an event per tile."""
        eng = self.eng
        if self.trace_on or not hasattr(eng, "copy_batch"):
            for key, ref in misses:
                self._fetch_resident(key, ref)
            return
        esz = self.esz
        directory = self.runtime.directory
        l2 = self.runtime.options.l2_enabled
        rows = array("q")
        new_h, new_p = [], []
        dm = self.dm
        for key, ref in misses:
            h, w = ref.phys_height, ref.phys_width
            ld = device_ld(h)
            nbytes = ld * w * esz
            try:
                off = self.arena.alloc(nbytes)
            except ArenaOutOfMemoryError:
                raise CapacityDeadlockError(
                    f"device {self.device_id}: resident arena exhausted (working-set estimate "
                    f"too small); set DeviceDesc.arena_capacity to use the evicting cache") from None
            blk = LruBlock(key, off, nbytes, ld, self.device_id)
            blk.reader = 1
            payload = h * w * esz
            src_id = directory.peer_source(key, self.device_id) if l2 else None
            src_blk = directory.cache_of(src_id)._blocks.get(key) if src_id is not None else None
            if src_blk is not None:
                wait = -1
                if src_blk.ready_ev is not None and not src_blk.ready_done:
                    if eng.done(src_blk.ready_ev):
                        src_blk.ready_done = True
                    else:
                        wait = src_blk.ready_ev
                rows.extend((1, off, ld, eng.slot(src_id), src_blk.offset, nbytes, 0, wait))
                new_p.append(blk)
                dm.d2d_in_bytes += payload
                self.runtime.add_d2d_out(src_id, payload)
                self.l2_hits += 1
            else:
                desc, r0, c0 = self._host_of(ref)
                rows.extend((esz << 8, off, ld, desc.element_address(r0, c0), desc.leading_dim,
                             h, w, -1))
                new_h.append(blk)
                dm.h2d_bytes += payload
                self.host_fetches += 1
        ev_h, ev_p = eng.copy_batch(self.slot, rows)
        for ev in (ev_h, ev_p):
            if ev >= 0:
                self._group_events.append(ev)
        pend = self._pending_keys
        blocks = self.cache._blocks
        with self.cache.lock:
            for blist, ev in ((new_h, ev_h), (new_p, ev_p)):
                for blk in blist:
                    blk.ready_ev = ev          # shared: owned by _group_events
                    blocks[blk.key] = blk
                    pend.add(blk.key)
        for blist in (new_h, new_p):
            for blk in blist:
                directory.add_holder(blk.key, self.device_id)
                self._permanent.append(blk)

    def _fetch_resident(self, key, ref):
        """Miss path of resident mode: allocate (never evicts), copy from the lowest-id peer
        holding the tile (L2 over NVLink) or from pinned host memory, register the block
        in the directory and pin it for the call."""
        h, w = ref.phys_height, ref.phys_width
        ld = device_ld(h)
        nbytes = ld * w * self.esz
        try:
            off = self.arena.alloc(nbytes)
        except ArenaOutOfMemoryError:
            raise CapacityDeadlockError(
                f"device {self.device_id}: resident arena exhausted (working-set estimate "
                f"too small); set DeviceDesc.arena_capacity to use the evicting cache") from None
        blk = LruBlock(key, off, nbytes, ld, self.device_id)
        blk.reader = 1
        payload = h * w * self.esz
        directory = self.runtime.directory
        src_id = directory.peer_source(key, self.device_id) if self.runtime.options.l2_enabled else None
        src_blk = None
        if src_id is not None:
            src_blk = directory.cache_of(src_id)._blocks.get(key)
        if src_blk is not None:
            waits = ()
            if src_blk.ready_ev is not None and not src_blk.ready_done:
                if self.eng.done(src_blk.ready_ev):
                    src_blk.ready_done = True
                else:
                    waits = (src_blk.ready_ev,)
            src_slot = self.eng.slot(src_id)
            blk.ready_ev = self._timed(LANE_P2P, lambda wt: self.eng.p2p(
                self.slot, off, src_slot, src_blk.offset, nbytes, wt), waits, "D2D", payload)
            self.dm.d2d_in_bytes += payload
            self.runtime.add_d2d_out(src_id, payload)
            self.l2_hits += 1
        else:
            desc, r0, c0 = self._host_of(ref)
            blk.ready_ev = self._timed(LANE_H2D, lambda wt: self.eng.h2d(
                self.slot, off, ld, desc, r0, c0, h, w, wt), (), "H2D", payload)
            self.dm.h2d_bytes += payload
            self.host_fetches += 1
        self._pending_keys.add(key)
        with self.cache.lock:
            self.cache._blocks[key] = blk
        directory.add_holder(key, self.device_id)
        self._permanent.append(blk)
        return blk

    def _resolve_uncached(self, task):
        """l1_enabled=False (scheduler.py:463-485): every step reference is a fresh host
        fetch into a transient buffer; a tile referenced by several steps of the task is
        fetched once per reference (counted as such) and the last copy is used."""
        out = {}
        for st in task.steps:
            for ref in st.input_refs():
                out[ref.key()] = self._resolve(ref)
        return out

    def _resolve(self, ref):
        """Uncached path (l1_enabled=False): every reference is a fresh host fetch."""
        act = self._cur
        h, w, ld, nbytes = self._tile_geom(ref)
        if True:
            off = self.cache.allocate_under_pressure(nbytes, self)
            act.scratch.append(off)
            desc, r0, c0 = self._host_of(ref)
            ev = self._timed(LANE_H2D, lambda wt: self.eng.h2d(self.slot, off, ld, desc, r0, c0,
                                                               h, w, wt), (), "H2D", h * w * self.esz)
            act.events.append(ev)
            self.dm.h2d_bytes += h * w * self.esz
            self.host_fetches += 1
            return off, ld, ev

    def _launched(self, act, ev) -> None:
        if ev is not None and ev >= 0:
            act.events.append(ev)
            act.last_ev = ev
        act.launched_pins.extend(act.pins)
        act.pins = []
        self.dm.kernel_launches += 1

    def _begin(self, entry, slot_index):
        """Issue a task's C buffer (and C move-in) and compile its launch program; the
        launches themselves are enqueued by ``_advance`` one launch group at a time."""
        task = entry.task
        opts = self.runtime.options
        act = _Active(entry, slot_index % self.n_streams, slot_index)
        self._cur = act
        try:
            out = task.out_ref
            h, w = out.phys_height, out.phys_width
            act.c_ld = device_ld(h)
            act.c_off = self.cache.allocate_under_pressure(act.c_ld * w * self.esz, self)
            # the C move-in is enqueued with the task's first launch group (_advance), so
            # the H2D queue interleaves a fresh batch's C tiles with its first panels
            act.c_pending = task.needs_c_move_in
            chunk = self.chunk_steps
            if self._ramp_left > 0:
                self._ramp_left -= 1
                act.ramp = True
                chunk = min(opts.ramp_chunk_steps, chunk)
            act.prog = compile_task(task, self.plan.call, chunk, opts.first_chunk_steps,
                                    opts.defer_c_move_in, opts.trsm_split_chain,
                                    opts.split_km)
            if act.prog.defer_c:
                # C0 gets its own buffer, fetched with the task's last launch group
                act.c_pending = False
                act.c0_off = self.cache.allocate_under_pressure(act.c_ld * w * self.esz, self)
                act.scratch.append(act.c0_off)
            act.lazy = opts.l1_enabled and not self.resident
            act.misses = 0
            act.misses_epoch = self._sync_epoch
            if not opts.l1_enabled:
                act.res = self._resolve_uncached(task)
            else:
                act.res = {}
            for i, n in enumerate(act.prog.scratch_n):
                ld = device_ld(n)
                off = self.cache.allocate_under_pressure(ld * n * self.esz, self)
                act.scratch.append(off)
                act.res[scratch_key(i)] = (off, ld, None)
            last = act.prog.ops[-1] if act.prog.ops else None
            if (type(last) is TrsmOp and self.resident and self._inv_wanted(task)
                    and os.environ.get("BX_TRSM_EARLY_INV", "1") != "0"):
                # start inv(E) of this task's diagonal tile now, on another stream, so it
                # overlaps the task's update GEMMs instead of following them
                out = task.out_ref
                n = out.phys_width if self.plan.call.side == "right" else out.phys_height
                if last.key not in self._inv:
                    act.res.update(self._resolve_resident(task, frozenset((last.key,))))
                    ao, al, aw = act.res[last.key]
                    self._trsm_inverse(last.key, ao, al, aw, (act.stream + 1) % self.n_streams, n)
            act.next_op = 0
            act.flops = task.flops
            if self.ic is not None:
                task_keys(task)
                self._ic_refs += task._bx_refs
        finally:
            self._cur = None
        self.active[slot_index] = act
        return act

    def _advance(self, act) -> bool:
        """Enqueue the task's next launch group (its tile fetches, then the launch); after
        the last group, enqueue the write-back.  Returns True once the task is fully
        issued.  Interleaving groups across freshly issued tasks orders the H2D queue
        k-major across them, so they share panel tiles early instead of one task
        fetching its whole k-range first."""
        task = act.entry.task
        call = self.plan.call
        opts = self.runtime.options
        ops = act.prog.ops
        eng, slot, stream = self.eng, self.slot, act.stream
        out = task.out_ref
        h, w = out.phys_height, out.phys_width
        self._cur = act
        self._task_misses = act.misses
        try:
            if act.c_pending:
                act.c_pending = False
                desc, r0, c0 = self._host_of(out)
                ev = self._timed(LANE_H2D, lambda wt: eng.h2d(
                    slot, act.c_off, act.c_ld, desc, r0, c0, h, w, wt), (), "H2D",
                    h * w * self.esz)
                act.events.append(ev)
                act.pending_waits.append(ev)
                self.dm.h2d_bytes += h * w * self.esz
            res = act.res
            i = act.next_op
            while i < len(ops):
                op = ops[i]
                i += 1
                if type(op) is AxpyOp:
                    pass
                elif act.lazy:
                    if act.misses_epoch != self._sync_epoch:
                        # a pressure sync released this task's earlier pins: forget them
                        for k in [k for k in res if k[0] != "#scratch"]:
                            del res[k]
                        act.misses_epoch = self._sync_epoch
                    res = act.res = self._resolve_op(task, op, res)
                    act.misses_epoch = self._sync_epoch
                elif self.ic is not None:
                    if type(op) is GemmOp:
                        last = i == len(ops)
                        steps, raw = ic_op_steps(task, act.prog, i - 1, res)
                        waits = act.pending_waits
                        act.pending_waits = []
                        ev = eng.ic_gemm(self.ic, self.ic_d, stream, self.f32, op.ta, op.tb, op.tri,
                                         h, w, steps, raw, op.alpha, op.beta, act.c_off, act.c_ld,
                                         waits, event=last)
                        self._launched(act, ev)
                        break
                    if op.key not in res:     # MatOp: its diagonal tile
                        offs, lds, wts = eng.ic_resolve(self.ic, self.ic_d,
                                                        array("i", (ic_tile_index(task, op.key),)))
                        res[op.key] = (offs[0], lds[0], wts[0] if wts else None)
                        if len(wts) > 1:
                            act.pending_waits.extend(wts[1:])
                elif opts.l1_enabled:
                    want = (op.keys if type(op) is GemmOp else frozenset((op.key,))) - res.keys()
                    if want:
                        res.update(self._resolve_resident(task, want))
                if type(op) is GemmOp:
                    steps = []
                    waits = []
                    for ak, bk, d, km in op.subs:
                        a_, b_ = res[ak], res[bk]
                        steps.append((a_[0], a_[1], b_[0], b_[1], d, km))
                        if a_[2] is not None:
                            waits.append(a_[2])
                        if b_[2] is not None:
                            waits.append(b_[2])
                    if waits:
                        waits = list(dict.fromkeys(waits))
                    waits += act.pending_waits
                    act.pending_waits = []
                    # only the task's last launch needs an event (its write-back waits on
                    # it); earlier launches are ordered by the task's stream
                    last = i == len(ops)
                    ev = self._timed(stream, lambda wt, op=op, steps=steps, last=last: eng.gemm(
                        slot, stream, op.ta, op.tb, op.tri, h, w, steps, op.alpha, op.beta,
                        act.c_off, act.c_ld, wt, f32=self.f32, event=last), waits, "KERNEL",
                        op.flops, op.k)
                    self._launched(act, ev)
                    break
                elif type(op) is MatOp:
                    ao, al, aw = res[op.key]
                    so, sl, _ = res[scratch_key(op.scratch)]
                    ev = self._timed(stream, lambda wt, op=op, ao=ao, al=al, so=so, sl=sl: eng.materialize(
                        slot, stream, op.sym, call.uplo == "upper",
                        False if op.sym else call.trans_a, (not op.sym) and call.diag == "unit",
                        op.n, ao, al, so, sl, wt, event=False), [aw] if aw is not None else [],
                        "KERNEL", 0, -1)
                    if ev is not None and ev >= 0:
                        act.events.append(ev)
                elif type(op) is AxpyOp:
                    desc, r0, c0 = self._host_of(out)
                    c0_ev = self._timed(LANE_H2D, lambda wt: eng.h2d(
                        slot, act.c0_off, act.c_ld, desc, r0, c0, h, w, wt), (), "H2D",
                        h * w * self.esz)
                    act.events.append(c0_ev)
                    self.dm.h2d_bytes += h * w * self.esz
                    ev = self._timed(stream, lambda wt, op=op: eng.axpy(
                        slot, stream, self.esz, h, w, op.beta, act.c0_off, act.c_ld, act.c_off,
                        act.c_ld, wt), [c0_ev], "KERNEL", 0, -1)
                    self._launched(act, ev)
                    break
                else:   # TrsmOp
                    ao, al, aw = res[op.key]
                    waits = ([aw] if aw is not None else []) + act.pending_waits
                    act.pending_waits = []
                    inv = self._trsm_inverse(op.key, ao, al, aw, stream, w if call.side == "right" else h)
                    if inv is not None:
                        # X = alpha inv(E) B into a fresh tile, which becomes the task's C
                        inv_off, inv_ld, inv_wait = inv
                        x_off = self.cache.allocate_under_pressure(act.c_ld * w * self.esz, self)
                        eff_upper = (call.uplo == "upper") != call.trans_a
                        ev = self._timed(stream, lambda wt, op=op, x_off=x_off: eng.trsm_apply(
                            slot, stream, call.side == "right", eff_upper, h, w, op.alpha, inv_off,
                            inv_ld, act.c_off, act.c_ld, x_off, act.c_ld, wt),
                            waits + ([inv_wait] if inv_wait is not None else []), "KERNEL",
                            op.flops, op.k)
                        act.scratch.append(act.c_off)
                        act.c_off = x_off
                    else:
                        ev = self._timed(stream, lambda wt, op=op, ao=ao, al=al: eng.trsm(
                            slot, stream, call.side == "right", call.uplo == "upper", call.trans_a,
                            call.diag == "unit", h, w, op.alpha, ao, al, act.c_off, act.c_ld, wt),
                            waits, "KERNEL", op.flops, op.k)
                    self._launched(act, ev)
                    break
            act.next_op = i
            act.misses = self._task_misses
            if i < len(ops):
                return False
            desc, r0, c0 = self._host_of(out)
            waits = [act.last_ev] + act.pending_waits
            act.pending_waits = []
            act.done_ev = self._timed(LANE_D2H, lambda wt: eng.d2h(
                slot, act.c_off, act.c_ld, desc, r0, c0, h, w, wt), waits, "D2H",
                h * w * self.esz)
            self.dm.d2h_bytes += h * w * self.esz
            act.events.append(act.done_ev)
            self._wb_order.append(act)
            if self._early_release and task.dependents:
                self._retain_on_issue(act)
            if act.lazy:
                self.l1_hits += task._bx_refs - act.misses
            act.res = None
            return True
        finally:
            self._cur = None

    def _retain_on_issue(self, act) -> None:
        """Release-on-issue: cache the task's solved tile now (state M: the device copy is
        the only up-to-date one until the write-back lands), with the event after the
        task's last kernel as its arrival event, and release the dependents.  A dependent
        on this GPU waits on that event on the GPU; one on a peer copies the tile over
        NVLink after it (the P2P copy waits on the same event).  The tile's value is final
        — TRSM writes each output tile once — so early readers see exactly what the
        write-back publishes."""
        task = act.entry.task
        key = task.out_ref.key()
        if act.last_ev is None or act.last_ev < 0 or self.cache.contains(key):
            return
        blk = LruBlock(key, act.c_off, act.c_ld * task.out_ref.phys_width * self.esz, act.c_ld,
                       self.device_id)
        blk.ready_ev = act.last_ev
        self.cache.insert_front(blk)
        self.cache.pin(blk)
        self._permanent.append(blk)
        self._pending_keys.add(key)
        act.retained = blk
        self.runtime.release_dependents(task)

    def _inv_wanted(self, task) -> bool:
        opts = self.runtime.options
        out = task.out_ref
        n = out.phys_width if self.plan.call.side == "right" else out.phys_height
        return bool(opts.trsm_inverse_min) and not self.f32 and n >= opts.trsm_inverse_min

    def _trsm_inverse(self, key, a_off, a_ld, a_wait, stream, n):
        """inv(E) of the diagonal tile ``key`` for the inverse-based TRSM diagonal step
        (resident arenas only): computed once per GPU and call by the first task that needs
        it, on that task's stream; later tasks wait on its event.  Returns (offset, ld,
        event to wait on or None), or None for the substitution path."""
        opts = self.runtime.options
        if (not self.resident or self.f32 or not opts.trsm_inverse_min
                or n < opts.trsm_inverse_min):
            return None
        ent = self._inv.get(key)
        if ent is None:
            ld = device_ld(n)
            try:
                off = self.arena.alloc(ld * n * self.esz)
            except ArenaOutOfMemoryError:
                return None
            call = self.plan.call
            ev = self._timed(stream, lambda wt: self.eng.trsm_inverse(
                self.slot, stream, call.uplo == "upper", call.trans_a, call.diag == "unit", n,
                a_off, a_ld, off, ld, wt), [a_wait] if a_wait is not None else [], "KERNEL",
                n * n * n // 3, -1)
            self._inv_events.append(ev)
            self._inv[key] = ent = [off, ld, ev, False]
        if not ent[3] and self.eng.done(ent[2]):
            ent[3] = True
        return ent[0], ent[1], None if ent[3] else ent[2]

    # ---- completion -----------------------------------------------------------------

    def in_flight(self) -> list:
        """The next write-back to complete (the D2H lane is in order, so no later task can
        complete before it)."""
        return [self._wb_order[0].done_ev] if self._wb_order else []

    def _retire(self, act) -> None:
        task = act.entry.task
        for cache, blk in act.pins + act.launched_pins:
            cache.unpin(blk)
        act.pins = act.launched_pins = []
        for off in act.scratch:
            self.arena.free(off)
        kept = act.retained
        if kept is not None:
            # cached at issue: the write-back has landed, so the solve has too.  Its event
            # id now belongs to the block (a peer may have read it as a wait) and is
            # released with the block when the call ends (release_all -> _on_evict)
            kept.ready_done = True
            act.events = [e for e in act.events if e != kept.ready_ev]
        self.eng.release_many(act.events)
        key = task.out_ref.key()
        if kept is not None:
            pass   # M -> E: the block (and peer copies of its final value) stay cached
        elif self._retain and self.runtime.options.l1_enabled and not self.cache.contains(key):
            self.runtime.directory.note_write_back(key)
            # write-back-then-retain: after the D2H the device copy equals
            # the host copy, so the tile moves M -> E instead of M -> I and dependents read
            # it from L1 / over NVLink instead of re-fetching it from the host
            out = task.out_ref
            blk = LruBlock(key, act.c_off, act.c_ld * out.phys_width * self.esz, act.c_ld,
                           self.device_id)
            blk.ready_done = True
            self.cache.insert_front(blk)
            if self.resident:
                self.cache.pin(blk)
                self._permanent.append(blk)
        else:
            self.runtime.directory.note_write_back(key)
            self.arena.free(act.c_off)
        if self.plan.call.kind == "trsm" and self.eng.singular(self.slot, reset=True):
            raise SingularMatrixError("zero on a non-unit triangular diagonal")
        self.tasks_done += 1
        self.dm.tasks += 1
        self.runtime.complete_task(task)

    def _retire_finished(self, block: bool) -> bool:
        """Retire completed tasks in write-back order: one event query per completed task
        plus one for the first still in flight, instead of one per active task."""
        got = False
        q = self._wb_order
        while q and self.eng.done(q[0].done_ev):
            act = q.popleft()
            self.active[act.slot_index] = None
            self._retire(act)
            got = True
        return got

    def poll(self) -> bool:
        return self._retire_finished(block=False)

    def idle(self) -> bool:
        return all(a is None for a in self.active)

    def ic_fold(self) -> None:
        """Add this GPU's resident issue engine counters to its metrics."""
        if self.ic is None:
            return
        met = self.ic.metrics[self.ic_d]
        self.dm.h2d_bytes += int(met[0])
        self.dm.d2d_in_bytes += int(met[1])
        self.host_fetches += int(met[2])
        self.l2_hits += int(met[3])
        self.l1_hits += self._ic_refs - int(met[2] + met[3])
        if met[4]:
            self.runtime.add_d2d_out(self.device_id, int(met[4]))

    def release_all(self) -> None:
        if self.ic is not None:
            if self.ic_d == 0:
                self.eng.ic_destroy(self.ic)
            self.arena.free(self._ic_region)
            self.ic, self.ic_d, self._ic_region = None, -1, -1
        for off, _ld, _ev, _landed in self._inv.values():
            self.arena.free(off)
        for ev in self._inv_events:
            self.eng.release(ev)
        self._inv, self._inv_events = {}, []
        if self._group_events:
            shared = set(self._group_events)
            for blk in self._permanent:
                if blk.ready_ev in shared:
                    blk.ready_ev = None
            for ev in self._group_events:
                self.eng.release(ev)
            self._group_events = []
        if self._permanent:
            self.cache.release(self._permanent)
            self._permanent = []
        for blk in self.cache.blocks():
            self._on_evict(blk)


def critical_path(task: Task, plan: TaskPlan) -> int:
    """Length of the longest chain of dependents below ``task`` (0 for a sink; TRSM only
    has dependency edges, routines.py:426-437).  Computed once per plan, cached on tasks."""
    cp = getattr(task, "_bx_cp", None)
    if cp is None:
        by_id = {t.task_id: t for t in plan.tasks}
        memo = {}   # explicit post-order DFS over the dependents DAG
        for root in plan.tasks:
            if root.task_id in memo:
                continue
            stack = [(root, False)]
            while stack:
                t, done = stack.pop()
                if t.task_id in memo:
                    continue
                if done:
                    memo[t.task_id] = max((1 + memo[d] for d in t.dependents), default=0)
                    continue
                stack.append((t, True))
                stack.extend((by_id[d], False) for d in t.dependents if d not in memo)
        for t in plan.tasks:
            t._bx_cp = memo[t.task_id]
        cp = task._bx_cp
    return cp


# ---- resident issue engine (engine.ic_*): tile ids and precompiled launch operands ----

IC_KINDS = ("gemm", "syrk", "syr2k", "symm")


def ic_index(plan: TaskPlan):
    """Input tiles of the plan's structure: (key -> tile id, [(key, phys h, phys w)]).
    Memoised on the (shared, immutable) tasks, so repeated calls of one shape reuse it."""
    if not plan.tasks:
        return {}, []
    hit = getattr(plan.tasks[0], "_bx_icmap", None)
    if hit is not None:
        return hit, plan.tasks[0]._bx_icgeom
    refs = {}
    for t in plan.tasks:
        for k, (ref, _m) in task_keys(t).items():
            refs.setdefault(k, ref)
    order = sorted(refs)
    tid = {k: i for i, k in enumerate(order)}
    geom = [(k, refs[k].phys_height, refs[k].phys_width) for k in order]
    for t in plan.tasks:
        t._bx_icmap = tid
        t._bx_icgeom = geom
    return tid, geom


def ic_task_tiles(task: Task):
    """The task's distinct input tile ids and per-tile reference counts (Eq. 3)."""
    hit = getattr(task, "_bx_ictiles", None)
    if hit is None:
        keys = task_keys(task)
        tmap = task._bx_icmap
        hit = (np.array([tmap[k] for k in keys], dtype=np.int64),
               np.array([m for _r, m in keys.values()], dtype=np.int64))
        task._bx_ictiles = hit
    return hit


def ic_tile_index(task: Task, key) -> int:
    return task._bx_icmap[key]


def ic_op_steps(task: Task, prog, index: int, res):
    """Launch ``index`` of the task's program as bx_ic_gemm step rows {a, b, depth, kmode}
    (scratch operand i -> id -(i+1), its (offset, ld) in the returned raw array)."""
    cache = getattr(task, "_bx_icsteps", None)
    if cache is None or cache[0] is not prog:
        cache = (prog, {})
        task._bx_icsteps = cache
    hit = cache[1].get(index)
    if hit is None:
        tmap = task._bx_icmap
        rows = array("i")
        scratch = False
        for ak, bk, d, km in prog.ops[index].subs:
            for k in (ak, bk):
                if k[0] == "#scratch":
                    rows.append(-(k[1] + 1))
                    scratch = True
                else:
                    rows.append(tmap[k])
            rows.append(d)
            rows.append(km)
        hit = cache[1][index] = (rows, scratch)
    rows, scratch = hit
    raw = None
    if scratch:
        raw = array("q")
        for i in range(len(prog.scratch_n)):
            off, ld, _ = res[scratch_key(i)]
            raw.append(off)
            raw.append(ld)
    return rows, raw


def _ic_setup(plan, options, workers, engine, topology) -> None:
    """Resident issue engine for this call: every GPU resident, L1 on, no tracing, one
    driver process, a routine whose programs are GEMM launches (+ materialise / axpy).
    Each GPU reserves a region of its arena for the call's input tiles."""
    if (not hasattr(engine, "ic_create") or options.record_trace or not options.l1_enabled
            or plan.call.kind not in IC_KINDS or plan.snapshot_alias is not None
            or os.environ.get("BX_IC", "1") == "0" or not plan.tasks
            or not all(w.resident for w in workers) or len(workers) > 32):
        return
    tmap, geom = ic_index(plan)
    esz = plan.dtype.itemsize
    t = plan.tile_size
    rows = array("q")
    region = 0
    for (mid, i, j), h, w in geom:
        desc = plan.matrices[mid]
        ld = device_ld(h)
        rows.extend((desc.element_address(i * t, j * t), desc.leading_dim, h, w, esz, ld))
        region += -(-ld * w * esz // 256) * 256
    offs = []
    try:
        for w in workers:
            offs.append(w.arena.alloc(region))
    except ArenaOutOfMemoryError:
        for w, off in zip(workers, offs):
            w.arena.free(off)
        return
    groups = {}
    gid = [groups.setdefault(topology.peer_group_of(w.desc), len(groups)) for w in workers]
    table = engine.ic_create([w.slot for w in workers], gid, rows, offs, [region] * len(workers),
                             options.l2_enabled)
    for d, (w, off) in enumerate(zip(workers, offs)):
        w.ic, w.ic_d, w._ic_region = table, d, off
        w._ic_group = sum(1 << e for e in range(len(workers)) if gid[e] == gid[d] and e != d)


SMALL_CALL_TASKS = 64    # below this a call has no start-up batch and may prefetch
LINK_BOUND_CALL_TASKS = 128   # ... and up to this many if its host traffic outlasts its math


def small_call(plan: TaskPlan, n_devices: int = 1) -> bool:
    """A call whose tasks can all be in flight at once: fewer than SMALL_CALL_TASKS, or up
    to LINK_BOUND_CALL_TASKS when it is host-link bound (its operand bytes at the ~54 GB/s
    of one host link take longer than its flops at the tensor rate: DGEMM 4096^3 at T=512,
    64 tasks, 11.0 -> 10.1 ms with the small-call rules; DGEMM 8192^3 at T=1024, 64 tasks
    but balanced, is better without them, profiles/small_call_ab_r02.txt)."""
    n = len(plan.tasks)
    if n < SMALL_CALL_TASKS:
        return True
    if n > LINK_BOUND_CALL_TASKS or n_devices > 1:
        return False
    esz = plan.dtype.itemsize
    call = plan.call
    nbytes = sum(m.rows * m.cols * esz for m in (call.a.matrix, call.b.matrix if call.b else None,
                                                   call.c.matrix) if m is not None)
    t_link = nbytes / 54e9
    t_math = plan.total_flops / (35e12 if esz == 8 else 600e12)
    return t_link > 1.5 * t_math


def _ic_prefetch(plan, options, workers, engine) -> None:
    """Small calls on one GPU (RunOptions.prefetch, auto: ``small_call``): enqueue every input tile's host load at the start, in the order the tasks will
    first read them (FIFO task order, then step order), one arrival event per task's new
    tiles.  The H2D lane then streams back to back instead of following the host's task
    issue rate; launches find the tiles present (or in flight: they wait on the arrival
    event).  Only with the resident issue engine on a single GPU: with several GPUs which
    GPU needs which tile is decided dynamically (stations, stealing), and a large call's
    C tiles would queue behind the whole prefetch on the one H2D lane."""
    want = options.prefetch
    if want < 0:
        want = small_call(plan)
    if len(workers) == 1 and workers[0].ic is not None and not want and options.prefetch_window_mb > 0:
        # large call: a window of first-use loads kept ahead of the tasks (prefetch_step)
        w = workers[0]
        seen, order = set(), []
        for task in plan.tasks:
            tids, _mult = ic_task_tiles(task)
            for t in tids:
                t = int(t)
                if t not in seen:
                    seen.add(t)
                    order.append(t)
        tile_bytes = device_ld(plan.tile_size) * plan.tile_size * plan.dtype.itemsize
        w._pf = (order, max(8, (options.prefetch_window_mb << 20) // tile_bytes))
        w._pf_next, w._pf_events = 0, []
        w.prefetch_step()
        return
    if not want or len(workers) != 1 or workers[0].ic is None:
        return
    w = workers[0]
    seen = set()
    for task in plan.tasks:
        tids, _mult = ic_task_tiles(task)
        new = [int(t) for t in tids if int(t) not in seen]
        if new:
            seen.update(new)
            engine.ic_resolve(w.ic, w.ic_d, array("i", new))


def task_keys(task: Task) -> dict:
    """Distinct input tiles of a task: key -> (ref, number of step references).  Cached on
    the (immutable) task together with its key set, total reference count and whether
    every tile is referenced once (the set-arithmetic priority fast path)."""
    keys = getattr(task, "_bx_keys", None)
    if keys is None:
        keys = {}
        for st in task.steps:
            for ref in st.input_refs():
                k = ref.key()
                hit = keys.get(k)
                keys[k] = (ref if hit is None else hit[0], 1 if hit is None else hit[1] + 1)
        task._bx_keys = keys
        task._bx_keyset = frozenset(keys)
        task._bx_refs = sum(m for _, m in keys.values())
        task._bx_single = task._bx_refs == len(keys)
    return keys


def _auto_arena_bytes(plan: TaskPlan, options: RunOptions, free_bytes: Optional[int]) -> int:
    """Enough for every tile of every input matrix plus the in-flight C / scratch buffers,
    capped at 90 % of free HBM (no eviction at BASELINE sizes on a 180 GB B200)."""
    esz = plan.dtype.itemsize
    t = plan.tile_size
    out_id = plan.call.c.matrix_id
    want = 0
    for mid, m in plan.matrices.items():
        if mid == out_id and plan.call.kind != "trsm":
            continue           # output tiles bypass the cache (except TRSM's solved tiles)
        rows_full, rem = divmod(m.rows, t)
        col_tiles = -(-m.cols // t)
        per_col_tile = rows_full * device_ld(t) + (device_ld(rem) if rem else 0)
        want += -(-per_col_tile * t * col_tiles * esz // 256) * 256 + 256 * col_tiles * (rows_full + 1)
    per_tile = device_ld(t) * t * esz
    slots = (options.n_streams * options.tasks_per_stream + max(0, options.ramp_tasks)
             + max(0, options.rampdown_tasks))
    want += (slots + 2) * 2 * per_tile + (64 << 20)
    if plan.call.kind == "trsm" and options.trsm_inverse_min:
        want += -(-plan.call.a.matrix.rows // t) * per_tile      # one inverse per diagonal tile
    if free_bytes is None:
        return want
    cap = int(free_bytes * 0.9) - (1 << 30)
    return max(min(want, cap), (WORKING_SET_TILES + 1) * per_tile)


def resolve_streams(plan: TaskPlan, options: RunOptions, n_devices: int,
                    bounded_arena: bool = False) -> RunOptions:
    """Auto launch shape.  chunk_steps=0: 8 k-steps per launch for GEMM/SYMM/SYR2K, 16
    otherwise (SYR2K 137.2 -> 130.3 ms; TRMM better at 16).
    n_streams=0: 4 compute streams (the reference's lanes, devices.py:36); GEMM/SYMM, TRSM
    and TRMM 8 (more independent launches in flight; latency-bound diagonal solves /
    materialisations leave SMs idle otherwise); SYRK 12 (its diagonal tasks run half-empty
    triangle kernels) — but never more in-flight tasks than a quarter of a GPU's share of
    the plan, so the dynamic schedule keeps tasks to balance at high GPU counts
    (profiles/streams_sweep_r01.txt, profiles/chunk_streams_sweep_r01.txt)."""
    import dataclasses
    kind = plan.call.kind
    if not options.chunk_steps:
        # GEMM-only tasks: 8-step launches interleave better across the streams than one
        # 16-step launch per task (cfg2 255.8 -> 252.4 ms with 8 streams)
        options = dataclasses.replace(options, chunk_steps=8 if kind in ("gemm", "symm", "syr2k") else 16)
    if options.n_streams:
        return options
    if n_devices == 1 and plan.tasks and small_call(plan) and not bounded_arena:
        # a small call on one GPU (auto-sized arena) has nothing to balance: one task per
        # stream, up to 16 (cfg1, 16 tasks: 2.7 -> 2.6 ms against the capped 4 streams,
        # profiles/small_call_ab_r02.txt)
        return dataclasses.replace(options, n_streams=min(16, len(plan.tasks)))
    want = {"trsm": 8, "trmm": 8, "syrk": 12, "gemm": 8, "symm": 8}.get(kind, 4)
    share = len(plan.tasks) // max(1, n_devices)
    cap = max(4, share // (4 * max(1, options.tasks_per_stream)))
    return dataclasses.replace(options, n_streams=min(want, cap) if want > 4 else want)


def resolve_ramp(plan: TaskPlan, options: RunOptions, n_devices: int) -> RunOptions:
    """ramp_tasks=-1 (auto): a start-up batch of up to 32 tasks per GPU, but at most a
    quarter of each GPU's share of the plan so the dynamic schedule (stations, stealing,
    L2 locality) keeps its freedom at high GPU counts.  No ramp for calls of fewer than 64
    tasks: their tasks are all issued at once anyway, and the first launches should carry
    whole tasks (cfg1, 16 tasks: 3.2 -> 2.9 ms without the ramp, profiles/ramp_ab_r02.txt)."""
    if options.ramp_tasks >= 0:
        return options
    import dataclasses
    ntasks = len(plan.tasks)
    ramp = min(32, ntasks // (4 * max(1, n_devices))) if not small_call(plan, n_devices) else 0
    return dataclasses.replace(options, ramp_tasks=ramp if ramp >= 4 else 0)


# One call at a time per process: every call carves its tiles out of the process-wide
# engine's per-GPU arena (offset 0 up) and shares the engine's streams, event pool and
# singular flag, so concurrent callers (threads, or C callers of libblasx.so with the GIL
# released inside ctypes) are serialised here.
_CALL_LOCK = threading.RLock()


def run_plan(plan: TaskPlan, topology: Optional[Topology] = None,
             options: Optional[RunOptions] = None, engine=None, _t_plan: float = 0.0) -> RunResult:
    """Execute a task plan on the topology's GPUs; the host output holds the result.
    Thread-safe: calls from several threads run one after another (``_CALL_LOCK``)."""
    with _CALL_LOCK:
        return _run_plan(plan, topology, options, engine, _t_plan)


def _run_plan(plan: TaskPlan, topology: Optional[Topology], options: Optional[RunOptions],
              engine, _t_plan: float) -> RunResult:
    from .engine import get_engine
    t_setup0 = time.perf_counter()
    options = options or RunOptions()
    if options.execution not in ("deterministic", "concurrent", "spmd"):
        raise ConfigError(f"unknown execution mode {options.execution!r}")
    if not 0 <= options.n_streams <= 16:
        raise ConfigError("n_streams must be in 1..16")
    if options.chunk_steps < 0:
        raise ConfigError("chunk_steps must be >= 1 (0 = auto)")
    if options.tasks_per_stream < 1:
        raise ConfigError("tasks_per_stream must be >= 1")
    if options.execution == "spmd":
        # one process per GPU: every rank of the session runs this same call (spmd.py)
        from . import spmd
        return spmd.run_plan_spmd(plan, options, engine, _t_plan=_t_plan)
    topology = topology or discover_topology()
    devs = topology.accelerators()
    bounded = bool(options.arena_bytes) or any(d.arena_capacity for d in devs)
    options = resolve_streams(plan, options, len(devs), bounded)
    options = resolve_ramp(plan, options, len(devs))
    if engine is None:
        engine = get_engine([d.device_id for d in devs], options.n_streams,
                            [d.device_id if d.cuda_ordinal is None else d.cuda_ordinal for d in devs])
    esz = plan.dtype.itemsize
    per_tile = device_ld(plan.tile_size) * plan.tile_size * esz
    caps = {}
    resident = {}
    for d in devs:
        slot = engine.slot(d.device_id)
        want = d.arena_capacity or options.arena_bytes
        resident[slot] = not want
        if not want:
            full = want = _auto_arena_bytes(plan, options, None)
            if want > engine.arena_capacity(slot):     # only then ask the driver (slow query)
                want = _auto_arena_bytes(plan, options, engine.free_bytes(slot)
                                         + engine.arena_capacity(slot))
            resident[slot] = want >= full              # out-of-core calls keep the full ALRU
        if want <= WORKING_SET_TILES * per_tile:
            raise ConfigError(
                f"device {d.device_id}: arena of {want} bytes cannot hold the "
                f"{WORKING_SET_TILES}-tile working set at tile size {plan.tile_size}")
        caps[slot] = want
    if not all(resident.values()):
        # one residency mode per call: a resident device copies from a peer's block without
        # pinning it, which is only safe if that peer can never evict (never reuse) the block
        resident = {s: False for s in resident}
    engine.ensure_arenas(caps)
    if plan.dtype.itemsize == 4 and hasattr(engine, "lib"):
        engine.lib.bx_set_sgemm_precise(int(sgemm_precise_for(plan, options)))
    if plan.snapshot_alias is not None and not _snapshot_alias_safe(
            plan, options, topology, devs, resident, caps, per_tile):
        # the reference's host copy (routines.py:393-400)
        from .tiling import MatrixDesc as _MD
        snap = plan.matrices[plan.snapshot_alias]
        plan.matrices[plan.snapshot_alias] = _MD(
            snap.matrix_id, snap.rows, snap.cols, snap.leading_dim, snap.storage.copy(),
            snap.base_offset)
        plan.snapshot_alias = None
    # Page-lock the operands for the DMA engine.  Buffers pinned by the caller beforehand
    # (``pin_host``; the paper excludes page-locking from timing) stay
    # pinned; the ones pinned here are unpinned when the call returns.
    pinned_here = [m.storage for m in plan.matrices.values() if engine.register_host(m.storage)]

    rt = _Runtime(plan, topology, options, engine)
    workers = [_GpuWorker(d, rt) for d in devs]
    for w in workers:
        w.resident = resident[w.slot] and options.l1_enabled
        # a dependent on another GPU must get the tile over L2 (the host copy is stale
        # until the write-back lands): one GPU, or L2 on with every GPU in one peer group
        w._early_release = (w.resident and w._retain and options.release_on_issue
                            and (len(devs) == 1 or (options.l2_enabled and w._one_group)))
        if (w.resident and len(devs) == 1 and options.rampdown_tasks > 0
                and plan.call.kind != "trsm"):
            w._rampdown = options.rampdown_tasks
        if not w.resident:
            w._ramp_left = 0      # the start-up batch is for resident arenas only
            # an evicting arena must hold every in-flight task's C and one launch's inputs
            tiles = caps[w.slot] // per_tile
            inflight = options.n_streams * options.tasks_per_stream
            w.chunk_steps = max(1, min(options.chunk_steps, (tiles - 2 * inflight) // 4))
        # an explicit capacity smaller than the reservation bounds the arena (eviction tests)
        if caps[w.slot] < w.arena.capacity:
            w.arena = Arena(caps[w.slot])
            w.cache.arena = w.arena
        w.runtime_trace = []
    rt.workers = workers
    _ic_setup(plan, options, workers, engine, topology)
    for w in workers:
        w.epoch = engine.record(w.slot, 0, timing=True)
    t0 = time.perf_counter()
    t_setup = t0 - t_setup0
    try:
        _ic_prefetch(plan, options, workers, engine)
        if options.execution == "deterministic":
            _drive_single(rt, workers)
        else:
            _drive_threads(rt, workers)
    except BaseException:
        for w in workers:
            try:
                engine.device_sync(w.slot)
            except Exception:
                pass
        if workers and workers[0].ic is not None:
            try:
                engine.ic_destroy(workers[0].ic)
            except Exception:
                pass
        _unpin(engine, pinned_here)
        raise
    wall = time.perf_counter() - t0
    t_fin0 = time.perf_counter()
    for w in workers:
        w.ic_fold()
    metrics = _finalize(rt, workers, wall)
    for w in workers:
        w.release_all()
    _unpin(engine, pinned_here)
    metrics.phases = {"plan_s": _t_plan, "setup_s": t_setup, "drive_s": wall,
                      "finalize_s": time.perf_counter() - t_fin0}
    return RunResult(metrics, sorted(rt.trace, key=lambda e: (e.time_start, e.device, e.time_end)),
                     {w.device_id: w.tasks_done for w in workers}, plan)


def _snapshot_alias_safe(plan, options, topology, devs, resident, caps, per_tile) -> bool:
    """TRMM reads its in-place operand through a snapshot (routines.py:393-400).  The
    snapshot may alias the live storage only if no snapshot tile can be fetched from the
    host after the task owning it has written it back.  That holds when the owner's own
    fetch (issued before its write-back) is the tile's only host fetch: every device keeps
    every tile it fetched (resident arenas, L1 on, room for the whole snapshot), and every
    other device gets the tile from a holder over L2 (L2 on, one peer group) — with one
    driver thread, so the directory sees each holder before the next lookup."""
    if options.execution != "deterministic" or not options.l1_enabled:
        return False
    if not all(resident.values()):
        return False
    if len(devs) > 1:
        if not options.l2_enabled:
            return False
        if len({topology.peer_group_of(d) for d in devs}) != 1:
            return False
    snap = plan.matrices[plan.snapshot_alias]
    snap_bytes = -(-snap.rows // plan.tile_size) * device_ld(plan.tile_size) * snap.cols * plan.dtype.itemsize
    return all(snap_bytes + 2 * WORKING_SET_TILES * per_tile <= c for c in caps.values())


def sgemm_precise_for(plan: TaskPlan, options: RunOptions) -> bool:
    """float32 calls: 3xTF32 (fp32-accurate split products) or plain TF32 inputs.
    ``sgemm_precise=None`` (auto) picks 3xTF32 when the call's reduction depth is below
    SGEMM_TF32_MIN_K: the TF32 rounding error (2^-11 per input) grows like sqrt(k) while the
    north-star bound grows like k (k * 2^-23), so plain TF32 meets the fp32 bound only for
    long reductions."""
    if options.sgemm_precise is not None:
        return bool(options.sgemm_precise)
    env = os.environ.get("BX_SGEMM_PRECISE")
    if env:
        return env != "0"
    return plan.dtype.itemsize == 4 and call_depth(plan.call) < SGEMM_TF32_MIN_K


def call_depth(call) -> int:
    """The reduction depth k of the north-star bound for a routine call."""
    a = call.a.matrix
    if call.kind in ("gemm", "syrk", "syr2k"):
        return a.rows if call.trans_a else a.cols
    return a.rows      # symm / trmm / trsm: the order of the square operand


def _unpin(engine, arrays) -> None:
    for arr in arrays:
        try:
            engine.unregister_host(arr)
        except Exception:
            pass


def _drive_single(rt: _Runtime, workers) -> None:
    eng = rt.engine
    while not rt.done():
        progressed = False
        for w in workers:
            progressed |= w.poll()
        for w in workers:
            progressed |= w.fill()
            if w._pf is not None:
                progressed |= w.prefetch_step()
        if rt.done():
            break
        if not progressed:
            evs = [e for w in workers for e in w.in_flight()]
            evs += [w._pf_events[0] for w in workers if w._pf_events and w._pf_next < len(w._pf[0])]
            if not evs:
                raise RuntimeError("runtime stalled: tasks remain but nothing is in flight")
            eng.wait_any(evs, spin_us=2000)


def _drive_threads(rt: _Runtime, workers) -> None:
    errors = []

    def drive(w):
        try:
            while not rt.done():
                p = w.poll()
                p |= w.fill()
                if not p:
                    evs = w.in_flight()
                    if evs:
                        rt.engine.wait_any(evs, spin_us=500)
                    else:
                        time.sleep(1e-4)
        except BaseException as exc:  # surfaced on the caller's thread
            errors.append(exc)
            with rt._lock:
                rt._done = rt.total

    threads = [threading.Thread(target=drive, args=(w,), daemon=True) for w in workers]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]


def _finalize(rt: _Runtime, workers, wall: float) -> Metrics:
    eng = rt.engine
    m = Metrics(total_flops=rt.plan.total_flops)
    span = 0.0
    for w in workers:
        end = eng.record(w.slot, LANE_D2H, timing=True)
        eng.sync(end)
        # every task ends with an in-order D2H on this lane, so `end` marks the last one
        elapsed = eng.elapsed_ms(w.epoch, end) / 1e3 if w.tasks_done else 0.0
        eng.release(end)
        dm = w.dm
        if rt.options.record_trace:
            kern, xfer = [], []
            for (kind, lane, e0, e1, amount, tid, k) in w.runtime_trace:
                s = eng.elapsed_ms(w.epoch, e0) / 1e3
                e = eng.elapsed_ms(w.epoch, e1) / 1e3
                rt.trace.append(TraceEvent(s, e, w.device_id, lane, kind, amount, tid, k))
                (kern if kind == "KERNEL" else xfer).append((s, e))
                eng.release(e0)
                eng.release(e1)
            dm.compt_seconds = sum(e - s for s, e in kern)
            dm.comm_unoverlapped_seconds = exposed_comm_time(xfer, kern)
            dm.other_seconds = max(0.0, elapsed - dm.compt_seconds - dm.comm_unoverlapped_seconds)
        else:
            dm.other_seconds = elapsed
        eng.release(w.epoch)
        m.l1_hits += w.l1_hits
        m.l2_hits += w.l2_hits
        m.host_fetches += w.host_fetches
        span = max(span, elapsed)
    m.makespan_seconds = span if span > 0 else wall
    m.wall_seconds = wall
    m.devices = dict(rt.device_metrics)
    return m


def run_call(call: RoutineCall, topology: Optional[Topology] = None,
             options: Optional[RunOptions] = None, engine=None) -> RunResult:
    """Plan and execute one routine call; on return the host output holds the result."""
    t0 = time.perf_counter()
    plan = generate_tasks(call, snapshot="alias")
    return run_plan(plan, topology, options, engine, _t_plan=time.perf_counter() - t0)
