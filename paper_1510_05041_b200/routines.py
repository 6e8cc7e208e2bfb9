"""Routine calls and their tile-task plans (the BLASX task DAG builder).

Semantics follow the reference planner step for step
(/root/reference/pkg/src/tileblas/routines.py:49-441) so the GPU runtime executes the
same tile steps in the same k order:

* one task per output tile C_ij (Eq. 2), numbered in Morton / Z order (routines.py:123-137);
* beta is applied exactly once, on a task's first step; later steps use beta = 1
  (routines.py:211-215); alpha multiplies every accumulation;
* transposes are flags on physical tiles (``logical_tile``), never copies;
* rank-k diagonal tasks always move C in (only the stored triangle is touched,
  routines.py:236-276);
* TRMM reads a snapshot of its input taken at plan time (routines.py:393-400);
* TRSM tasks carry dependency edges to the tasks that produce the solved tiles they
  read (routines.py:426-437); their first gemm step has beta = alpha and alpha = -1
  (routines.py:358-380).

The plan is data only; ``scheduler.run_plan`` turns each task into DMA transfers and
tile-kernel launches on the GPUs.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import NamedTuple, Optional

import numpy as np

from .errors import InvalidArgumentError
from .tiling import MatrixDesc, TiledMatrix, TileRef, logical_tile, transpose_ref

ROUTINES = ("gemm", "syrk", "syr2k", "symm", "trmm", "trsm")

GEMM_UPDATE = "gemm_update"
SYRK_UPDATE = "syrk_update"
SYR2K_UPDATE = "syr2k_update"
TRSM_SOLVE = "trsm_solve"
TRMM_DIAG = "trmm_diag"
SYMM_DIAG = "symm_diag"
KERNEL_KINDS = (GEMM_UPDATE, SYRK_UPDATE, SYR2K_UPDATE, TRSM_SOLVE, TRMM_DIAG, SYMM_DIAG)


def step_flops(kind: str, h: int, w: int, d: int) -> int:
    """Algorithmic flops of one tile step (reference kernels.py:214-231)."""
    if kind in (GEMM_UPDATE, SYMM_DIAG):
        return 2 * h * w * d
    if kind == SYRK_UPDATE:
        return h * (h + 1) * d
    if kind == SYR2K_UPDATE:
        return 2 * h * (h + 1) * d
    if kind in (TRSM_SOLVE, TRMM_DIAG):
        return d * d * (w if d == h else h)
    raise InvalidArgumentError(f"unknown kernel kind {kind!r}")


@dataclass
class RoutineCall:
    """One level-3 call.  ``c`` is the output; trmm/trsm work in place on ``c`` (b is None)."""

    kind: str
    a: TiledMatrix
    c: TiledMatrix
    b: Optional[TiledMatrix] = None
    alpha: float = 1.0
    beta: float = 0.0
    trans_a: bool = False
    trans_b: bool = False
    uplo: str = "upper"
    side: str = "left"
    diag: str = "non-unit"


class TaskStep(NamedTuple):
    k: int
    kind: str
    a: TileRef
    b: Optional[TileRef]
    alpha: float
    beta: float
    flops: int

    def input_refs(self):
        return (self.a,) if self.b is None else (self.a, self.b)


@dataclass
class Task:
    task_id: int
    i: int
    j: int
    out_ref: TileRef
    steps: tuple
    flops: int
    needs_c_move_in: bool
    deps_remaining: int = 0
    dependents: tuple = ()

    @property
    def k_lo(self) -> int:
        return self.steps[0].k

    @property
    def k_hi(self) -> int:
        return self.steps[-1].k


@dataclass
class TaskPlan:
    call: RoutineCall
    tile_size: int
    tasks: list
    matrices: dict
    total_flops: int = 0
    dtype: np.dtype = field(default_factory=lambda: np.dtype(np.float64))
    snapshot_alias: Optional[str] = None   # TRMM snapshot id when it aliases live storage

    def initially_ready(self) -> list:
        return [t for t in self.tasks if t.deps_remaining == 0]


def degree_of_parallelism(rows: int, cols: int, tile_size: int) -> int:
    """Independent output-tile tasks of a rows x cols output (Eq. 2)."""
    if rows < 1 or cols < 1 or tile_size < 1:
        raise InvalidArgumentError("rows, cols and tile_size must be >= 1")
    return -(-rows // tile_size) * -(-cols // tile_size)


def morton_key(i: int, j: int) -> int:
    """Interleave bits: j in even positions, i in odd (Z order over the tile grid)."""
    key, shift = 0, 0
    while i or j:
        key |= (j & 1) << shift | (i & 1) << (shift + 1)
        i, j, shift = i >> 1, j >> 1, shift + 2
    return key


# --------------------------------------------------------------------- validation

def _require(ok: bool, msg: str) -> None:
    if not ok:
        raise InvalidArgumentError(msg)


def _op_shape(tm: TiledMatrix, trans: bool):
    r, c = tm.matrix.rows, tm.matrix.cols
    return (c, r) if trans else (r, c)


def validate(call: RoutineCall) -> None:
    """Argument checks of the reference (routines.py:145-195), plus dtype rules."""
    _require(call.kind in ROUTINES, f"unknown routine {call.kind!r}")
    _require(call.uplo in ("upper", "lower"), f"bad uplo {call.uplo!r}")
    _require(call.side in ("left", "right"), f"bad side {call.side!r}")
    _require(call.diag in ("unit", "non-unit"), f"bad diag {call.diag!r}")
    if call.kind != "gemm":
        _require(not call.trans_b, f"{call.kind} has a single transpose switch; "
                                   f"trans_b does not apply")
    if call.kind == "symm":
        _require(not call.trans_a, "symm does not take a transpose")
    ops = [x for x in (call.a, call.c, call.b) if x is not None]
    t = call.c.tile_size
    seen = set()
    for tm in ops:
        _require(tm.tile_size == t, "operands tiled with different tile sizes")
        _require(tm.matrix_id not in seen, f"operands alias matrix {tm.matrix_id!r}")
        seen.add(tm.matrix_id)
    dts = {tm.matrix.storage.dtype for tm in ops}
    _require(len(dts) == 1, "operands mix float32 and float64")
    if np.dtype(np.float32) in dts:
        _require(call.kind == "gemm", "float32 operands are supported for gemm (sgemm) only")
    m, n = call.c.matrix.rows, call.c.matrix.cols
    ar, ac = call.a.matrix.rows, call.a.matrix.cols
    if call.kind == "gemm":
        _require(call.b is not None, "gemm needs a b operand")
        oa, ob = _op_shape(call.a, call.trans_a), _op_shape(call.b, call.trans_b)
        _require(oa[0] == m and ob[1] == n and oa[1] == ob[0],
                 f"gemm shapes op(a)={oa} op(b)={ob} c=({m},{n})")
    elif call.kind in ("syrk", "syr2k"):
        _require(m == n, "rank-k output must be square")
        oa = _op_shape(call.a, call.trans_a)
        _require(oa[0] == n, f"op(a) rows {oa[0]} != output order {n}")
        if call.kind == "syr2k":
            _require(call.b is not None, "syr2k needs a b operand")
            _require((call.b.matrix.rows, call.b.matrix.cols) == (ar, ac),
                     "syr2k operands a and b must have identical shape")
        else:
            _require(call.b is None, "syrk takes no b operand")
    elif call.kind == "symm":
        _require(call.b is not None, "symm needs a b operand")
        order = m if call.side == "left" else n
        _require(ar == ac == order, f"symmetric operand must be {order}x{order}, got {ar}x{ac}")
        _require((call.b.matrix.rows, call.b.matrix.cols) == (m, n),
                 "symm b operand must match the output shape")
    else:
        _require(call.b is None, f"{call.kind} takes no separate b operand")
        order = m if call.side == "left" else n
        _require(ar == ac == order, f"triangular operand must be {order}x{order}, got {ar}x{ac}")


# --------------------------------------------------------------------- planners
# Each planner yields (k, kind, a_ref, b_ref, depth) for output tile (i, j); the scalar
# policy (alpha/beta per step) is applied by ``_scalars``.

_TR_MEMO = {}


def _tr(ref: TileRef) -> TileRef:
    out = _TR_MEMO.get(ref)
    if out is None:
        if len(_TR_MEMO) > 1 << 16:
            _TR_MEMO.clear()
        out = _TR_MEMO[ref] = transpose_ref(ref)
    return out


def _k_tiles(tm: TiledMatrix, trans: bool) -> int:
    return tm.tile_rows if trans else tm.tile_cols


def _gemm_steps(call, i, j, _snap, lt):
    for k in range(_k_tiles(call.a, call.trans_a)):
        a = lt(call.a, i, k, call.trans_a)
        yield k, GEMM_UPDATE, a, lt(call.b, k, j, call.trans_b), a.width


def _syrk_steps(call, i, j, _snap, lt):
    ta = call.trans_a
    for k in range(_k_tiles(call.a, ta)):
        a = lt(call.a, i, k, ta)
        if i == j:
            yield k, SYRK_UPDATE, a, None, a.width
        else:
            yield k, GEMM_UPDATE, a, _tr(lt(call.a, j, k, ta)), a.width


def _syr2k_steps(call, i, j, _snap, lt):
    ta = call.trans_a
    for k in range(_k_tiles(call.a, ta)):
        a = lt(call.a, i, k, ta)
        b = lt(call.b, i, k, ta)
        if i == j:
            yield k, SYR2K_UPDATE, a, b, a.width
        else:
            yield k, GEMM_UPDATE, a, _tr(lt(call.b, j, k, ta)), a.width
            yield k, GEMM_UPDATE, b, _tr(lt(call.a, j, k, ta)), b.width


def _sym_tile(call, r, c, lt) -> TileRef:
    """Tile (r, c) of the symmetric extension of the stored triangle (routines.py:279-284)."""
    in_stored = c > r if call.uplo == "upper" else c < r
    if in_stored:
        return lt(call.a, r, c, False)
    return _tr(lt(call.a, c, r, False))


def _symm_steps(call, i, j, _snap, lt):
    left = call.side == "left"
    for k in range(call.a.tile_rows):
        if left:
            b = lt(call.b, k, j, False)
            if k == i:
                d = lt(call.a, i, i, False)
                yield k, SYMM_DIAG, d, b, d.height
            else:
                a = _sym_tile(call, i, k, lt)
                yield k, GEMM_UPDATE, a, b, a.width
        else:
            a = lt(call.b, i, k, False)
            if k == j:
                d = lt(call.a, j, j, False)
                yield k, SYMM_DIAG, d, a, d.height
            else:
                yield k, GEMM_UPDATE, a, _sym_tile(call, k, j, lt), a.width


def _eff_upper(call) -> bool:
    return (call.uplo == "upper") != call.trans_a


def _trmm_steps(call, i, j, snap, lt):
    nt = call.a.tile_rows
    if call.side == "left":
        diag_k = i
        ks = range(i, nt) if _eff_upper(call) else range(i + 1)
    else:
        diag_k = j
        ks = range(j + 1) if _eff_upper(call) else range(j, nt)
    for k in ks:
        if k == diag_k:
            d = lt(call.a, k, k, False)
            yield k, TRMM_DIAG, d, lt(snap, i, j, False), d.height
        elif call.side == "left":
            a = lt(call.a, i, k, call.trans_a)
            yield k, GEMM_UPDATE, a, lt(snap, k, j, False), a.width
        else:
            s = lt(snap, i, k, False)
            yield k, GEMM_UPDATE, s, lt(call.a, k, j, call.trans_a), s.width


def trsm_producers(call, i: int, j: int) -> range:
    """k indices of the solved tiles task (i, j) consumes (routines.py:350-356)."""
    nt = call.a.tile_rows
    if call.side == "left":
        return range(i + 1, nt) if _eff_upper(call) else range(i)
    return range(j) if _eff_upper(call) else range(j + 1, nt)


def _trsm_steps(call, i, j, _snap, lt):
    for k in trsm_producers(call, i, j):
        if call.side == "left":
            a = lt(call.a, i, k, call.trans_a)
            yield k, GEMM_UPDATE, a, lt(call.c, k, j, False), a.width
        else:
            x = lt(call.c, i, k, False)
            yield k, GEMM_UPDATE, x, lt(call.a, k, j, call.trans_a), x.width
    dk = i if call.side == "left" else j
    d = lt(call.a, dk, dk, False)
    yield dk, TRSM_SOLVE, d, None, d.height


_PLANNERS = dict(gemm=_gemm_steps, syrk=_syrk_steps, syr2k=_syr2k_steps, symm=_symm_steps,
                 trmm=_trmm_steps, trsm=_trsm_steps)


def _scalars(call, index: int, kind: str, n_gemm_before: int):
    """(alpha, beta) of the index-th step of a task."""
    if call.kind == "trmm":
        return call.alpha, (0.0 if index == 0 else 1.0)
    if call.kind == "trsm":
        if kind == TRSM_SOLVE:
            return (call.alpha if n_gemm_before == 0 else 1.0), 1.0
        return -1.0, (call.alpha if index == 0 else 1.0)
    return call.alpha, (call.beta if index == 0 else 1.0)


def _needs_c(call, i, j) -> bool:
    if call.kind == "trmm":
        return False
    if call.kind == "trsm":
        return True
    if call.kind in ("syrk", "syr2k"):
        return call.beta != 0.0 or i == j
    return call.beta != 0.0


def _output_pairs(call):
    mt, nt = call.c.tile_rows, call.c.tile_cols
    if call.kind in ("syrk", "syr2k"):
        if call.uplo == "upper":
            return [(i, j) for i in range(mt) for j in range(i, nt)]
        return [(i, j) for i in range(mt) for j in range(i + 1)]
    return [(i, j) for i in range(mt) for j in range(nt)]


_PLAN_CACHE = {}
_PLAN_CACHE_MAX = 8


def _structure_key(call: RoutineCall) -> tuple:
    """Everything a plan's task structure depends on (shapes, tiling, flags, scalars and
    matrix ids) — but not the operand values or storage."""
    def shape(tm):
        return None if tm is None else (tm.matrix_id, tm.matrix.rows, tm.matrix.cols)
    return (call.kind, shape(call.a), shape(call.b), shape(call.c), call.c.tile_size,
            call.alpha, call.beta, call.trans_a, call.trans_b, call.uplo, call.side, call.diag,
            str(call.c.matrix.storage.dtype))


def generate_tasks(call: RoutineCall, cache: bool = True, snapshot: str = "copy") -> TaskPlan:
    """Expand a call into its task plan (reference routines.py:383-441).

    The task structure is a pure function of shapes / flags / scalars, so it is memoised
    (``cache``): a repeated call of the same shape rebinds the cached tasks to the new
    operand storage instead of re-planning.

    TRMM reads a snapshot of its in-place operand.  ``snapshot="copy"`` takes a host copy
    (the reference, routines.py:393-400); ``"alias"`` lets the snapshot descriptor share
    the live storage — valid only for an executor that fetches every snapshot tile before
    the task owning that tile writes it back and never re-fetches it afterwards (the GPU
    runtime pins snapshot tiles on device for the whole call, see scheduler.py)."""
    validate(call)
    t = call.c.tile_size
    matrices = {tm.matrix_id: tm.matrix for tm in (call.a, call.c, call.b) if tm is not None}
    snap = None
    if call.kind == "trmm":
        src = call.c.matrix
        if snapshot not in ("copy", "alias"):
            raise InvalidArgumentError(f"bad snapshot mode {snapshot!r}")
        sd = MatrixDesc(src.matrix_id + ".snapshot", src.rows, src.cols, src.leading_dim,
                        src.storage.copy() if snapshot == "copy" else src.storage,
                        src.base_offset)
        snap = TiledMatrix(sd, t, call.c.tile_rows, call.c.tile_cols)
        matrices[sd.matrix_id] = sd
    skey = _structure_key(call) if cache else None
    hit = _PLAN_CACHE.get(skey) if cache else None
    if hit is not None:
        tasks, total = hit
        plan = TaskPlan(call, t, tasks, matrices, total, call.c.matrix.storage.dtype)
        plan.snapshot_alias = snap.matrix_id if (snap is not None and snapshot == "alias") else None
        return plan
    planner = _PLANNERS[call.kind]
    memo = {}

    def lt(tm, i, j, trans=False):
        # every input tile is referenced by many tasks: build each TileRef once per plan
        key = (tm.matrix_id, i, j, trans)
        ref = memo.get(key)
        if ref is None:
            ref = memo[key] = logical_tile(tm, i, j, trans)
        return ref
    pairs = sorted(_output_pairs(call), key=lambda p: morton_key(*p))
    tasks = []
    for tid, (i, j) in enumerate(pairs):
        out = logical_tile(call.c, i, j, False)
        steps = []
        n_gemm = 0
        for idx, (k, kind, a, b, d) in enumerate(planner(call, i, j, snap, lt)):
            alpha, beta = _scalars(call, idx, kind, n_gemm)
            n_gemm += kind == GEMM_UPDATE
            steps.append(TaskStep(k, kind, a, b, alpha, beta,
                                  step_flops(kind, out.height, out.width, d)))
        tasks.append(Task(tid, i, j, out, tuple(steps), sum(s.flops for s in steps),
                          _needs_c(call, i, j)))
    if call.kind == "trsm":
        by_coord = {(x.i, x.j): x for x in tasks}
        deps = {x.task_id: [] for x in tasks}
        for x in tasks:
            ks = trsm_producers(call, x.i, x.j)
            x.deps_remaining = len(ks)
            for k in ks:
                prod = by_coord[(k, x.j) if call.side == "left" else (x.i, k)]
                deps[prod.task_id].append(x.task_id)
        for x in tasks:
            x.dependents = tuple(sorted(deps[x.task_id]))
    total = sum(x.flops for x in tasks)
    if cache:
        if len(_PLAN_CACHE) >= _PLAN_CACHE_MAX:
            _PLAN_CACHE.pop(next(iter(_PLAN_CACHE)))
        _PLAN_CACHE[skey] = (tasks, total)
    plan = TaskPlan(call, t, tasks, matrices, total, call.c.matrix.storage.dtype)
    plan.snapshot_alias = snap.matrix_id if (snap is not None and snapshot == "alias") else None
    return plan


def gemm_flop_fraction(plan: TaskPlan) -> float:
    """Share of the plan's flops in plain gemm accumulation steps (Table I)."""
    total = sum(s.flops for t in plan.tasks for s in t.steps)
    gemm = sum(s.flops for t in plan.tasks for s in t.steps if s.kind == GEMM_UPDATE)
    return gemm / total if total else 0.0
