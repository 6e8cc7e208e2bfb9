"""Compile a planner Task into the launch program the GPU runtime issues.

Data only (no device state): consecutive tile steps that share a kernel configuration
are fused into one GEMM launch of up to ``chunk_steps`` sub-steps (accumulators stay in
registers across them); rank-k diagonal steps become triangle-epilogue GEMMs; SYRK
diagonal steps pair a tile with its own transpose, SYR2K diagonal steps expand into the
two products alpha(A B^T + B A^T) (kernels.py:67-102); TRMM / SYMM diagonal steps first
materialise op(tri(A)) / sym(A) into a scratch tile (kernels.py:164-211); TRSM ends with
the triangular solve (kernels.py:105-161).  Programs depend only on the task structure,
so they are cached on the (immutable) Task.
"""

from __future__ import annotations

from typing import NamedTuple

from .routines import (GEMM_UPDATE, SYMM_DIAG, SYR2K_UPDATE, SYRK_UPDATE, TRMM_DIAG,
                       TRSM_SOLVE, Task)


class GemmOp(NamedTuple):
    ta: bool
    tb: bool
    tri: int             # 0 full, 1 lower, 2 upper
    alpha: float
    beta: float
    subs: tuple          # ((a_key, b_key, depth, kmode), ...); kmode: triangular operand
                         # (KM_* below) whose zero half the kernel's CTAs skip
    k: int
    flops: int
    keys: frozenset = frozenset()   # the input tiles the launch reads (scratch excluded)


KM_NONE, KM_A_LOWER, KM_A_UPPER, KM_B_UPPER, KM_B_LOWER = 0, 1, 2, 3, 4


class MatOp(NamedTuple):
    sym: bool
    key: tuple           # diagonal tile key
    n: int
    scratch: int         # scratch slot index


class TrsmOp(NamedTuple):
    key: tuple
    alpha: float
    k: int
    flops: int


class AxpyOp(NamedTuple):
    beta: float          # C += beta * C0 (C0 = the output tile's host values, fetched late)


class Program(NamedTuple):
    ops: tuple
    scratch_n: tuple     # order of each scratch tile
    defer_c: bool = False  # C move-in deferred to a final AxpyOp (first GEMM runs beta=0)


def scratch_key(i: int) -> tuple:
    return ("#scratch", i)


def compile_task(task: Task, call, chunk_steps: int, first_chunk: int = 0,
                 defer_c: bool = False, split_chain: bool = False,
                 split_km: bool = False) -> Program:
    """``first_chunk`` (if > 0) caps the task's first GEMM launch so its kernel can start
    as soon as the first few input tiles have landed (pipeline ramp-up).

    ``defer_c``: for a task whose C tile must be moved in only for the beta*C term (plain
    GEMM updates, no triangle epilogue, no solve), the first GEMM launch runs with beta = 0
    (C is not read, kernels.py:40-41) and a final AxpyOp adds beta*C0 from a separately
    fetched copy — beta is still applied exactly once (routines.py:211-215), but the
    task's kernels no longer wait for the C tile's host copy.

    ``split_chain`` (TRSM): when the task's last update step reads the tile its chain
    predecessor solves (k adjacent to the diagonal: left/lower and right/upper, whose
    updates run towards the diagonal, routines.py:347-375), that step gets a launch of its
    own.  The earlier updates read tiles solved long before, so their launch can start
    while the predecessor's solve is still running; only the one-step launch and the solve
    wait for it.  Same steps, same order, same beta: the numerics are unchanged.

    ``split_km``: a triangular-operand step (TRMM diagonal) never shares a launch with
    plain steps, so the plain steps run the kernel instantiation without per-step k-range
    bookkeeping (bx_gemm_dmma.cuh KM template) — same steps and order."""
    ckey = (chunk_steps, first_chunk, defer_c, split_chain, split_km)
    cache = getattr(task, "_bx_prog", None)
    if cache is not None and cache[0] == ckey:
        return cache[1]
    h, w = task.out_ref.phys_height, task.out_ref.phys_width
    tri = 1 if call.uplo == "lower" else 2
    ops = []
    scratch = []
    cur = None          # [ta, tb, tri, alpha, beta, subs, k]

    def flush():
        nonlocal cur
        if cur is not None:
            subs = tuple(cur[5])
            ops.append(GemmOp(cur[0], cur[1], cur[2], cur[3], cur[4], subs, cur[6],
                              sum(2 * h * w * d for _, _, d, _ in subs),
                              frozenset(k for ak, bk, _, _ in subs for k in (ak, bk)
                                        if k[0] != "#scratch")))
            cur = None

    def add(ta, tb, tr, alpha, beta, a, b, d, k, km=KM_NONE):
        nonlocal cur
        cap = chunk_steps
        if first_chunk and not any(type(o) is GemmOp for o in ops):
            cap = min(first_chunk, chunk_steps)
        if (cur is None or (cur[0], cur[1], cur[2], cur[3]) != (ta, tb, tr, alpha)
                or beta != 1.0 or len(cur[5]) >= cap
                or (split_km and (km != KM_NONE) != (cur[5][-1][3] != KM_NONE))):
            flush()
            cur = [ta, tb, tr, alpha, beta, [], k]
        cur[5].append((a, b, d, km))

    split_at = -1
    if split_chain and len(task.steps) >= 3 and task.steps[-1].kind == TRSM_SOLVE:
        last = task.steps[-2]
        if last.kind == GEMM_UPDATE and abs(last.k - task.steps[-1].k) == 1:
            split_at = len(task.steps) - 2
    for si, st in enumerate(task.steps):
        kind = st.kind
        if si == split_at:
            flush()
        if kind == GEMM_UPDATE:
            add(st.a.transposed, st.b.transposed, 0, st.alpha, st.beta, st.a.key(), st.b.key(),
                st.a.width, st.k)
        elif kind == SYRK_UPDATE:
            ka = st.a.key()
            add(st.a.transposed, not st.a.transposed, tri, st.alpha, st.beta, ka, ka,
                st.a.width, st.k)
        elif kind == SYR2K_UPDATE:
            ka, kb = st.a.key(), st.b.key()
            add(st.a.transposed, not st.b.transposed, tri, st.alpha, st.beta, ka, kb,
                st.a.width, st.k)
            add(st.b.transposed, not st.a.transposed, tri, st.alpha, 1.0, kb, ka,
                st.a.width, st.k)
        elif kind in (TRMM_DIAG, SYMM_DIAG):
            n = st.a.phys_height
            idx = len(scratch)
            scratch.append(n)
            ops.append(MatOp(kind == SYMM_DIAG, st.a.key(), n, idx))
            sk = scratch_key(idx)
            # op(tri(A)) is triangular (zeros materialised): the kernel skips its zero half
            eff_upper = (call.uplo == "upper") != call.trans_a
            tri_op = kind == TRMM_DIAG
            if call.side == "left":
                km = (KM_A_UPPER if eff_upper else KM_A_LOWER) if tri_op else KM_NONE
                add(False, st.b.transposed, 0, st.alpha, st.beta, sk, st.b.key(), n, st.k, km)
            else:
                km = (KM_B_UPPER if eff_upper else KM_B_LOWER) if tri_op else KM_NONE
                add(st.b.transposed, False, 0, st.alpha, st.beta, st.b.key(), sk, n, st.k, km)
        elif kind == TRSM_SOLVE:
            flush()
            ops.append(TrsmOp(st.a.key(), st.alpha, st.k, st.flops))
        else:
            raise ValueError(f"unknown step kind {kind!r}")
    flush()
    deferred = False
    if defer_c and task.needs_c_move_in:
        gemms = [i for i, o in enumerate(ops) if type(o) is GemmOp]
        if (gemms and all(type(o) is not TrsmOp for o in ops)
                and all(ops[i].tri == 0 for i in gemms) and ops[gemms[0]].beta != 0.0):
            g = ops[gemms[0]]
            ops[gemms[0]] = g._replace(beta=0.0)
            ops.append(AxpyOp(g.beta))
            deferred = True
    prog = Program(tuple(ops), tuple(scratch), deferred)
    task._bx_prog = (ckey, prog)
    return prog
