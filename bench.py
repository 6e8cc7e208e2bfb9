#!/usr/bin/env python
"""Benchmark: host-resident tiled level-3 BLAS on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config cfg2|cfg1|dgemm32768|cfg3_syrk|cfg3_syr2k|cfg4_trsm|cfg4_trmm|cfg5_sgemm]

Prints ONE JSON line (rank 0).  A "step" is one routine call over the config's seeded
host-resident operands (BASELINE.json: "host-resident operands").  Legs:
  value     ``run_call`` (the reference's API, scheduler.py:665-669) on the host buffers:
            every step plans, loads tiles over the host link (H2D), computes on the FP64
            tensor cores, writes C back (D2H); timed on the device with CUDA events, max over
            ranks; whole-job TFLOP/s (plan.total_flops / time);
  e2e       the cblas-style public API (``dgemm``/``dsyrk``/... on the caller's column-major
            buffers, blas.py) timed by the host clock around the call, max over ranks, with
            the H2D/D2H bytes each step moved;
  roofline  the dominant kernel (the FP64 DMMA task GEMM; tcgen05 TF32 for SGEMM) timed
            alone on device-resident operands of the config's shape, vs the FP64 DMMA peak
            measured live (MEASURED_PEAKS.json has no FP64 entry); plus the north-star
            roofline max(t_tensor, t_link) of the value leg with the host-link / NVLink
            bandwidths measured in this run with all N GPUs active (``links``);
  parity    the output of the last timed e2e step checked against the sampled-block oracle
            (oracle/sampled.py; test infrastructure used as the checker only) with the
            north-star bound restricted to each block;
  cpu_baseline  the oracle port of the reference's tiled runtime (numpy + OpenBLAS, all
            host cores) on sampled output blocks of the same routine and operands.
``--gpus N``: one process per GPU (spmd.py: shared task queue, stations with stealing, L2
tile cache over peer HBM through CUDA IPC, no collectives) — under torchrun every rank runs
this file; without torchrun the script launches the N ranks itself.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

# torchrun exports OMP_NUM_THREADS=1 to every rank; the CPU baseline / reference arm should
# use all host cores (OpenBLAS reads OPENBLAS_NUM_THREADS before OMP_NUM_THREADS at import)
if "OPENBLAS_NUM_THREADS" not in os.environ:
    os.environ["OPENBLAS_NUM_THREADS"] = str(os.cpu_count() or 1)

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "cfg1": dict(kind="gemm", m=2048, n=2048, k=2048, tile=512, alpha=1.0, beta=1.0,
                 desc="DGEMM 2048x2048x2048 NN, tile 512, alpha=1 beta=1 (BASELINE configs[0])"),
    "cfg2": dict(kind="gemm", m=16384, n=16384, k=16384, tile=1024, alpha=1.0, beta=1.0,
                 desc="DGEMM 16384^3 NN host-resident, tile 1024, alpha=1 beta=1 (BASELINE configs[1])"),
    "dgemm32768": dict(kind="gemm", m=32768, n=32768, k=32768, tile=1024, alpha=1.0, beta=1.0,
                       desc="DGEMM 32768^3 NN host-resident, tile 1024 (north-star target)"),
    "cfg3_syrk": dict(kind="syrk", m=16384, n=16384, k=8192, tile=1024, alpha=1.0, beta=1.0,
                      uplo="lower", desc="DSYRK N=16384 K=8192 lower, tile 1024 (configs[2])"),
    "cfg3_syr2k": dict(kind="syr2k", m=16384, n=16384, k=8192, tile=1024, alpha=1.0, beta=1.0,
                       uplo="lower", desc="DSYR2K N=16384 K=8192 lower, tile 1024 (configs[2])"),
    "cfg4_trsm": dict(kind="trsm", m=16384, n=16384, k=16384, tile=1024, alpha=1.0, beta=0.0,
                      uplo="lower", desc="DTRSM left/lower/notrans 16384, tile 1024 (configs[3])"),
    "cfg4_trmm": dict(kind="trmm", m=16384, n=16384, k=16384, tile=1024, alpha=1.0, beta=0.0,
                      uplo="lower", desc="DTRMM left/lower/notrans 16384, tile 1024 (configs[3])"),
    "cfg5_sgemm": dict(kind="gemm", m=32768, n=32768, k=32768, tile=2048, alpha=1.0, beta=1.0,
                       dtype="f32", sweep=(512, 1024, 2048, 4096),
                       desc="SGEMM 32768^3 NN host-resident on tcgen05 (TF32), tile 2048 + tile sweep "
                            "512-4096 (BASELINE configs[4])"),
}
METRIC = "DGEMM TFLOP/s at 1/2/4/8 B200 (host-resident operands), % of FP64 peak"
METRIC_F32 = "SGEMM TFLOP/s (host-resident operands, tcgen05 kind::tf32), % of TF32 tensor peak"
PARITY_BLOCKS = {"gemm": 16, "syrk": 16, "syr2k": 16, "trsm": 2, "trmm": 2}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", ",".join(str(g) for g in self.gpus)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                clk, cmax = float(f[1]), float(f[2])
            except ValueError:
                continue
            mx.append(cmax)
            if clk > 0.5 * cmax:   # under load
                sm.append(clk)
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.lines)}


# ----------------------------------------------------------------------------- helpers

def make_operands(cfg, seed=0, tile=None):
    from paper_1510_05041_b200.operands import build_call
    kw = {}
    if "uplo" in cfg:
        kw["uplo"] = cfg["uplo"]
    if cfg.get("dtype") == "f32":
        kw["dtype"] = np.float32
    return build_call(cfg["kind"], m=cfg["m"], n=cfg["n"], k=cfg["k"], tile_size=tile or cfg["tile"],
                      seed=seed, alpha=cfg["alpha"], beta=cfg["beta"],
                      trsm_scaled=cfg["kind"] in ("trsm", "trmm"), **kw)


def retile(call, tile):
    """Same operands, another tile size."""
    from paper_1510_05041_b200 import RoutineCall
    from paper_1510_05041_b200.tiling import make_tiled
    return RoutineCall(call.kind, a=make_tiled(call.a.matrix, tile),
                       b=None if call.b is None else make_tiled(call.b.matrix, tile),
                       c=make_tiled(call.c.matrix, tile), alpha=call.alpha, beta=call.beta,
                       trans_a=call.trans_a, trans_b=call.trans_b, uplo=call.uplo, side=call.side,
                       diag=call.diag)


def tf32_peak_tflops():
    """tcgen05 kind::tf32 issues at half the kind::f16 rate: use half of the driver-measured
    dense bf16 peak (MEASURED_PEAKS.json), else half of the profiling guide's fallback."""
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return mp["bf16_tflops"] / 2.0, "MEASURED_PEAKS.json bf16_tflops / 2 (kind::tf32 = half the f16 rate)"
    except (OSError, ValueError, KeyError):
        return 1590.0 / 2.0, "fallback 1.59 PF bf16 / 2 (B200_PROFILING.md)"


def tf32_sustained_tflops():
    """Half of MEASURED_PEAKS.json's sustained (back-to-back, power-capped) bf16 rate, or None."""
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return mp["bf16_tflops_sustained"] / 2.0
    except (OSError, ValueError, KeyError):
        return None


def config_dict(cfg, args):
    """The ``config`` object — identical for both arms (same routine, shape and scalars)."""
    return {"workload": cfg["desc"], "routine": cfg["kind"], "m": cfg["m"], "n": cfg["n"],
            "k": cfg["k"], "tile": cfg["tile"], "alpha": cfg["alpha"], "beta": cfg["beta"],
            **({"uplo": cfg["uplo"]} if "uplo" in cfg else {}),
            "dtype": "f32" if cfg.get("dtype") == "f32" else "f64",
            "operands": "host-resident, column-major, seeded uniform[-1,1) (reference build_call)",
            "l2_flush": "none needed: every step streams > 2 GiB of operands through a 126 MB L2"}


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))


def block_flops(kind, blk, cfg):
    """Algorithmic flops of one sampled output block (plan.total_flops restricted)."""
    t, k, m, n = cfg["tile"], cfg["k"], cfg["m"], cfg["n"]
    if kind in ("trsm", "trmm"):
        if blk[0] == "col":       # side left: an m x w strip against the m x m triangle
            return float(m) * m * min(t, n - blk[1] * t)
        return float(n) * n * min(t, m - blk[1] * t)
    i, j = blk
    h, w = min(t, m - i * t), min(t, n - j * t)
    if kind == "gemm":
        return 2.0 * h * w * k
    mult = 2.0 if kind == "syr2k" else 1.0
    return mult * (h * (h + 1) * k if i == j else 2.0 * h * w * k)


def cpu_sample(cfg, call, target_s=12.0, seed=1):
    """The oracle port of the reference tiled runtime (oracle/sampled.py: the same step
    sequences as routines.py:227-380 run with the kernels.py numerics, execute_task_on_host
    routines.py:482-492) on random output blocks of this routine and these operands, all
    host threads (OpenBLAS), for about ``target_s`` seconds."""
    from oracle import sampled
    try:   # all host threads, whatever the launcher exported
        from threadpoolctl import threadpool_limits
        threadpool_limits(os.cpu_count(), user_api="blas")
    except Exception:
        pass
    kind = cfg["kind"]
    every = sampled.call_blocks(call, 10 ** 6, seed=seed)
    rng = np.random.default_rng(seed)
    a = call.a.matrix.as_2d()
    b = call.b.matrix.as_2d() if call.b is not None else None
    c = call.c.matrix.as_2d()

    def one(blk):
        c0 = sampled.snapshot_blocks(c, [blk], cfg["tile"])[blk]
        sampled.compute_block(kind, a, b, c0, blk, tile=cfg["tile"], alpha=cfg["alpha"],
                              beta=cfg["beta"], uplo=cfg.get("uplo", "upper"))
    one(every[0])     # warm-up (OpenBLAS thread start)
    t0 = time.perf_counter()
    flops, done = 0.0, 0
    while time.perf_counter() - t0 < target_s or done == 0:
        blk = every[int(rng.integers(0, len(every)))]
        one(blk)
        flops += block_flops(kind, blk, cfg)
        done += 1
    dt = time.perf_counter() - t0
    unit_name = "tile columns" if kind in ("trsm", "trmm") else f"{cfg['tile']}x{cfg['tile']} output tiles"
    return dict(value=flops / dt / 1e12, unit="TFLOP/s", cores=os.cpu_count(), kind="port",
                seconds=dt,
                sample=f"{done} random {unit_name} of {cfg['desc']} ({flops / 1e9:.0f} GFLOP) "
                       f"with the reference's step sequence, oracle/sampled.py (numpy + OpenBLAS, "
                       f"{os.cpu_count()} threads)")


def api_call(call, options=None, topology=None):
    """The cblas-style public entry point (blas.py) over the call's column-major buffers."""
    from paper_1510_05041_b200 import blas
    a, c = call.a.matrix, call.c.matrix
    t = call.c.tile_size
    kw = dict(tile_size=t, options=options, topology=topology)
    tr = "T" if call.trans_a else "N"
    up = "U" if call.uplo == "upper" else "L"
    if call.kind == "gemm":
        b = call.b.matrix
        m, n = c.rows, c.cols
        k = a.rows if call.trans_a else a.cols
        fn = blas.sgemm if c.storage.dtype == np.float32 else blas.dgemm
        return fn(tr, "T" if call.trans_b else "N", m, n, k, call.alpha, a.storage, a.leading_dim,
                  b.storage, b.leading_dim, call.beta, c.storage, c.leading_dim, **kw)
    if call.kind == "syrk":
        k = a.rows if call.trans_a else a.cols
        return blas.dsyrk(up, tr, c.rows, k, call.alpha, a.storage, a.leading_dim, call.beta,
                          c.storage, c.leading_dim, **kw)
    if call.kind == "syr2k":
        b = call.b.matrix
        k = a.rows if call.trans_a else a.cols
        return blas.dsyr2k(up, tr, c.rows, k, call.alpha, a.storage, a.leading_dim, b.storage,
                           b.leading_dim, call.beta, c.storage, c.leading_dim, **kw)
    fn = blas.dtrsm if call.kind == "trsm" else blas.dtrmm
    return fn("L" if call.side == "left" else "R", up, tr, "U" if call.diag == "unit" else "N",
              c.rows, c.cols, call.alpha, a.storage, a.leading_dim, c.storage, c.leading_dim, **kw)


def parity_check(call, c0_blocks):
    """North-star bound on the sampled blocks of the last timed step (oracle/sampled.py)."""
    from oracle import sampled, tolerance
    t0 = time.perf_counter()
    worst, per = sampled.call_check(call, c0_blocks)
    eps = float(np.finfo(call.c.matrix.storage.dtype).eps)
    return {"max_ratio": worst, "bound": tolerance.BOUND, "pass": bool(worst <= tolerance.BOUND),
            "blocks": len(per),
            "block_kind": "tile columns (independent sub-problems)" if call.kind in ("trsm", "trmm")
            else f"{call.c.tile_size}x{call.c.tile_size} output tiles",
            "eps": eps, "checked": "output of the last timed e2e step vs oracle/sampled.py "
                                   "(reference step sequence), bound restricted to each block",
            "seconds": time.perf_counter() - t0}


# ----------------------------------------------------------------------------- reference arm

def run_reference(args, cfg):
    """The reference's CPU path (oracle port of its tiled runtime, all host cores) on the
    same routine, operands and scalars; each step is a bounded sample of the workload."""
    call = make_operands(cfg, seed=0)
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_sample(cfg, call, target_s=args.ref_seconds, seed=1 + i)
        if i >= args.warmup:
            vals.append(r)
    v = statistics.median([r["value"] for r in vals])
    sec = statistics.median([r["seconds"] for r in vals])
    return {"metric": METRIC_F32 if cfg.get("dtype") == "f32" else METRIC, "value": v,
            "unit": "TFLOP/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32" if cfg.get("dtype") == "f32" else "f64",
            "data": "synthetic (seeded uniform[-1,1), reference build_call generator)",
            "config": config_dict(cfg, args),
            "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": vals[0]["cores"],
                             "kind": "port", "sample": vals[0]["sample"]},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ----------------------------------------------------------------------------- kernel leg

def kernel_shape(cfg):
    """(m, n, k) of the device-resident launch of the dominant kernel: the config's own GEMM
    shape; for the rank-k / triangular routines the GEMM their tasks are made of."""
    if cfg["kind"] in ("syrk", "syr2k"):
        return cfg["n"], cfg["n"], cfg["k"]
    if cfg["kind"] in ("trsm", "trmm"):
        return cfg["m"], cfg["n"], cfg["m"]
    return cfg["m"], cfg["n"], cfg["k"]


def kernel_leg(args, cfg, eng, lib, slot, cols, seed, sync_all=None):
    """The dominant kernel alone: one device-resident launch per step over this GPU's column
    panel, timed with CUDA events on the launching stream (compute lane 0)."""
    from paper_1510_05041_b200 import _native as NN
    m, _, k = kernel_shape(cfg)
    f32 = cfg.get("dtype") == "f32"
    esz = 4 if f32 else 8
    ptrs = []
    for i, nelem in enumerate((m * k, k * cols, m * cols)):
        p = C.c_uint64()
        NN.check(lib.bx_dev_alloc(slot, nelem * esz, C.byref(p)), "alloc")
        fill = lib.bx_dev_fill_uniform_f32 if f32 else lib.bx_dev_fill_uniform
        NN.check(fill(slot, p.value, nelem, seed + i, 0), "fill")
        ptrs.append(p.value)
    eng.device_sync(slot)
    a, b, c = ptrs

    def launch():
        if f32:
            NN.check(lib.bx_sgemm_device(slot, 0, 0, 0, m, cols, k, 1.0, a, m, b, k, 0.0, c, m), "sgemm")
        else:
            NN.check(lib.bx_dgemm_device(slot, 0, 0, 0, m, cols, k, 1.0, a, m, b, k, 1.0, c, m), "dgemm")
    for _ in range(max(1, min(args.warmup, 3))):
        launch()
    eng.device_sync(slot)
    n0 = eng.launches()
    times = []
    for _ in range(max(1, min(args.steps, 5))):
        if sync_all:
            sync_all()
        e0 = eng.record(slot, 0, timing=True)
        launch()
        e1 = eng.record(slot, 0, timing=True)
        eng.sync(e1)
        times.append(eng.elapsed_ms(e0, e1))
        eng.release(e0)
        eng.release(e1)
    launches = eng.launches() - n0
    for p in ptrs:
        lib.bx_dev_free(slot, p)
    ms = statistics.mean(times)
    fl = 2.0 * m * cols * k
    return dict(ms=ms, flops=fl, tflops=fl / (ms / 1e3) / 1e12, launches=launches,
                shape=[m, cols, k])


# ----------------------------------------------------------------------------- links

def link_probe(eng, lib, slot, nbytes=256 << 20, reps=4, peers=None, sync_all=None):
    """Pinned host->device / device->host bandwidth of this GPU's copy lanes (one 2-d tile
    copy of ``nbytes`` into/out of the arena, the engine's own bx_h2d_tile / bx_d2h_tile),
    timed with events on the copy lane; ``sync_all`` (a cross-GPU barrier) makes every GPU
    copy at once, so the figures are per-GPU bandwidths with N GPUs active.  ``peers``:
    [(src_ptr or slot, kind)] for the peer-to-peer figure (CUDA IPC or cudaMemcpyPeer)."""
    from paper_1510_05041_b200.engine import LANE_D2H, LANE_H2D, LANE_P2P
    rows = 8192
    # small calls have small arenas: copy what fits (>= 16 MB still saturates the link)
    nbytes = min(nbytes, eng.arena_capacity(slot) // 2)
    cols = nbytes // (rows * 8)
    if cols < 256:
        return None
    nbytes = rows * cols * 8
    host = np.empty(rows * cols, dtype=np.float64)
    host[:] = 1.0
    eng.register_host(host)

    class _Desc:      # the h2d/d2h wrappers take a MatrixDesc-like source
        leading_dim = rows
        itemsize = 8

        @staticmethod
        def element_address(r, c):
            return host.ctypes.data + 8 * (r + c * rows)
    out = {}
    try:
        for name, lane in (("h2d", LANE_H2D), ("d2h", LANE_D2H)):
            ts = []
            for _ in range(reps):
                if sync_all:
                    sync_all()
                e0 = eng.record(slot, lane, timing=True)
                if name == "h2d":
                    ev = eng.h2d(slot, 0, rows, _Desc, 0, 0, rows, cols)
                else:
                    ev = eng.d2h(slot, 0, rows, _Desc, 0, 0, rows, cols)
                e1 = eng.record(slot, lane, timing=True)
                eng.sync(e1)
                ts.append(eng.elapsed_ms(e0, e1))
                for e in (ev, e0, e1):
                    eng.release(e)
            out[name + "_gbs"] = nbytes / (min(ts) / 1e3) / 1e9
        if peers:
            ts = []
            for _ in range(reps):
                if sync_all:
                    sync_all()
                e0 = eng.record(slot, LANE_P2P, timing=True)
                evs = []
                for src, kind in peers:
                    if kind == "ipc":
                        evs.append(eng.copy_remote(slot, nbytes, src, nbytes))
                    else:
                        evs.append(eng.p2p(slot, nbytes, src, 0, nbytes))
                e1 = eng.record(slot, LANE_P2P, timing=True)
                eng.sync(e1)
                ts.append(eng.elapsed_ms(e0, e1))
                for e in evs + [e0, e1]:
                    eng.release(e)
            out["p2p_in_gbs"] = len(peers) * nbytes / (min(ts) / 1e3) / 1e9
    finally:
        eng.unregister_host(host)
    out["bytes_per_copy"] = nbytes
    return out


# ----------------------------------------------------------------------------- the line

TRAFFIC_FILE = os.path.join(ROOT, "profiles", "ncu_kernel_traffic_r02.json")


def kernel_traffic(f32, shape):
    """DRAM bytes (read + write) per launch of this exact kernel-leg launch (dtype and
    m x n x k) from its committed ncu --set full capture (tools/kernel_traffic.py), or None
    when no capture of this shape exists (a traffic figure is never borrowed from another
    kernel or shape)."""
    try:
        tab = json.load(open(TRAFFIC_FILE))
    except (OSError, ValueError):
        return None, None
    key = f"{'f32' if f32 else 'f64'} {'x'.join(str(int(x)) for x in shape)}"
    ent = tab.get(key)
    if not ent:
        return None, None
    return ent["traffic_bytes"], f"profiles/{os.path.basename(TRAFFIC_FILE)}[{key!r}] ({ent['source']})"


def result_line(args, cfg, val, e2e, kern, peak_measured, clk, cpu, links, parity,
                execution="single process"):
    """The bench JSON line (shared by the single-process and one-process-per-GPU paths)."""
    f32 = cfg.get("dtype") == "f32"
    n = args.gpus
    flops = val["flops"]
    peak_tf, peak_src = peak_measured, ("measured live: register-only DMMA.8x8x4 loop "
                                        "(bx_fp64_peak_probe); MEASURED_PEAKS.json has no FP64 entry")
    if f32:
        peak_tf, peak_src = tf32_peak_tflops()
    # north-star roofline: slower of aggregate tensor time and the bytes this run moved over
    # the host links / NVLink at the bandwidths measured in this run with all N GPUs active
    t_tensor = flops / (n * peak_tf * 1e12)
    t_link = None
    if links and links.get("h2d_gbs"):
        per_dev = val["per_device"]
        h2d_max = max(d["h2d"] for d in per_dev.values())
        p2p_max = max(d["d2d_in"] for d in per_dev.values())
        d2h_max = max(d.get("d2h", 0) for d in per_dev.values())
        # the host link is full duplex: H2D and D2H overlap, the slower direction bounds
        t_link = h2d_max / (links["h2d_gbs"] * 1e9)
        if d2h_max and links.get("d2h_gbs"):
            t_link = max(t_link, d2h_max / (links["d2h_gbs"] * 1e9))
        if p2p_max:
            t_link += p2p_max / (links["p2p_in_gbs"] * 1e9) if links.get("p2p_in_gbs") else float("nan")
    t_meas = val["ms"] / 1e3
    roof = max(t_tensor, t_link or 0.0)
    esz = 4 if f32 else 8
    traffic, traffic_src = kernel_traffic(f32, kern["shape"])
    out = {
        "metric": METRIC_F32 if f32 else METRIC,
        "value": val["value"], "unit": "TFLOP/s",
        "n_gpus": n, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": val["ms"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 (tf32 MMA, f32 accumulate)" if f32 else "f64",
        "data": "synthetic: seeded uniform[-1,1) host operands (reference build_call generator); "
                "device-filled uniform[-1,1) for the kernel-alone roofline leg",
        "config": config_dict(cfg, args),
        "frac_of_tensor_peak": val["value"] / (n * peak_tf),
        "e2e": {"value": e2e["value"], "unit": "TFLOP/s", "ms_per_step": e2e["ms"],
                "api": e2e["api"],
                "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"],
                "p2p_bytes_per_step": e2e["p2p"]},
        "cache": {"h2d_bytes": val["h2d"], "p2p_bytes": val["p2p"], "d2h_bytes": val["d2h"],
                  "l1_hits": val["l1"], "l2_hits": val["l2"], "host_fetches": val["host"],
                  "per_device": val["per_device"]},
        "roofline": {"bound": "tensor", "achieved": kern["tflops"], "peak": peak_tf,
                     "unit": "TFLOP/s", "frac": kern["tflops"] / peak_tf,
                     "frac_of_sustained_peak": (kern["tflops"] / tf32_sustained_tflops()
                                                if f32 and tf32_sustained_tflops() else None),
                     "traffic": traffic,
                     "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": esz * (kern["shape"][0] * kern["shape"][2]
                                                            + kern["shape"][2] * kern["shape"][1]
                                                            + (1 if f32 else 2) * kern["shape"][0] * kern["shape"][1]),
                     "kernel": ("bx::sgemm_tc2c_kernel (tcgen05.mma.cta_group::2 kind::tf32, 256x256 "
                                "pair tiles taken by cluster launch control, double-buffered TMEM "
                                "accumulators, TMA)" if f32 else
                                "bx::gemm_task_mb_kernel (FP64 DMMA m8n8k4, mbarrier cp.async ring)"),
                     "kernel_shape": kern["shape"], "flops_per_launch": kern["flops"],
                     "avg_launch_ms": kern["ms"], "peak_source": peak_src,
                     "fp64_dmma_peak_measured": peak_measured,
                     "north_star": {"t_tensor_s": t_tensor, "t_link_s": t_link,
                                    "t_measured_s": t_meas, "frac": roof / t_meas,
                                    "bound": "link" if (t_link or 0) > t_tensor else "tensor",
                                    "links_measured": links}},
        "parity": parity,
        "gpu_launches": val["launches"] + e2e["launches"] + kern["launches"],
        "gpu_launches_detail": {"value_leg": val["launches"], "e2e_leg": e2e["launches"],
                                "kernel_leg": kern["launches"]},
        **({"tile_sweep": val["sweep"]} if val.get("sweep") else {}),
        "clocks": clk.summary() if clk else None,
        "execution": execution,
    }
    if cpu:
        out["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
    return out


def _metrics_summary(res):
    mt = res.metrics
    return dict(h2d=mt.total_h2d_bytes(), d2h=mt.total_d2h_bytes(), p2p=mt.total_d2d_bytes(),
                l1=mt.l1_hits, l2=mt.l2_hits, host=mt.host_fetches,
                per_device={str(d): dict(h2d=v.h2d_bytes, d2h=v.d2h_bytes, d2d_in=v.d2d_in_bytes,
                                          tasks=v.tasks)
                            for d, v in mt.devices.items()})


# ----------------------------------------------------------------------------- one process

def single_bench(args, cfg):
    """N GPUs driven from this process (the reference's shape; N=1 by default)."""
    from paper_1510_05041_b200 import RunOptions, _native as NN, run_call
    from paper_1510_05041_b200.devices import DeviceDesc, Topology
    from paper_1510_05041_b200.engine import get_engine
    from oracle import sampled
    lib = NN.load()
    NN.require_gpu()
    eng = get_engine(list(range(args.gpus)), 4)
    peak = C.c_double()
    NN.check(lib.bx_fp64_peak_probe(0, 40000, C.byref(peak)), "peak probe")
    call = make_operands(cfg, seed=0)
    topo = Topology([DeviceDesc(g, peer_group="nvlink") for g in range(args.gpus)])
    opts = RunOptions(chunk_steps=args.chunk, n_streams=args.streams,
                      tasks_per_stream=args.tasks_per_stream, trsm_inverse_min=args.trsm_inverse_min,
                      release_on_issue=bool(args.release_on_issue),
                      owner_prefetch=args.owner_prefetch_mb > 0,
                      owner_prefetch_mb=max(1, args.owner_prefetch_mb))
    for mt in (call.a, call.b, call.c):
        if mt is not None:
            eng.register_host(mt.matrix.storage)   # page-locking excluded
    for _ in range(args.warmup):
        run_call(call, topo, opts)
    slots = [eng.slot(g) for g in range(args.gpus)]
    links = link_probe(eng, lib, slots[0],
                       peers=[(s, "peer") for s in slots[1:]] if len(slots) > 1 else None)

    def all_sync():
        for s in slots:
            eng.device_sync(s)

    with ClockSampler(list(range(args.gpus))) as clk:
        # value: run_call (RoutineCall API), device-event timed
        n0 = eng.launches()
        times = []
        res = None
        for _ in range(args.steps):
            all_sync()
            e0 = eng.record(slots[0], 0, timing=True)
            res = run_call(call, topo, opts)
            e1 = eng.record(slots[0], 0, timing=True)
            eng.sync(e1)
            all_sync()
            times.append(eng.elapsed_ms(e0, e1))
            eng.release(e0)
            eng.release(e1)
        v_launch = eng.launches() - n0
        ms = statistics.mean(times)
        val = dict(value=res.plan.total_flops / (ms / 1e3) / 1e12, ms=ms, flops=res.plan.total_flops,
                   launches=v_launch, **_metrics_summary(res))
        # e2e: the cblas-style public API, host clock
        blocks = sampled.call_blocks(call, PARITY_BLOCKS[cfg["kind"]], seed=1)
        n0 = eng.launches()
        wall = []
        c0 = None
        for s in range(args.steps):
            if s == args.steps - 1:
                c0 = sampled.call_snapshot(call, blocks)
            all_sync()
            t0 = time.perf_counter()
            r2 = api_call(call, opts, topo)
            wall.append((time.perf_counter() - t0) * 1e3)
        e_launch = eng.launches() - n0
        ms2 = statistics.mean(wall)
        ms_e2e = _metrics_summary(r2)
        e2e = dict(value=r2.plan.total_flops / (ms2 / 1e3) / 1e12, ms=ms2, launches=e_launch,
                   api=f"blas.{ 's' if cfg.get('dtype') == 'f32' else 'd'}{cfg['kind']} (cblas-style, "
                       f"caller's column-major host buffers)", **ms_e2e)
        kern = kernel_leg(args, cfg, eng, lib, slots[0], kernel_shape(cfg)[1], 1234)
    parity = parity_check(call, c0)
    sweep = []
    for t in cfg.get("sweep", ()):
        c2 = retile(call, t)
        run_call(c2, topo, opts)
        all_sync()
        e0 = eng.record(slots[0], 0, timing=True)
        r3 = run_call(c2, topo, opts)
        e1 = eng.record(slots[0], 0, timing=True)
        eng.sync(e1)
        tms = eng.elapsed_ms(e0, e1)
        eng.release(e0)
        eng.release(e1)
        m3 = r3.metrics
        sweep.append(dict(tile=t, ms=tms, tflops=r3.plan.total_flops / (tms / 1e3) / 1e12,
                          h2d_bytes=m3.total_h2d_bytes(), p2p_bytes=m3.total_d2d_bytes(),
                          d2h_bytes=m3.total_d2h_bytes(), tasks=len(r3.plan.tasks),
                          l1_hits=m3.l1_hits, l2_hits=m3.l2_hits, host_fetches=m3.host_fetches))
    val["sweep"] = sweep
    cpu = None if args.no_cpu_baseline else cpu_sample(cfg, call, target_s=args.cpu_seconds)
    line = result_line(args, cfg, val, e2e, kern, peak.value, clk, cpu, links, parity,
                       execution=f"single process, {args.gpus} GPU(s)")
    print(json.dumps(line), flush=True)
    return line


# ----------------------------------------------------------------------------- one process per GPU

def spmd_bench(args, cfg):
    """One process per GPU (torchrun, or ``launch_ranks``): every rank drives its own GPU
    through the SPMD runtime (paper_1510_05041_b200/spmd.py).  Each step is bracketed by a
    session barrier and a device sync on every rank; step time = max over ranks of each
    rank's CUDA-event time.  Returns rank 0's line (None elsewhere)."""
    from paper_1510_05041_b200 import RunOptions, run_call, spmd
    from paper_1510_05041_b200 import _native as NN
    from paper_1510_05041_b200.engine import get_engine
    from oracle import sampled
    sess = spmd.init(device=0 if args.ranks_share_gpu else None)
    r, W = sess.rank, sess.world
    lib = NN.load()
    NN.require_gpu()
    eng = get_engine([r], 4, [sess.device])
    slot = eng.slot(r)
    peak = C.c_double()
    NN.check(lib.bx_fp64_peak_probe(slot, 40000, C.byref(peak)), "peak probe")
    peak_v = float(sess.allgather(peak.value).min())

    def barrier_sync():
        sess.barrier("step start")
        eng.device_sync(slot)

    call = make_operands(cfg, seed=0) if r == 0 else None
    call = sess.share_call(call)
    for mt in (call.a, call.b, call.c):
        if mt is not None:
            eng.register_host(mt.matrix.storage)   # page-locking excluded from timing
    opts = RunOptions(execution="spmd", chunk_steps=args.chunk, n_streams=args.streams,
                      tasks_per_stream=args.tasks_per_stream, trsm_inverse_min=args.trsm_inverse_min,
                      release_on_issue=bool(args.release_on_issue),
                      owner_prefetch=args.owner_prefetch_mb > 0,
                      owner_prefetch_mb=max(1, args.owner_prefetch_mb))
    for _ in range(args.warmup):
        run_call(call, options=opts)
    # links with all ranks active: H2D/D2H of this rank's lanes, P2P from the next rank's
    # arena over CUDA IPC (a ring: every GPU reads one peer at once)
    bases = sess.peer_bases(eng, slot)
    nxt = (r + 1) % W
    links = link_probe(eng, lib, slot, peers=[(bases[nxt], "ipc")] if W > 1 else None,
                       sync_all=lambda: sess.barrier("link probe"))
    if links:
        agg = {k: float(sess.allgather(links.get(k) or 0.0).min()) for k in ("h2d_gbs", "d2h_gbs", "p2p_in_gbs")}
        links.update(agg)
        links["note"] = "per GPU, minimum over ranks, all ranks copying at once"

    clk = ClockSampler([sess.device] if args.ranks_share_gpu else list(range(W))) if r == 0 else None
    if clk:
        clk.__enter__()
    try:
        n0 = eng.launches()
        times = []
        res = None
        for _ in range(args.steps):
            barrier_sync()
            e0 = eng.record(slot, 0, timing=True)
            res = run_call(call, options=opts)
            e1 = eng.record(slot, 0, timing=True)
            eng.sync(e1)
            eng.device_sync(slot)
            times.append(sess.allreduce_max(eng.elapsed_ms(e0, e1)))
            eng.release(e0)
            eng.release(e1)
        v_launch = int(sess.allgather(eng.launches() - n0).sum())
        ms = statistics.mean(times)
        val = dict(value=res.plan.total_flops / (ms / 1e3) / 1e12, ms=ms, flops=res.plan.total_flops,
                   launches=v_launch, **_metrics_summary(res))
        # e2e: the public run_call in spmd mode on the shared host buffers, host clock
        blocks = sampled.call_blocks(call, PARITY_BLOCKS[cfg["kind"]], seed=1) if r == 0 else None
        n0 = eng.launches()
        wall = []
        c0 = None
        r2 = None
        for s in range(args.steps):
            if s == args.steps - 1 and r == 0:
                c0 = sampled.call_snapshot(call, blocks)
            barrier_sync()
            t0 = time.perf_counter()
            r2 = run_call(call, options=opts)
            wall.append(sess.allreduce_max((time.perf_counter() - t0) * 1e3))
        e_launch = int(sess.allgather(eng.launches() - n0).sum())
        ms2 = statistics.mean(wall)
        e2e = dict(value=r2.plan.total_flops / (ms2 / 1e3) / 1e12, ms=ms2, launches=e_launch,
                   api="run_call(call, options=RunOptions(execution='spmd')) on node-shared host "
                       "buffers, every rank", **_metrics_summary(r2))
        m, n, k = kernel_shape(cfg)
        cols = [n // W + (1 if g < n % W else 0) for g in range(W)]
        kern = kernel_leg(args, cfg, eng, lib, slot, cols[r], 1234 + 7 * r,
                          sync_all=lambda: sess.barrier("kernel step"))
        kern["tflops"] = float(sess.allgather(kern["tflops"]).mean())
        kern["launches"] = int(sess.allgather(kern["launches"]).sum())
    finally:
        if clk:
            clk.__exit__(None, None, None)
    line = None
    if r == 0:
        parity = parity_check(call, c0)
        line = result_line(args, cfg, val, e2e, kern, peak_v, clk, None, links, parity,
                           execution=f"one process per GPU ({W} ranks, spmd runtime, input tiles "
                                     f"dealt to the ranks' host links: owner prefetch)")
        if not args.no_cpu_baseline and W == 1:
            line["cpu_baseline"] = {k: v for k, v in cpu_sample(cfg, call, args.cpu_seconds).items()
                                    if k in ("value", "unit", "cores", "kind", "sample")}
    sess.barrier("bench end")
    spmd.shutdown()
    return line


def _rank_main(argv):
    """Entry point of a rank started by ``launch_ranks`` (module-level: spawn imports it)."""
    args = parse_args(argv)
    line = spmd_bench(args, CONFIGS_FOR(args))
    return line


def launch_ranks(args, argv):
    """``--gpus N`` without torchrun: start one process per GPU (spmd.launch) running the
    same bench, and print rank 0's line."""
    import bench as this      # importable by name in the spawned ranks (ROOT is on sys.path)
    from paper_1510_05041_b200 import spmd
    devices = [0] * args.gpus if args.ranks_share_gpu else list(range(args.gpus))
    outs = spmd.launch(args.gpus, this._rank_main, argv, devices=devices, timeout=3600)
    print(json.dumps(outs[0]), flush=True)


# ----------------------------------------------------------------------------- main

def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--chunk", type=int, default=0, help="k-steps per launch (0 = auto)")
    ap.add_argument("--streams", type=int, default=0)
    ap.add_argument("--tasks-per-stream", type=int, default=2)
    ap.add_argument("--trsm-inverse-min", type=int, default=128,
                    help="TRSM: inverse-based diagonal step from this tile order (0 = substitution)")
    ap.add_argument("--release-on-issue", type=int, default=0, choices=[0, 1],
                    help="TRSM: release dependents when a solve is enqueued (1) or after its "
                         "write-back (0, the reference's rule)")
    ap.add_argument("--owner-prefetch-mb", type=int, default=64,
                    help="one process per GPU: owner loads in flight per rank (0 = plain "
                         "first-holder fetches)")
    ap.add_argument("--ref-seconds", type=float, default=8.0)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--single-process", action="store_true",
                    help="--gpus N>1 from one process (the reference's shape) instead of N ranks")
    ap.add_argument("--ranks-share-gpu", action="store_true",
                    help="N ranks all on GPU 0 (functional check of the multi-process path)")
    ap.add_argument("--tile", type=int, default=0, help="override the config's tile size")
    args = ap.parse_args(argv)
    args.steps = max(1, args.steps)
    return args


def CONFIGS_FOR(args):
    cfg = CONFIGS[args.config]
    if args.tile:
        cfg = dict(cfg, tile=args.tile, desc=cfg["desc"].replace(f"tile {cfg['tile']}", f"tile {args.tile}"))
    return cfg


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    args = parse_args(argv)
    cfg = CONFIGS_FOR(args)
    rank, world = dist_env()
    if world > 1 and args.gpus != world:
        log(f"bench: --gpus {args.gpus} but WORLD_SIZE {world}; using WORLD_SIZE")
        args.gpus = world
    if args.impl == "reference":
        # the reference's CPU path: rank 0 alone runs it, the other ranks exit without work
        if rank == 0:
            print(json.dumps(run_reference(args, cfg)), flush=True)
        return
    if world > 1:
        line = spmd_bench(args, cfg)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if args.gpus > 1 and not args.single_process:
        launch_ranks(args, argv)
        return
    single_bench(args, cfg)


if __name__ == "__main__":
    main()
