#!/usr/bin/env python
"""Benchmark: host-resident tiled DGEMM on B200 (BASELINE.json configs[1]).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config cfg2|cfg1|dgemm32768|cfg3_syrk|cfg3_syr2k|cfg4_trsm|cfg4_trmm]

Prints ONE JSON line (rank 0).  Legs:
  value     device-resident DGEMM over the same workload (inputs already in HBM; the
            dominant tile kernel, FP64 DMMA) — whole-job TFLOP/s over the N GPUs;
  e2e       the public API call (``dgemm`` / ``run_call``) on host-resident numpy buffers,
            H2D tile loads + D2H write-back inside the timed region — the headline;
  roofline  dominant kernel: flops per launch / CUDA-event launch time vs the FP64 DMMA
            peak measured live (MEASURED_PEAKS.json has no FP64 figure);
  cpu_baseline  the oracle port of the reference tiled runtime (numpy/OpenBLAS, all host
            cores) on a bounded sample of the same workload.
Under torchrun (WORLD_SIZE>1) every rank drives its own GPU (LOCAL_RANK) through the
one-process-per-GPU runtime (spmd.py): shared task queue, stations with stealing, and the
L2 tile cache over peer HBM via CUDA IPC; steps are bracketed by session barriers and the
step time is the max over ranks.  ``--gpus N`` without torchrun drives N GPUs from one
process (the single-address-space runtime).
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
                 "-lms", "200", "-i", ",".join(str(g) for g in range(self.gpus))],
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


def cpu_sample(cfg, call, target_s=12.0):
    """Oracle port of the reference tiled runtime (routines.py:482-492 execute_task_on_host)
    on sampled output tiles of the same workload, all host threads (OpenBLAS)."""
    from oracle import tiled
    a, b, c = (x.matrix.as_2d() for x in (call.a, call.b, call.c))
    t = cfg["tile"]
    kt = -(-cfg["k"] // t)
    tiles = []
    rng = np.random.default_rng(1)
    nt = -(-cfg["m"] // t)
    flops_per_tile = 2 * t * t * cfg["k"]
    try:   # all host threads, whatever the launcher exported
        from threadpoolctl import threadpool_limits
        threadpool_limits(os.cpu_count(), user_api="blas")
    except Exception:
        pass
    # warm-up one tile (OpenBLAS init), then as many tiles as fit target_s
    tiled.run_tiles_subset("gemm", a, c, b, tile_size=t, tiles=[(0, 0)], alpha=cfg["alpha"],
                           beta=cfg["beta"])
    t0 = time.perf_counter()
    done = 0
    while time.perf_counter() - t0 < target_s:
        ij = (int(rng.integers(0, nt)), int(rng.integers(0, nt)))
        tiled.run_tiles_subset("gemm", a, c, b, tile_size=t, tiles=[ij], alpha=cfg["alpha"],
                               beta=cfg["beta"])
        tiles.append(ij)
        done += 1
    dt = time.perf_counter() - t0
    return dict(value=done * flops_per_tile / dt / 1e12, unit="TFLOP/s", cores=os.cpu_count(),
                kind="port", seconds=dt,
                sample=f"{done} sampled {t}x{t} output tiles x {kt} k-steps of {cfg['desc']} "
                       f"({done * flops_per_tile / 1e9:.0f} GFLOP), oracle/tiled.py numpy+OpenBLAS")


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))


# ----------------------------------------------------------------------------- legs

def run_reference(args, cfg):
    call = make_operands(CONFIGS["cfg2"] if cfg["kind"] != "gemm" else cfg, seed=0)
    cfg_g = cfg if cfg["kind"] == "gemm" else CONFIGS["cfg2"]
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_sample(cfg_g, call, target_s=args.ref_seconds)
        if i >= args.warmup:
            vals.append(r)
    v = statistics.median([r["value"] for r in vals])
    sec = statistics.median([r["seconds"] for r in vals])
    return {"metric": METRIC, "value": v, "unit": "TFLOP/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded uniform[-1,1))",
            "config": {"workload": cfg_g["desc"], "m": cfg_g["m"], "n": cfg_g["n"], "k": cfg_g["k"],
                       "tile": cfg_g["tile"]},
            "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": vals[0]["cores"],
                             "kind": "port", "sample": vals[0]["sample"]},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def device_value_leg(args, cfg, eng, lib, N):
    """Device-resident DGEMM of the same shape, sharded by column panels over the GPUs."""
    from paper_1510_05041_b200 import _native as NN
    m, n, k = cfg["m"], cfg["n"], cfg["k"]
    f32 = cfg.get("dtype") == "f32"
    esz = 4 if f32 else 8
    ngpu = args.gpus
    cols = [n // ngpu + (1 if g < n % ngpu else 0) for g in range(ngpu)]
    bufs = []
    for g in range(ngpu):
        slot = eng.slot(g)
        ptrs = []
        for nelem in (m * k, k * cols[g], m * cols[g]):
            p = C.c_uint64()
            NN.check(lib.bx_dev_alloc(slot, nelem * esz, C.byref(p)), "alloc")
            if f32:
                NN.check(lib.bx_dev_fill_uniform_f32(slot, p.value, nelem, 1234 + len(ptrs), 0), "fill")
            else:
                NN.check(lib.bx_dev_fill_uniform(slot, p.value, nelem, 1234 + len(ptrs), 0), "fill")
            ptrs.append(p.value)
        bufs.append(ptrs)
    for g in range(ngpu):
        eng.device_sync(eng.slot(g))

    def launch(g):
        s = eng.slot(g)
        a, b, c = bufs[g]
        if f32:
            NN.check(lib.bx_sgemm_device(s, 0, 0, 0, m, cols[g], k, 1.0, a, m, b, k, 0.0, c, m), "sgemm")
        else:
            NN.check(lib.bx_dgemm_device(s, 0, 0, 0, m, cols[g], k, 1.0, a, m, b, k, 1.0, c, m), "dgemm")

    for _ in range(args.warmup):
        for g in range(ngpu):
            launch(g)
    for g in range(ngpu):
        eng.device_sync(eng.slot(g))
    per_launch = []
    evs = []
    n0 = eng.launches()
    t_steps = []
    for _ in range(args.steps):
        pairs = []
        for g in range(ngpu):
            s = eng.slot(g)
            e0 = eng.record(s, 0, timing=True)
            launch(g)
            e1 = eng.record(s, 0, timing=True)
            pairs.append((s, e0, e1))
        step_ms = 0.0
        for s, e0, e1 in pairs:
            eng.sync(e1)
            ms = eng.elapsed_ms(e0, e1)
            per_launch.append((ms, 2.0 * m * cols[s] * k))
            step_ms = max(step_ms, ms)
            eng.release(e0)
            eng.release(e1)
        t_steps.append(step_ms)
    launches = eng.launches() - n0
    for g in range(ngpu):
        s = eng.slot(g)
        for p in bufs[g]:
            lib.bx_dev_free(s, p)
    ms_step = statistics.mean(t_steps)
    flops = 2.0 * m * n * k
    avg_launch_ms = statistics.mean(x[0] for x in per_launch)
    avg_launch_flops = statistics.mean(x[1] for x in per_launch)
    return dict(value=flops / (ms_step / 1e3) / 1e12, ms_per_step=ms_step, launches=launches,
                kernel_tflops=avg_launch_flops / (avg_launch_ms / 1e3) / 1e12,
                avg_launch_ms=avg_launch_ms, flops_per_launch=avg_launch_flops)


def e2e_leg(args, cfg, eng):
    from paper_1510_05041_b200 import RunOptions, run_call
    from paper_1510_05041_b200.devices import DeviceDesc, Topology
    call = make_operands(cfg, seed=0)
    topo = Topology([DeviceDesc(g, peer_group="nvlink") for g in range(args.gpus)])
    opts = RunOptions(chunk_steps=args.chunk, n_streams=args.streams,
                      tasks_per_stream=args.tasks_per_stream)
    for m in (call.a, call.b, call.c):
        if m is not None:
            eng.register_host(m.matrix.storage)   # page-locking excluded from timing
    res = None
    for _ in range(args.warmup):
        res = run_call(call, topo, opts)
    times, metrics = [], []
    n0 = eng.launches()
    for _ in range(args.steps):
        e0 = eng.record(0, 0, timing=True)
        res = run_call(call, topo, opts)
        e1 = eng.record(0, 0, timing=True)
        eng.sync(e1)
        times.append(eng.elapsed_ms(e0, e1))
        eng.release(e0)
        eng.release(e1)
        metrics.append(res.metrics)
    launches = eng.launches() - n0
    ms = statistics.mean(times)
    flops = res.plan.total_flops
    mt = metrics[-1]
    sweep = []
    for t in cfg.get("sweep", ()):
        c2 = retile(call, t)
        run_call(c2, topo, opts)
        e0 = eng.record(0, 0, timing=True)
        r2 = run_call(c2, topo, opts)
        e1 = eng.record(0, 0, timing=True)
        eng.sync(e1)
        tms = eng.elapsed_ms(e0, e1)
        eng.release(e0)
        eng.release(e1)
        m2 = r2.metrics
        sweep.append(dict(tile=t, ms=tms, tflops=flops / (tms / 1e3) / 1e12,
                          h2d_bytes=m2.total_h2d_bytes(), p2p_bytes=m2.total_d2d_bytes(),
                          d2h_bytes=m2.total_d2h_bytes(), tasks=len(r2.plan.tasks),
                          l1_hits=m2.l1_hits, l2_hits=m2.l2_hits, host_fetches=m2.host_fetches))
    return dict(value=flops / (ms / 1e3) / 1e12, ms=ms, flops=flops, launches=launches, sweep=sweep,
                h2d=mt.total_h2d_bytes(), d2h=mt.total_d2h_bytes(), p2p=mt.total_d2d_bytes(),
                l1=mt.l1_hits, l2=mt.l2_hits, host=mt.host_fetches,
                per_device={str(d): dict(h2d=v.h2d_bytes, d2d_in=v.d2d_in_bytes, tasks=v.tasks)
                            for d, v in mt.devices.items()}, call=call)


def result_line(args, cfg, val, e2e, peak_measured, clk, cpu, f32, execution="single process"):
    """The bench JSON line (shared by the single-process and one-process-per-GPU paths)."""
    flops = e2e["flops"]
    h2d_bw, p2p_bw = 53.0e9, 700e9      # measured (profiles/peaks_r01.json); P2P: nominal-measured
    peak_tf = peak_measured
    peak_src = ("measured live: register-only DMMA.8x8x4 loop (bx_fp64_peak_probe); "
                "MEASURED_PEAKS.json has no FP64 entry")
    if f32:
        peak_tf, peak_src = tf32_peak_tflops()
    t_a = flops / (args.gpus * peak_tf * 1e12)
    t_b = e2e["h2d"] / (h2d_bw * args.gpus) + e2e["p2p"] / (p2p_bw * args.gpus)
    prof = os.path.join(ROOT, "profiles", "ncu_dgemm_traffic_r01.json")
    traffic = None
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    kernel_tf = val["kernel_tflops"] if val else e2e["value"]
    out = {
        "metric": METRIC if not f32 else "SGEMM TFLOP/s (host-resident operands, tcgen05 kind::tf32), % of TF32 tensor peak",
        "value": val["value"] if val else e2e["value"],
        "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": val["ms_per_step"] if val else e2e["ms"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 (tf32 MMA, f32 accumulate)" if f32 else "f64",
        "data": "synthetic: seeded uniform[-1,1) (reference build_call generator) for e2e; "
                "device-filled uniform[-1,1) for the HBM-resident leg",
        "config": {"workload": cfg["desc"], "m": cfg["m"], "n": cfg["n"], "k": cfg["k"],
                   "tile": cfg["tile"], "alpha": cfg["alpha"], "beta": cfg["beta"],
                   "l2_flush": "none needed: every step streams > 6 GiB of operands through a 126 MB L2",
                   "chunk_steps": args.chunk or "auto (GEMM/SYMM/SYR2K 8, others 16)"},
        "e2e": {"value": e2e["value"], "unit": "TFLOP/s", "ms_per_step": e2e["ms"],
                "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"],
                "p2p_bytes_per_step": e2e["p2p"],
                "frac_of_tensor_peak": e2e["value"] / (args.gpus * peak_tf),
                "cache": {"l1_hits": e2e["l1"], "l2_hits": e2e["l2"], "host_fetches": e2e["host"]},
                "per_device": e2e["per_device"],
                "roofline_north_star": {"t_tensor_s": t_a, "t_link_s": t_b,
                                        "frac": max(t_a, t_b) / (e2e["ms"] / 1e3),
                                        "h2d_gbs_assumed": h2d_bw / 1e9, "p2p_gbs_assumed": p2p_bw / 1e9}},
        "roofline": {"bound": "tensor", "achieved": kernel_tf, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": kernel_tf / peak_tf, "traffic": None if f32 else traffic,
                     "kernel": ("bx::sgemm_tc2_kernel (tcgen05.mma.cta_group::2 kind::tf32, 256x256 pair tile, TMEM accumulators, TMA)"
                                if f32 else "bx::gemm_task_mb_kernel (FP64 DMMA m8n8k4, mbarrier cp.async ring)"),
                     "peak_source": peak_src,
                     "fp64_dmma_peak_measured": peak_measured,
                     "flops_per_launch": val["flops_per_launch"] if val else None,
                     "avg_launch_ms": val["avg_launch_ms"] if val else None},
        "gpu_launches": e2e["launches"] + (val["launches"] if val else 0),
        **({"tile_sweep": e2e["sweep"]} if e2e["sweep"] else {}),
        "gpu_launches_e2e": e2e["launches"],
        "clocks": clk.summary(),
    }
    if cpu:
        out["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
    out["execution"] = execution
    return out


# ----------------------------------------------------------------------------- one process per GPU

def spmd_bench(args, cfg):
    """WORLD_SIZE > 1 (torchrun): every rank drives its own GPU (LOCAL_RANK) through the SPMD
    runtime (paper_1510_05041_b200/spmd.py: shared task queue, stations with stealing, IPC
    peer tile cache).  Each step is bracketed by a session barrier and a device sync on
    every rank; the step time is the max over ranks of the rank's CUDA-event time."""
    from paper_1510_05041_b200 import RunOptions, run_call, spmd
    from paper_1510_05041_b200 import _native as NN
    from paper_1510_05041_b200.engine import get_engine
    # --ranks-share-gpu: every rank on GPU 0 (exercises the multi-process path on a 1-GPU box)
    sess = spmd.init(device=0 if args.ranks_share_gpu else None)
    r, W = sess.rank, sess.world
    lib = NN.load()
    NN.require_gpu()
    f32 = cfg.get("dtype") == "f32"
    eng = get_engine([r], 4, [sess.device])
    slot = eng.slot(r)
    peak = C.c_double()
    NN.check(lib.bx_fp64_peak_probe(slot, 40000, C.byref(peak)), "peak probe")
    peak_v = float(sess.allgather(peak.value).min())

    def timed(fn):
        sess.barrier("step start")
        eng.device_sync(slot)
        e0 = eng.record(slot, 0, timing=True)
        out = fn()
        e1 = eng.record(slot, 0, timing=True)
        eng.sync(e1)
        eng.device_sync(slot)
        ms = eng.elapsed_ms(e0, e1)
        eng.release(e0)
        eng.release(e1)
        return sess.allreduce_max(ms), ms, out

    clk = ClockSampler(W) if r == 0 else None
    if clk:
        clk.__enter__()
    try:
        val = None
        if cfg["kind"] == "gemm":
            m, n, k = cfg["m"], cfg["n"], cfg["k"]
            esz = 4 if f32 else 8
            cols = [n // W + (1 if g < n % W else 0) for g in range(W)]
            mine = cols[r]
            ptrs = []
            for i, nelem in enumerate((m * k, k * mine, m * mine)):
                p = C.c_uint64()
                NN.check(lib.bx_dev_alloc(slot, nelem * esz, C.byref(p)), "alloc")
                fill = lib.bx_dev_fill_uniform_f32 if f32 else lib.bx_dev_fill_uniform
                NN.check(fill(slot, p.value, nelem, 1234 + 7 * r + i, 0), "fill")
                ptrs.append(p.value)
            eng.device_sync(slot)
            a, b, c = ptrs

            def launch():
                if f32:
                    NN.check(lib.bx_sgemm_device(slot, 0, 0, 0, m, mine, k, 1.0, a, m, b, k, 0.0, c, m), "sgemm")
                else:
                    NN.check(lib.bx_dgemm_device(slot, 0, 0, 0, m, mine, k, 1.0, a, m, b, k, 1.0, c, m), "dgemm")
            for _ in range(args.warmup):
                launch()
            n0 = eng.launches()
            steps, mine_ms = [], []
            for _ in range(args.steps):
                t, own, _ = timed(launch)
                steps.append(t)
                mine_ms.append(own)
            launches = int(sess.allgather(eng.launches() - n0).sum())
            for p in ptrs:
                lib.bx_dev_free(slot, p)
            ms_step = statistics.mean(steps)
            own_ms = statistics.mean(mine_ms)
            flops_mine = 2.0 * m * mine * k
            # dominant-kernel roofline: rank-average launch time and flops
            avg_ms = float(sess.allgather(own_ms).mean())
            avg_fl = float(sess.allgather(flops_mine).mean())
            val = dict(value=2.0 * m * n * k / (ms_step / 1e3) / 1e12, ms_per_step=ms_step,
                       launches=launches, kernel_tflops=avg_fl / (avg_ms / 1e3) / 1e12,
                       avg_launch_ms=avg_ms, flops_per_launch=avg_fl)

        call = make_operands(cfg, seed=0) if r == 0 else None
        call = sess.share_call(call)
        for mt in (call.a, call.b, call.c):
            if mt is not None:
                eng.register_host(mt.matrix.storage)   # page-locking excluded from timing
        opts = RunOptions(execution="spmd", chunk_steps=args.chunk, n_streams=args.streams,
                          tasks_per_stream=args.tasks_per_stream)
        res = None
        for _ in range(args.warmup):
            res = run_call(call, options=opts)
        n0 = eng.launches()
        times = []
        for _ in range(args.steps):
            t, _, res = timed(lambda: run_call(call, options=opts))
            times.append(t)
        launches = int(sess.allgather(eng.launches() - n0).sum())
    finally:
        if clk:
            clk.__exit__(None, None, None)
    ms = statistics.mean(times)
    mt = res.metrics
    e2e = dict(value=res.plan.total_flops / (ms / 1e3) / 1e12, ms=ms, flops=res.plan.total_flops,
               launches=launches, sweep=[], h2d=mt.total_h2d_bytes(), d2h=mt.total_d2h_bytes(),
               p2p=mt.total_d2d_bytes(), l1=mt.l1_hits, l2=mt.l2_hits, host=mt.host_fetches,
               per_device={str(d): dict(h2d=v.h2d_bytes, d2d_in=v.d2d_in_bytes, tasks=v.tasks)
                           for d, v in mt.devices.items()})
    sess.barrier("bench end")
    if r == 0:
        line = result_line(args, cfg, val, e2e, peak_v, clk, None, f32,
                           execution=f"one process per GPU ({W} ranks, spmd runtime)")
        print(json.dumps(line), flush=True)
    sess.barrier("bench printed")
    spmd.shutdown()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--chunk", type=int, default=0, help="k-steps per launch (0 = auto)")
    ap.add_argument("--streams", type=int, default=0)
    ap.add_argument("--tasks-per-stream", type=int, default=2)
    ap.add_argument("--ref-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ranks-share-gpu", action="store_true",
                    help="torchrun test mode: all ranks use GPU 0 (numbers are not scaling)")
    ap.add_argument("--tile", type=int, default=0, help="override the config's tile size")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.tile:
        cfg = dict(cfg, tile=args.tile, desc=cfg["desc"].replace(f"tile {cfg['tile']}", f"tile {args.tile}"))
    rank, world = dist_env()
    if args.gpus != world and world > 1:
        log(f"bench: --gpus {args.gpus} but WORLD_SIZE {world}; using WORLD_SIZE")
        args.gpus = world

    if args.impl == "reference":
        # the reference's CPU path: rank 0 alone runs it, the other ranks exit without work
        if rank == 0:
            print(json.dumps(run_reference(args, cfg)), flush=True)
        return

    if world > 1:
        spmd_bench(args, cfg)
        return

    from paper_1510_05041_b200 import _native as NN
    from paper_1510_05041_b200.engine import get_engine
    lib = NN.load()
    NN.require_gpu()
    f32 = cfg.get("dtype") == "f32"
    eng = get_engine(list(range(args.gpus)), 4)
    if os.environ.get("BX_TRSM_LEAF"):
        NN.check(lib.bx_set_trsm_leaf(int(os.environ["BX_TRSM_LEAF"])), "trsm leaf")
    peak = C.c_double()
    NN.check(lib.bx_fp64_peak_probe(0, 40000, C.byref(peak)), "peak probe")

    with ClockSampler(args.gpus) as clk:
        if cfg["kind"] == "gemm":
            val = device_value_leg(args, cfg, eng, lib, NN)
        else:
            val = None
        e2e = e2e_leg(args, cfg, eng)

    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_sample(cfg if cfg["kind"] == "gemm" else CONFIGS["cfg2"],
                         e2e["call"] if cfg["kind"] == "gemm" else make_operands(CONFIGS["cfg2"]),
                         target_s=10.0)

    print(json.dumps(result_line(args, cfg, val, e2e, peak.value, clk, cpu, f32)), flush=True)


if __name__ == "__main__":
    main()
