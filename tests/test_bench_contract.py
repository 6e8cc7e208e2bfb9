"""bench.py's JSON line (the driver's contract) assembled from synthetic leg results on CPU,
and the runtime's automatic launch-shape resolution."""

import json
import os
import sys
import types

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1510_05041_b200 import RunOptions, build_call  # noqa: E402
from paper_1510_05041_b200.routines import generate_tasks  # noqa: E402
from paper_1510_05041_b200.scheduler import resolve_ramp, resolve_streams  # noqa: E402

REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
            "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "clocks",
            "roofline"]


class _Clk:
    def summary(self):
        return {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0, "reasons": [], "samples": 3}


def _legs():
    per_dev = {"0": dict(h2d=6.44e9, d2d_in=0, tasks=256)}
    val = dict(value=34.9, ms=252.0, flops=8.8e12, launches=1536, h2d=6.44e9, d2h=2.15e9, p2p=0,
               l1=7680, l2=0, host=512, per_device=per_dev)
    e2e = dict(value=34.5, ms=255.0, launches=1536, api="blas.dgemm", h2d=6.44e9, d2h=2.15e9,
               p2p=0, l1=7680, l2=0, host=512, per_device=per_dev)
    kern = dict(ms=246.0, flops=8.8e12, tflops=35.7, launches=3, shape=[16384, 16384, 16384])
    cpu = dict(value=0.45, unit="TFLOP/s", cores=16, kind="port", sample="x", seconds=10.0)
    links = {"h2d_gbs": 53.0, "d2h_gbs": 54.0, "bytes_per_copy": 1 << 28}
    parity = {"max_ratio": 0.01, "bound": 10.0, "pass": True, "blocks": 16}
    return val, e2e, kern, cpu, links, parity


def test_result_line_has_the_contract_keys():
    args = types.SimpleNamespace(gpus=1, steps=3, warmup=3, chunk=0)
    cfg = bench.CONFIGS["cfg2"]
    val, e2e, kern, cpu, links, parity = _legs()
    line = bench.result_line(args, cfg, val, e2e, kern, 37.1, _Clk(), cpu, links, parity)
    json.dumps(line)
    assert [k for k in REQUIRED if k not in line] == []
    # value = the host-resident run_call (the BASELINE metric), not the kernel alone
    assert line["value"] == 34.9 and line["ms_per_step"] == 252.0
    assert line["e2e"]["h2d_bytes_per_step"] == 6.44e9 and line["e2e"]["unit"] == "TFLOP/s"
    r = line["roofline"]
    assert r["bound"] == "tensor" and r["frac"] == pytest.approx(35.7 / 37.1)
    ns = r["north_star"]
    assert ns["t_link_s"] == pytest.approx(6.44e9 / 53e9)
    assert ns["frac"] == pytest.approx(max(ns["t_tensor_s"], ns["t_link_s"]) / 0.252)
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] == 16
    assert line["higher_is_better"] is True and line["vs_baseline"] is None
    assert line["parity"]["pass"] and line["gpu_launches"] == 1536 * 2 + 3


def test_reference_arm_reports_the_same_config():
    """Both arms describe the same routine, shape and scalars (same_config)."""
    args = types.SimpleNamespace(gpus=1, steps=3, warmup=3, chunk=0)
    for name in ("cfg2", "cfg3_syrk", "cfg4_trsm"):
        cfg = bench.CONFIGS[name]
        val, e2e, kern, cpu, links, parity = _legs()
        ours = bench.result_line(args, cfg, val, e2e, kern, 37.1, _Clk(), cpu, links, parity)
        assert ours["config"] == bench.config_dict(cfg, args)
        assert "alpha" in ours["config"] and "beta" in ours["config"]


@pytest.mark.parametrize("name", ["cfg2", "cfg3_syrk", "cfg3_syr2k", "cfg4_trsm", "cfg4_trmm"])
def test_cpu_sample_runs_the_configs_routine(name, monkeypatch):
    """The CPU baseline / reference arm samples blocks of the config's OWN routine (small
    shape here), and counts their algorithmic flops."""
    cfg = dict(bench.CONFIGS[name], m=256, n=256, k=256 if name != "cfg3_syrk" else 128, tile=64)
    call = bench.make_operands(cfg, seed=0)
    r = bench.cpu_sample(cfg, call, target_s=0.05)
    assert r["value"] > 0 and r["kind"] == "port"
    unit = "tile columns" if cfg["kind"] in ("trsm", "trmm") else "output tiles"
    assert unit in r["sample"]


def test_block_flops_sum_to_plan_flops():
    from oracle import sampled
    from paper_1510_05041_b200.routines import generate_tasks
    for name in ("cfg2", "cfg3_syrk", "cfg3_syr2k", "cfg4_trsm", "cfg4_trmm"):
        cfg = dict(bench.CONFIGS[name], m=300, n=300, k=200, tile=64)
        call = bench.make_operands(cfg, seed=0)
        blocks = sampled.call_blocks(call, 10 ** 6)
        total = sum(bench.block_flops(cfg["kind"], b, cfg) for b in blocks)
        assert total == pytest.approx(generate_tasks(call).total_flops, rel=1e-12), name


@pytest.mark.parametrize("kind,k,ndev,chunk,streams", [
    ("gemm", 1024, 1, 8, 8), ("gemm", 1024, 8, 8, 4), ("symm", 1024, 1, 8, 8),
    ("syrk", 512, 1, 16, 12), ("syrk", 512, 8, 16, 4), ("trsm", 1024, 1, 16, 8),
    ("trmm", 1024, 1, 16, 8), ("syr2k", 512, 1, 8, 4)])
def test_auto_launch_shape(kind, k, ndev, chunk, streams):
    # the BASELINE task grids (16 x 16 tiles; K = 16 or 8 steps) at a small element count
    call = build_call(kind, m=1024, n=1024, k=k, tile_size=64, seed=0, uplo="lower",
                      beta=1.0 if kind in ("gemm", "syrk", "syr2k", "symm") else 0.0)
    plan = generate_tasks(call)
    o = resolve_ramp(plan, resolve_streams(plan, RunOptions(), ndev), ndev)
    assert (o.chunk_steps, o.n_streams) == (chunk, streams)
    assert 0 <= o.ramp_tasks <= max(0, len(plan.tasks) // (4 * ndev))
    if kind == "gemm":
        assert o.ramp_tasks == min(32, 256 // (4 * ndev))
    # explicit values are kept
    o2 = resolve_streams(plan, RunOptions(chunk_steps=3, n_streams=2), ndev)
    assert (o2.chunk_steps, o2.n_streams) == (3, 2)


def test_no_start_up_batch_for_small_calls():
    """cfg1-sized calls (16 tasks) issue whole-task launches from the start."""
    call = build_call("gemm", m=256, n=256, k=256, tile_size=64, seed=0, beta=1.0)
    plan = generate_tasks(call)
    assert len(plan.tasks) == 16
    assert resolve_ramp(plan, RunOptions(), 1).ramp_tasks == 0
    assert resolve_ramp(plan, RunOptions(ramp_tasks=4), 1).ramp_tasks == 4


def test_small_call_one_stream_per_task():
    """Small calls (< 64 tasks) on one GPU with an auto-sized arena: one task per compute
    stream (up to 16); bounded arenas and several GPUs keep the capped default."""
    call = build_call("gemm", m=256, n=256, k=256, tile_size=64, seed=0, beta=1.0)
    plan = generate_tasks(call)
    assert resolve_streams(plan, RunOptions(), 1).n_streams == 16
    assert resolve_streams(plan, RunOptions(), 1, bounded_arena=True).n_streams == 4
    assert resolve_streams(plan, RunOptions(), 2).n_streams == 4
    assert resolve_streams(plan, RunOptions(n_streams=3), 1).n_streams == 3
    tiny = generate_tasks(build_call("gemm", m=128, n=64, k=64, tile_size=64, seed=0))
    assert resolve_streams(tiny, RunOptions(), 1).n_streams == len(tiny.tasks) == 2


@pytest.mark.gpu
def test_bench_runs_end_to_end_on_the_gpu():
    """The driver's command shape on a B200 (small config, one step): one JSON line with the
    contract keys, the parity check passing, kernels launched, the traffic field sourced."""
    import subprocess
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "cfg1",
                          "--steps", "2", "--warmup", "3", "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    for k in REQUIRED + ["parity", "cache"]:
        assert k in d, k
    assert d["parity"]["pass"] and d["parity"]["max_ratio"] <= 10
    assert d["gpu_launches"] > 0 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["roofline"]["traffic"] and "ncu_kernel_traffic" in d["roofline"]["traffic_source"]
    assert d["warmup"] >= 3


def test_small_call_rule_counts_link_bound_mid_size_calls():
    """64-128 tasks count as small on one GPU only when host-link bound: DGEMM 4096^3 at
    T=512 (64 tasks, 0.38 GB for 0.14 TFLOP) yes, 8192^3 at T=1024 (64 tasks, balanced) no."""
    from paper_1510_05041_b200.scheduler import small_call
    from paper_1510_05041_b200 import RoutineCall
    from paper_1510_05041_b200.tiling import MatrixDesc, make_tiled
    import numpy as np

    def plan_of(n, t):
        buf = np.zeros(n * n)      # one buffer for all three operands: only geometry matters
        return generate_tasks(RoutineCall("gemm", a=make_tiled(MatrixDesc("A", n, n, n, buf), t),
                                          b=make_tiled(MatrixDesc("B", n, n, n, buf), t),
                                          c=make_tiled(MatrixDesc("C", n, n, n, buf), t), beta=1.0))
    p1 = plan_of(4096, 512)
    p2 = plan_of(8192, 1024)
    assert len(p1.tasks) == len(p2.tasks) == 64
    assert small_call(p1) and not small_call(p2)
    assert not small_call(p1, n_devices=2)
    assert resolve_ramp(p1, RunOptions(), 1).ramp_tasks == 0
    assert resolve_ramp(p2, RunOptions(), 1).ramp_tasks == 16
    assert resolve_streams(p1, RunOptions(), 1).n_streams == 16
