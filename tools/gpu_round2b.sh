#!/bin/bash
# round 2: whole GPU suite with the inverse-based TRSM step + cfg4 TRSM both ways
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/status_b.txt
timeout 900 python bench.py --config cfg4_trsm --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_trsm_inv.json 2> gpurun_out/bench_trsm_inv.err
echo "trsm inv rc=$?" >> gpurun_out/status_b.txt
timeout 900 python bench.py --config cfg4_trsm --steps 5 --warmup 3 --no-cpu-baseline --trsm-inverse-min 0 > gpurun_out/bench_trsm_sub.json 2> gpurun_out/bench_trsm_sub.err
echo "trsm sub rc=$?" >> gpurun_out/status_b.txt
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_all.log 2>&1
echo "pytest rc=$?" >> gpurun_out/status_b.txt
