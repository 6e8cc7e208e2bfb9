#!/bin/bash
# round 2: new GPU tests (full-size parity, SGEMM auto precision) + bench lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
free -g >> gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt; df -h /dev/shm >> gpurun_out/smi.txt
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -s > gpurun_out/pytest_full.log 2>&1
echo "fullsize rc=$?" >> gpurun_out/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "sgemm" > gpurun_out/pytest_sgemm.log 2>&1
echo "sgemm rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
echo "bench rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --gpus 2 --ranks-share-gpu --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_spmd2.json 2> gpurun_out/bench_spmd2.err
echo "spmd2 rc=$?" >> gpurun_out/status.txt
