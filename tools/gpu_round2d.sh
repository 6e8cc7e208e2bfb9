#!/bin/bash
# round 2: sanitizers over every kernel, failure-path tests, TRSM/TRMM after the k-range /
# early-inverse changes
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/status_d.txt
timeout 600 python tools/sanitize_small.py > gpurun_out/san_plain.txt 2>&1
echo "plain rc=$?" >> gpurun_out/status_d.txt
for c in cfg4_trsm cfg4_trmm; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "bench $c rc=$?" >> gpurun_out/status_d.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_spmd.py -m gpu -q -k "capacity or singular or trmm or trsm" > gpurun_out/pytest_fail.log 2>&1
echo "pytest rc=$?" >> gpurun_out/status_d.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_small.py > gpurun_out/san_$tool.txt 2>&1
  echo "sanitizer $tool rc=$?" >> gpurun_out/status_d.txt
done
