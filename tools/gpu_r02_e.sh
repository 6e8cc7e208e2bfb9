#!/bin/bash
# round 2, part E: resident issue engine + release-on-issue fix on hardware: GPU suite,
# bench lines, TRSM A/B, host issue rate, logical-device runs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
S=gpurun_out/status_e.txt; rm -f $S
timeout 2700 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_e.log 2>&1
echo "pytest rc=$?" >> $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_e.log 2>&1
echo "smoke rc=$?" >> $S
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_e.json 2> gpurun_out/bench_cfg2_e.err
echo "bench cfg2 rc=$?" >> $S
timeout 900 python bench.py --config cfg1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg1_e.json 2> gpurun_out/bench_cfg1_e.err
echo "bench cfg1 rc=$?" >> $S
for r in 1 2; do
  for e in 1 0; do
    timeout 900 python bench.py --config cfg4_trsm --steps 3 --warmup 2 --no-cpu-baseline --release-on-issue $e > gpurun_out/trsm_e_roi${e}_$r.json 2> gpurun_out/trsm_e_roi${e}_$r.err
    echo "trsm roi=$e r=$r rc=$?" >> $S
  done
done
timeout 900 python bench.py --config cfg3_syrk --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_syrk_e.json 2> gpurun_out/bench_syrk_e.err
echo "bench syrk rc=$?" >> $S
timeout 600 python tools/host_rate_gpu.py 512 1,8 > gpurun_out/host_rate_e.txt 2>&1
echo "host rate rc=$?" >> $S
BX_IC=0 timeout 600 python tools/host_rate_gpu.py 512 1,8 > gpurun_out/host_rate_e_noic.txt 2>&1
echo "host rate noic rc=$?" >> $S
timeout 900 python tools/logical_e2e.py 16384 1024 1 8 > gpurun_out/logical_e.txt 2>&1
echo "logical rc=$?" >> $S
