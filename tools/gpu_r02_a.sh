#!/bin/bash
# round 2 evidence, part A: whole GPU suite, smoke, every config's bench line (both arms for cfg2)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
S=gpurun_out/status_a.txt; rm -f $S
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt
nproc >> gpurun_out/smi.txt; free -g >> gpurun_out/smi.txt
timeout 2700 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> $S
timeout 900 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
echo "bench cfg2 rc=$?" >> $S
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_cfg2.json 2> gpurun_out/bench_ref_cfg2.err
echo "bench ref rc=$?" >> $S
for c in cfg1 cfg3_syrk cfg3_syr2k cfg4_trsm cfg4_trmm dgemm32768 cfg5_sgemm; do
  timeout 1200 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "bench $c rc=$?" >> $S
done
