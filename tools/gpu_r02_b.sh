#!/bin/bash
# round 2 evidence, part B: DGEMM kernel A/B against the round-1 build, launch list of the
# default bench, ncu --set full of the task GEMM, TRSM timeline, host issue rate, sanitizers
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
S=gpurun_out/status_b.txt; rm -f $S
for r in 1 2 3; do
  for lib in tools/_ab/libblasx_cuda_r1.so tools/_ab/libblasx_cuda_pre_kmode.so paper_1510_05041_b200/libblasx_cuda.so; do
    timeout 300 python tools/ab_dgemm.py $lib 16384 3 >> gpurun_out/ab_dgemm.txt 2>&1
  done
done
echo "ab rc=$?" >> $S
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.json 2>&1
echo "launches rc=$?" >> $S
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_task -s 1 -c 1 -o gpurun_out/ncu_dgemm_16384 python tools/prof_gemm.py 16384 0 0 2 > gpurun_out/ncu_dgemm.log 2>&1
echo "ncu dgemm rc=$?" >> $S
BX_KIND=trsm timeout 600 python tools/trace_e2e.py 16384 1024 16 2 > gpurun_out/trace_trsm.txt 2>&1
echo "trace trsm rc=$?" >> $S
timeout 600 python tools/host_rate_gpu.py 512 1,8 > gpurun_out/host_rate.txt 2>&1
echo "host rate rc=$?" >> $S
timeout 600 python tools/sanitize_small.py > gpurun_out/san_plain.txt 2>&1
echo "san plain rc=$?" >> $S
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_small.py > gpurun_out/san_$tool.txt 2>&1
  echo "sanitizer $tool rc=$?" >> $S
done
