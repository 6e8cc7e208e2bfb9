#!/bin/bash
# round 2, part C: DGEMM kernel with the KM template split (A/B vs pre-kmode build), cfg2 /
# cfg4 TRMM bench, ncu capture + launch list of the fixed kernel, sanitizer follow-ups
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
S=gpurun_out/status_c.txt; rm -f $S gpurun_out/ab_dgemm_c.txt
for r in 1 2 3; do
  for lib in tools/_ab/libblasx_cuda_pre_kmode.so tools/_ab/libblasx_cuda_km.so; do
    timeout 300 python tools/ab_dgemm.py $lib 16384 3 >> gpurun_out/ab_dgemm_c.txt 2>&1
  done
done
echo "ab rc=$?" >> $S
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_c.json 2> gpurun_out/bench_cfg2_c.err
echo "bench cfg2 rc=$?" >> $S
timeout 900 python bench.py --config cfg4_trmm --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_trmm_c.json 2> gpurun_out/bench_trmm_c.err
echo "bench trmm rc=$?" >> $S
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_c.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu_c.json 2>&1
echo "launches rc=$?" >> $S
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_task -s 1 -c 1 -o gpurun_out/ncu_dgemm_16384_c python tools/prof_gemm.py 16384 0 0 2 > gpurun_out/ncu_dgemm_c.log 2>&1
echo "ncu dgemm rc=$?" >> $S
BX_SAN_SGEMM=0,2 timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/san_synccheck_no2sm.txt 2>&1
echo "synccheck no 2-SM rc=$?" >> $S
BX_GEMM_VARIANT=1 BX_SAN_SGEMM= timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/san_racecheck_variant1.txt 2>&1
echo "racecheck variant1 rc=$?" >> $S
