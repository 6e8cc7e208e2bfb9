#!/bin/bash
# round 2, part D: 2-SM SGEMM producer tail under synccheck, SGEMM GPU tests, TRSM
# release-on-issue A/B (cfg4), cfg5 / cfg1 / TRSM timelines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
S=gpurun_out/status_d.txt; rm -f $S
BX_SAN_ONLY_SGEMM=1 BX_SAN_SGEMM=0,1,2 timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/san_synccheck_sgemm.txt 2>&1
echo "synccheck sgemm rc=$?" >> $S
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sgemm" > gpurun_out/pytest_sgemm_d.log 2>&1
echo "pytest sgemm rc=$?" >> $S
for r in 1 2; do
  for e in 1 0; do
    timeout 900 python bench.py --config cfg4_trsm --steps 3 --warmup 2 --no-cpu-baseline --release-on-issue $e > gpurun_out/trsm_roi${e}_$r.json 2> gpurun_out/trsm_roi${e}_$r.err
    echo "trsm roi=$e r=$r rc=$?" >> $S
  done
done
BX_KIND=trsm timeout 600 python tools/trace_e2e.py 16384 1024 16 2 > gpurun_out/trace_trsm_d.txt 2>&1
echo "trace trsm rc=$?" >> $S
BX_F32=1 timeout 600 python tools/trace_e2e.py 32768 2048 8 2 > gpurun_out/trace_cfg5.txt 2>&1
echo "trace cfg5 rc=$?" >> $S
timeout 600 python tools/trace_e2e.py 2048 512 8 2 > gpurun_out/trace_cfg1.txt 2>&1
echo "trace cfg1 rc=$?" >> $S
timeout 900 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg1_d.json 2> gpurun_out/bench_cfg1_d.err
echo "bench cfg1 rc=$?" >> $S
