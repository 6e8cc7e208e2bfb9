#!/bin/bash
# round 2: host issue rate after event skipping (+ profile), TRSM early-inverse A/B,
# sanitizer follow-ups (synccheck per kernel family, racecheck on the __syncthreads GEMM)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/status_e.txt
BX_PROF=1 timeout 600 python tools/host_rate_gpu.py 512 1,8 > gpurun_out/host_rate_new2.txt 2>&1
echo "hr rc=$?" >> gpurun_out/status_e.txt
for r in 1 2 3; do
  for e in 0 1; do
    BX_TRSM_EARLY_INV=$e timeout 900 python bench.py --config cfg4_trsm --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/trsm_ab_${e}_$r.json 2>/dev/null
  done
done
echo "ab done" >> gpurun_out/status_e.txt
BX_SAN_SGEMM=0 timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/san_synccheck_v0.txt 2>&1
echo "synccheck v0 rc=$?" >> gpurun_out/status_e.txt
BX_SAN_ONLY_SGEMM=1 BX_SAN_SGEMM=2 timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/san_synccheck_v2.txt 2>&1
echo "synccheck v2 rc=$?" >> gpurun_out/status_e.txt
BX_GEMM_VARIANT=1 BX_SAN_SGEMM= timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/san_racecheck_variant1.txt 2>&1
echo "racecheck variant1 rc=$?" >> gpurun_out/status_e.txt
