#!/bin/bash
# round 2: host issue rate before/after (round-1 runtime in tools/_r1pkg vs this tree),
# logical-device DGEMM, TRSM timeline
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/status_c.txt
timeout 600 python tools/host_rate_gpu.py 512 1,8 > gpurun_out/host_rate_new.txt 2>&1
echo "hr new rc=$?" >> gpurun_out/status_c.txt
BX_PKG_ROOT=tools/_r1pkg timeout 600 python tools/host_rate_gpu.py 512 1,8 > gpurun_out/host_rate_r1.txt 2>&1
echo "hr r1 rc=$?" >> gpurun_out/status_c.txt
timeout 600 python tools/logical_e2e.py 16384 1024 1 8 > gpurun_out/logical_new.txt 2>&1
echo "logical rc=$?" >> gpurun_out/status_c.txt
BX_KIND=trsm timeout 600 python tools/trace_e2e.py 16384 1024 16 2 0 > gpurun_out/trace_trsm.txt 2>&1
echo "trace rc=$?" >> gpurun_out/status_c.txt
for c in cfg3_syrk cfg3_syr2k cfg4_trmm dgemm32768; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "bench $c rc=$?" >> gpurun_out/status_c.txt
done
