#!/bin/bash
# round 2, part Q: SGEMM 32768^3 DRAM traffic: K split into chained launches and raster group
cd "$(dirname "$0")/.."
O=gpurun_out/q; mkdir -p $O
timeout 900 python tools/sgemm_ksplit.py 32768 4 1,2,4 2,4,8 > $O/ksplit.txt 2>&1
BX_ONCE=1 timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second \
  --clock-control none -k regex:sgemm_tc2c --csv --log-file $O/ncu_ksplit.csv python tools/sgemm_ksplit.py 32768 1 1,2,4 4,8 > $O/ncu.log 2>&1
BX_F32=1 timeout 600 python tools/trace_e2e.py 32768 2048 > $O/trace_cfg5.txt 2>&1
echo done > $O/status.txt
