#!/bin/bash
# round 2, part J: tcgen05 SGEMM vs cuBLAS TF32 (comparator) at 16384^3 and 32768^3,
# alternating launches; ncu DRAM traffic / clock of both at 16384^3
cd "$(dirname "$0")/.."
O=gpurun_out/j; mkdir -p $O
timeout 900 python tools/sgemm_vs_cublas.py 16384,32768 6 > $O/sgemm_vs_cublas.txt 2>&1
BX_ONCE=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum \
  --clock-control none --csv --log-file $O/ncu_sgemm_vs_cublas.csv python tools/sgemm_vs_cublas.py 16384 > $O/ncu_run.log 2>&1
nvidia-smi -q -d POWER > $O/power.txt 2>&1
echo done > $O/status.txt
