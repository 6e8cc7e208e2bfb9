#!/bin/bash
# round 2, part F: where the rank-k / triangular routines and the small cfg1 call lose time:
# host cost per task on the box's CPU (no-op ABI), traced timelines (kernel concurrency,
# H2D busy) and link-stubbed runs per routine
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/f; mkdir -p $O
lscpu > $O/lscpu.txt 2>&1
timeout 300 python tools/host_cost.py 2048 512 1 > $O/host_cost.txt 2>&1
timeout 300 python tools/host_cost.py 16384 1024 1 >> $O/host_cost.txt 2>&1
timeout 300 python tools/host_cost.py 16384 1024 8 >> $O/host_cost.txt 2>&1
BX_KIND=gemm timeout 300 python tools/trace_e2e.py 2048 512 > $O/trace_cfg1.txt 2>&1
BX_KIND=gemm timeout 600 python tools/trace_e2e.py 16384 1024 > $O/trace_cfg2.txt 2>&1
BX_KIND=trsm timeout 600 python tools/trace_e2e.py 16384 1024 > $O/trace_trsm.txt 2>&1
BX_KIND=trmm timeout 600 python tools/trace_e2e.py 16384 1024 > $O/trace_trmm.txt 2>&1
BX_KIND=syrk BX_K=8192 timeout 600 python tools/trace_e2e.py 16384 1024 > $O/trace_syrk.txt 2>&1
BX_KIND=syr2k BX_K=8192 timeout 600 python tools/trace_e2e.py 16384 1024 > $O/trace_syr2k.txt 2>&1
for k in trsm trmm; do BX_IC=0 BX_KIND=$k timeout 900 python tools/nolink_e2e.py 16384 > $O/nolink_$k.txt 2>&1; done
BX_IC=0 BX_KIND=syrk BX_K=8192 timeout 900 python tools/nolink_e2e.py 16384 > $O/nolink_syrk.txt 2>&1
echo done > $O/status.txt
