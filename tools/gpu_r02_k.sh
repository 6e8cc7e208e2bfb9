#!/bin/bash
# round 2, part K: start-up batch (ramp) and launch-shape A/B for cfg2, cfg1, SYRK, TRMM, TRSM
cd "$(dirname "$0")/.."
O=gpurun_out/k; mkdir -p $O
timeout 900 python tools/opts_ab.py gemm 16384 16384 1024 6 'dict()' 'dict(ramp_tasks=64)' 'dict(ramp_tasks=48)' \
  'dict(ramp_tasks=64, ramp_chunk_steps=2)' 'dict(ramp_tasks=16)' 'dict(ramp_chunk_steps=2)' 'dict(ramp_tasks=0)' > $O/ab_cfg2.txt 2>&1
timeout 900 python tools/opts_ab.py gemm 2048 2048 512 30 'dict()' 'dict(ramp_chunk_steps=1)' 'dict(ramp_chunk_steps=2)' \
  'dict(ramp_tasks=0)' 'dict(ramp_tasks=16, ramp_chunk_steps=1)' 'dict(n_streams=4)' 'dict(chunk_steps=2)' \
  'dict(defer_c_move_in=False)' 'dict(ramp_tasks=16, ramp_chunk_steps=2)' > $O/ab_cfg1.txt 2>&1
timeout 900 python tools/opts_ab.py syrk 16384 8192 1024 6 'dict()' 'dict(ramp_chunk_steps=2)' 'dict(ramp_tasks=0)' \
  'dict(ramp_tasks=16)' 'dict(n_streams=16, ramp_chunk_steps=2)' > $O/ab_syrk.txt 2>&1
timeout 900 python tools/opts_ab.py trmm 16384 16384 1024 6 'dict()' 'dict(ramp_chunk_steps=2)' 'dict(ramp_tasks=0)' \
  'dict(ramp_tasks=64)' 'dict(chunk_steps=8)' > $O/ab_trmm.txt 2>&1
timeout 900 python tools/opts_ab.py trsm 16384 16384 1024 6 'dict()' 'dict(ramp_chunk_steps=2)' 'dict(ramp_tasks=0)' \
  'dict(release_on_issue=False)' 'dict(chunk_steps=8)' 'dict(critical_path_weight=4)' > $O/ab_trsm.txt 2>&1
echo done > $O/status.txt
