#!/bin/bash
# round 2, part I: TRSM chain split / lookahead, TRMM KM split, SYRK launch shape (interleaved A/B)
cd "$(dirname "$0")/.."
O=gpurun_out/i; mkdir -p $O
timeout 900 python tools/opts_ab.py trsm 16384 16384 1024 8 'dict(trsm_split_chain=False)' 'dict()' \
  'dict(tasks_per_stream=3)' 'dict(tasks_per_stream=4)' 'dict(n_streams=12)' 'dict(n_streams=12, tasks_per_stream=3)' \
  'dict(trsm_split_chain=False, tasks_per_stream=3)' > $O/ab_trsm.txt 2>&1
timeout 900 python tools/opts_ab.py trmm 16384 16384 1024 8 'dict()' 'dict(split_km=True)' \
  'dict(split_km=True, tasks_per_stream=3)' 'dict(n_streams=12)' 'dict(split_km=True, n_streams=12)' > $O/ab_trmm.txt 2>&1
timeout 900 python tools/opts_ab.py syrk 16384 8192 1024 8 'dict()' 'dict(n_streams=16)' 'dict(tasks_per_stream=3)' \
  'dict(chunk_steps=8)' 'dict(n_streams=8)' > $O/ab_syrk.txt 2>&1
echo done > $O/status.txt
