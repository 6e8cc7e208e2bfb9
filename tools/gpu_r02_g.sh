#!/bin/bash
# round 2, part G: host-link bandwidth per tile shape / copy streams; the inverse-based TRSM
# diagonal step (correctness, ncu --set full of its kernels); the cfg4 TRSM call's launch list
cd "$(dirname "$0")/.."
O=gpurun_out/g; mkdir -p $O
timeout 300 ./tools/h2d_tiles > $O/h2d_tiles.txt 2>&1
timeout 300 python tools/prof_trsm_inv.py 1024 3 > $O/trsm_inv.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_trsm.csv \
  python bench.py --config cfg4_trsm --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_trsm_under_ncu.json 2>&1
python tools/summarize_launches.py $O/launches_trsm.csv > $O/launches_trsm.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -s 9 -c 12 -o $O/ncu_trsm_inv \
  python tools/prof_trsm_inv.py 1024 3 > $O/ncu_trsm_inv.log 2>&1
echo done > $O/status.txt
