#!/bin/bash
# round 2, part H: every config's bench line at HEAD (with cpu_baseline), the reference arm
cd "$(dirname "$0")/.."
O=gpurun_out/h; mkdir -p $O
for c in cfg2 cfg1 cfg3_syrk cfg3_syr2k cfg4_trsm cfg4_trmm dgemm32768 cfg5_sgemm; do
  st=5; [ $c = cfg1 ] && st=20; [ $c = dgemm32768 ] && st=3; [ $c = cfg5_sgemm ] && st=3
  timeout 1500 python bench.py --config $c --steps $st --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
  echo "$c rc=$?" >> $O/status.txt
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_cfg2.json 2> $O/bench_ref_cfg2.err
echo "ref rc=$?" >> $O/status.txt
