#!/bin/bash
# round 2, closing evidence at HEAD: three default bench runs (run-to-run spread of the
# headline), every other config once, the reference arm
cd "$(dirname "$0")/.."
O=gpurun_out/final2; mkdir -p $O
for r in 1 2 3; do
  timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_cfg2_run$r.json 2> $O/bench_cfg2_run$r.err
  echo "cfg2 run $r rc=$?" >> $O/status.txt
done
for c in cfg1 cfg3_syrk cfg3_syr2k cfg4_trsm cfg4_trmm dgemm32768 cfg5_sgemm; do
  st=5; [ $c = cfg1 ] && st=20; [ $c = dgemm32768 ] && st=3; [ $c = cfg5_sgemm ] && st=3
  timeout 1500 python bench.py --config $c --steps $st --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
  echo "$c rc=$?" >> $O/status.txt
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_cfg2.json 2> $O/bench_ref_cfg2.err
echo "ref rc=$?" >> $O/status.txt
