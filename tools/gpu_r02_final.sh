#!/bin/bash
# round 2, final evidence at HEAD: GPU suite + smoke, every config's bench line (with
# cpu_baseline), the reference arm, the default bench's ncu launch list
cd "$(dirname "$0")/.."
O=gpurun_out/final; mkdir -p $O
timeout 2700 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/status.txt
for c in cfg2 cfg1 cfg3_syrk cfg3_syr2k cfg4_trsm cfg4_trmm dgemm32768 cfg5_sgemm; do
  st=5; [ $c = cfg1 ] && st=20; [ $c = dgemm32768 ] && st=3; [ $c = cfg5_sgemm ] && st=3
  timeout 1500 python bench.py --config $c --steps $st --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
  echo "$c rc=$?" >> $O/status.txt
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_cfg2.json 2> $O/bench_ref_cfg2.err
echo "ref rc=$?" >> $O/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_under_ncu.json 2>&1
python tools/summarize_launches.py $O/launches_cfg2.csv > $O/launches_cfg2.txt 2>&1
echo "ncu rc=$?" >> $O/status.txt
