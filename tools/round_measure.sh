# Round evidence for profiles/ (run under gpurun): every config's bench line, the default
# bench's launch list, and ncu --set full captures of the dominant kernels.
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
for c in cfg1 cfg3_syrk cfg3_syr2k cfg4_trmm cfg4_trsm; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
for t in 1024 2048; do
  timeout 900 python bench.py --config dgemm32768 --tile $t --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_dgemm32768_t$t.json 2> gpurun_out/bench_dgemm32768_t$t.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_task -s 1 -c 1 -o gpurun_out/ncu_dgemm_16384 python tools/prof_gemm.py 16384 0 0 2 > gpurun_out/ncu_dgemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trsm_panel -s 2 -c 1 -o gpurun_out/ncu_trsm_panel python tools/prof_trsm.py 1024 256 > gpurun_out/ncu_trsm.log 2>&1
for f in gpurun_out/bench_*.json; do echo "$f"; python -c "
import json,sys
d=json.load(open('$f')); e=d['e2e']
print('  value %.2f e2e %.2f TF/s %.1f ms frac %.3f clocks %s' % (d['value'], e['value'], e['ms_per_step'], d['roofline']['frac'], d.get('clocks')))" 2>/dev/null; done
