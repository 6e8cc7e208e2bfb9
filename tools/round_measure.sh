# bench + ncu evidence for profiles/ (run under gpurun)
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 1500 python bench.py --config cfg5_sgemm --steps 2 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
cat gpurun_out/bench_cfg5.json; tail -3 gpurun_out/bench_cfg5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_task -s 1 -c 1 -o gpurun_out/prof_gemm_16384 python tools/prof_gemm.py 16384 0 0 2 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgemm_tc -s 1 -c 1 -o gpurun_out/prof_sgemm_16384 python tools/kernel_check.py --sgemm-only-perf > gpurun_out/ncu_sgemm.log 2>&1
tail -2 gpurun_out/ncu_full.log gpurun_out/ncu_sgemm.log
