mkdir -p gpurun_out
free -g > gpurun_out/free.txt; nproc >> gpurun_out/free.txt
for t in 1024 2048; do
timeout 900 python bench.py --config dgemm32768 --tile $t --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b32k_$t.json 2> gpurun_out/b32k_$t.err
cat gpurun_out/b32k_$t.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($t, d['value'], d['e2e']['value'], d['e2e']['ms_per_step'], d['clocks'])"
done
timeout 900 python tools/logical_e2e.py 16384 1024 1 2 4 8 > gpurun_out/logical_16k.txt 2>&1
timeout 900 python tools/logical_e2e.py 32768 2048 1 8 > gpurun_out/logical_32k.txt 2>&1
cat gpurun_out/logical_16k.txt gpurun_out/logical_32k.txt
