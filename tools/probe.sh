set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/probe_clocks.csv &
SMI=$!
./tools/probe_peaks > gpurun_out/probe_peaks.json 2>&1
true #python tools/cublas_dgemm_ref.py > gpurun_out/cublas_dgemm.json 2>&1
kill $SMI
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
nvidia-smi -q | head -80 > gpurun_out/smi_q.txt
lscpu > gpurun_out/lscpu.txt
cat gpurun_out/probe_peaks.json gpurun_out/cublas_dgemm.json
