#!/bin/bash
# round 2, part N: small-call prefetch A/B (cfg1), GPU tests touching it, spmd fixed cost
cd "$(dirname "$0")/.."
O=gpurun_out/n; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "launch_shape or medium or cfg1 or variants_match" > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/status.txt
timeout 900 python tools/opts_ab.py gemm 2048 2048 512 40 'dict(prefetch=0)' 'dict()' 'dict(prefetch=0, ramp_tasks=4)' > $O/ab_cfg1.txt 2>&1
timeout 900 python tools/opts_ab.py gemm 4096 4096 1024 20 'dict(prefetch=0)' 'dict()' > $O/ab_4096.txt 2>&1
timeout 900 python tools/opts_ab.py syrk 4096 2048 512 20 'dict(prefetch=0)' 'dict()' > $O/ab_syrk4096.txt 2>&1
timeout 900 python bench.py --config cfg1 --steps 20 --warmup 3 > $O/bench_cfg1.json 2> $O/bench_cfg1.err
echo "cfg1 rc=$?" >> $O/status.txt
timeout 900 python bench.py --config cfg1 --gpus 2 --ranks-share-gpu --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg1_spmd2.json 2> $O/bench_cfg1_spmd2.err
echo "spmd2 rc=$?" >> $O/status.txt
timeout 900 python bench.py --gpus 2 --ranks-share-gpu --steps 3 --warmup 2 --no-cpu-baseline > $O/bench_cfg2_spmd2.json 2> $O/bench_cfg2_spmd2.err
echo "spmd2 cfg2 rc=$?" >> $O/status.txt
