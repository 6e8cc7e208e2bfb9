#!/bin/bash
# round 2, part M: GPU suite + smoke with the CLC SGEMM default and the small-call ramp rule;
# cfg5 / cfg1 / cfg2 bench lines; synccheck of the CLC kernel
cd "$(dirname "$0")/.."
O=gpurun_out/m; mkdir -p $O
timeout 2700 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/status.txt
timeout 1500 python bench.py --config cfg5_sgemm --steps 3 --warmup 3 > $O/bench_cfg5_sgemm.json 2> $O/bench_cfg5_sgemm.err
echo "cfg5 rc=$?" >> $O/status.txt
timeout 900 python bench.py --config cfg1 --steps 20 --warmup 3 > $O/bench_cfg1.json 2> $O/bench_cfg1.err
echo "cfg1 rc=$?" >> $O/status.txt
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
echo "cfg2 rc=$?" >> $O/status.txt
BX_SAN_ONLY_SGEMM=1 BX_SAN_SGEMM=3 timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_small.py > $O/synccheck_v3.txt 2>&1
echo "synccheck rc=$?" >> $O/status.txt
BX_SAN_ONLY_SGEMM=1 BX_SAN_SGEMM=3 timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_small.py > $O/racecheck_v3.txt 2>&1
echo "racecheck rc=$?" >> $O/status.txt
