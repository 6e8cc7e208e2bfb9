#!/bin/bash
# round 2, part O: the one-process-per-GPU path as the driver launches it (torchrun), ranks
# sharing GPU 0 (functional: contexts time-slice), for every routine family
cd "$(dirname "$0")/.."
O=gpurun_out/o; mkdir -p $O
timeout 1200 python -m pytest tests/test_spmd.py -m gpu -q -x > $O/pytest_spmd.log 2>&1
echo "pytest spmd rc=$?" >> $O/status.txt
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 2 --master-port 29511 bench.py --gpus 2 --ranks-share-gpu --config cfg4_trsm --steps 2 --warmup 1 --no-cpu-baseline > $O/trsm_2.json 2> $O/trsm_2.err
echo "trsm 2 rc=$?" >> $O/status.txt
timeout 900 $TR --nproc-per-node 2 --master-port 29512 bench.py --gpus 2 --ranks-share-gpu --config cfg4_trmm --steps 2 --warmup 1 --no-cpu-baseline > $O/trmm_2.json 2> $O/trmm_2.err
echo "trmm 2 rc=$?" >> $O/status.txt
timeout 900 $TR --nproc-per-node 3 --master-port 29513 bench.py --gpus 3 --ranks-share-gpu --config cfg3_syrk --steps 2 --warmup 1 --no-cpu-baseline > $O/syrk_3.json 2> $O/syrk_3.err
echo "syrk 3 rc=$?" >> $O/status.txt
timeout 900 $TR --nproc-per-node 2 --master-port 29514 bench.py --gpus 2 --ranks-share-gpu --config cfg3_syr2k --steps 2 --warmup 1 --no-cpu-baseline > $O/syr2k_2.json 2> $O/syr2k_2.err
echo "syr2k 2 rc=$?" >> $O/status.txt
timeout 1500 $TR --nproc-per-node 2 --master-port 29515 bench.py --gpus 2 --ranks-share-gpu --config cfg5_sgemm --steps 1 --warmup 1 --no-cpu-baseline > $O/sgemm_2.json 2> $O/sgemm_2.err
echo "sgemm 2 rc=$?" >> $O/status.txt
timeout 900 $TR --nproc-per-node 4 --master-port 29516 bench.py --gpus 4 --ranks-share-gpu --steps 2 --warmup 1 --no-cpu-baseline > $O/cfg2_4.json 2> $O/cfg2_4.err
echo "cfg2 4 rc=$?" >> $O/status.txt
timeout 600 $TR --nproc-per-node 2 --master-port 29517 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > $O/ref_2.json 2> $O/ref_2.err
echo "ref 2 rc=$?" >> $O/status.txt
