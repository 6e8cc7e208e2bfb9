#!/bin/bash
# round 2, part L: cluster-launch-control persistent SGEMM (variant 3): correctness, memcheck,
# rate vs variant 1 and vs cuBLAS TF32 (alternating), ncu at 16384^3
cd "$(dirname "$0")/.."
O=gpurun_out/l; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sgemm_tcgen05" > $O/pytest_sgemm.log 2>&1
echo "pytest rc=$?" >> $O/status.txt
BX_SAN_ONLY_SGEMM=1 BX_SAN_SGEMM=3 timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_small.py > $O/memcheck_v3.txt 2>&1
echo "memcheck rc=$?" >> $O/status.txt
BX_LAYOUTS=00,10,01,11 BX_REPS=2 timeout 600 python tools/sgemm_variants.py 16384 1 3 > $O/variants_16384.txt 2>&1
echo "variants rc=$?" >> $O/status.txt
BX_LAYOUTS=00 BX_REPS=2 timeout 600 python tools/sgemm_variants.py 32768 1 3 > $O/variants_32768.txt 2>&1
BX_SGEMM_VARIANT=3 timeout 900 python tools/sgemm_vs_cublas.py 16384,32768 6 > $O/v3_vs_cublas.txt 2>&1
timeout 900 python tools/sgemm_vs_cublas.py 16384,32768 6 > $O/v1_vs_cublas.txt 2>&1
BX_SGEMM_VARIANT=3 BX_ONCE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgemm_tc2c -c 1 -o $O/ncu_sgemm_v3_16384 python tools/sgemm_vs_cublas.py 16384 > $O/ncu_v3.log 2>&1
echo done >> $O/status.txt
