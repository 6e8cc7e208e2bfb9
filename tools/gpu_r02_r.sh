#!/bin/bash
# round 2, part R: batched C loads in the SGEMM / FP64 epilogues — A/B against the previous
# build on host-resident calls, SGEMM K-split / raster group sweep, SGEMM GPU tests
cd "$(dirname "$0")/.."
O=gpurun_out/r; mkdir -p $O
NEW=paper_1510_05041_b200/libblasx_cuda.so; OLD=tools/_ab/libblasx_cuda_prev.so
for r in 1 2 3; do
  for L in $OLD $NEW; do
    timeout 300 python tools/ab_call.py $L gemm 16384 16384 1024 5 >> $O/ab_cfg2.txt 2>&1
    timeout 300 python tools/ab_call.py $L trsm 16384 16384 1024 5 >> $O/ab_trsm.txt 2>&1
    timeout 300 python tools/ab_call.py $L trmm 16384 16384 1024 5 >> $O/ab_trmm.txt 2>&1
    timeout 300 python tools/ab_call.py $L syrk 16384 8192 1024 5 >> $O/ab_syrk.txt 2>&1
  done
done
for r in 1 2; do
  for L in $OLD $NEW; do
    BX_F32=1 timeout 600 python - $L >> $O/ab_sgemm_ksplit.txt 2>&1 <<'PY'
import sys, statistics, ctypes as C
sys.path.insert(0, ".")
from paper_1510_05041_b200 import _native as N
N.load(sys.argv[1])
from paper_1510_05041_b200.engine import get_engine
eng = get_engine([0]); lib = eng.lib
n = 32768
ptrs = []
for i in range(3):
    p = C.c_uint64(); N.check(lib.bx_dev_alloc(0, n * n * 4, C.byref(p)))
    N.check(lib.bx_dev_fill_uniform_f32(0, p.value, n * n, 11 + i, 0)); ptrs.append(p.value)
a, b, c = ptrs
def run(split):
    kc = n // split
    for s in range(split):
        N.check(lib.bx_sgemm_device(0, 0, 0, 0, n, n, kc, 1.0, a + 4 * s * kc * n, n, b + 4 * s * kc, n, 0.0 if s == 0 else 1.0, c, n))
for sp in (1, 2):
    run(sp); eng.device_sync(0)
    ts = []
    for _ in range(3):
        e0 = eng.record(0, 0, timing=True); run(sp); e1 = eng.record(0, 0, timing=True); eng.sync(e1)
        ts.append(eng.elapsed_ms(e0, e1))
    print(f"{sys.argv[1].split('/')[-1]} sgemm 32768^3 K split {sp}: median {statistics.median(ts):.2f} ms {2*n**3/statistics.median(ts)/1e9:.1f} TF/s", flush=True)
PY
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sgemm or medium or variants_match or launch_shape" > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/status.txt
