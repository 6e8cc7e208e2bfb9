"""Comparator: the repo's tcgen05 SGEMM (bx_sgemm_device, TF32 inputs, 2-SM kernel) vs cuBLAS
TF32 (torch matmul with allow_tf32; comparator only, not product code) on the same uniform
[-1,1) operands, alternating launches so both see the same power-cap state.
python tools/sgemm_vs_cublas.py [n,...] [rounds]     (BX_ONCE=1: one launch each, for ncu)"""
import os
import statistics
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1510_05041_b200 import _native as N  # noqa: E402
from paper_1510_05041_b200.engine import get_engine  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = True
sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "16384,32768").split(",")]
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 5
once = os.environ.get("BX_ONCE") == "1"
eng = get_engine([0])
lib = eng.lib
for n in sizes:
    g = torch.Generator(device="cuda").manual_seed(n)
    a = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
    b = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
    c = torch.empty(n, n, device="cuda")
    torch.cuda.synchronize()

    def ours():
        N.check(lib.bx_sgemm_device(0, 0, 0, 0, n, n, n, 1.0, a.data_ptr(), n, b.data_ptr(), n, 0.0,
                                    c.data_ptr(), n), "sgemm")

    def theirs():
        torch.matmul(a, b, out=c)

    if once:
        ours()
        eng.device_sync(0)
        theirs()
        torch.cuda.synchronize()
        continue
    ours(); eng.device_sync(0); theirs(); torch.cuda.synchronize()     # warm-up
    t_ours, t_cub = [], []
    for _ in range(rounds):
        e0 = eng.record(0, 0, timing=True)
        ours()
        e1 = eng.record(0, 0, timing=True)
        eng.sync(e1)
        t_ours.append(eng.elapsed_ms(e0, e1))
        eng.release(e0)
        eng.release(e1)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        theirs()
        s1.record()
        torch.cuda.synchronize()
        t_cub.append(s0.elapsed_time(s1))
    fl = 2.0 * n ** 3
    print(f"n={n}: ours median {statistics.median(t_ours):.2f} ms = {fl / statistics.median(t_ours) / 1e9:.1f} TF/s; "
          f"cuBLAS TF32 median {statistics.median(t_cub):.2f} ms = {fl / statistics.median(t_cub) / 1e9:.1f} TF/s "
          f"(rounds {rounds}, alternating)", flush=True)
