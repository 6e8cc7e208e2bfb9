"""Comparator only (never on the product path): cuBLAS DGEMM through torch.matmul on
float64, to put the FP64 DMMA probe next to the vendor library's achieved rate."""
import json, time, torch

def run(n, reps=5):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return {"n": n, "ms": best, "tflops": 2 * n ** 3 / best / 1e9}

out = {"cublas_dgemm": [run(n) for n in (1024, 4096, 8192, 16384)]}
print(json.dumps(out))
