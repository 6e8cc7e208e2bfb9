"""Comparator only: cuBLAS TF32 SGEMM via torch (allow_tf32) on random data."""
import json
import torch
torch.backends.cuda.matmul.allow_tf32 = True
out = []
for n in (8192, 16384):
    a = torch.rand(n, n, device="cuda") * 2 - 1
    b = torch.rand(n, n, device="cuda") * 2 - 1
    c = a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out.append({"n": n, "ms": best, "tflops": 2 * n ** 3 / best / 1e9})
print(json.dumps({"cublas_tf32": out}))
