"""Measure the FP64 GEMM peak (cuBLAS DGEMM via torch.matmul) used as the roofline denominator."""
import json, torch
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
for _ in range(3): torch.matmul(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(json.dumps({"dgemm_n": n, "ms": best, "fp64_tflops": 2 * n**3 / best / 1e9}))
