"""cuBLAS DGEMM ceiling probe (reference only, never on the product path)."""
import json, torch
torch.backends.cuda.matmul.allow_tf32 = False
for n in (2048, 4096, 8192):
    a = torch.rand(n, n, dtype=torch.float64, device="cuda")
    b = torch.rand(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(json.dumps({"kind": "cublas_dgemm", "n": n, "ms": best, "tflops": 2 * n**3 / best / 1e9}))
