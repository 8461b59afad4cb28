"""cuBLAS DGEMM (torch.matmul float64) as the FP64 sanity bar for the DMMA roofline."""
import json, torch
torch.backends.cuda.matmul.allow_tf32 = False
res = {}
for n in (4096, 8192, 16384):
    a = torch.rand(n, n, dtype=torch.float64, device="cuda")
    b = torch.rand(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); torch.matmul(a, b); e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e))
    res[f"cublas_dgemm_{n}_tflops"] = round(2 * n**3 / best / 1e9, 2)
print(json.dumps(res))
