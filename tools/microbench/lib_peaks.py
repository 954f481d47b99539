"""Measurement only: library GEMM peaks used as roofline denominators
(cuBLAS DGEMM and TF32 GEMM via torch).  Never on the product path."""
import json, torch

def bench(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best

out = {}
n = 8192
a = torch.randn(n, n, device="cuda", dtype=torch.float64); b = torch.randn_like(a)
ms = bench(lambda: a @ b); out["dgemm_8192_tflops"] = 2 * n**3 / ms / 1e9
# syrk-shaped: A^T A via matmul
ms = bench(lambda: a.t() @ a); out["dgemm_AtA_8192_tflops"] = 2 * n**3 / ms / 1e9
torch.backends.cuda.matmul.allow_tf32 = True
af = torch.randn(n, n, device="cuda", dtype=torch.float32); bf = torch.randn_like(af)
ms = bench(lambda: af @ bf); out["tf32_8192_tflops"] = 2 * n**3 / ms / 1e9
at = torch.randn(1048576 // 4, 2048, device="cuda", dtype=torch.float32)
ms = bench(lambda: at.t() @ at); out["tf32_AtA_262144x2048_tflops"] = 2 * at.shape[0] * 2048**2 / ms / 1e9
print(json.dumps(out))
