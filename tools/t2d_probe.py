import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2110_13042_b200 as P
case = sys.argv[1]
m = 300
if case == "aligned_ragged":   off, n, k, ld = 0, 129, 77, 214
elif case == "aligned_16":     off, n, k, ld = 0, 128, 64, 214
elif case == "mis_16":         off, n, k, ld = 1, 128, 64, 214
elif case == "aligned_even":   off, n, k, ld = 0, 130, 78, 214
elif case == "mis_even":       off, n, k, ld = 1, 130, 78, 214
else:                          off, n, k, ld = 1, 129, 77, 214
big = torch.rand(m, ld, dtype=torch.float64, device="cuda")
a = big[:, off:off + n]; b = big[:, off + n + (off + n) % 2: off + n + (off + n) % 2 + k] if case == "aligned_16" else big[:, off + n:off + n + k]
C = torch.zeros((n, k), dtype=torch.float64, device="cuda")
P.naive_gemm_atb(a, b, C, 1.0)
torch.cuda.synchronize()
ref = a.cpu().numpy().T @ b.cpu().numpy()
print(case, np.abs(C.cpu().numpy() - ref).max())
