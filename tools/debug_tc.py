"""Debug harness for the tcgen05 TF32 kernel: small structured GEMMs, prints
where the result deviates from the fp64 reference."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2110_13042_b200 import planner, engine, _native as nat

def run(a, b):
    m, n = a.shape; k = b.shape[1]
    A = torch.from_numpy(a).cuda(); B = torch.from_numpy(b).cuda()
    C = torch.full((n, k), float("nan"), device="cuda")
    pb = planner.PlanBuilder("t")
    pb.product("gemm", m, n, k, [(planner.Win(0, 0, n, m, n), 1.0)], [(planner.Win(3, 0, k, m, k), 1.0)],
               [(planner.Win(1, 0, k, n, k), 1.0)], accumulate=0, group=1)
    engine.run_plan(pb.finish(), nat.ATA_TF32, A.data_ptr(), A.numel(), C.data_ptr(), C.numel(), 1.0,
                    B=B.data_ptr(), b_elems=B.numel())
    torch.cuda.synchronize()
    return C.cpu().numpy()

np.set_printoptions(linewidth=200, precision=3, suppress=True)
m, n, k = 32, 128, 256
# case 1: A = e_0 outer (row 0 all ones) ... use A[l, i] = (l == 0) * (i + 1), B[l, j] = (l == 0) * 1
a = np.zeros((m, n), np.float32); b = np.zeros((m, k), np.float32)
a[0, :] = np.arange(1, n + 1); b[0, :] = 1.0
c = run(a, b)
ref = a.T.astype(np.float64) @ b
print("case1 max|c|", np.abs(c).max(), "err", np.abs(c - ref).max())
print("c[:8,:8]\n", c[:8, :8]); print("ref rows 0..7 col0", ref[:8, 0])
# where do values land? for each row i of ref (value i+1), find rows in c containing i+1
nz = np.argwhere(np.abs(c) > 0)
print("nonzeros", len(nz), nz[:10])
# case 2: B varies along cols
a = np.zeros((m, n), np.float32); b = np.zeros((m, k), np.float32)
a[0, :] = 1.0; b[0, :] = np.arange(1, k + 1)
c = run(a, b)
print("case2 err", np.abs(c - (a.T.astype(np.float64) @ b)).max(), "c[0,:40]", c[0, :40])
# case 3: contraction structure: a[l, 0] = 1 for all l, b[l, 0] = l+1
a = np.zeros((m, n), np.float32); b = np.zeros((m, k), np.float32)
a[:, 0] = 1.0; b[:, 0] = np.arange(1, m + 1)
c = run(a, b)
print("case3 c[0,0]", c[0, 0], "ref", (a.T.astype(np.float64) @ b)[0, 0])
# random
a = np.random.default_rng(0).standard_normal((m, n)).astype(np.float32)
b = np.random.default_rng(1).standard_normal((m, k)).astype(np.float32)
c = run(a, b); ref = a.T.astype(np.float64) @ b
print("random rel err", np.linalg.norm(c - ref) / np.linalg.norm(ref))

# stage-0 smem dump of the first k-block (needs ATA_TC_DEBUG=1): case a[l,i] = 1000*l + i
import ctypes
if os.environ.get("ATA_TC_DEBUG"):
    m, n, k = 32, 128, 256
    a = (1000.0 * np.arange(m)[:, None] + np.arange(n)[None, :]).astype(np.float32)
    b = (-(1000.0 * np.arange(m)[:, None] + np.arange(k)[None, :])).astype(np.float32)
    run(a, b)
    lib = nat.load()
    buf = np.zeros(12288, dtype=np.float32)
    rc = lib.ata_tc_debug_copy(buf.ctypes.data_as(ctypes.c_void_p), 12288)
    print("debug copy rc", rc)
    A_s = buf[:4096]
    print("A smem first 40:", A_s[:40])
    print("A smem [256:296]:", A_s[256:296])
    print("A smem [1024:1064]:", A_s[1024:1064])
    B_s = buf[4096:]
    print("B smem first 40:", B_s[:40])
    buf = np.zeros(12288 + 4096, dtype=np.float32)
    lib.ata_tc_debug_copy(buf.ctypes.data_as(ctypes.c_void_p), 12288 + 4096)
    T = buf[12288:].reshape(128, 32)
    ref = a.T.astype(np.float64) @ b
    print("TMEM rows 0..3, cols 0..7:\n", T[:4, :8]); print("ref:\n", ref[:4, :8])
    print("TMEM max abs", np.abs(T).max())
