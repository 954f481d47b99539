"""e2e of the pinned-host pipeline (c4 shape), wall time of ata() on host A/C."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_13042_b200 as P
m, n = int(sys.argv[1]), int(sys.argv[2])
hA = torch.empty((m, n), dtype=torch.float64).pin_memory(); hA.uniform_(-1, 1)
hC = torch.zeros((n, n), dtype=torch.float64).pin_memory()
ts = []
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    P.ata(hA, hC, 1.0, threshold="auto"); torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(f"zero_c={os.environ.get('ATA_PIPE_ZERO_C','0')} {m}x{n}: " + " ".join(f"{1e3*t:.1f}" for t in ts) + " ms", flush=True)
