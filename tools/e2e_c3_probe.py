"""e2e probe at the c3 shape (16384^2 fp64, pinned host A and C through ata()):
wall time per geometric-pipeline setting (min ratio, block count)."""
import os, sys, time, importlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_13042_b200 as P
mod = importlib.import_module("paper_2110_13042_b200.ata")
m = n = 16384
hA = torch.empty((m, n), dtype=torch.float64).pin_memory(); hA.uniform_(-1, 1)
hC = torch.zeros((n, n), dtype=torch.float64).pin_memory()
for thr, R in ((4.0, 3), (2.0, 2), (4.0, 3), (2.0, 2)):
    mod.PIPELINE_GEOMETRIC_MIN_RATIO = mod.PIPELINE_GEOMETRIC_MIN_RATIO2 = thr; mod.PIPELINE_GEOMETRIC_BLOCKS = R
    ts = []
    for _ in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        P.ata(hA, hC, 1.0, threshold="auto", auto_params=os.environ.get("AUTO_PARAMS")); torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(thr, R, [b for _, b in mod._row_blocks(m, n, 8, False)], " ".join(f"{1e3*t:.1f}" for t in ts), flush=True)
