"""e2e (host pinned A and C through ata()) with uniform vs geometric row
blocks of the host pipeline (ata._row_blocks).  python tools/e2e_ab.py m n"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_13042_b200 as P  # noqa: E402
import importlib  # noqa: E402
mod = importlib.import_module("paper_2110_13042_b200.ata")

m, n = int(sys.argv[1]), int(sys.argv[2])
hA = torch.empty((m, n), dtype=torch.float64).pin_memory()
hA.uniform_(-1, 1)
hC = torch.zeros((n, n), dtype=torch.float64).pin_memory()
for geo, blocks in ((False, 0), (True, 3), (True, 4), (True, 5)):
    mod.PIPELINE_GEOMETRIC = geo
    if blocks:
        mod.PIPELINE_GEOMETRIC_BLOCKS = blocks
    P.ata(hA, hC, 1.0, threshold="auto")
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.ata(hA, hC, 1.0, threshold="auto")
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    print(f"geometric={geo} R={blocks or 'uniform'}: {t * 1e3:8.1f} ms  {m * n * n / t / 1e12:6.2f} TF/s "
          f"blocks={[b for _, b in mod._row_blocks(m, n, 8, False)]}", flush=True)
