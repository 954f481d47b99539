"""e2e (host pinned A and C through ata()) vs the pipeline's row-block size.

  python tools/e2e_sweep.py m n GB [GB ...]
"""
import importlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_13042_b200 as P  # noqa: E402


def main():
    m, n = int(sys.argv[1]), int(sys.argv[2])
    sizes = [float(x) for x in sys.argv[3:]] or [4.0]
    mod = importlib.import_module("paper_2110_13042_b200.ata")
    hA = torch.empty((m, n), dtype=torch.float64).pin_memory()
    hA.uniform_(-1, 1)
    hC = torch.zeros((n, n), dtype=torch.float64).pin_memory()
    for gb in sizes:
        mod.PIPELINE_BLOCK_BYTES = int(gb * (1 << 30))
        P.ata(hA, hC, 1.0, threshold="auto")
        ts = []
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            P.ata(hA, hC, 1.0, threshold="auto")
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        t = min(ts)
        print(f"block {gb:5.1f} GB: {t * 1e3:8.1f} ms  {m * n * n / t / 1e12:6.2f} TF/s", flush=True)


if __name__ == "__main__":
    main()
