"""e2e (host pinned A and C through ata()) per row-block layout of the host pipeline:
each argument is a comma-separated list of block row counts summing to m.

  python tools/e2e_blocks.py m n 3346,12849,49341 8192,57344 ...
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
    layouts = [[int(x) for x in arg.split(",")] for arg in sys.argv[3:]]
    mod = importlib.import_module("paper_2110_13042_b200.ata")
    hA = torch.empty((m, n), dtype=torch.float64).pin_memory()
    hA.uniform_(-1, 1)
    hC = torch.zeros((n, n), dtype=torch.float64).pin_memory()
    default = mod._row_blocks
    for rows in [None] + layouts:
        if rows is None:
            mod._row_blocks = default
            name = "default " + ",".join(str(r) for _, r in default(m, n, 8, False))
        else:
            assert sum(rows) == m, rows
            cuts, r0 = [], 0
            for r in rows:
                cuts.append((r0, r))
                r0 += r
            mod._row_blocks = lambda *a, cuts=cuts: list(cuts)
            name = ",".join(str(r) for r in rows)
        try:
            P.ata(hA, hC, 1.0, threshold="auto")
            ts = []
            for _ in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                P.ata(hA, hC, 1.0, threshold="auto")
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t0)
            t = sorted(ts)[1]
            print(f"blocks {name}: {t * 1e3:8.1f} ms  {m * n * n / t / 1e12:6.2f} TF/s", flush=True)
        except Exception as e:      # e.g. out of memory for a layout
            print(f"blocks {name}: failed {type(e).__name__}: {str(e)[:200]}", flush=True)
        P.release_cached_buffers()


if __name__ == "__main__":
    main()
