"""Accumulation bias of the f32 product paths on long contractions: relative
error of the Gram diagonal (all-positive sums) vs fp64, per precision mode.

  python tools/acc_bias.py [m n]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2110_13042_b200 as P  # noqa: E402


def main():
    m, n = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) >= 3 else (1 << 20, 256)
    a = torch.randn(m, n, device="cuda")
    ref = (a.double() ** 2).sum(0).cpu().numpy()
    for prec in ("fp32", "tf32"):
        C = torch.zeros(n, n, device="cuda")
        P.ata(a, C, 1.0, threshold="auto", precision=prec)
        d = torch.diagonal(C).double().cpu().numpy()
        rel = (d - ref) / ref
        print(f"{prec}: diag rel error mean {rel.mean():+.2e}  max|.| {np.abs(rel).max():.2e}", flush=True)


if __name__ == "__main__":
    main()
