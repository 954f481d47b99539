"""Riding operand sums (ATA_OPF_RIDE): correctness of forced depth-first auto
plans against the BLAS Gram, and that product launches actually carried sums."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import atamul_oracle as O
import paper_2110_13042_b200 as P
from paper_2110_13042_b200 import _native as nat
from paper_2110_13042_b200.auto_plan import AutoParams

rng = np.random.default_rng(11)
lib = nat.load()
for (m, n, kw) in [(4096, 2048, dict(leaf_cols=256, min_dim=128, ws_budget_gb=0.02, max_depth=3, hbm_gbs=1e9, ride_gbs=1e12)),
                   (3000, 1536, dict(leaf_cols=256, min_dim=128, ws_budget_gb=0.01, max_depth=3, hbm_gbs=1e9, ride_gbs=1e12)),
                   (2050, 1100, dict(leaf_cols=256, min_dim=128, ws_budget_gb=0.005, max_depth=3, hbm_gbs=1e9, ride_gbs=1e12)),
                   (8192, 4096, dict(ws_budget_gb=0.2))]:
    A = torch.from_numpy(rng.uniform(-1, 1, (m, n))).cuda()
    want = O.gram_blas(A.cpu().numpy())
    for rep in range(3):
        C = torch.zeros(n, n, dtype=torch.float64, device="cuda")
        r0 = lib.ata_ride_count()
        P.ata(A, C, 1.0, threshold="auto", auto_params=AutoParams(**kw))
        torch.cuda.synchronize()
        err = O.rel_frobenius_lower(C.cpu().numpy(), want)
        print(f"ride_check {m}x{n} rep {rep}: rel err {err:.2e}, rides {lib.ata_ride_count() - r0}", flush=True)
        assert err < 1e-12, err
print("ride_check ok")
