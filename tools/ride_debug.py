"""Bisect an auto plan's GPU execution against the NumPy interpreter
(tests/plan_interp.py): python tools/ride_debug.py m n budget_gb ride_sums(0/1)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import plan_interp  # noqa: E402
from paper_2110_13042_b200 import engine, _native as nat  # noqa: E402
from paper_2110_13042_b200.auto_plan import plan_ata_auto, AutoParams  # noqa: E402


class Sub:
    def __init__(self, ops):
        self.ops = ops


def main():
    m, n = int(sys.argv[1]), int(sys.argv[2])
    budget, ride = float(sys.argv[3]), bool(int(sys.argv[4]))
    a = np.random.default_rng(0).standard_normal((m, n))
    plan = plan_ata_auto(m, n, n, n, AutoParams(leaf_cols=256, min_dim=128, ws_budget_gb=budget, max_depth=3,
                                                hbm_gbs=1e9, ride_sums=ride))
    ws_n = max(1, plan.ws_scalars)
    A = torch.from_numpy(a).cuda()

    def diverged(end):
        c = np.zeros((n, n))
        ws = np.zeros(ws_n)
        plan_interp.run(plan.ops[:end], a, c, 1.0, WS=ws)
        C = torch.zeros(n, n, dtype=torch.float64, device="cuda")
        W = torch.zeros(ws_n, dtype=torch.float64, device="cuda")
        engine.run_plan(Sub(np.ascontiguousarray(plan.ops[:end])), nat.ATA_F64, A.data_ptr(), A.numel(),
                        C.data_ptr(), C.numel(), 1.0, ws=W.data_ptr(), ws_elems=W.numel())
        torch.cuda.synchronize()
        dc = np.abs(np.tril(C.cpu().numpy()) - np.tril(c)).max()
        dw = np.abs(W.cpu().numpy() - ws).max()
        return dc > 1e-9 or dw > 1e-9, dc, dw

    print(len(plan.ops), "ops, ride flags", int((plan.ops["flags"] & 1).sum()), "rides so far", nat.load().ata_ride_count())
    lo, hi = 0, len(plan.ops)
    bad, dc, dw = diverged(hi)
    if not bad:
        print("no divergence", dc, dw)
        return
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if diverged(mid)[0]:
            hi = mid
        else:
            lo = mid
    _, dc, dw = diverged(hi)
    op = plan.ops[hi - 1]
    print(f"first divergence after op {hi - 1}: type {int(op['type'])} group {int(op['group'])} flags {int(op['flags'])} "
          f"m,n,k=({int(op['m'])},{int(op['n'])},{int(op['k'])}) dC={dc:.3e} dWS={dw:.3e}")
    for o in plan.ops[max(0, hi - 6):hi + 2]:
        print(int(o["type"]), int(o["group"]), int(o["flags"]), int(o["m"]), int(o["n"]), int(o["k"]),
              [(int(r["base"]), int(r["off"]), int(r["ld"]), int(r["rows"]), int(r["cols"])) for r in o["s"][:int(o["ns"])]],
              [(int(r["base"]), int(r["off"]), int(r["ld"]), int(r["rows"]), int(r["cols"])) for r in o["t"][:int(o["nt"])]],
              [(int(r["base"]), int(r["off"]), int(r["ld"]), int(r["rows"]), int(r["cols"]), int(r["region"])) for r in o["d"][:int(o["nd"])]])


if __name__ == "__main__":
    main()
