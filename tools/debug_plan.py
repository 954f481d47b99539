"""Bisect a plan's GPU execution against the NumPy interpreter (tests/plan_interp.py):
runs growing prefixes of the op list on both and reports the first op after
which C or the workspace differ.

  python tools/debug_plan.py m n threshold
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import plan_interp  # noqa: E402
from paper_2110_13042_b200 import engine, ref_bfs, _native as nat  # noqa: E402


class Sub:
    def __init__(self, ops):
        self.ops = ops


def main():
    m, n, t = (int(x) for x in sys.argv[1:4])
    a = np.random.default_rng(0).standard_normal((m, n))
    plan = ref_bfs.plan_ata_reference_bfs(m, n, n, n, t)
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
        dc = np.abs(C.cpu().numpy() - np.tril(c)).max()
        dw = np.abs(W.cpu().numpy() - ws).max()
        return dc > 1e-9 or dw > 1e-9, dc, dw

    print(len(plan.ops), "ops")
    lo, hi = 0, len(plan.ops)          # invariant: prefix lo agrees, prefix hi diverges
    if not diverged(hi)[0]:
        print("no divergence")
        return
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if diverged(mid)[0]:
            hi = mid
        else:
            lo = mid
    for end in [hi]:
        _, dc, dw = diverged(end)
        if True:
            op = plan.ops[end - 1]
            print(f"first divergence after op {end - 1}: type {int(op['type'])} group {int(op['group'])} "
                  f"m,n,k=({int(op['m'])},{int(op['n'])},{int(op['k'])}) dC={dc:.3e} dWS={dw:.3e}")
            print(op)
            prev = plan.ops[max(0, end - 4):end - 1]
            print("previous ops types/groups:", [(int(o["type"]), int(o["group"])) for o in prev])


if __name__ == "__main__":
    main()
