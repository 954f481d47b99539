"""Profiling driver: a few launches of the product kernels on representative
shapes (used under ncu; also prints CUDA-event timings when run plainly).

  python tools/prof_kernel.py [gemm|syrk|fused|all] [m n k] [reps]
"""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_13042_b200 as P  # noqa: E402
from paper_2110_13042_b200 import auto_plan, planner, engine, _native as nat  # noqa: E402


def timed(fn, reps, flops, name):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name}: {ms:.3f} ms  {flops / ms / 1e9:.2f} TFLOP/s", flush=True)


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    m, n, k = (int(x) for x in sys.argv[2:5]) if len(sys.argv) >= 5 else (8192, 4096, 4096)
    reps = int(sys.argv[5]) if len(sys.argv) >= 6 else 3
    dt = torch.float64
    A = torch.rand(m, n, dtype=dt, device="cuda") * 2 - 1
    B = torch.rand(m, k, dtype=dt, device="cuda") * 2 - 1
    if what in ("gemm", "all"):
        C = torch.zeros(n, k, dtype=dt, device="cuda")
        timed(lambda: P.naive_gemm_atb(A, B, C, 1.0), reps, 2.0 * m * n * k, f"gemm {m}x{n}x{k}")
    if what in ("syrk", "all"):
        C = torch.zeros(n, n, dtype=dt, device="cuda")
        timed(lambda: P.naive_syrk_lower(A, C, 1.0), reps, 1.0 * m * n * (n + 1), f"syrk {m}x{n}")
    if what in ("fused", "all"):
        # one Strassen level of C21 += A_r^T A_l, all 7 fused products
        N = n
        C = torch.zeros(N, N, dtype=dt, device="cuda")
        plan = auto_plan.plan_ata_auto(m, N, N, N, auto_plan.AutoParams(leaf_cols=N // 2, max_depth=1, min_dim=1, hbm_gbs=1e9))
        keep = [int(o["type"]) != nat.OP_SYRK for o in plan.ops]

        class SP:
            ops = plan.ops[keep]
        fl = sum(2.0 * int(o["m"]) * int(o["n"]) * int(o["k"]) for o in SP.ops
                 if int(o["type"]) == nat.OP_GEMM)
        ws = torch.empty(max(1, plan.ws_scalars), dtype=dt, device="cuda")
        timed(lambda: engine.run_plan(SP, nat.ATA_F64, int(A.data_ptr()), A.numel(),
                                      int(C.data_ptr()), C.numel(), 1.0, ws=int(ws.data_ptr()),
                                      ws_elems=ws.numel()), reps, fl,
              f"strassen level m={m} n={N} (2 combo4 + 7 products), executed-flop rate")


if __name__ == "__main__":
    main()
