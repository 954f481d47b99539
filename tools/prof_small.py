"""Throughput of many small leaf products in one group (the breadth-first
reference plans' leaf phase): 1-term vs 2-term (fused Strassen sum) operands.

  python tools/prof_small.py [count m n k]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_13042_b200 import engine, planner, _native as nat  # noqa: E402
from paper_2110_13042_b200.planner import Win  # noqa: E402


def main():
    cnt, m, n, k = (int(x) for x in sys.argv[1:5]) if len(sys.argv) >= 5 else (2048, 188, 128, 128)
    A = torch.randn(cnt * m * (n + k), dtype=torch.float64, device="cuda")
    C = torch.zeros(cnt * n * k, dtype=torch.float64, device="cuda")
    for terms in (1, 2):
        pb = planner.PlanBuilder("t")
        g = pb.new_group()
        for i in range(cnt):
            base = i * m * (n + k)
            a = Win(nat.BASE_A, base, n + k, m, n)
            b = Win(nat.BASE_A, base + n, n + k, m, k)
            S = [(a, 1.0)] + ([(a, -1.0)] if terms == 2 else [])
            T = [(b, 1.0)] + ([(b, 1.0)] if terms == 2 else [])
            pb.product("gemm", m, n, k, S, T, [(Win(nat.BASE_C, i * n * k, k, n, k), 1.0)], accumulate=0, group=g)
        plan = pb.finish()
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            engine.run_plan(plan, nat.ATA_F64, A.data_ptr(), A.numel(), C.data_ptr(), C.numel(), 1.0)
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"{cnt} products {m}x{n}x{k}, {terms}-term operands: {ms:.3f} ms, "
              f"{2.0 * cnt * m * n * k / ms / 1e9:.2f} TFLOP/s, {ms * 1e3 / cnt * 148 / 1.0:.1f} us per tile-wave",
              flush=True)


if __name__ == "__main__":
    main()
