"""Riding-sums throughput probe: one FP64 product group (nprod products of
m x 1024 x 1024) carrying `nodes` operand-sum nodes of rows x cols quadrants,
timed with CUDA events; nprod = 0 runs the ride behind one 128^3 product (the
ride alone).  Run once per library variant (ATA_LIB_PATH):

  python tools/ride_ab.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_13042_b200 import _native as nat, engine, planner  # noqa: E402
from paper_2110_13042_b200.planner import Win  # noqa: E402

S_COEFS = [(1, 0, 0, 1), (0, 1, 0, 1), (1, 0, 1, 0), (-1, 1, 0, 0), (0, 0, 1, -1)]


def plan_for(nprod, m, nodes, rows, cols, lda=32768):
    w = 1024
    pb = planner.PlanBuilder("ride-ab")
    ws_top = 0
    moved = 0
    # operand-sum nodes: quadrants of windows of A -> five sums each in the workspace
    for i in range(nodes):
        r0 = (i % 2) * 2 * rows
        c0 = ((i // 2) * 2 * cols) % (lda - 2 * cols)
        X = [Win(nat.BASE_A, (r0 + dr * rows) * lda + c0 + dc * cols, lda, rows, cols) for dr in (0, 1) for dc in (0, 1)]
        outs = []
        for coef in S_COEFS:
            outs.append((Win(nat.BASE_WS, ws_top, cols, rows, cols), coef))
            ws_top += rows * cols
        pb.combo4(X, outs)
        moved += 9 * rows * cols * 8
    ride_ops = len(pb.rows)
    g = pb.new_group()
    if nprod == 0:
        a = Win(nat.BASE_A, 0, lda, 128, 128)
        pb.product("gemm", 128, 128, 128, [(a, 1.0)], [(a, 1.0)], [(Win(nat.BASE_WS, ws_top, 128, 128, 128), 1.0)],
                   accumulate=0, group=g)
        ws_top += 128 * 128
    for i in range(nprod):
        r0 = (i % 4) * m
        c0 = (i * w) % (lda - 2 * w)
        a = Win(nat.BASE_A, r0 * lda + c0, lda, m, w)
        b = Win(nat.BASE_A, r0 * lda + c0 + w, lda, m, w)
        pb.product("gemm", m, w, w, [(a, 1.0)], [(b, 1.0)], [(Win(nat.BASE_WS, ws_top, w, w, w), 1.0)],
                   accumulate=0, group=g)
        ws_top += w * w
    p = pb.finish()
    p.ops["flags"][:ride_ops] |= nat.OPF_RIDE
    p.ws_scalars = ws_top
    return p, moved


def main():
    lda, m = 32768, 4096
    A = torch.rand(4 * m, lda, dtype=torch.float64, device="cuda")
    C = torch.empty(1, dtype=torch.float64, device="cuda")
    lib = nat.load()
    cases = [(58, 0, 0, 0), (0, 16, 4096, 1024), (58, 16, 4096, 1024), (58, 32, 4096, 1024),
             (58, 48, 4096, 1024), (0, 64, 2048, 512), (58, 64, 2048, 512)]
    if len(sys.argv) > 1 and sys.argv[1] == "bound":
        cases = [(58, 48, 4096, 1024), (58, 64, 4096, 1024)]
    if len(sys.argv) > 1 and sys.argv[1] == "bound2":
        cases = [(58, 64, 4096, 1024), (58, 96, 4096, 1024), (58, 128, 4096, 1024), (58, 192, 4096, 1024)]
    for (nprod, nodes, rows, cols) in cases:
        plan, moved = plan_for(nprod, m, nodes, rows, cols, lda)
        ws = torch.empty(max(1, plan.ws_scalars), dtype=torch.float64, device="cuda")

        def run():
            engine.run_plan(plan, nat.ATA_F64, A.data_ptr(), A.numel(), C.data_ptr(), 1, 1.0,
                            ws=ws.data_ptr(), ws_elems=ws.numel())
        r0 = lib.ata_ride_count()
        run()
        torch.cuda.synchronize()
        rides = lib.ata_ride_count() - r0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"{os.environ.get('ATA_LIB_PATH', 'base')} prods {nprod} nodes {nodes} ({rows}x{cols}, {moved / 1e9:.2f} GB) "
              f"rides {rides}: {ms:.3f} ms" + (f"  ride rate if bound: {moved / ms / 1e9:.2f} TB/s" if nodes else ""),
              flush=True)
        del ws


if __name__ == "__main__":
    main()
