"""FP64 leaf-kernel A/B timing: one persistent launch of a c4-like leaf group
(products of 4096 x 1024 x 1024 over quadrant windows of A into private
buffers, like the breadth-first Strassen leaves of the c4 plan), timed with
CUDA events; optionally a SYRK group.  Run once per library variant:

  ATA_LIB_PATH=_ab/v1.so python tools/f64_ab.py [nprod] [m] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_13042_b200 import _native as nat, engine, planner  # noqa: E402
from paper_2110_13042_b200.planner import Win  # noqa: E402


def group_plan(nprod, m, w, kind="gemm", lda=32768):
    pb = planner.PlanBuilder("ab")
    g = pb.new_group()
    for i in range(nprod):
        r0 = (i % 4) * m
        c0 = (i * w) % (lda - 2 * w)
        a = Win(nat.BASE_A, r0 * lda + c0, lda, m, w)
        b = Win(nat.BASE_A, r0 * lda + c0 + w, lda, m, w)
        out = Win(nat.BASE_WS, i * w * w, w, w, w)
        pb.product(kind, m, w, w, [(a, 1.0)], [] if kind == "syrk" else [(b, 1.0)], [(out, 1.0)],
                   accumulate=0, group=g)
    p = pb.finish()
    p.ws_scalars = nprod * w * w
    return p


def main():
    nprod = int(sys.argv[1]) if len(sys.argv) > 1 else 58
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    w, lda = 1024, 32768
    A = torch.rand(4 * m, lda, dtype=torch.float64, device="cuda")
    for kind in ("gemm", "syrk"):
        plan = group_plan(nprod, m, w, kind, lda)
        ws = torch.empty(plan.ws_scalars, dtype=torch.float64, device="cuda")
        C = torch.empty(1, dtype=torch.float64, device="cuda")

        def run():
            engine.run_plan(plan, nat.ATA_F64, A.data_ptr(), A.numel(), C.data_ptr(), 1, 1.0,
                            ws=ws.data_ptr(), ws_elems=ws.numel())
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        flops = nprod * (2.0 * m * w * w if kind == "gemm" else 1.0 * m * w * (w + 1))
        tiles = nprod * (64 if kind == "gemm" else 36)
        print(f"{os.environ.get('ATA_LIB_PATH', 'base')} {kind}: {nprod} x {m}x{w}x{w} ({tiles} tiles) "
              f"{ms:.3f} ms {flops / ms / 1e9:.2f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
