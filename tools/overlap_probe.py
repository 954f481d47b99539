"""Probe: does the c5 TF32 rounding pass co-run with the tcgen05 product
launch on the same SMs (separate streams)?  Times round-then-products on one
stream against the two issued on two streams (timing only, device randn)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_13042_b200 import auto_plan, engine, _native as nat

m, n = 1 << 20, 2048
A = torch.randn(m, n, device="cuda")
C = torch.zeros(n, n, device="cuda")
plan = auto_plan.plan_ata_auto(m, n, n, n, auto_plan.AutoParams(), round_tf32=True)
ws = torch.empty(max(1, plan.ws_scalars), device="cuda")


class Part:
    def __init__(self, ops):
        self.ops = ops


r_ops = Part(plan.ops[:1])
p_ops = Part(plan.ops[1:])
assert int(plan.ops[0]["type"]) == nat.OP_ROUND
s1 = torch.cuda.Stream()
s2 = torch.cuda.Stream()


def run(part, stream):
    with torch.cuda.stream(stream):
        engine.run_plan(part, nat.ATA_TF32, A.data_ptr(), A.numel(), C.data_ptr(), C.numel(), 1.0,
                        ws=ws.data_ptr(), ws_elems=ws.numel(), stream=int(stream.cuda_stream))


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def seq():
    cur = torch.cuda.current_stream()
    run(r_ops, cur)
    run(p_ops, cur)


def conc():
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(cur)
    s1.wait_event(ev)
    s2.wait_event(ev)
    run(p_ops, s1)
    run(r_ops, s2)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


for f in (seq, conc, seq, conc):
    f()
for name, f in (("round only", lambda: run(r_ops, torch.cuda.current_stream())),
                ("products only", lambda: run(p_ops, torch.cuda.current_stream())),
                ("sequential", seq), ("two streams", conc)):
    ts = sorted(timed(f) for _ in range(5))
    print(f"{name:14s} {ts[2]:.3f} ms", flush=True)
