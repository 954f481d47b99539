"""Fused-rounding diagnostics for single-pass TF32 plans (config c5 shape):
time of the product launch with the rounding fused and the moment the last
rounding item completed, read back from the sync buffer (sync[2], sync[3]).

  python tools/round_diag.py [m n]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_13042_b200 import auto_plan, engine, _native as nat  # noqa: E402


def main():
    m, n = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) >= 3 else (1048576, 2048)
    A = torch.randn(m, n, device="cuda")
    C = torch.zeros(n, n, device="cuda")
    plan = auto_plan.plan_ata_auto(m, n, n, n, round_tf32=True)
    ws = torch.empty(plan.ws_scalars, device="cuda")
    need = engine.sync_ints_needed(plan, nat.ATA_TF32)
    sync = engine.sync_buffer(torch.device("cuda", 0), need)
    for rep in range(4):
        sync.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        engine.run_plan(plan, nat.ATA_TF32, A.data_ptr(), A.numel(), C.data_ptr(), C.numel(), 1.0,
                        ws=ws.data_ptr(), ws_elems=ws.numel(), sync=sync)
        e1.record()
        torch.cuda.synchronize()
        s = sync[:8].cpu().tolist()
        wait_ns = (s[6] & 0xffffffff) | (s[7] << 32)
        done_ms = ((s[2] - s[3]) % (1 << 31)) / 1e6
        print(f"rep {rep}: plan {e0.elapsed_time(e1):.3f} ms, rounding done {done_ms:.3f} ms after "
              f"the product kernel started (items done {s[1]}), producer wait {wait_ns / 1e6:.1f} ms summed "
              f"over CTAs", flush=True)


if __name__ == "__main__":
    main()
