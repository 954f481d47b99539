"""A/B timing of the c5 single-pass-TF32 plan (A 2^20 x 2048 fp32, device
randn -- timing only) for library variants built by tools/ab_build.py.

  python tools/tf32_ab.py [lib.so ...]     (no args: the in-tree library)
Prints one line per variant: ms per plan run (median of 5) and the product
launch share is reported by bench.py --dump-units; this is the quick loop.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, torch
sys.path.insert(0, %r)
from paper_2110_13042_b200 import auto_plan, engine, _native as nat
m, n = 1 << 20, 2048
torch.manual_seed(0)
A = torch.randn(m, n, device="cuda")
C = torch.zeros(n, n, device="cuda")
import os
plan = auto_plan.plan_ata_auto(m, n, n, n, auto_plan.AutoParams(tf32_ring=os.environ.get("TF32_RING", "1") == "1"),
                               round_tf32=True)
ws = torch.empty(max(1, plan.ws_scalars), device="cuda")
run = lambda: engine.run_plan(plan, nat.ATA_TF32, A.data_ptr(), A.numel(), C.data_ptr(), C.numel(), 1.0,
                              ws=ws.data_ptr(), ws_elems=ws.numel())
for _ in range(2):
    run()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
# sustained: 200 runs back to back (the TF32 launch hits the board power cap)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200):
    run()
e1.record(); torch.cuda.synchronize()
sus = e0.elapsed_time(e1) / 200
g = C.double()
print("ms %%.3f  TF/s %%.1f  sustained ms %%.3f TF/s %%.1f  diag[0] %%.6e" %% (
    ts[2], m * n * n / ts[2] / 1e9, sus, m * n * n / sus / 1e9, g[0, 0].item()), flush=True)
''' % ROOT

libs = sys.argv[1:] or [""]
for lib in libs:
    env = dict(os.environ)
    if lib:
        env["ATA_LIB_PATH"] = lib
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
    out = (r.stdout.strip().splitlines() or [""])[-1] if r.returncode == 0 else "FAILED " + r.stderr[-400:]
    print(f"{os.path.basename(lib) or 'in-tree'}: {out}", flush=True)
