"""Timeline of the pinned-host pipeline (ata._pipelined_host_ata) on a config:
CUDA-event marks on the copy and compute streams, in ms from the start.

  python tools/e2e_timeline.py [c4]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import importlib  # noqa: E402

import torch  # noqa: E402

import paper_2110_13042_b200 as P  # noqa: E402
from paper_2110_13042_b200.measure import CONFIGS, config_matrix, bench_plan_params  # noqa: E402

A_mod = importlib.import_module("paper_2110_13042_b200.ata")
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = CONFIGS[name]
a = config_matrix(name)
hA = torch.from_numpy(a).pin_memory()
hC = torch.zeros((cfg["n"], cfg["n"]), dtype=hA.dtype).pin_memory()
params, precision = bench_plan_params(name, a.shape[0], torch.device("cuda", 0))
kw = dict(threshold=cfg["threshold"], precision=precision, auto_params=params)
P.ata(hA, hC, 1.0, **kw)
for rep in range(2):
    A_mod.PIPE_TRACE = []
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record()
    P.ata(hA, hC, 1.0, **kw)
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record()
    torch.cuda.synchronize()
    print(f"--- rep {rep}: total {e0.elapsed_time(e1):.1f} ms")
    for label, ev in A_mod.PIPE_TRACE:
        print(f"{e0.elapsed_time(ev):9.1f}  {label}")
A_mod.PIPE_TRACE = None
