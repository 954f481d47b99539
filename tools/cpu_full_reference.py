"""One full-size run of the reference's own CPU path (unmodified atamul from
oracle/_ref: SharedRunner on every host core, prepare() untimed, run() timed,
as the reference's bench does) on a BASELINE config -- context for the
bench's sampled reference arm.  Writes one JSON line.

  python tools/cpu_full_reference.py c4 [threshold]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.cpu_baseline import cpu_model, reference_module  # noqa: E402
from paper_2110_13042_b200.measure import CONFIGS, config_matrix  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
threshold = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 19
ref = reference_module()
if ref is None:
    raise SystemExit("oracle/_ref missing: run oracle/build_ref.sh")
cfg = CONFIGS[name]
t0 = time.perf_counter()
a = config_matrix(name)
gen = time.perf_counter() - t0
procs = min(os.cpu_count() or 1, 128)
runner = ref.SharedRunner(a, procs, threshold)
t0 = time.perf_counter()
runner.prepare()
prep = time.perf_counter() - t0
t0 = time.perf_counter()
res = runner.run()
dt = time.perf_counter() - t0
m, n = a.shape
print(json.dumps({"config": name, "impl": "reference atamul.SharedRunner (oracle/_ref, unmodified)",
                  "m": m, "n": n, "procs": procs, "threshold": threshold, "cpu": cpu_model(),
                  "run_s": dt, "prepare_s": prep, "input_gen_s": gen,
                  "eff_gflops": m * n * n / dt / 1e9}), flush=True)
