"""Generate tests/golden/ fixtures for the reference's executors by running the
REFERENCE (build container only; the reference tree is absent on the GPU box):

    python tools/make_golden_exec.py /root/reference/pkg/src

* ``distsim.json``: for a grid of (P, m, n), the reference ``ata_d`` run
  (leaf kernels "naive" and "fast", seeded uniform input): the CommStats
  counters per process, the message trace (src, dst, [(kind, region, words)]),
  the ``verify_comm_bounds`` report, the exact multiplication count and
  row sums / Frobenius norm of the result; the result matrices go to
  ``exec_results.npz``.
* ``shared.json``: ``ata_s`` / ``SharedRunner`` results (same checksums, per
  worker max multiplication count with count_mults=True).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True
import numpy as np

REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
sys.path.insert(0, REF)
import atamul as R  # noqa: E402  (reference, read-only)

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def region(r):
    return [r.row_offset, r.col_offset, r.rows, r.cols]


arrays = {}
dist_cases = []
for (p, m, n, t, kern) in [(1, 40, 30, 64, "naive"), (2, 40, 30, 64, "fast"), (3, 37, 29, 64, "fast"),
                           (5, 64, 48, 256, "naive"), (6, 50, 44, 64, "fast"), (7, 61, 53, 128, "naive"),
                           (8, 64, 64, 64, "fast"), (11, 96, 80, 256, "fast"), (16, 128, 96, 512, "naive"),
                           (36, 128, 128, 1024, "fast")]:
    a = R.gen_matrix(m, n, seed=p).a
    cnt = R.MultCounter()
    trace = []
    res, st = R.ata_d(a, p, threshold=t, leaf_kernel=kern, counter=cnt, trace=trace, scheduler_seed=3)
    rep = R.verify_comm_bounds(st, n, p)
    key = f"dist_{p}_{m}_{n}"
    arrays[key] = res.a
    dist_cases.append({
        "p": p, "m": m, "n": n, "threshold": t, "leaf_kernel": kern, "seed": p, "key": key,
        "sent_messages": st.sent_messages, "sent_words": st.sent_words,
        "recv_messages": st.recv_messages, "recv_words": st.recv_words,
        "critical_path_messages": st.critical_path_messages, "total_words": st.total_words,
        "trace": [[s, d, [[k, region(r), w] for (k, r, w) in parts]] for (s, d, parts) in trace],
        "report": {"levels": rep.levels, "latency_bound": rep.latency_bound,
                   "words_bound": rep.words_bound, "ok": rep.ok, "summary": rep.summary()},
        "mults": cnt.scalar_mults})
bounds = [{"p": p, "n": n, "latency": R.distsim.comm_bound_latency(p),
           "words": R.distsim.comm_bound_words(n, p)}
          for p in (1, 2, 5, 6, 7, 36, 37, 64, 216) for n in (8, 100, 4097)]
(OUT / "distsim.json").write_text(json.dumps({"cases": dist_cases, "bounds": bounds}))

shared_cases = []
for (p, m, n, t) in [(1, 40, 30, 64), (2, 33, 31, 64), (3, 64, 48, 256), (4, 37, 29, 64), (7, 96, 80, 512),
                     (9, 50, 60, 128)]:
    a = R.gen_matrix(m, n, seed=100 + p).a
    runner = R.SharedRunner(a, p, threshold=t, count_mults=True)
    runner.prepare()
    res = runner.run()
    key = f"shared_{p}_{m}_{n}"
    arrays[key] = res.a
    shared_cases.append({"p": p, "m": m, "n": n, "threshold": t, "seed": 100 + p, "key": key,
                         "max_worker_mults": runner.max_worker_mults,
                         "worker_mults": [c.scalar_mults for c in runner.counters]})
(OUT / "shared.json").write_text(json.dumps({"cases": shared_cases}))
np.savez_compressed(OUT / "exec_results.npz", **arrays)
print(f"{len(dist_cases)} ata_d cases, {len(shared_cases)} SharedRunner cases -> {OUT}")
