"""Generate tests/golden/ fixtures for the callers and data formats either
side of the hot path by running the REFERENCE:

    python tools/make_golden_cli.py /root/reference/pkg/src

* task trees: ``render_tree`` text and the per-process leaf tasks of
  ``build_tree_distributed`` / ``build_tree_shared`` (scheduler.py) for a
  grid of (P, m, n), plus ``levels_*`` for P = 1..130;
* ATAM files written by ``write_matrix`` (matrix.py:383-417), f32 and f64;
* the benchmark CSV header and one formatted row (bench.py:30-31, :50-54).
Build container only: the reference tree does not exist on the GPU box.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True
import numpy as np

REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
sys.path.insert(0, REF)
from atamul import bench as rbench  # noqa: E402  (reference, read-only)
from atamul import scheduler as rs  # noqa: E402
from atamul.matrix import DenseMatrix, write_matrix  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
OUT.mkdir(parents=True, exist_ok=True)


def region(r):
    return None if r is None else [r.row_offset, r.col_offset, r.rows, r.cols]


def tree_case(mode, p, m, n):
    build = rs.build_tree_distributed if mode == "distributed" else rs.build_tree_shared
    try:
        t = build(p, m, n)
    except Exception as e:  # unsplittable shapes: record the error class
        return {"mode": mode, "p": p, "m": m, "n": n, "error": type(e).__name__}
    leaves = []
    for q in range(p):
        task = rs.leaf_task(t, q)
        leaves.append([task.computation.value, region(task.a_region), region(task.b_region),
                       region(task.c_region), task.parent, task.owner])
    chains = [[node.id for node in rs.path_to_root(t, q)] for q in range(p)]
    return {"mode": mode, "p": p, "m": m, "n": n, "depth": t.depth, "render": rs.render_tree(t),
            "leaves": leaves, "chains": chains}


cases = []
for mode in ("distributed", "shared"):
    for p in list(range(1, 13)) + [16, 24, 32, 36, 64]:
        for (m, n) in [(65536, 32768), (1048576, 2048), (8, 8), (37, 29), (6001, 4097), (3, 40)]:
            cases.append(tree_case(mode, p, m, n))
levels = {"distributed": [rs.levels_distributed(p) for p in range(1, 131)],
          "shared": [rs.levels_shared(p) for p in range(1, 131)]}
(OUT / "trees.json").write_text(json.dumps({"cases": cases, "levels": levels}))

rng = np.random.default_rng(5)
write_matrix(str(OUT / "ref_f64.atam"), DenseMatrix(rng.uniform(-1, 1, (7, 5))))
write_matrix(str(OUT / "ref_f32.atam"), DenseMatrix(rng.standard_normal((3, 11)).astype(np.float32)))

rec = rbench.BenchRecord(mode="seq", m=1024, n=1024, procs=1, threshold=4096, reps=5,
                         median_s=0.123456789, eff_gflops=8.6975e3, max_abs_err=1.25e-13,
                         mult_count=362086400)
rec2 = rbench.BenchRecord(mode="oracle", m=7, n=5, procs=1, threshold=32768, reps=1,
                          median_s=3.0e-05, eff_gflops=0.0058333)
(OUT / "cli_csv.json").write_text(json.dumps({"header": rbench.CSV_HEADER,
                                              "rows": [rec.csv_row(), rec2.csv_row()],
                                              "tolerance_f64_7x5": rbench.check_tolerance(
                                                  np.full((7, 5), 0.5)),
                                              "tolerance_f32_3x11": rbench.check_tolerance(
                                                  np.full((3, 11), 2.0, dtype=np.float32))}))
print("wrote", OUT)
