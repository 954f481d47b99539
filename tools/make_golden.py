"""Generate tests/golden/ fixtures by running the REFERENCE implementation.

Run in the build container only (the reference tree does not exist on the
GPU box):

    python tools/make_golden.py /root/reference/pkg/src

It imports the reference package read-only (no bytecode written) and records
its outputs for seeded inputs: leaf-kernel known answers, exact
multiplication counts, workspace level sizes, full AtA / Strassen results on
small shapes (including odd and degenerate ones), and checksummed results for
config c1 at the parity cutoff.  The committed .npz/.json files are what the
oracle and the GPU path are pinned against.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True
import numpy as np

REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
sys.path.insert(0, REF)
import atamul  # noqa: E402  (reference, read-only)
from atamul.matrix import MultCounter, mirror_lower_to_upper, naive_gemm_atb, naive_syrk_lower, pack_lower  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
OUT.mkdir(parents=True, exist_ok=True)


def ref_ata(a, t, alpha=1.0, sentinel=None):
    n = a.shape[1]
    c = np.zeros((n, n), dtype=a.dtype)
    if sentinel is not None:
        c[np.triu_indices(n, 1)] = sentinel
    cnt = MultCounter()
    atamul.ata(a, c, alpha, threshold=t, counter=cnt)
    return c, cnt.scalar_mults


def ref_strassen(a, b, t, c0=None, alpha=1.0):
    c = np.zeros((a.shape[1], b.shape[1]), dtype=a.dtype) if c0 is None else c0.copy()
    cnt = MultCounter()
    atamul.fast_strassen(a, b, c, alpha, atamul.workspace_for(a.shape[0], a.shape[1], b.shape[1], t,
                                                             dtype=c.dtype), t, cnt)
    return c, cnt.scalar_mults


def main():
    meta = {"reference": "atamul " + atamul.__version__, "numpy": np.__version__}
    arrays = {}

    # ---- known-answer tests (tests/test_matrix.py:140-185, test_ata.py:16-19) ----
    kat = {}
    c = np.zeros((2, 2)); naive_syrk_lower(np.array([[1.0, 2.0], [3.0, 4.0]]), c, 1.0)
    kat["syrk_2x2"] = [c[0, 0], c[1, 0], c[1, 1]]
    c = np.zeros((2, 1)); naive_gemm_atb(np.array([[1.0, 0.0], [0.0, 2.0]]), np.array([[3.0], [4.0]]), c, 1.0)
    kat["gemm_2x2x1"] = c.ravel().tolist()
    c = np.zeros((1, 1)); atamul.ata(np.array([[2.0]]), c, 1.0, threshold=4)
    kat["ata_1x1"] = float(c[0, 0])
    c = np.zeros((3, 3)); naive_syrk_lower(np.array([[2.0, -3.0, 5.0]]), c, 1.0)
    kat["syrk_row_vector_packed"] = pack_lower(c).data.tolist()
    meta["kat"] = kat

    # ---- exact multiplication counts ----
    counts = {}
    for n in [1, 2, 4, 8, 16, 32]:
        _, cnt = ref_ata(np.ones((n, n)), 1)
        counts[f"ata_square_{n}_t1"] = cnt
        _, cnt = ref_strassen(np.ones((n, n)), np.ones((n, n)), 1)
        counts[f"strassen_cube_{n}_t1"] = cnt
    for (m, n, t) in [(6, 4, 1), (12, 9, 4), (50, 37, 64), (300, 17, 512), (129, 65, 1024),
                      (1024, 1024, 4096), (1024, 1024, 32768), (6001, 4097, 65536)]:
        # counts depend only on shapes: use a cheap shape-only walk through the
        # reference by running it on zeros for small shapes, and on the
        # reference's own workspace planner only for the big ones.
        if m * n <= 2_000_000:
            _, cnt = ref_ata(np.zeros((m, n)), t)
            counts[f"ata_{m}x{n}_t{t}"] = cnt
    meta["counts"] = counts

    # ---- workspace sizes (tests/test_strassen.py:124-151) ----
    ws = {}
    for (m, n, k, t) in [(8, 8, 8, 2), (16, 16, 16, 1), (64, 64, 64, 1), (256, 256, 256, 1),
                         (32, 32, 32, 4), (16, 20, 9, 4), (23, 17, 19, 8), (1, 64, 64, 1)]:
        w = atamul.workspace_for(m, n, k, t)
        ws[f"strassen_{m}_{n}_{k}_t{t}"] = {
            "levels": [[lv.prod.size, lv.lhs.size, lv.rhs.size] for lv in w.levels],
            "base": [w.base_acc.size, w.base_lhs.size, w.base_rhs.size],
            "total": w.total_scalars}
    for (m, n, t) in [(8, 8, 64), (64, 64, 64), (12, 9, 4), (1024, 1024, 4096), (300, 17, 512),
                      (6001, 4097, 65536), (100, 80, 64)]:
        w = atamul.workspace_for_ata(m, n, t)
        ws[f"ata_{m}_{n}_t{t}"] = {
            "levels": [[lv.prod.size, lv.lhs.size, lv.rhs.size] for lv in w.levels],
            "base": [w.base_acc.size, w.base_lhs.size, w.base_rhs.size],
            "total": w.total_scalars}
    meta["workspace"] = ws

    # ---- full results on small shapes ----
    cases = []
    rng = np.random.default_rng(20240811)
    ata_shapes = [(6, 4, 1), (12, 9, 4), (7, 5, 1), (1, 8, 4), (8, 1, 4), (1, 1, 4), (2, 2, 1),
                  (50, 37, 1), (50, 37, 64), (50, 37, 4096), (33, 21, 8), (64, 64, 16), (63, 65, 16),
                  (512, 32, 512), (300, 17, 512), (129, 65, 1024), (101, 101, 1024), (40, 25, 32),
                  (17, 64, 16), (3, 3, 1)]
    for i, (m, n, t) in enumerate(ata_shapes):
        a = rng.uniform(-1, 1, (m, n))
        c, cnt = ref_ata(a, t, sentinel=1.2345e67)
        key = f"ata{i}"
        arrays[key + "_A"] = a
        arrays[key + "_C"] = c
        cases.append({"kind": "ata", "key": key, "m": m, "n": n, "threshold": t, "alpha": 1.0,
                      "mults": cnt})
    # alpha != 1 and float32
    a = rng.uniform(-1, 1, (23, 19)); c, cnt = ref_ata(a, 16, alpha=-2.5)
    arrays["ata_alpha_A"] = a; arrays["ata_alpha_C"] = c
    cases.append({"kind": "ata", "key": "ata_alpha", "m": 23, "n": 19, "threshold": 16,
                  "alpha": -2.5, "mults": cnt})
    a = rng.uniform(-1, 1, (100, 80)).astype(np.float32); c, cnt = ref_ata(a, 64)
    arrays["ata_f32_A"] = a; arrays["ata_f32_C"] = c
    cases.append({"kind": "ata", "key": "ata_f32", "m": 100, "n": 80, "threshold": 64,
                  "alpha": 1.0, "mults": cnt})
    st_shapes = [(7, 5, 6, 1), (6, 4, 3, 8), (9, 6, 7, 4), (23, 17, 19, 8), (64, 64, 64, 16),
                 (33, 1, 20, 16), (1, 9, 9, 1), (45, 30, 31, 16), (2, 2, 2, 1)]
    for i, (m, n, k, t) in enumerate(st_shapes):
        a = rng.uniform(-1, 1, (m, n)); b = rng.uniform(-1, 1, (m, k)); c0 = rng.uniform(-1, 1, (n, k))
        c, cnt = ref_strassen(a, b, t, c0=c0)
        key = f"st{i}"
        arrays[key + "_A"] = a; arrays[key + "_B"] = b; arrays[key + "_C0"] = c0; arrays[key + "_C"] = c
        cases.append({"kind": "strassen", "key": key, "m": m, "n": n, "k": k, "threshold": t,
                      "mults": cnt})
    meta["cases"] = cases

    # ---- config c1 at the parity cutoff (t = 64^2): checksums + sampled entries ----
    a = np.random.default_rng(0).uniform(-1.0, 1.0, (1024, 1024))
    c, cnt = ref_ata(a, 4096)
    il, jl = np.tril_indices(1024)
    vals = c[il, jl]
    srng = np.random.default_rng(99)
    pick = srng.choice(vals.size, 4096, replace=False)
    arrays["c1_sample_idx"] = pick
    arrays["c1_sample_val"] = vals[pick]
    meta["c1"] = {"m": 1024, "n": 1024, "seed": 0, "threshold": 4096, "mults": cnt,
                  "lower_fro": float(np.linalg.norm(vals)), "lower_sum": float(vals.sum())}
    arrays["c1_row_sums"] = np.array([c[i, :i + 1].sum() for i in range(1024)])

    np.savez_compressed(OUT / "reference_cases.npz", **arrays)
    (OUT / "reference_meta.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
