"""Host planner logic on the CPU: workspace sizes and exact multiplication
counts against the reference's golden values, and plan semantics through the
NumPy plan interpreter against the oracle."""
import numpy as np
import pytest
from hypothesis import given
from hypothesis import strategies as st

import plan_interp
from oracle import atamul_oracle as O
from paper_2110_13042_b200 import auto_plan, planner, ref_bfs
from paper_2110_13042_b200.workspace import ata_calls, calls_sizes, workspace_for_calls
from paper_2110_13042_b200.strassen import workspace_for
from paper_2110_13042_b200.ata import workspace_for_ata


def _ata_plan(m, n, t, fuse=True):
    ws = workspace_for_ata(m, n, t)
    return planner.plan_ata_reference(m, n, n, n, t, ws.level_offsets(), fuse=fuse), ws


def _interp_ata(plan, ws, a, alpha=1.0, sentinel=None):
    n = a.shape[1]
    c = np.zeros((n, n), dtype=a.dtype)
    if sentinel is not None:
        c[np.triu_indices(n, 1)] = sentinel
    wsbuf = np.zeros(max(1, ws.total_scalars), dtype=a.dtype)
    plan_interp.run(plan.ops, a, c, alpha, WS=wsbuf)
    return c


def test_workspace_sizes_match_reference(golden):
    meta, _ = golden
    for key, want in meta["workspace"].items():
        parts = key.split("_")
        if parts[0] == "strassen":
            m, n, k, t = int(parts[1]), int(parts[2]), int(parts[3]), int(parts[4][1:])
            ws = workspace_for(m, n, k, t)
        else:
            m, n, t = int(parts[1]), int(parts[2]), int(parts[3][1:])
            ws = workspace_for_ata(m, n, t)
        got = [[lv.prod.size, lv.lhs.size, lv.rhs.size] for lv in ws.levels]
        assert got == want["levels"], key
        assert list(ws.base_sizes) == want["base"], key


def test_space_bound():
    for n in (16, 64, 256):
        assert workspace_for(n, n, n, 1).total_scalars <= 1.5 * n * n


def test_covers():
    ws = workspace_for(32, 32, 32, 4)
    assert ws.covers(32, 32, 32, 4) and ws.covers(16, 16, 16, 4)
    assert not ws.covers(33, 32, 32, 4)
    assert not ws.covers(16, 20, 9, 4)
    assert workspace_for(16, 20, 9, 4).covers(16, 20, 9, 4)


@pytest.mark.parametrize("fuse", [True, False])
def test_reference_plan_counts(golden, fuse):
    meta, _ = golden
    for key, want in meta["counts"].items():
        parts = key.split("_")
        if parts[0] == "ata" and parts[1] == "square":
            n, t = int(parts[2]), int(parts[3][1:])
            m = n
        elif parts[0] == "ata":
            m, n = map(int, parts[1].split("x"))
            t = int(parts[2][1:])
        else:
            n = int(parts[2])
            ws = workspace_for(n, n, n, 1)
            p = planner.plan_strassen_reference(n, n, n, n, n, n, 1, ws.level_offsets(), fuse=fuse)
            assert p.mults == want, key
            continue
        p, _ = _ata_plan(m, n, t, fuse)
        assert p.mults == want, key


@pytest.mark.parametrize("fuse", [True, False])
def test_reference_plan_semantics(golden, fuse):
    meta, arrays = golden
    for case in meta["cases"]:
        key = case["key"]
        if case["kind"] == "ata":
            a = arrays[key + "_A"]
            m, n = a.shape
            p, ws = _ata_plan(m, n, case["threshold"], fuse)
            c = _interp_ata(p, ws, a, case["alpha"], sentinel=1.0e30)
            ref = arrays[key + "_C"]
            il, jl = np.tril_indices(n)
            tol = 1e-12 if a.dtype == np.float64 else 1e-5
            assert O.rel_frobenius_lower(c, ref) <= tol, key
            assert np.all(c[np.triu_indices(n, 1)] == 1.0e30), key
        else:
            a, b, c0 = arrays[key + "_A"], arrays[key + "_B"], arrays[key + "_C0"]
            m, n = a.shape
            k = b.shape[1]
            ws = workspace_for(m, n, k, case["threshold"])
            p = planner.plan_strassen_reference(m, n, k, n, k, k, case["threshold"],
                                                ws.level_offsets(), fuse=fuse)
            c = c0.copy()
            plan_interp.run(p.ops, a, c, 1.0, WS=np.zeros(max(1, ws.total_scalars)), B=b)
            ref = arrays[key + "_C"]
            assert np.abs(c - ref).max() <= 1e-12 * m, key


def test_fused_plan_has_fewer_ops():
    p_f, _ = _ata_plan(256, 256, 1024, True)
    p_u, _ = _ata_plan(256, 256, 1024, False)
    assert p_f.mults == p_u.mults
    assert len(p_f.ops) < len(p_u.ops)


@given(m=st.integers(1, 300), n=st.integers(1, 300), leaf=st.sampled_from([8, 16, 33, 64]),
       mind=st.sampled_from([2, 4, 16, 10**9]), depth=st.sampled_from([1, 2, 3]),
       seed=st.integers(0, 2**16))
def test_auto_plan_semantics(m, n, leaf, mind, depth, seed):
    a = np.random.default_rng(seed).uniform(-1, 1, (m, n))
    params = auto_plan.AutoParams(leaf_cols=leaf, min_dim=mind, max_depth=depth, hbm_gbs=1e9)
    p = auto_plan.plan_ata_auto(m, n, n, n, params)
    c = np.zeros((n, n))
    c[np.triu_indices(n, 1)] = 7.0
    plan_interp.run(p.ops, a, c, 1.0, WS=np.zeros(max(1, p.ws_scalars)))
    assert np.all(c[np.triu_indices(n, 1)] == 7.0)
    assert O.rel_frobenius_lower(c, O.gram(a)) <= 1e-12


def _dest_cells(op, n_ld):
    """(base, element) -> region id of every destination element of an op."""
    cells = {}
    for j in range(int(op["nd"])):
        d = op["d"][j]
        rows, cols, off, ld = int(d["rows"]), int(d["cols"]), int(d["off"]), int(d["ld"])
        for r in range(rows):
            for c in range(cols):
                if int(op["type"]) == 1 and c > r:
                    continue
                cells[(int(d["base"]), off + r * ld + c)] = int(d["region"])
    return cells


def test_auto_plan_groups_write_disjoint():
    p = auto_plan.plan_ata_auto(200, 150, 150, 150,
                                auto_plan.AutoParams(leaf_cols=16, min_dim=4, hbm_gbs=1e9))
    groups = {}
    for op in p.ops:
        g = int(op["group"])
        if g < 0:
            continue
        groups.setdefault(g, []).append(op)
    assert groups
    for g, ops in groups.items():
        seen = {}
        for op in ops:
            cells = _dest_cells(op, 150)
            for cell, region in cells.items():
                if cell in seen:
                    # a shared cell must belong to the same ordered region in both ops
                    assert region > 0 and seen[cell] == region, f"group {g}: unordered overlap"
                seen[cell] = region


def test_auto_plan_tf32_round_and_split_contraction():
    """Single-pass-TF32 plans round A once into the workspace and split the
    contraction of tall-skinny groups; checked through the interpreter."""
    m, n = 6000, 96
    a = np.random.default_rng(3).standard_normal((m, n)).astype(np.float32)
    p = auto_plan.plan_ata_auto(m, n, n, n, auto_plan.AutoParams(leaf_cols=32, min_chunk=512),
                                round_tf32=True)
    types = [int(o["type"]) for o in p.ops]
    assert types[0] == 7 and 5 in types          # ROUND first, combo4 partial sums present
    c = np.zeros((n, n), dtype=np.float32)
    c[np.triu_indices(n, 1)] = 5.0
    plan_interp.run(p.ops, a, c, 1.0, WS=np.full(max(1, p.ws_scalars), np.nan, dtype=np.float32))
    assert np.all(c[np.triu_indices(n, 1)] == 5.0)
    assert O.rel_frobenius_lower(c, O.gram_blas(a)) <= 1e-4


# ---------------------------------------------------------- breadth-first reference plans

def _bfs_plan(m, n, t, budget=ref_bfs.DEFAULT_BUDGET):
    return ref_bfs.plan_ata_reference_bfs(m, n, n, n, t, budget)


def test_bfs_reference_plan_counts(golden):
    """Same recursion tree as the reference: the exact MultCounter totals."""
    meta, _ = golden
    for key, want in meta["counts"].items():
        parts = key.split("_")
        if parts[0] == "ata" and parts[1] == "square":
            n, t = int(parts[2]), int(parts[3][1:])
            m = n
        elif parts[0] == "ata":
            m, n = map(int, parts[1].split("x"))
            t = int(parts[2][1:])
        else:
            n = int(parts[2])
            p = ref_bfs.plan_strassen_reference_bfs(n, n, n, n, n, n, 1)
            assert p.mults == want, key
            continue
        assert _bfs_plan(m, n, t).mults == want, key
        # a tiny scratch budget forces the depth-first fallback: same tree
        assert _bfs_plan(m, n, t, budget=64).mults == want, key


@pytest.mark.parametrize("budget", [ref_bfs.DEFAULT_BUDGET, 200])
def test_bfs_reference_plan_semantics(golden, budget):
    """Every golden AtA / Strassen case through the interpreter: reference
    results (1e-12 / 1e-5), strict upper triangle untouched."""
    meta, arrays = golden
    for case in meta["cases"]:
        key = case["key"]
        if case["kind"] == "ata":
            a = arrays[key + "_A"]
            m, n = a.shape
            p = _bfs_plan(m, n, case["threshold"], budget)
            c = np.zeros((n, n), dtype=a.dtype)
            c[np.triu_indices(n, 1)] = 1.0e30
            plan_interp.run(p.ops, a, c, case["alpha"],
                            WS=np.full(max(1, p.ws_scalars), np.nan, dtype=a.dtype))
            tol = 1e-12 if a.dtype == np.float64 else 1e-5
            assert O.rel_frobenius_lower(c, arrays[key + "_C"]) <= tol, key
            assert np.all(c[np.triu_indices(n, 1)] == 1.0e30), key
        else:
            a, b, c0 = arrays[key + "_A"], arrays[key + "_B"], arrays[key + "_C0"]
            m, n = a.shape
            k = b.shape[1]
            p = ref_bfs.plan_strassen_reference_bfs(m, n, k, n, k, k, case["threshold"], budget)
            c = c0.copy()
            plan_interp.run(p.ops, a, c, 1.0, WS=np.full(max(1, p.ws_scalars), np.nan), B=b)
            assert np.abs(c - arrays[key + "_C"]).max() <= 1e-12 * m, key


@pytest.mark.parametrize("shape", [(97, 83, 64), (50, 37, 1), (50, 37, 64), (33, 17, 2), (9, 40, 3)])
def test_bfs_reference_plan_groups_write_disjoint(shape):
    """Within one launch group no two ops write the same element (rounds),
    including nested diagonal leaves of uneven splits (threshold 1)."""
    p = _bfs_plan(*shape)
    groups = {}
    for op in p.ops:
        g = int(op["group"])
        if g >= 0:
            groups.setdefault(g, []).append(op)
    assert len(groups) >= 1
    for g, ops in groups.items():
        seen = set()
        for op in ops:
            cells = set(_dest_cells(op, shape[1]))
            assert not (cells & seen), f"group {g}: two writers"
            seen |= cells


def test_bfs_reference_plan_launches():
    """c2-shaped recursion: far fewer launches than the depth-first executor."""
    m, n, t = 6001, 4097, 256 * 256
    p = _bfs_plan(m, n, t)
    d = planner.plan_ata_reference(m, n, n, n, t, workspace_for_ata(m, n, t).level_offsets())
    assert p.mults == d.mults
    assert p.launches * 10 < d.launches


def test_tf32_ring_plan_reads_raw_rows():
    """Single-pass TF32 tall-skinny plans whose chunks fit the CTA-pair kernel's
    waves use the L2 rounding ring: no HBM rounding pass (ROUND op with
    accumulate = 2, a small ring scratch), products read A itself; the other
    shapes keep the rounding pass.  The ring plan computes the same Gram."""
    m, n = 1 << 17, 2048
    p = auto_plan.plan_ata_auto(m, n, n, n, auto_plan.AutoParams(), round_tf32=True)
    assert int(p.ops[0]["type"]) == 7 and int(p.ops[0]["accumulate"]) == 2
    prods = [o for o in p.ops if int(o["type"]) in (0, 1)]
    assert prods and all(int(o["s"][0]["base"]) == 0 for o in prods)
    q = auto_plan.plan_ata_auto(m, n, n, n, auto_plan.AutoParams(tf32_ring=False), round_tf32=True)
    assert int(q.ops[0]["accumulate"]) == 0 and int(q.ops[1]["s"][0]["base"]) == 2
    small = auto_plan.plan_ata_auto(6000, 96, 96, 96, auto_plan.AutoParams(leaf_cols=32, min_chunk=512),
                                    round_tf32=True)
    assert int(small.ops[0]["accumulate"]) == 0
    a = np.random.default_rng(9).standard_normal((m, n)).astype(np.float32)[:, :n]
    c = np.zeros((n, n), dtype=np.float32)
    plan_interp.run(p.ops, a, c, 1.0, WS=np.full(p.ws_scalars, np.nan, dtype=np.float32))
    assert O.rel_frobenius_lower(c, O.gram_blas(a)) <= 1e-5


def test_host_pipeline_row_blocks_regimes():
    """ata._row_blocks: three geometric blocks for compute-bound fp64 shapes (c3,
    c4), the first less than half the second (C starts at zero on the device);
    equal blocks when PCIe bound."""
    import importlib
    A = importlib.import_module("paper_2110_13042_b200.ata")
    for m, n, es, tc, nb, grow in ((65536, 32768, 8, False, 3, True), (16384, 16384, 8, False, 3, True),
                                   (1 << 20, 2048, 4, True, 2, False), (6001, 4097, 8, False, 2, False)):
        blocks = A._row_blocks(m, n, es, tc)
        assert len(blocks) == nb
        assert blocks[0][0] == 0 and sum(b for _, b in blocks) == m
        assert all(r0 + b == r1 for (r0, b), (r1, _) in zip(blocks, blocks[1:]))
        sizes = [b for _, b in blocks]
        assert (sizes == sorted(sizes) and 2 * sizes[0] < sizes[1]) if grow else (max(sizes) - min(sizes) <= 1)
