"""Riding operand sums (ATA_OPF_RIDE, auto_plan._hoist_sums): the reordered
plans keep their sequential meaning, every flagged COMBO4 sits directly in
front of a product group and is element-wise independent of it (the executor
runs it concurrently with that group's launch)."""
import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import atamul_oracle as O
from paper_2110_13042_b200 import _native as nat
from paper_2110_13042_b200 import auto_plan

import plan_interp


def _cells(ref, lower=False):
    rows, cols, off, ld = int(ref["rows"]), int(ref["cols"]), int(ref["off"]), int(ref["ld"])
    if rows == 0 or cols == 0:
        return set()
    r, c = np.meshgrid(np.arange(rows), np.arange(cols), indexing="ij")
    keep = (c <= r) if lower else np.ones_like(r, dtype=bool)
    return {(int(ref["base"]), int(e)) for e in (off + r * ld + c)[keep].ravel()}


def _reads_writes(op):
    t = int(op["type"])
    reads, writes = set(), set()
    for j in range(int(op["ns"])):
        reads |= _cells(op["s"][j])
    if t in (nat.OP_GEMM, nat.OP_POSTADD7):
        for j in range(int(op["nt"])):
            reads |= _cells(op["t"][j])
    for j in range(int(op["nd"])):
        writes |= _cells(op["d"][j])
    return reads, writes


def _ride_runs(ops):
    """[(first, last, group_first, group_last)]: maximal runs of flagged ops and
    the product group that follows each."""
    out, i, n = [], 0, len(ops)
    while i < n:
        if int(ops[i]["flags"]) & nat.OPF_RIDE:
            j = i
            while j < n and int(ops[j]["flags"]) & nat.OPF_RIDE:
                j += 1
            k = j
            while k < n and int(ops[k]["type"]) in (nat.OP_GEMM, nat.OP_SYRK) and \
                    int(ops[k]["group"]) == int(ops[j]["group"]):
                k += 1
            out.append((i, j, j, k))
            i = j
        else:
            i += 1
    return out


# (ride_gbs: no capacity limit -- these toy products are far too short to hide anything)
FORCED_DFS = dict(leaf_cols=16, min_dim=4, max_depth=3, hbm_gbs=1e9, ws_budget_gb=2e-5, ride_gbs=1e12)


@settings(max_examples=25, deadline=None)
@given(m=st.integers(40, 260), n=st.integers(40, 200), seed=st.integers(0, 2**16),
       budget=st.sampled_from([4e-6, 2e-5, 1e-4]))
def test_hoisted_plan_semantics(m, n, seed, budget):
    a = np.random.default_rng(seed).uniform(-1, 1, (m, n))
    params = auto_plan.AutoParams(**{**FORCED_DFS, "ws_budget_gb": budget})
    p = auto_plan.plan_ata_auto(m, n, n, n, params)
    c = np.zeros((n, n))
    c[np.triu_indices(n, 1)] = 7.0
    plan_interp.run(p.ops, a, c, 1.0, WS=np.zeros(max(1, p.ws_scalars)))
    assert np.all(c[np.triu_indices(n, 1)] == 7.0)
    assert O.rel_frobenius_lower(c, O.gram(a)) <= 1e-12
    # same multiplications and ops as the plan without riding sums
    q = auto_plan.plan_ata_auto(m, n, n, n, auto_plan.AutoParams(**{**FORCED_DFS, "ws_budget_gb": budget,
                                                                    "ride_sums": False}))
    assert q.mults == p.mults and len(q.ops) == len(p.ops)
    assert not (q.ops["flags"] & nat.OPF_RIDE).any()


@pytest.mark.parametrize("m,n", [(192, 160), (257, 131), (300, 96)])
def test_ride_ops_precede_a_group_and_are_independent_of_it(m, n):
    p = auto_plan.plan_ata_auto(m, n, n, n, auto_plan.AutoParams(**FORCED_DFS))
    ops = p.ops
    runs = _ride_runs(ops)
    assert runs, "the forced depth-first plan has riding sums"
    assert int((ops["flags"] & nat.OPF_RIDE).sum()) == sum(j - i for i, j, _, _ in runs)
    for (i, j, g0, g1) in runs:
        assert g1 > g0, "a riding run is followed by a product group"
        assert all(int(ops[q]["type"]) == nat.OP_COMBO4 and int(ops[q]["accumulate"]) == 0 for q in range(i, j))
        g_reads, g_writes = set(), set()
        for q in range(g0, g1):
            r, w = _reads_writes(ops[q])
            g_reads |= r
            g_writes |= w
        for q in range(i, j):
            r, w = _reads_writes(ops[q])
            assert not (w & g_reads) and not (w & g_writes) and not (r & g_writes), (q, g0, g1)


def test_c4_plan_rides_most_operand_sums():
    """Config c4: every leaf group except each tree's first carries the next group's sums."""
    p = auto_plan.plan_ata_auto(65536, 32768, 32768, 32768, auto_plan.AutoParams())
    ops = p.ops
    combo = ops["type"] == nat.OP_COMBO4
    ride = (ops["flags"] & nat.OPF_RIDE) != 0
    assert not (ride & ~combo).any()
    assert ride.sum() >= 0.85 * combo.sum()      # (the rest: each later tree's first group, and what exceeds ride_gbs)
    # (plans with riding sums split at gain_ride = 1.0: the same tree without riding sums)
    q = auto_plan.plan_ata_auto(65536, 32768, 32768, 32768, auto_plan.AutoParams(ride_sums=False, gain=1.0))
    assert q.mults == p.mults
    assert p.mults < 0.64 * 65536 * 32768 * 32769 // 2
    assert p.ws_scalars * 8 <= 115e9     # alternating regions + the second top-level arena (65.1 GB without arenas)


def test_ride_capacity_limits_what_a_group_carries():
    """A product group carries at most ride_gbs x its own duration of additions."""
    base = dict(leaf_cols=256, min_dim=128, max_depth=3, hbm_gbs=1e9, ws_budget_gb=0.02)
    free = auto_plan.plan_ata_auto(4096, 2048, 2048, 2048, auto_plan.AutoParams(**base, ride_gbs=1e12))
    tight = auto_plan.plan_ata_auto(4096, 2048, 2048, 2048, auto_plan.AutoParams(**base, ride_gbs=800.0))
    none = auto_plan.plan_ata_auto(4096, 2048, 2048, 2048, auto_plan.AutoParams(**base, ride_gbs=0.0))
    count = lambda p: int(((p.ops["flags"] & nat.OPF_RIDE) != 0).sum())
    assert count(free) > count(tight) >= count(none) == 0
    for (i, j, g0, g1) in _ride_runs(tight.ops):
        flops = sum(2.0 * int(o["m"]) * int(o["n"]) * int(o["k"]) if int(o["type"]) == nat.OP_GEMM
                    else 1.0 * int(o["m"]) * int(o["n"]) * (int(o["n"]) + 1) for o in tight.ops[g0:g1])
        moved = sum(auto_plan._op_bytes(o) for o in tight.ops[i:j])
        assert moved <= 800e9 * flops / (auto_plan.AutoParams().dmma_tflops * 1e12) + 1


# looking back across groups, row bands of large sums, alternating top-level arenas
SPREAD = dict(ride_lookback=16, ride_band_gb=2e-6, ride_arenas=True)


@settings(max_examples=25, deadline=None)
@given(m=st.integers(40, 400), n=st.integers(40, 260), seed=st.integers(0, 2**16),
       budget=st.sampled_from([4e-6, 2e-5, 1e-4]), gbs=st.sampled_from([1e12, 3e6, 3e5]),
       arenas=st.booleans(), band=st.sampled_from([0.0, 2e-6, 2e-5]))
def test_spread_hoist_keeps_plan_semantics(m, n, seed, budget, gbs, arenas, band):
    """Sums riding several groups early, cut into row bands, frames in two arenas:
    the op list still computes lower(A^T A) sequentially, with the same products."""
    a = np.random.default_rng(seed).uniform(-1, 1, (m, n))
    kw = {**FORCED_DFS, "ws_budget_gb": budget, "ride_gbs": gbs, "ride_lookback": 16,
          "ride_band_gb": band, "ride_arenas": arenas}
    p = auto_plan.plan_ata_auto(m, n, n, n, auto_plan.AutoParams(**kw))
    c = np.zeros((n, n))
    c[np.triu_indices(n, 1)] = 7.0
    plan_interp.run(p.ops, a, c, 1.0, WS=np.zeros(max(1, p.ws_scalars)))
    assert np.all(c[np.triu_indices(n, 1)] == 7.0)
    assert O.rel_frobenius_lower(c, O.gram(a)) <= 1e-12
    q = auto_plan.plan_ata_auto(m, n, n, n, auto_plan.AutoParams(**{**FORCED_DFS, "ws_budget_gb": budget,
                                                                    "ride_sums": False}))
    assert q.mults == p.mults
    is_prod = lambda o: np.isin(o["type"], (nat.OP_GEMM, nat.OP_SYRK))
    assert int(is_prod(p.ops).sum()) == int(is_prod(q.ops).sum())
    if band == 0.0:
        assert len(p.ops) == len(q.ops)


@pytest.mark.parametrize("m,n", [(192, 160), (257, 131), (300, 96), (520, 300)])
def test_spread_ride_ops_are_independent_of_their_group(m, n):
    p = auto_plan.plan_ata_auto(m, n, n, n, auto_plan.AutoParams(**{**FORCED_DFS, **SPREAD}))
    ops = p.ops
    runs = _ride_runs(ops)
    assert runs
    assert int((ops["flags"] & nat.OPF_RIDE).sum()) == sum(j - i for i, j, _, _ in runs)
    for (i, j, g0, g1) in runs:
        assert g1 > g0
        g_reads, g_writes = set(), set()
        for q in range(g0, g1):
            r, w = _reads_writes(ops[q])
            g_reads |= r
            g_writes |= w
        for q in range(i, j):
            assert int(ops[q]["type"]) == nat.OP_COMBO4 and int(ops[q]["accumulate"]) == 0
            r, w = _reads_writes(ops[q])
            assert not (w & g_reads) and not (w & g_writes) and not (r & g_writes), (q, g0, g1)


def test_spread_hoist_hides_more_than_the_adjacent_one():
    """Config c4: with look-back, row bands and two arenas almost every operand sum rides
    (146.8 GB exposed -> 2.4 GB), no group above its capacity."""
    def exposed(**kw):
        p = auto_plan.plan_ata_auto(65536, 32768, 32768, 32768, auto_plan.AutoParams(**kw))
        ops = p.ops
        e = sum(auto_plan._op_bytes(o) for o in ops
                if int(o["type"]) == nat.OP_COMBO4 and not int(o["flags"]) & nat.OPF_RIDE)
        return e, p
    old = dict(ride_gbs=800.0, gain_ride=1.25)       # the tree and capacity the hoist was first measured on
    e0, p0 = exposed(**old, ride_lookback=0, ride_band_gb=0.0, ride_arenas=False)
    e1, p1 = exposed(**old, ride_lookback=64, ride_band_gb=1.25, ride_arenas=False)
    e2, p2 = exposed(**old, ride_lookback=64, ride_band_gb=1.25, ride_arenas=True)
    assert e0 > e1 > e2 and e2 < 5e9
    assert p0.mults == p1.mults == p2.mults
    assert p1.ws_scalars == p0.ws_scalars and p2.ws_scalars * 8 <= 80e9
    for (i, j, g0, g1) in _ride_runs(p2.ops):
        flops = sum(2.0 * int(o["m"]) * int(o["n"]) * int(o["k"]) if int(o["type"]) == nat.OP_GEMM
                    else 1.0 * int(o["m"]) * int(o["n"]) * (int(o["n"]) + 1) for o in p2.ops[g0:g1])
        moved = sum(auto_plan._op_bytes(o) for o in p2.ops[i:j])
        assert moved <= 800e9 * flops / (auto_plan.AutoParams().dmma_tflops * 1e12) + 1


@pytest.mark.parametrize("m,n,private", [(260, 200, True), (333, 170, True), (260, 200, False)])
def test_private_tail_of_a_large_group(m, n, private):
    """A leaf group too large for a shared-destination launch (> MAX_BATCH_NARROW
    products) K-splits its trailing products into private partials summed by combo4
    passes behind the group: same result, same multiplications, no regions."""
    a = np.random.default_rng(m * n).uniform(-1, 1, (m, n))
    kw = dict(leaf_cols=16, min_dim=4, max_depth=3, hbm_gbs=1e9, ws_budget_gb=1.0, min_tail_rows=2,
              tail_private=private)
    p = auto_plan.plan_ata_auto(m, n, n, n, auto_plan.AutoParams(**kw))
    q = auto_plan.plan_ata_auto(m, n, n, n, auto_plan.AutoParams(**{**kw, "tail_split": False}))
    ops = p.ops
    prod = np.isin(ops["type"], (nat.OP_GEMM, nat.OP_SYRK))
    sizes = {}
    for o in ops[prod]:
        sizes[int(o["group"])] = sizes.get(int(o["group"]), 0) + 1
    big = [g for g, c in sizes.items() if c > auto_plan.MAX_BATCH_NARROW]
    assert big, "the breadth-first tree has a group beyond one shared-destination launch"
    regions = {g: any(int(d["region"]) > 0 for o in ops[prod & (ops["group"] == g)] for d in o["d"][:int(o["nd"])])
               for g in big}
    assert not any(regions.values())
    if private:
        assert int(prod.sum()) > int(np.isin(q.ops["type"], (nat.OP_GEMM, nat.OP_SYRK)).sum())
    assert p.mults == q.mults
    c = np.zeros((n, n))
    c[np.triu_indices(n, 1)] = 7.0
    plan_interp.run(ops, a, c, 1.0, WS=np.zeros(max(1, p.ws_scalars)))
    assert np.all(c[np.triu_indices(n, 1)] == 7.0)
    assert O.rel_frobenius_lower(c, O.gram(a)) <= 1e-12
