"""Multi-GPU units partition (auto_plan.partition_units / plan_units,
dist.reduce_regions) on CPU: the top level's two AtA sub-problems and the
seven Strassen products of its C21 node as row-range segments on P ranks.

* every rank's plan, run by the NumPy plan interpreter (tests/plan_interp.py),
  summed over the ranks equals the oracle's classical Gram (odd shapes, P = 1..8);
* the balance: at config c4 the critical path (max executed multiplications
  per rank) is below the row-shard partition's for P = 4 and 8;
* world size 2 over gloo: each rank computes only its segments from the rows
  it needs, the regions are reduced to rank 0 with the real region groups,
  and rank 0's lower triangle matches the oracle."""
import os
import socket

import numpy as np
import pytest

import plan_interp
from oracle import atamul_oracle as O
from paper_2110_13042_b200 import auto_plan as ap
from paper_2110_13042_b200 import dist as pdist

SMALL = ap.AutoParams(leaf_cols=16, min_dim=4, hbm_gbs=1e9, max_depth=3)


def _interp(segments, a, params=SMALL):
    m, n = a.shape
    plan = ap.plan_units(segments, m, n, n, n, params)
    C = np.zeros((n, n))
    WS = np.zeros(max(1, plan.ws_scalars))
    plan_interp.run(plan.ops, a.copy(), C, 1.0, WS)
    return C, plan


@pytest.mark.parametrize("m,n", [(96, 80), (101, 77), (64, 131), (257, 66)])
@pytest.mark.parametrize("procs", [1, 2, 3, 5, 8])
def test_units_sum_to_gram(m, n, procs):
    a = np.random.default_rng(m * n + procs).uniform(-1, 1, (m, n))
    parts = ap.partition_units(m, n, procs, SMALL, align=4)
    assert len(parts) == procs
    # each unit's contraction rows are covered exactly once, in order
    for u in ap.UNITS:
        spans = sorted((r0, r1) for segs in parts for (uu, r0, r1) in segs if uu == u)
        rows = ap.unit_rows(u, m, n)
        assert spans[0][0] == 0 and spans[-1][1] == rows
        assert all(x[1] == y[0] for x, y in zip(spans, spans[1:]))
    total = np.zeros((n, n))
    for segs in parts:
        C, _ = _interp(segs, a)
        total += C
    ref = O.gram(a)
    assert O.rel_frobenius_lower(total, ref) <= 1e-12
    # the strict upper triangle is never written
    assert np.all(total[np.triu_indices(n, 1)] == 0.0)


def test_rows_needed_cover_reads():
    """A rank only needs the rows a_rows_needed names: zeroing every other
    row leaves its plan's result unchanged."""
    m, n = 101, 77
    a = np.random.default_rng(1).uniform(-1, 1, (m, n))
    for segs in ap.partition_units(m, n, 5, SMALL, align=4):
        full, _ = _interp(segs, a)
        part = np.zeros_like(a)
        for lo, hi in ap.a_rows_needed(segs, m, n):
            part[lo:hi] = a[lo:hi]
        got, _ = _interp(segs, part)
        assert np.array_equal(got, full)


def test_c4_balance_beats_row_shards():
    m, n = 65536, 32768
    costs = ap.unit_costs(m, n)
    single = ap.plan_ata_auto(m, n, n, n).mults
    assert abs(sum(costs[u] * ap.unit_rows(u, m, n) for u in ap.UNITS) - single) <= 1e-9 * single
    for P in (4, 8):
        loads = [ap.plan_units(s, m, n, n, n).mults for s in ap.partition_units(m, n, P, costs=costs)]
        rows_shard = ap.plan_ata_auto(m // P, n, n, n).mults
        assert max(loads) < 0.975 * rows_shard, (P, max(loads), rows_shard)
        assert max(loads) <= 1.02 * sum(loads) / P


def test_region_members():
    parts = [[("ata_l", 0, 10)], [("ata_l", 10, 20), ("ata_r", 0, 5)], [("ata_r", 5, 20), ("p1", 0, 3)],
             [("p1", 3, 10), ("p7", 0, 10)]]
    mem = pdist.region_members(parts)
    assert mem == {"c11": [0, 1], "c22": [0, 1, 2], "c21": [0, 2, 3]}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, m, n, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch
    import torch.distributed as dist
    from exec_host import HostBlocks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = np.random.default_rng(7).uniform(-1, 1, (m, n))
    parts = ap.partition_units(m, n, world, SMALL, align=4)
    mine = parts[rank]
    a = np.zeros_like(full)                       # only the rows this rank needs
    for lo, hi in ap.a_rows_needed(mine, m, n):
        a[lo:hi] = full[lo:hi]
    C, _ = _interp(mine, a)
    Ct = torch.from_numpy(C)
    groups, members = pdist.make_region_groups(parts)
    pdist.reduce_regions(Ct, n, rank, groups, members, HostBlocks())
    if rank == 0:
        out.put(Ct.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_units_reduce(world):
    import torch.multiprocessing as mp
    m, n = 101, 77
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = np.random.default_rng(7).uniform(-1, 1, (m, n))
    assert O.rel_frobenius_lower(got, O.gram(a)) <= 1e-12
