"""Host logic of the distribute-compute-retrieve executor (distsim.py) on CPU:
the per-process program, the seeded in-process scheduler, the message
accounting (CommStats), the bounds (verify_comm_bounds) and the
torch.distributed transport over gloo with world size 2 and 3.  Every case is
pinned to the reference's own ata_d run (tests/golden/distsim.json, written by
tools/make_golden_exec.py): identical counters, identical message trace,
identical multiplication count and the same result.  Block operations and
leaves are the CPU stand-ins of tests/exec_host.py (oracle arithmetic); the
device versions are covered by tests/test_gpu_executors.py."""
import json
import os
import socket

import numpy as np
import pytest
import torch

from exec_host import HostBlocks, oracle_leaf
from paper_2110_13042_b200 import distsim as D
from paper_2110_13042_b200.errors import ProtocolError
from paper_2110_13042_b200.measure import gen_matrix
from paper_2110_13042_b200.tasktree import Region, build_tree_distributed

from conftest import GOLDEN

CASES = json.loads((GOLDEN / "distsim.json").read_text())
RESULTS = np.load(GOLDEN / "exec_results.npz")


def _region(r):
    return [r.row_offset, r.col_offset, r.rows, r.cols]


def _simulate(case, seed):
    p, m, n = case["p"], case["m"], case["n"]
    a = torch.from_numpy(gen_matrix(m, n, case["seed"]).a.copy())
    tree = build_tree_distributed(p, m, n)
    count = [0]
    leaf = oracle_leaf(case["threshold"], case["leaf_kernel"], count)
    ops = HostBlocks()
    gens = {q: D.process_program(q, tree, a if q == 0 else None, ops, leaf) for q in range(p)}
    stats, trace = D.CommStats(p), []
    done = D.run_processes(gens, stats, trace, seed)
    return done[0][0].numpy(), stats, trace, count[0]


@pytest.mark.parametrize("case", CASES["cases"], ids=lambda c: f"P{c['p']}_{c['m']}x{c['n']}")
def test_program_matches_reference_run(case):
    got, st, trace, mults = _simulate(case, seed=3)
    assert st.sent_messages == case["sent_messages"] and st.sent_words == case["sent_words"]
    assert st.recv_messages == case["recv_messages"] and st.recv_words == case["recv_words"]
    assert st.critical_path_messages == case["critical_path_messages"]
    assert st.total_words == case["total_words"]
    assert [[s, d, [[k, _region(r), w] for (k, r, w) in parts]] for (s, d, parts) in trace] == case["trace"]
    assert mults == case["mults"]
    ref = RESULTS[case["key"]]
    n = case["n"]
    il = np.tril_indices(n)
    np.testing.assert_allclose(got[il], ref[il], rtol=1e-12, atol=1e-12 * case["m"])
    rep = D.verify_comm_bounds(st, n, case["p"])
    assert rep.ok == case["report"]["ok"] and rep.summary() == case["report"]["summary"]
    assert rep.latency_bound == case["report"]["latency_bound"]
    assert rep.words_bound == case["report"]["words_bound"]


@pytest.mark.parametrize("case", [c for c in CASES["cases"] if c["p"] in (6, 8, 11)],
                         ids=lambda c: f"P{c['p']}")
def test_interleaving_independence(case):
    """Any scheduler seed: the same result bits and the same counters."""
    base, st0, _, _ = _simulate(case, seed=0)
    for seed in (1, 7, 123):
        got, st, _, _ = _simulate(case, seed)
        assert np.array_equal(got, base)
        assert st.sent_words == st0.sent_words and st.recv_messages == st0.recv_messages


def test_bounds_match_reference():
    for b in CASES["bounds"]:
        assert D.comm_bound_latency(b["p"]) == b["latency"]
        assert D.comm_bound_words(b["n"], b["p"]) == pytest.approx(b["words"], rel=1e-15, abs=0)


def test_comm_stats_csv(tmp_path):
    st = D.CommStats(3, [1, 2, 3], [10, 20, 30], [3, 2, 1], [30, 20, 10])
    path = tmp_path / "c.csv"
    st.write_csv(path)
    lines = path.read_text().splitlines()
    assert lines[0] == "process,sent_messages,sent_words,recv_messages,recv_words"
    assert lines[1] == "0,1,10,3,30" and lines[-1] == "critical_path,1,10,3,30"
    assert st.critical_path_messages == 4 and st.total_messages == 6 and st.total_words == 60


def test_protocol_errors():
    ops = HostBlocks()
    with pytest.raises(ProtocolError):
        D.MessagePart("rect", Region(0, 0, 2, 3), torch.zeros(5))
    with pytest.raises(ProtocolError):
        D.MessagePart("packed", Region(0, 0, 3, 3), torch.zeros(9))

    def waits_forever():
        yield ("recv", 1, [("rect", Region(0, 0, 1, 1))])

    def silent():
        return None
        yield  # pragma: no cover

    with pytest.raises(ProtocolError, match="deadlock"):
        D.run_processes({0: waits_forever(), 1: silent()}, D.CommStats(2))

    def sends_unread():
        yield ("send", D.Message(0, 1, [D.MessagePart("rect", Region(0, 0, 1, 1), ops.zeros(1, 1).view(-1))]))

    with pytest.raises(ProtocolError, match="undelivered"):
        D.run_processes({0: sends_unread(), 1: silent()}, D.CommStats(2))

    def wrong_region():
        yield ("recv", 0, [("rect", Region(0, 0, 2, 2))])

    def sends_small():
        yield ("send", D.Message(0, 1, [D.MessagePart("rect", Region(0, 0, 1, 1), ops.zeros(1, 1).view(-1))]))

    with pytest.raises(ProtocolError, match="expected"):
        D.run_processes({0: sends_small(), 1: wrong_region()}, D.CommStats(2))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_worker(rank, world, port, case, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist
    from exec_host import HostBlocks, oracle_leaf
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, n = case["m"], case["n"]
    tree = build_tree_distributed(world, m, n)
    a = torch.from_numpy(gen_matrix(m, n, case["seed"]).a.copy()) if rank == 0 else None
    ops = HostBlocks()
    count = [0]
    st = D.CommStats(world)
    res, _ = D.run_rank(rank, D.process_program(rank, tree, a, ops, oracle_leaf(case["threshold"],
                                                                                 case["leaf_kernel"], count)),
                        D._GroupLink(None, ops), st)
    full = D._gather_stats(st, None, torch.device("cpu"))
    mults = torch.tensor([count[0]], dtype=torch.int64)
    dist.all_reduce(mults)
    if rank == 0:
        out.put((res.numpy().copy(), full.sent_messages, full.sent_words, full.recv_messages,
                 full.recv_words, int(mults.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_ranks_match_reference(world):
    """One OS process per rank over torch.distributed (gloo): the operand
    blocks really travel from rank 0 and the partials back."""
    import torch.multiprocessing as mp
    case = next(c for c in CASES["cases"] if c["p"] == world)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, sm, sw, rm, rw, mults = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert (sm, sw, rm, rw) == (case["sent_messages"], case["sent_words"], case["recv_messages"],
                                case["recv_words"])
    assert mults == case["mults"]
    ref = RESULTS[case["key"]]
    il = np.tril_indices(case["n"])
    np.testing.assert_allclose(got[il], ref[il], rtol=1e-12, atol=1e-12 * case["m"])
