"""GPU executors behind the reference names (shared.py, distsim.py,
execute.py): ata_s / SharedRunner (leaves on concurrent CUDA streams),
ata_d / CommStats / verify_comm_bounds (distribute-compute-retrieve, simulated
on one GPU), execute_leaf, and MatrixView operands.  Checked against the
reference's own runs (tests/golden/shared.json, distsim.json,
exec_results.npz from tools/make_golden_exec.py) and the CPU oracle."""
import json

import numpy as np
import pytest

from oracle import atamul_oracle as O

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

SHARED = json.loads((GOLDEN / "shared.json").read_text())["cases"]
DIST = json.loads((GOLDEN / "distsim.json").read_text())["cases"]
RESULTS = np.load(GOLDEN / "exec_results.npz")


def _close(got, ref, tol=1e-12):
    got = np.asarray(got)
    assert O.rel_frobenius_lower(got, ref) <= tol
    # ata_s / ata_d return the full symmetric matrix (mirrored)
    assert np.array_equal(got, got.T)


@pytest.mark.parametrize("case", SHARED, ids=lambda c: f"P{c['p']}_{c['m']}x{c['n']}")
def test_shared_runner_matches_reference(case):
    import paper_2110_13042_b200 as P
    a = P.gen_matrix(case["m"], case["n"], case["seed"]).a
    runner = P.SharedRunner(a, case["p"], threshold=case["threshold"], count_mults=True)
    runner.prepare()
    res = runner.run()
    assert isinstance(res.a, np.ndarray)
    _close(res.a, RESULTS[case["key"]])
    assert runner.max_worker_mults == case["max_worker_mults"]
    assert [c.scalar_mults for c in runner.counters] == case["worker_mults"]
    # a second run reuses the tree, workspaces and streams
    res2 = runner.run()
    assert np.array_equal(res.a, res2.a)


def test_ata_s_device_input_and_errors():
    import torch
    import paper_2110_13042_b200 as P
    A = torch.from_numpy(P.gen_matrix(700, 513, 9).a).cuda()
    res = P.ata_s(A, 5, threshold="auto")
    assert res.a.is_cuda
    ref = O.gram_blas(A.cpu().numpy())
    assert O.rel_frobenius_lower(res.a.cpu().numpy(), ref) <= 1e-13
    with pytest.raises(P.TooManyWorkersError):
        P.SharedRunner(A, 129)
    with pytest.raises(ValueError):
        P.SharedRunner(A, 0)


@pytest.mark.parametrize("case", DIST, ids=lambda c: f"P{c['p']}_{c['m']}x{c['n']}")
def test_ata_d_matches_reference(case):
    import paper_2110_13042_b200 as P
    a = P.gen_matrix(case["m"], case["n"], case["seed"]).a
    cnt = P.MultCounter()
    trace = []
    res, st = P.ata_d(a, case["p"], threshold=case["threshold"], leaf_kernel=case["leaf_kernel"],
                      scheduler_seed=3, counter=cnt, trace=trace)
    _close(res.a, RESULTS[case["key"]])
    assert (st.sent_messages, st.sent_words, st.recv_messages, st.recv_words) == \
        (case["sent_messages"], case["sent_words"], case["recv_messages"], case["recv_words"])
    assert len(trace) == len(case["trace"])
    assert cnt.scalar_mults == case["mults"]
    assert st.compute_seconds > 0
    rep = P.verify_comm_bounds(st, case["n"], case["p"])
    assert rep.summary() == case["report"]["summary"]


def test_ata_d_auto_threshold_device():
    import torch
    import paper_2110_13042_b200 as P
    A = torch.from_numpy(P.gen_matrix(2048, 1536, 4).a).cuda()
    res, st = P.ata_d(A, 8, threshold="auto")
    assert res.a.is_cuda
    ref = O.gram_blas(A.cpu().numpy())
    assert O.rel_frobenius_lower(res.a.cpu().numpy(), ref) <= 1e-13
    assert st.total_messages == sum(st.recv_messages)


def test_execute_leaf_covers_shared_tree_host_buffers():
    """Every leaf of a shared tree through execute_leaf into one HOST C
    (staged through the device and written back in place): the union is
    lower(A^T A) (the covering property of scheduler.py)."""
    import paper_2110_13042_b200 as P
    from paper_2110_13042_b200.tasktree import build_tree_shared, leaf_task
    m, n, procs = 301, 203, 7
    a = P.gen_matrix(m, n, 11).a
    tree = build_tree_shared(procs, m, n)
    c = np.zeros((n, n))
    c[np.triu_indices(n, 1)] = 3.5
    cnt = P.MultCounter()
    for p in range(procs):
        task = leaf_task(tree, p)
        P.execute_leaf(task, a, c, 4096, cnt, "fast", P.workspace_for_leaf(task, 4096))
    assert np.all(c[np.triu_indices(n, 1)] == 3.5)
    assert O.rel_frobenius_lower(c, O.gram_blas(a)) <= 1e-13
    c2 = np.zeros((n, n))
    for p in range(procs):
        P.execute_leaf(leaf_task(tree, p), a, c2, 4096, None, "naive")
    assert O.rel_frobenius_lower(c2, O.gram_blas(a)) <= 1e-13
    with pytest.raises(ValueError):
        P.execute_leaf(leaf_task(tree, 0), a, c2, 4096, None, "blas")


def test_matrix_view_operands():
    """MatrixView inputs (matrix.py:107-150): A and C as windows of larger
    DenseMatrix buffers, host and device; only the window's lower triangle
    changes."""
    import torch
    import paper_2110_13042_b200 as P
    rng = np.random.default_rng(3)
    baseA = P.DenseMatrix(rng.uniform(-1, 1, (400, 300)))
    baseC = P.DenseMatrix.zeros(260, 260)
    av = baseA.view(17, 31, 351, 203)
    cv = baseC.view(40, 50, 203, 203)
    P.ata(av, cv, 1.0, threshold=2048)
    ref = O.gram_blas(av.a)
    assert O.rel_frobenius_lower(cv.a, ref) <= 1e-13
    touched = np.zeros((260, 260), dtype=bool)
    touched[40:243, 50:253] = np.tril(np.ones((203, 203), dtype=bool))
    assert np.all(baseC.a[~touched] == 0.0)
    # fast_strassen on views of one device base, quadrants from split4
    dA = P.DenseMatrix(torch.from_numpy(baseA.a).cuda())
    q = P.split4(dA.view(0, 0, 400, 300))
    out = P.DenseMatrix.zeros(150, 150, device="cuda")
    P.fast_strassen(q[0], q[1], out.view(), 1.0, threshold=4096)
    want = baseA.a[:200, :150].T @ baseA.a[:200, 150:300]
    assert np.abs(out.a.cpu().numpy() - want).max() <= 1e-12 * 200
