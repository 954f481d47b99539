"""Acceptance-style parity on the GPU (the reference's criteria):
a seeded sweep of 200 shapes through the reference recursion (integer
thresholds, exact multiplication counts) and the auto plan, with the
reference's tolerance 1e-9 * m * max|A|^2 and the strict upper triangle
untouched; all-ones inputs give every Gram entry exactly m (also through
Strassen and the distributed task tree); threshold independence."""
import numpy as np
import pytest

from oracle import atamul_oracle as O

pytestmark = pytest.mark.gpu
SENT = 1.2345e67


def _run(a, t, alpha=1.0):
    import torch
    import paper_2110_13042_b200 as P
    n = a.shape[1]
    C = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    iu = torch.triu_indices(n, n, 1, device="cuda")
    C[iu[0], iu[1]] = SENT
    cnt = P.MultCounter()
    P.ata(torch.from_numpy(a).cuda(), C, alpha, threshold=t, counter=cnt)
    return C.cpu().numpy(), cnt.scalar_mults


def test_acceptance_sweep_200_shapes():
    rng = np.random.default_rng(1234)
    thresholds = [1, 16, 64, 4096, "auto"]
    for case in range(200):
        t = thresholds[case % len(thresholds)]
        hi = 25 if t == 1 else 97          # t = 1 recurses to 1x1 leaves: keep those small
        m, n = int(rng.integers(1, hi)), int(rng.integers(1, hi))
        a = rng.uniform(-1, 1, (m, n))
        got, mults = _run(a, t)
        ref = O.gram_blas(a)
        tol = 1e-9 * m * max(float(np.abs(a).max()), 1e-30) ** 2
        il = np.tril_indices(n)
        assert np.abs(got[il] - ref[il]).max() <= tol, (case, m, n, t)
        assert np.all(got[np.triu_indices(n, 1)] == SENT), (case, m, n, t)
        if t != "auto":
            want = [0]
            O.ata_lower(a, np.zeros((n, n)), 1.0, t, want)
            assert mults == want[0], (case, m, n, t, mults, want[0])


@pytest.mark.parametrize("t", [1, 64, 4096, 1 << 15, "auto"])
def test_all_ones_exact(t):
    m, n = (41, 37) if t == 1 else (301, 257)
    got, _ = _run(np.ones((m, n)), t)
    il = np.tril_indices(n)
    assert np.all(got[il] == float(m))


def test_all_ones_exact_strassen_and_tree():
    import torch
    import paper_2110_13042_b200 as P
    from paper_2110_13042_b200 import dist
    from paper_2110_13042_b200.auto_plan import AutoParams
    m, n, k = 1031, 700, 650
    A = torch.ones((m, n), dtype=torch.float64, device="cuda")
    B = torch.ones((m, k), dtype=torch.float64, device="cuda")
    for t in (1 << 15, "auto"):
        C = torch.zeros((n, k), dtype=torch.float64, device="cuda")
        P.fast_strassen(A, B, C, 1.0, threshold=t,
                        auto_params=AutoParams(min_dim=64, hbm_gbs=1e9) if t == "auto" else None)
        assert bool((C == m).all()), t
    for procs in (2, 6, 8):
        C = torch.zeros((n, n), dtype=torch.float64, device="cuda")
        dist.ata_tree(lambda r: A[r.row_offset:r.row_offset + r.rows, r.col_offset:r.col_offset + r.cols],
                      m, n, C, 1.0, "auto", procs=procs)
        il = torch.tril_indices(n, n, device="cuda")
        assert bool((C[il[0], il[1]] == m).all()), procs


def test_threshold_independence():
    for (m, n, ts) in ((60, 45, (1, 64, 4096, "auto")), (300, 170, (64, 4096, "auto"))):
        a = np.random.default_rng(7).standard_normal((m, n))
        ref = O.gram_blas(a)
        for t in ts:
            got, _ = _run(a, t)
            assert O.rel_frobenius_lower(got, ref) <= 1e-13, (m, n, t)
