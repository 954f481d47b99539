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


def test_random_windows_products_vs_numpy():
    """Randomised leaf products through the native executor: random shapes,
    pitches (even / odd), column offsets (16-byte aligned, 8-byte aligned),
    GEMM and SYRK, one or two terms per operand -- so every operand path of
    the FP64 product kernels (TMA 3-D maps, TMA 2-D maps, cp.async) and the
    diagonal-tile patterns get exercised -- against NumPy in fp64."""
    import torch
    from paper_2110_13042_b200 import _native as nat, engine, planner
    from paper_2110_13042_b200.planner import Win
    rng = np.random.default_rng(2024)
    for case in range(40):
        m = int(rng.integers(1, 700))
        n = int(rng.integers(1, 400))
        k = int(rng.integers(1, 400))
        ld = int(rng.integers(n + k + 4, n + k + 40))
        off = int(rng.integers(0, 4))
        kind = "syrk" if rng.random() < 0.3 else "gemm"
        two = rng.random() < 0.3 and kind == "gemm"
        A = rng.uniform(-1, 1, (2 * m + 2, ld))
        dA = torch.from_numpy(A).cuda()
        pb = planner.PlanBuilder("rand")
        g = pb.new_group()
        s0 = Win(nat.BASE_A, off, ld, m, n)
        t0 = Win(nat.BASE_A, off + n + 1, ld, m, k)
        S, T = [(s0, 1.0)], [(t0, 1.0)]
        Sn = A[:m, off:off + n].copy()
        Tn = A[:m, off + n + 1:off + n + 1 + k].copy()
        if two:
            s1 = Win(nat.BASE_A, (m + 1) * ld + off, ld, m, n)
            S.append((s1, -1.0))
            Sn = Sn - A[m + 1:2 * m + 1, off:off + n]
        kk = n if kind == "syrk" else k
        C = torch.full((n, kk), 0.5, dtype=torch.float64, device="cuda")
        out = Win(nat.BASE_C, 0, kk, n, kk)
        pb.product(kind, m, n, kk, S, [] if kind == "syrk" else T, [(out, 1.0)], accumulate=1, group=g)
        plan = pb.finish()
        engine.run_plan(plan, nat.ATA_F64, dA.data_ptr(), dA.numel(), C.data_ptr(), C.numel(), 2.0)
        got = C.cpu().numpy()
        ref = 0.5 + 2.0 * (Sn.T @ (Sn if kind == "syrk" else Tn))
        if kind == "syrk":
            il = np.tril_indices(n)
            assert np.all(got[np.triu_indices(n, 1)] == 0.5), case
            got, ref = got[il], ref[il]
        assert np.abs(got - ref).max() <= 1e-12 * max(1, m), (case, m, n, k, ld, off, kind, two)
