"""Riding operand sums on the GPU (ATA_OPF_RIDE): forced depth-first auto plans
whose Strassen operand sums execute inside the previous leaf group's product
launch (the FP64 TMA kernel's spare warps) must match the BLAS Gram of the
same input, the launches must actually have carried sums, and sums that cannot
ride (odd windows) must run as ordinary passes with the same result."""
import numpy as np
import pytest

from oracle import atamul_oracle as O

pytestmark = pytest.mark.gpu
SENT = 1.2345e67

# (ride_gbs: no capacity limit, so these small plans exercise the riding path)
DEEP = dict(leaf_cols=256, min_dim=128, max_depth=3, hbm_gbs=1e9, ride_gbs=1e12)


def _ata(a, params, alpha=1.0):
    import torch
    import paper_2110_13042_b200 as P
    from paper_2110_13042_b200 import _native as nat
    n = a.shape[1]
    C = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    iu = torch.triu_indices(n, n, 1, device="cuda")
    C[iu[0], iu[1]] = SENT
    lib = nat.load()
    r0 = lib.ata_ride_count()
    P.ata(torch.from_numpy(a).cuda(), C, alpha, threshold="auto", auto_params=params)
    torch.cuda.synchronize()
    return C.cpu().numpy(), lib.ata_ride_count() - r0


@pytest.mark.parametrize("m,n,budget,rides", [(4096, 2048, 0.02, True), (3000, 1536, 0.01, True),
                                              (1024, 1024, 0.004, True), (8192, 4096, 0.2, True),
                                              # odd quadrant windows: the sums cannot ride and run as passes
                                              (2050, 1100, 0.005, False), (1537, 1030, 0.003, False)])
def test_riding_sums_match_blas(m, n, budget, rides):
    from paper_2110_13042_b200.auto_plan import AutoParams, plan_ata_auto
    from paper_2110_13042_b200 import _native as nat
    params = AutoParams(**{**DEEP, "ws_budget_gb": budget})
    plan = plan_ata_auto(m, n, n, n, params)
    assert (plan.ops["flags"] & nat.OPF_RIDE).any(), "the plan has riding sums"
    a = np.random.default_rng(m + n).uniform(-1, 1, (m, n))
    want = O.gram_blas(a)
    got, carried = _ata(a, params)
    assert np.all(got[np.triu_indices(n, 1)] == SENT)
    assert O.rel_frobenius_lower(got, want) <= 1e-12
    if rides:
        assert carried > 0, "no product launch carried operand sums"
    # the plan without riding sums: same ops (scratch addresses differ, and with them the
    # alignment-dependent choice between the TMA and cp.async leaf kernels)
    import dataclasses
    plain, none = _ata(a, dataclasses.replace(params, ride_sums=False))
    assert none == 0
    assert O.rel_frobenius_lower(got, np.tril(plain)) <= 1e-14


def test_riding_is_deterministic_and_alpha_linear():
    from paper_2110_13042_b200.auto_plan import AutoParams
    params = AutoParams(**{**DEEP, "ws_budget_gb": 0.02})
    a = np.random.default_rng(5).standard_normal((4096, 2048))
    c1, r1 = _ata(a, params)
    c2, r2 = _ata(a, params)
    assert r1 > 0 and r1 == r2
    assert np.array_equal(np.tril(c1), np.tril(c2))
    c3, _ = _ata(a, params, alpha=-2.0)
    assert np.array_equal(np.tril(c3), -2.0 * np.tril(c1))


def test_narrow_odd_window_products_are_zero_extended():
    """Regression: a product operand window with an odd width narrower than the
    product (odd Strassen quadrants, 137 of 138 columns) must read zeros past
    its last column; the TMA 2-D map would have delivered the next column."""
    from paper_2110_13042_b200.auto_plan import AutoParams
    a = np.random.default_rng(0).standard_normal((2050, 1100))
    got, _ = _ata(a, AutoParams(**{**DEEP, "ws_budget_gb": 0.005, "ride_sums": False}))
    assert O.rel_frobenius_lower(got, O.gram_blas(a)) <= 1e-12


@pytest.mark.parametrize("m,n,budget", [(4096, 2048, 0.02), (8192, 4096, 0.05), (3000, 1536, 0.01)])
@pytest.mark.parametrize("arenas", [False, True])
def test_spread_riding_sums_match_blas(m, n, budget, arenas):
    """Sums hoisted several groups early, cut into row bands, top-level frames in
    two arenas (auto_plan._hoist_sums lookback / _split_bands / _enter_frame)."""
    from paper_2110_13042_b200.auto_plan import AutoParams, plan_ata_auto
    from paper_2110_13042_b200 import _native as nat
    params = AutoParams(**{**DEEP, "ws_budget_gb": budget, "ride_lookback": 16, "ride_band_gb": 1e-3,
                           "ride_arenas": arenas, "ride_gbs": 3e4})
    near = plan_ata_auto(m, n, n, n, AutoParams(**{**DEEP, "ws_budget_gb": budget, "ride_gbs": 3e4,
                                                   "ride_lookback": 0, "ride_band_gb": 0.0, "ride_arenas": False}))
    plan = plan_ata_auto(m, n, n, n, params)
    riding = lambda p: int(((p.ops["flags"] & nat.OPF_RIDE) != 0).sum())
    assert riding(plan) > riding(near) > 0
    a = np.random.default_rng(m + n + 1).uniform(-1, 1, (m, n))
    got, carried = _ata(a, params)
    assert carried > 0
    assert np.all(got[np.triu_indices(n, 1)] == SENT)
    assert O.rel_frobenius_lower(got, O.gram_blas(a)) <= 1e-12


def test_private_tail_split_matches_blas():
    """A 343-leaf group (one launch, beyond the shared-destination batch size):
    its trailing products are K-split into private partials (AutoParams.tail_private)."""
    from paper_2110_13042_b200.auto_plan import AutoParams, plan_ata_auto, MAX_BATCH_NARROW
    from paper_2110_13042_b200 import _native as nat
    m, n = 8192, 4096
    params = AutoParams(leaf_cols=2048, min_dim=128, max_depth=3, hbm_gbs=1e9, ws_budget_gb=4.0, min_tail_rows=128)
    plan = plan_ata_auto(m, n, n, n, params)
    prod = np.isin(plan.ops["type"], (nat.OP_GEMM, nat.OP_SYRK))
    groups = np.unique(plan.ops["group"][prod], return_counts=True)
    assert groups[1].max() > MAX_BATCH_NARROW + 20
    import dataclasses
    plain = plan_ata_auto(m, n, n, n, dataclasses.replace(params, tail_split=False))
    assert int(prod.sum()) > int(np.isin(plain.ops["type"], (nat.OP_GEMM, nat.OP_SYRK)).sum())
    a = np.random.default_rng(11).uniform(-1, 1, (m, n))
    got, _ = _ata(a, params)
    assert np.all(got[np.triu_indices(n, 1)] == SENT)
    assert O.rel_frobenius_lower(got, O.gram_blas(a)) <= 1e-12
