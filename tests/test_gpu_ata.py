"""GPU parity of the AtA / Strassen drop-ins against the reference's golden
outputs and the oracle: reference-faithful plans (exact counts), auto plans,
odd and degenerate shapes, workspace semantics, determinism, configs c1/c2."""
import numpy as np
import pytest

from oracle import atamul_oracle as O

pytestmark = pytest.mark.gpu


def test_golden_cases(golden):
    import paper_2110_13042_b200 as P
    meta, arrays = golden
    for case in meta["cases"]:
        key = case["key"]
        if case["kind"] == "ata":
            a = arrays[key + "_A"]
            n = a.shape[1]
            c = np.zeros((n, n), dtype=a.dtype)
            sentinel = 1.2345e67 if a.dtype == np.float64 else 3.0e30
            c[np.triu_indices(n, 1)] = sentinel
            cnt = P.MultCounter()
            P.ata(a, c, case["alpha"], threshold=case["threshold"], counter=cnt)
            assert cnt.scalar_mults == case["mults"], key
            assert np.all(c[np.triu_indices(n, 1)] == sentinel), key
            tol = 1e-10 if a.dtype == np.float64 else 1e-4
            assert O.rel_frobenius_lower(c, arrays[key + "_C"]) <= tol, key
        else:
            a, b, c0 = arrays[key + "_A"], arrays[key + "_B"], arrays[key + "_C0"]
            c = c0.copy()
            cnt = P.MultCounter()
            P.fast_strassen(a, b, c, 1.0, None, case["threshold"], cnt)
            assert cnt.scalar_mults == case["mults"], key
            ref = arrays[key + "_C"]
            assert np.linalg.norm(c - ref) <= 1e-10 * max(np.linalg.norm(ref), 1.0), key


def test_exact_counts_power_of_two(rng):
    import paper_2110_13042_b200 as P
    for n in [1, 2, 4, 8, 16, 32]:
        cnt = P.MultCounter()
        P.ata(rng.uniform(-1, 1, (n, n)), np.zeros((n, n)), 1.0, threshold=1, counter=cnt)
        assert cnt.scalar_mults == P.ata_mult_count(n)
        cnt = P.MultCounter()
        P.fast_strassen(rng.normal(size=(n, n)), rng.normal(size=(n, n)), np.zeros((n, n)), 1.0,
                        P.workspace_for(n, n, n, 1), 1, cnt)
        assert cnt.scalar_mults == P.strassen_mult_count(n)


@pytest.mark.parametrize("shape,t", [((1, 8), 4), ((8, 1), 4), ((63, 65), 16), ((512, 32), 512),
                                     ((300, 17), 512), ((129, 65), 1), ((1000, 999), 4096)])
def test_reference_plan_vs_oracle(shape, t, rng):
    import paper_2110_13042_b200 as P
    a = rng.uniform(-1, 1, shape)
    got = P.ata_full(a, threshold=t).a
    ref = O.gram(a)
    assert np.abs(got - ref).max() <= 1e-9 * shape[0]
    assert np.array_equal(got, got.T)


@pytest.mark.parametrize("shape", [(1, 1), (3, 300), (1000, 1), (2000, 2500), (4097, 1537),
                                   (5000, 3001)])
def test_auto_plan_vs_oracle(shape, rng):
    torch = pytest.importorskip("torch")
    import paper_2110_13042_b200 as P
    from paper_2110_13042_b200.auto_plan import AutoParams
    a = rng.standard_normal(shape)
    n = shape[1]
    for params in (AutoParams(), AutoParams(leaf_cols=256, min_dim=128, hbm_gbs=1e9),
                   AutoParams(leaf_cols=256, min_dim=128, hbm_gbs=1e9, fuse_leaf_sums=True)):
        A = torch.from_numpy(a).cuda()
        C = torch.triu(torch.full((n, n), 7.0, dtype=torch.float64, device="cuda"), 1)
        P.ata(A, C, 1.0, threshold="auto", auto_params=params)
        got = C.cpu().numpy()
        assert np.all(got[np.triu_indices(n, 1)] == 7.0)
        assert O.rel_frobenius_lower(got, O.gram_blas(a)) <= 1e-13


def test_workspace_reuse_zero_alloc_and_determinism(rng):
    import paper_2110_13042_b200 as P
    a, b = rng.uniform(-1, 1, (96, 80)), rng.uniform(-1, 1, (96, 70))
    ws = P.workspace_for(96, 80, 70, 64)
    c1 = np.zeros((80, 70))
    P.fast_strassen(a, b, c1, 1.0, ws, threshold=64)
    c2 = np.zeros((80, 70))
    with P.count_allocations() as tr:
        P.fast_strassen(a, b, c2, 1.0, ws, threshold=64)
    assert tr["count"] == 0
    assert np.array_equal(c1, c2)
    c3 = np.zeros((80, 70))
    P.fast_strassen(a, b, c3, 2.0, ws, threshold=64)
    assert np.array_equal(c3, 2.0 * c1)


def test_workspace_undersized_and_shape_errors():
    import paper_2110_13042_b200 as P
    ws = P.workspace_for_ata(8, 8, threshold=64)
    with pytest.raises(P.WorkspaceUndersizedError):
        P.ata(np.zeros((64, 64)), np.zeros((64, 64)), 1.0, threshold=64, ws=ws)
    with pytest.raises(P.ShapeMismatchError):
        P.ata(np.zeros((4, 3)), np.zeros((4, 4)))
    ws = P.workspace_for(8, 8, 8, threshold=32)
    with pytest.raises(P.WorkspaceUndersizedError):
        P.fast_strassen(np.zeros((8, 8)), np.zeros((8, 8)), np.zeros((8, 8)), 1.0, ws, threshold=1)


def test_workspace_dtype_differs_from_c(rng):
    """A workspace sized for f32 handed to an f64 call (legal in the
    reference: NumPy casts on assignment) computes the f64 result in an f64
    arena of the same scalar count -- no overrun of a half-sized buffer."""
    import torch
    import paper_2110_13042_b200 as P
    a = rng.uniform(-1, 1, (301, 203))
    ws = P.workspace_for_ata(301, 203, 4096, dtype=np.float32)
    c = np.zeros((203, 203))
    P.ata(a, c, 1.0, threshold=4096, ws=ws)
    assert ws.buffer.dtype == torch.float64
    assert ws.buffer.numel() * 8 >= ws.total_scalars * 8
    ref = np.zeros((203, 203))
    O.ata_lower(a, ref, 1.0, 4096)
    assert O.rel_frobenius_lower(c, ref) <= 1e-13
    b = rng.uniform(-1, 1, (301, 150))
    ws2 = P.workspace_for(301, 203, 150, 4096, dtype=np.float32)
    c2 = np.zeros((203, 150))
    P.fast_strassen(a, b, c2, 1.0, ws2, threshold=4096)
    assert np.allclose(c2, a.T @ b, rtol=0, atol=1e-11)


def test_config_c1_golden(golden):
    """c1 (1024^2 U[-1,1], seed 0) at the parity cutoff t = 64^2: exact count,
    sampled entries and checksums against the reference's own run."""
    import paper_2110_13042_b200 as P
    meta, arrays = golden
    info = meta["c1"]
    a = P.gen_matrix(1024, 1024, 0).a
    c = np.zeros((1024, 1024))
    cnt = P.MultCounter()
    P.ata(a, c, 1.0, threshold=info["threshold"], counter=cnt)
    assert cnt.scalar_mults == info["mults"]
    il, jl = np.tril_indices(1024)
    vals = c[il, jl]
    samp = arrays["c1_sample_val"]
    got = vals[arrays["c1_sample_idx"]]
    assert np.linalg.norm(got - samp) / np.linalg.norm(samp) <= 1e-12
    assert abs(np.linalg.norm(vals) - info["lower_fro"]) <= 1e-12 * info["lower_fro"]
    rows = np.array([c[i, :i + 1].sum() for i in range(1024)])
    assert np.linalg.norm(rows - arrays["c1_row_sums"]) <= 1e-11 * np.linalg.norm(arrays["c1_row_sums"])


def test_config_c2_full_parity():
    """c2 (6001x4097 N(0,1), seed 1, cutoff 256 -> t = 256^2): odd sizes on
    every level, checked on the stored triangle against the oracle."""
    import paper_2110_13042_b200 as P
    from paper_2110_13042_b200.measure import config_matrix
    a = config_matrix("c2")
    c = np.zeros((4097, 4097))
    P.ata(a, c, 1.0, threshold=256 * 256)
    assert O.rel_frobenius_lower(c, O.gram_blas(a)) <= 1e-10


@pytest.mark.parametrize("dtype,precision,geometric", [("f64", "fp32", False), ("f32", "tf32", False),
                                                       ("f64", "fp32", True)])
def test_pipelined_host_ata(monkeypatch, dtype, precision, geometric):
    """Pinned host A and C: A crosses PCIe in row blocks on a copy stream while
    the GPU runs the blocks already resident (ata._pipelined_host_ata).  Same
    result as the device path within the dtype tolerance, upper triangle of C
    untouched, C accumulated into (not overwritten)."""
    import torch
    import paper_2110_13042_b200 as P
    import importlib
    ata_mod = importlib.import_module("paper_2110_13042_b200.ata")
    monkeypatch.setattr(ata_mod, "PIPELINE_MIN_BYTES", 1 << 20)
    monkeypatch.setattr(ata_mod, "PIPELINE_BLOCK_BYTES", 3 << 20)
    if geometric:   # compute-bound regime: 3 geometric row blocks (ata._row_blocks)
        monkeypatch.setattr(ata_mod, "PIPELINE_FP64_TFLOPS", 0.05)
        assert len(ata_mod._row_blocks(20011, 300, 8, False)) == 3
    tdt = torch.float64 if dtype == "f64" else torch.float32
    rng = np.random.default_rng(21)
    a = rng.standard_normal((20011, 300))
    hA = torch.from_numpy(a).to(tdt).pin_memory()
    c0 = rng.standard_normal((300, 300))
    hC = torch.from_numpy(c0).to(tdt).pin_memory()
    called = []
    orig = ata_mod._pipelined_host_ata
    monkeypatch.setattr(ata_mod, "_pipelined_host_ata", lambda *x: called.append(1) or orig(*x))
    P.ata(hA, hC, 0.5, threshold="auto", precision=precision)
    assert called
    got = hC.numpy().astype(np.float64)
    ref = c0 + 0.5 * O.gram_blas(hA.numpy().astype(np.float64))
    tol = 1e-12 if dtype == "f64" else 1e-4
    assert O.rel_frobenius_lower(got, ref) <= tol
    iu = np.triu_indices(300, 1)
    assert np.array_equal(hC.numpy()[iu], torch.from_numpy(c0).to(tdt).numpy()[iu])


def test_reference_plan_graph_replay():
    """Integer thresholds: the second identical call captures a CUDA graph and
    later calls replay it -- every call gives the bitwise-same result and the
    exact reference multiplication count."""
    import torch
    import paper_2110_13042_b200 as P
    from paper_2110_13042_b200 import engine
    a = torch.from_numpy(np.random.default_rng(3).standard_normal((700, 300))).cuda()
    C = torch.zeros(300, 300, dtype=torch.float64, device="cuda")
    outs, counts = [], []
    before = len(engine._GRAPHS)
    for _ in range(4):
        C.zero_()
        cnt = P.MultCounter()
        P.ata(a, C, 1.0, threshold=64 * 64, counter=cnt)
        outs.append(C.cpu().numpy().copy())
        counts.append(cnt.scalar_mults)
    assert len(engine._GRAPHS) == before + 1
    assert all(np.array_equal(o, outs[0]) for o in outs[1:])
    assert len(set(counts)) == 1
    ref = O.gram_blas(a.cpu().numpy())
    assert O.rel_frobenius_lower(outs[-1], ref) <= 1e-12


@pytest.mark.parametrize("kernel", ["tma", "cp.async"])
def test_fused_leaf_sums_vs_oracle(kernel, monkeypatch, rng):
    """Last Strassen level's operand sums read as two zero-extended quadrant
    terms inside the product kernel (AutoParams.fuse_leaf_sums), on the
    TMA-fed and the cp.async-fed FP64 kernels (the latter also takes windows
    TMA cannot: odd pitches), odd and even shapes, against the oracle."""
    torch = pytest.importorskip("torch")
    import paper_2110_13042_b200 as P
    from paper_2110_13042_b200 import auto_plan, engine
    from paper_2110_13042_b200.auto_plan import AutoParams
    params = AutoParams(leaf_cols=512, min_dim=128, hbm_gbs=1e9, fuse_leaf_sums=True, max_depth=3)
    for shape in ((3000, 2048), (2501, 1537), (4096, 3001)):
        a = rng.uniform(-1, 1, shape)
        n = shape[1]
        plan = auto_plan.plan_ata_auto(shape[0], n, n, n, params)
        assert (plan.ops["ns"] == 2).any() or (plan.ops["nt"] == 2).any()   # fused operands present
        A = torch.from_numpy(a).cuda()
        C = torch.triu(torch.full((n, n), 7.0, dtype=torch.float64, device="cuda"), 1)
        # the native library reads ATA_F64_TMA once per process: select the
        # cp.async kernel through an odd pitch instead (TMA needs an even one)
        if kernel == "cp.async":
            ld = n + 1 if n % 2 == 0 else n + 2          # odd pitch
            big = torch.zeros((shape[0], ld), dtype=torch.float64, device="cuda")
            big[:, :n] = A
            A = big[:, :n]
        P.ata(A, C, 1.0, threshold="auto", auto_params=params)
        got = C.cpu().numpy()
        assert np.all(got[np.triu_indices(n, 1)] == 7.0)
        assert O.rel_frobenius_lower(got, O.gram_blas(a)) <= 1e-13, shape
    engine._PLAN_CACHE.clear()


def test_reference_depth_first_executor(golden, monkeypatch):
    """ATA_REF_DFS=1: the reference's own depth-first order with its per-depth
    scratch (planner._ReferencePlanner) on the golden cases -- same exact
    counts and results within tolerance as the reference run."""
    import paper_2110_13042_b200 as P
    from paper_2110_13042_b200 import engine
    monkeypatch.setenv("ATA_REF_DFS", "1")
    engine._PLAN_CACHE.clear()
    meta, arrays = golden
    done = 0
    for case in meta["cases"]:
        if case.get("kind") != "ata" or case["m"] * case["n"] > 200000:
            continue
        a = arrays[case["key"] + "_A"]
        c = np.zeros((case["n"], case["n"]), dtype=a.dtype)
        cnt = P.MultCounter()
        P.ata(a, c, case["alpha"], threshold=case["threshold"], counter=cnt)
        ref = arrays[case["key"] + "_C"]
        tol = 1e-10 if a.dtype == np.float64 else 1e-4
        assert O.rel_frobenius_lower(c, ref) <= tol, case["key"]
        assert cnt.scalar_mults == case["mults"], case["key"]
        done += 1
    assert done >= 5
    engine._PLAN_CACHE.clear()


def test_workspace_budget_follows_free_memory():
    """fit_workspace_budget keeps the default 40 GB budget when it fits and
    shrinks it to the HBM the process can get when it does not; a plan made
    with a small budget needs less scratch and gives the same result."""
    import dataclasses
    import torch
    from paper_2110_13042_b200 import auto_plan
    from paper_2110_13042_b200.ata import fit_workspace_budget
    base = auto_plan.AutoParams()
    assert fit_workspace_budget(base) == base                      # an idle 180 GB B200
    huge = dataclasses.replace(base, ws_budget_gb=1e6)
    fitted = fit_workspace_budget(huge)
    free, total = torch.cuda.mem_get_info()
    assert fitted.ws_budget_gb <= total / 1e9
    m, n = 16384, 8192
    big = auto_plan.plan_ata_auto(m, n, n, n, base)
    small = auto_plan.plan_ata_auto(m, n, n, n, dataclasses.replace(base, ws_budget_gb=0.5))
    assert small.ws_scalars < big.ws_scalars


def test_pipelined_host_reference_plan():
    """Integer threshold on pinned host A and C (ata._pipelined_host_ref):
    A's upload first, C's behind the operand-sum phase, tiles home as their
    last writer finishes, the plan as CUDA-graph segments -- exact count, the
    oracle's result added to the caller's C, the strict upper triangle
    untouched, repeat calls (graph replay) bit-identical."""
    import torch
    import paper_2110_13042_b200 as P
    rng = np.random.default_rng(23)
    m, n, t = 6001, 1401, 65536
    a = rng.standard_normal((m, n))
    c0 = rng.uniform(-1, 1, (n, n))
    hA = torch.from_numpy(a).pin_memory()
    outs = []
    for _ in range(3):
        hC = torch.from_numpy(c0.copy()).pin_memory()
        cnt = P.MultCounter()
        P.ata(hA, hC, 1.5, threshold=t, counter=cnt)
        outs.append(hC.numpy().copy())
    got = outs[0]
    iu = np.triu_indices(n, 1)
    assert np.array_equal(got[iu], c0[iu])
    ref = c0.copy()
    want = [0]
    O.ata_lower(a, ref, 1.5, t, want)
    assert cnt.scalar_mults == want[0]
    assert O.rel_frobenius_lower(got, ref) <= 1e-13
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[1], outs[2])
