"""GPU parity of the leaf and elementwise kernels against the oracle
(known answers from the reference tests, random and odd shapes, alpha,
upper-triangle sentinel, f32/TF32)."""
import numpy as np
import pytest

from oracle import atamul_oracle as O

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def test_kat_values(golden):
    import paper_2110_13042_b200 as P
    meta, _ = golden
    kat = meta["kat"]
    c = np.zeros((2, 2))
    P.naive_syrk_lower(np.array([[1.0, 2.0], [3.0, 4.0]]), c, 1.0)
    assert [c[0, 0], c[1, 0], c[1, 1]] == kat["syrk_2x2"]
    c = np.zeros((2, 1))
    P.naive_gemm_atb(np.array([[1.0, 0.0], [0.0, 2.0]]), np.array([[3.0], [4.0]]), c, 1.0)
    assert c.ravel().tolist() == kat["gemm_2x2x1"]
    c = np.zeros((1, 1))
    P.ata(np.array([[2.0]]), c, 1.0, threshold=4)
    assert c[0, 0] == kat["ata_1x1"]
    c = np.zeros((3, 3))
    P.naive_syrk_lower(np.array([[2.0, -3.0, 5.0]]), c, 1.0)
    assert np.asarray(P.pack_lower(c).data).tolist() == kat["syrk_row_vector_packed"]


@pytest.mark.parametrize("shape", [(1, 1, 1), (5, 4, 3), (64, 64, 64), (129, 130, 131),
                                   (300, 257, 3), (1000, 17, 250), (2049, 255, 129)])
def test_gemm_atb_f64(shape, rng):
    import paper_2110_13042_b200 as P
    m, n, k = shape
    a, b = rng.uniform(-1, 1, (m, n)), rng.uniform(-1, 1, (m, k))
    c0 = rng.uniform(-1, 1, (n, k))
    got = c0.copy()
    P.naive_gemm_atb(a, b, got, -1.5)
    ref = c0.copy()
    O.gemm_atb(a, b, ref, -1.5)
    assert np.abs(got - ref).max() <= 1e-12 * m


@pytest.mark.parametrize("shape", [(1, 1), (9, 7), (128, 128), (129, 257), (700, 300), (33, 1000)])
def test_syrk_lower_f64_sentinel(shape, rng):
    import paper_2110_13042_b200 as P
    m, n = shape
    a = rng.uniform(-1, 1, (m, n))
    c = np.zeros((n, n))
    iu = np.triu_indices(n, 1)
    c[iu] = 1.2345e67
    P.naive_syrk_lower(a, c, 1.0)
    assert np.all(c[iu] == 1.2345e67)
    ref = np.zeros((n, n))
    O.syrk_lower(a, ref)
    assert O.rel_frobenius_lower(c, ref) <= 1e-14


def test_device_tensor_zero_copy_and_strided_views(rng):
    torch = _torch()
    import paper_2110_13042_b200 as P
    big = torch.from_numpy(rng.uniform(-1, 1, (300, 211))).cuda()
    a = big[7:290, 3:200]          # strided view, odd offsets -> 8-byte loads
    cbig = torch.zeros((250, 250), dtype=torch.float64, device="cuda")
    c = cbig[5:202, 9:206]
    P.naive_syrk_lower(a, c, 2.0)
    ref = np.zeros((197, 197))
    O.syrk_lower(a.cpu().numpy(), ref, 2.0)
    got = c.cpu().numpy()
    assert O.rel_frobenius_lower(got, ref) <= 1e-14
    assert np.all(np.triu(got, 1) == 0)
    assert float(cbig[:5].abs().sum()) == 0.0


def test_f32_tf32_leaves(rng):
    import paper_2110_13042_b200 as P
    a = rng.standard_normal((4000, 300)).astype(np.float32)
    c = np.zeros((300, 300), dtype=np.float32)
    P.naive_syrk_lower(a, c, 1.0)
    ref = np.zeros((300, 300))
    O.syrk_lower(a.astype(np.float64), ref)
    assert O.rel_frobenius_lower(c, ref) <= 1e-4
    b = rng.standard_normal((4000, 77)).astype(np.float32)
    c = np.zeros((300, 77), dtype=np.float32)
    P.naive_gemm_atb(a, b, c, 1.0)
    ref = a.astype(np.float64).T @ b.astype(np.float64)
    assert np.linalg.norm(c - ref) / np.linalg.norm(ref) <= 1e-4


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_add_truncated_mirror_pack(dtype, rng):
    import paper_2110_13042_b200 as P
    d = rng.uniform(-1, 1, (37, 41)).astype(dtype)
    s = rng.uniform(-1, 1, (38, 40)).astype(dtype)
    ref = d.copy()
    O.add_truncated(ref, s, -1.0)
    got = d.copy()
    P.add_truncated(got, s, -1.0)
    assert np.array_equal(got, ref)
    c = rng.uniform(-1, 1, (77, 77)).astype(dtype)
    ref = c.copy()
    O.mirror(ref)
    got = c.copy()
    P.mirror_lower_to_upper(got)
    assert np.array_equal(got, ref)
    pk = P.pack_lower(c)
    assert np.array_equal(np.asarray(pk.data), O.pack_lower(c))
    tgt = np.zeros_like(c)
    P.unpack_lower(pk, tgt)
    assert np.array_equal(np.tril(tgt), np.tril(c))
    P.unpack_lower(pk, tgt, accumulate=True)
    assert np.array_equal(np.tril(tgt), np.tril(2 * c))
    with pytest.raises(P.ShapeMismatchError):
        P.add_truncated(np.zeros((4, 4), dtype), np.zeros((6, 4), dtype))


def test_alpha_zero_is_noop(rng):
    import paper_2110_13042_b200 as P
    a, b = rng.normal(size=(4, 3)), rng.normal(size=(4, 5))
    c = rng.normal(size=(3, 5))
    before = c.copy()
    P.naive_gemm_atb(a, b, c, 0.0)
    assert np.array_equal(c, before)


def test_large_mirror_pack_roundtrip():
    torch = _torch()
    import paper_2110_13042_b200 as P
    n = 4097
    c = torch.randn(n, n, dtype=torch.float64, device="cuda")
    pk = P.pack_lower(c)
    il = torch.tril_indices(n, n, device="cuda")
    assert torch.equal(pk.data, c[il[0], il[1]])
    P.mirror_lower_to_upper(c)
    assert torch.equal(c, c.T)


def _tf32_round(x):
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return (((b + 0x1000) & ~np.uint64(0x1FFF)).astype(np.uint32)).view(np.float32)


@pytest.mark.parametrize("tc", ["2", "1", "0"])
def test_tf32_products_tcgen05_and_legacy(tc, rng, monkeypatch):
    """Single-pass TF32 plain products through run_plan: the tcgen05/TMA kernel
    (ATA_TF32_TC=1, default) and the mma.sync kernel agree with an fp64 product
    of the TF32-rounded operands (GEMM and SYRK kinds, ragged edges)."""
    import subprocess, sys, json, os
    code = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, "%s")
from paper_2110_13042_b200 import planner, engine, _native as nat
rng = np.random.default_rng(11)
out = {}
for (m, n, k) in [(3000, 300, 520), (777, 129, 257), (4096, 1024, 1024)]:
    a = rng.standard_normal((m, n)).astype(np.float32); b = rng.standard_normal((m, k)).astype(np.float32)
    ar = a.view(np.uint32).astype(np.uint64); ar = (((ar + 0x1000) & ~np.uint64(0x1FFF)).astype(np.uint32)).view(np.float32)
    br = b.view(np.uint32).astype(np.uint64); br = (((br + 0x1000) & ~np.uint64(0x1FFF)).astype(np.uint32)).view(np.float32)
    A = torch.from_numpy(ar).cuda(); B = torch.from_numpy(br).cuda()
    pb = planner.PlanBuilder("t")
    C = torch.zeros(n, k, device="cuda")
    pb.product("gemm", m, n, k, [(planner.Win(0, 0, n, m, n), 1.0)], [(planner.Win(3, 0, k, m, k), 1.0)],
               [(planner.Win(1, 0, k, n, k), 1.0)], accumulate=0, group=1)
    engine.run_plan(pb.finish(), nat.ATA_TF32, A.data_ptr(), A.numel(), C.data_ptr(), C.numel(), 1.0,
                    B=B.data_ptr(), b_elems=B.numel())
    ref = ar.astype(np.float64).T @ br.astype(np.float64)
    g = np.linalg.norm(C.cpu().numpy() - ref) / np.linalg.norm(ref)
    pb = planner.PlanBuilder("t")
    S = torch.full((n, n), 3.0, device="cuda")
    pb.product("syrk", m, n, n, [(planner.Win(0, 0, n, m, n), 1.0)], [], [(planner.Win(1, 0, n, n, n), -1.0)],
               accumulate=1, group=1)
    engine.run_plan(pb.finish(), nat.ATA_TF32, A.data_ptr(), A.numel(), S.data_ptr(), S.numel(), 2.0)
    s = S.cpu().numpy(); refs = 3.0 - 2.0 * (ar.astype(np.float64).T @ ar.astype(np.float64))
    il = np.tril_indices(n)
    e = np.linalg.norm(s[il] - refs[il]) / np.linalg.norm(refs[il])
    up = bool(np.all(s[np.triu_indices(n, 1)] == 3.0))
    out[f"{m}x{n}x{k}"] = [g, e, up]
print(json.dumps(out))
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, ATA_TF32_TC=tc)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for key, (g, e, up) in res.items():
        assert g <= 5e-5, (key, g)     # fp32 accumulation of TF32 products
        assert e <= 5e-5, (key, e)
        assert up, key


def test_ata_tf32_tall_skinny():
    """Config-c5-shaped (scaled) single-pass TF32 AtA: rel-Frobenius <= 1e-4
    against the fp64 Gram of the fp32 input (the c5 tolerance)."""
    import torch
    import paper_2110_13042_b200 as P
    a = np.random.default_rng(4).standard_normal((200000, 640)).astype(np.float32)
    A = torch.from_numpy(a).cuda()
    C = torch.zeros(640, 640, dtype=torch.float32, device="cuda")
    P.ata(A, C, 1.0, threshold="auto", precision="tf32")
    got = C.cpu().numpy()
    assert np.all(np.triu(got, 1) == 0)
    assert O.rel_frobenius_lower(got, O.gram_blas(a)) <= 1e-4



def test_tf32_l2_ring_matches_rounding_pass():
    """Single-pass TF32 through the CTA-pair kernel's L2 rounding ring (rounder
    warps round 96-row pieces of A into two small rings, TMA reads them back)
    gives bit-for-bit the result of the HBM rounding pass: same cvt.rna
    rounding, same products in the same order."""
    import torch
    from paper_2110_13042_b200 import auto_plan, engine, _native as nat
    m, n = 1 << 17, 2048
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn((m, n), device="cuda", generator=g)
    out = []
    for ring in (True, False):
        plan = auto_plan.plan_ata_auto(m, n, n, n, auto_plan.AutoParams(tf32_ring=ring), round_tf32=True)
        assert (int(plan.ops[0]["accumulate"]) == 2) == ring
        ws = torch.empty(plan.ws_scalars, device="cuda")
        C = torch.zeros((n, n), device="cuda")
        for _ in range(2):   # second run: flags and ring reused
            C.zero_()
            engine.run_plan(plan, nat.ATA_TF32, A.data_ptr(), A.numel(), C.data_ptr(), C.numel(), 1.0,
                            ws=ws.data_ptr(), ws_elems=ws.numel())
        torch.cuda.synchronize()
        out.append(C.clone())
    assert torch.equal(out[0], out[1])
    ref = O.gram_blas(A.double().cpu().numpy())
    assert O.rel_frobenius_lower(out[0].cpu().numpy(), ref) <= 1e-4


def test_tf32_l2_ring_under_sm_contention():
    """The L2-ring launch needs every CTA resident at once (CTAs wait on one
    another's rounding items); it is a cooperative launch, so work on another
    stream that holds SMs delays it instead of leaving resident CTAs spinning.
    Run the ring plan while a second stream keeps the SMs busy with GEMMs and
    check it completes with the same bits as on an idle GPU."""
    import torch
    from paper_2110_13042_b200 import auto_plan, engine, _native as nat
    m, n = 1 << 17, 2048
    g = torch.Generator(device="cuda").manual_seed(6)
    A = torch.randn((m, n), device="cuda", generator=g)
    plan = auto_plan.plan_ata_auto(m, n, n, n, auto_plan.AutoParams(tf32_ring=True), round_tf32=True)
    assert int(plan.ops[0]["accumulate"]) == 2
    ws = torch.empty(plan.ws_scalars, device="cuda")

    def run(C, stream):
        engine.run_plan(plan, nat.ATA_TF32, A.data_ptr(), A.numel(), C.data_ptr(), C.numel(), 1.0,
                        ws=ws.data_ptr(), ws_elems=ws.numel(), stream=int(stream.cuda_stream))

    main = torch.cuda.current_stream()
    C0 = torch.zeros((n, n), device="cuda")
    run(C0, main)
    torch.cuda.synchronize()
    hog = torch.cuda.Stream()
    x = torch.randn((4096, 4096), device="cuda", dtype=torch.bfloat16)
    C1 = torch.zeros((n, n), device="cuda")
    with torch.cuda.stream(hog):
        for _ in range(40):
            x = (x @ x).clamp_(-1, 1)
    run(C1, main)            # queued while the hog stream occupies SMs
    with torch.cuda.stream(hog):
        for _ in range(40):
            x = (x @ x).clamp_(-1, 1)
    torch.cuda.synchronize()
    assert torch.equal(C0, C1)


def test_graph_replay_survives_descriptor_cache_churn(monkeypatch):
    """A CUDA graph captured over TMA / device-descriptor launches keeps the
    descriptor blobs it baked in: entries used under capture are pinned, so a
    later flood of other launches (with a tiny cache budget forcing eviction)
    cannot free them, and replays stay bit-identical to the eager run."""
    import torch
    from paper_2110_13042_b200 import auto_plan, engine, _native as nat
    m, n = 4096, 2048
    params = auto_plan.AutoParams(leaf_cols=512, min_dim=128, hbm_gbs=1e9)
    plan = auto_plan.plan_ata_auto(m, n, n, n, params)
    A = torch.rand(m, n, dtype=torch.float64, device="cuda")
    C = torch.zeros(n, n, dtype=torch.float64, device="cuda")
    ws = torch.empty(max(1, plan.ws_scalars), dtype=torch.float64, device="cuda")
    args = (plan, nat.ATA_F64, A.data_ptr(), A.numel(), C.data_ptr(), C.numel(), 1.0)
    kw = dict(ws=ws.data_ptr(), ws_elems=ws.numel())
    engine.run_plan(*args, **kw)                 # eager: blobs uploaded
    torch.cuda.synchronize()
    ref = C.clone()
    g = engine.PlanGraph(*args, **kw)            # captured: blobs pinned
    monkeypatch.setenv("ATA_DESC_CACHE_KB", "1")
    for i in range(12):                          # churn: new blobs evict everything unpinned
        Ai = torch.rand(m + 16 * (i + 1), n, dtype=torch.float64, device="cuda")
        Ci = torch.zeros(n, n, dtype=torch.float64, device="cuda")
        pi = auto_plan.plan_ata_auto(Ai.shape[0], n, n, n, params)
        wi = torch.empty(max(1, pi.ws_scalars), dtype=torch.float64, device="cuda")
        engine.run_plan(pi, nat.ATA_F64, Ai.data_ptr(), Ai.numel(), Ci.data_ptr(), Ci.numel(), 1.0,
                        ws=wi.data_ptr(), ws_elems=wi.numel())
    torch.cuda.synchronize()
    for _ in range(2):
        C.zero_()
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(C, ref)


@pytest.mark.parametrize("m,n", [(2048, 1024), (777, 1040), (4096, 256), (129, 16)])
def test_tma_syrk_diagonal_tiles(m, n):
    """SYRK leaves on the TMA-fed FP64 kernel (16-column-multiple windows):
    diagonal tiles compute only their on/below-diagonal 8x8 blocks with the
    permuted warp map; the stored triangle matches the oracle and the strict
    upper triangle keeps its sentinel."""
    import torch
    import paper_2110_13042_b200 as P
    rng = np.random.default_rng(m + n)
    a = rng.uniform(-1, 1, (m, n))
    A = torch.from_numpy(a).cuda()
    C = torch.triu(torch.full((n, n), 5.0, dtype=torch.float64, device="cuda"), 1)
    P.naive_syrk_lower(A, C, 2.0)
    got = C.cpu().numpy()
    assert np.all(got[np.triu_indices(n, 1)] == 5.0)
    ref = np.zeros((n, n))
    O.syrk_lower(a, ref, 2.0)
    assert O.rel_frobenius_lower(got, ref) <= 1e-14


_CFG_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2110_13042_b200 as P
from oracle import atamul_oracle as O
from paper_2110_13042_b200.auto_plan import AutoParams
rng = np.random.default_rng(3)
for shape in ((700, 333), (1500, 1024)):
    a = rng.uniform(-1, 1, shape)
    n = shape[1]
    for thr, kw in ((4096, {}), ("auto", {"auto_params": AutoParams(leaf_cols=256, min_dim=128, hbm_gbs=1e9)})):
        C = torch.triu(torch.full((n, n), 7.0, dtype=torch.float64, device="cuda"), 1)
        P.ata(torch.from_numpy(a).cuda(), C, 1.0, threshold=thr, **kw)
        got = C.cpu().numpy()
        assert np.all(got[np.triu_indices(n, 1)] == 7.0)
        err = O.rel_frobenius_lower(got, O.gram_blas(a))
        assert err <= 1e-13, (shape, thr, err)
print("OK")
"""


@pytest.mark.parametrize("cfg", ["0", "1", "2", "3"])
def test_legacy_f64_configurations(cfg):
    """The non-default FP64 product-kernel configurations kept for A/B
    comparison (ATA_F64_CFG = 0..3: CTA-per-tile kernels of gemm_f64.cu) give
    the oracle's result on reference and auto plans (fresh process: the
    configuration is read once)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, ATA_F64_CFG=cfg)
    r = subprocess.run([sys.executable, "-c", _CFG_SCRIPT, root], capture_output=True, text=True, env=env,
                       timeout=600, cwd=root)
    assert r.returncode == 0 and "OK" in r.stdout, r.stderr[-3000:]


@pytest.mark.parametrize("m,n,k,off", [(300, 129, 77, 1), (1000, 200, 300, 3), (64, 16, 1, 1), (513, 255, 257, 0),
                                       (300, 130, 77, 0), (777, 18, 129, 2)])
def test_tma_2d_maps_unaligned_windows(m, n, k, off):
    """Ragged widths and 8-byte-aligned starts: 16-byte-aligned even-pitch
    windows with any width go through the TMA-fed kernel's 2-D maps (extents
    bounded at the window's last row), windows starting 8 bytes into a
    16-byte unit through the cp.async kernel -- GEMM and SYRK leaves against
    NumPy, destinations outside the windows untouched."""
    import torch
    import paper_2110_13042_b200 as P
    rng = np.random.default_rng(m + n + k)
    ld = 2 * ((n + k + off + 8) // 2)                 # even pitch
    big = torch.from_numpy(rng.uniform(-1, 1, (m, ld))).cuda()
    a = big[:, off:off + n]
    b = big[:, off + n:off + n + k]
    C = torch.full((n, k), 2.5, dtype=torch.float64, device="cuda")
    P.naive_gemm_atb(a, b, C, 1.0)
    an, bn = a.cpu().numpy(), b.cpu().numpy()
    assert np.abs(C.cpu().numpy() - (2.5 + an.T @ bn)).max() <= 1e-12 * m
    S = torch.triu(torch.full((n, n), 9.0, dtype=torch.float64, device="cuda"), 1)
    P.naive_syrk_lower(a, S, -1.0)
    got = S.cpu().numpy()
    assert np.all(got[np.triu_indices(n, 1)] == 9.0)
    il = np.tril_indices(n)
    assert np.abs(got[il] + (an.T @ an)[il]).max() <= 1e-12 * m


def test_even_pitch_relayout_reference_plan():
    """An odd-pitch fp64 operand (config c2's 4097 columns) is re-laid out with
    an even pitch inside ata() (ata.even_pitch) and the reference tree runs on
    the TMA-fed kernel: exact count and the oracle's result, repeat calls
    (graph replay) identical."""
    import torch
    import paper_2110_13042_b200 as P
    rng = np.random.default_rng(17)
    a = rng.standard_normal((1501, 1025))
    A = torch.from_numpy(a).cuda()
    outs = []
    for _ in range(3):
        C = torch.zeros(1025, 1025, dtype=torch.float64, device="cuda")
        cnt = P.MultCounter()
        P.ata(A, C, 1.0, threshold=128 * 128, counter=cnt)
        outs.append(C.cpu().numpy())
    ref = np.zeros((1025, 1025))
    want = [0]
    O.ata_lower(a, ref, 1.0, 128 * 128, want)
    assert cnt.scalar_mults == want[0]
    assert O.rel_frobenius_lower(outs[0], ref) <= 1e-13
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[1], outs[2])
