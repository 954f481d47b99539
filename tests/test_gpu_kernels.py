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
