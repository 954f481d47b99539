"""Full-size BASELINE configs c3, c4, c5 on the GPU, checked through
size-independent properties against the CPU oracle (the full CPU Gram of c4 /
c5 would take hours): the checksum identity C 1 = A^T (A 1) over the whole
symmetric result (every entry contributes), and classical products of sampled
256-column block pairs of the stored lower triangle (oracle gemm_atb /
syrk_lower on the same seeded inputs).  Tolerances: 1e-10 rel-Frobenius for
fp64 (north_star), 1e-4 for the single-pass TF32 config c5."""
import numpy as np
import pytest

from oracle import atamul_oracle as O

pytestmark = pytest.mark.gpu


def _check(a, C, tol, blocks=8, width=256, seed=0, offdiag_tol=None):
    """C: device result (lower triangle valid).  a: host input (float64 or float32).
    The stored triangle's rel-Frobenius error is dominated by the diagonal
    blocks (A^T A's diagonal is ~m, off-diagonal entries ~sqrt(m)); the checksum
    and the diagonal blocks are held to `tol`, off-diagonal blocks to
    `offdiag_tol` (TF32 operands carry a 2^-11 rounding: ~4e-4 relative on
    entries that are sums of signed terms)."""
    offdiag_tol = tol if offdiag_tol is None else offdiag_tol
    import torch
    import paper_2110_13042_b200 as P
    n = a.shape[1]
    P.mirror_lower_to_upper(C)
    ones = torch.ones(n, dtype=torch.float64, device=C.device)
    got_rows = (C.double() @ ones).cpu().numpy()
    # A^T (A 1) in fp64 on the host, blockwise to bound memory
    ref_rows = np.zeros(n)
    step = 1 << 14
    for r0 in range(0, a.shape[0], step):
        blk = a[r0:r0 + step].astype(np.float64, copy=False)
        w = blk @ np.ones(n)
        ref_rows += blk.T @ w
    assert np.linalg.norm(got_rows - ref_rows) <= tol * np.linalg.norm(ref_rows)
    rng = np.random.default_rng(seed)
    starts = np.arange(0, n - width + 1, width)
    for _ in range(blocks):
        i, j = sorted(rng.choice(starts, 2, replace=True))[::-1]   # i >= j: lower triangle
        ai = a[:, i:i + width].astype(np.float64)
        aj = a[:, j:j + width].astype(np.float64)
        # classical fp64 products of the blocks (BLAS: the oracle's gram_blas path)
        if i == j:
            ref = np.tril(ai.T @ ai)
            got = np.tril(C[i:i + width, j:j + width].double().cpu().numpy())
        else:
            ref = ai.T @ aj
            got = C[i:i + width, j:j + width].double().cpu().numpy()
        lim = tol if i == j else offdiag_tol
        assert np.linalg.norm(got - ref) <= lim * np.linalg.norm(ref), (i, j)


def _run(name, precision="fp32"):
    import torch
    import paper_2110_13042_b200 as P
    from paper_2110_13042_b200.measure import CONFIGS, config_matrix
    cfg = CONFIGS[name]
    a = config_matrix(name)
    A = torch.from_numpy(a).cuda()
    C = torch.zeros((cfg["n"], cfg["n"]), dtype=A.dtype, device="cuda")
    P.ata(A, C, 1.0, threshold=cfg["threshold"], precision=precision)
    del A
    torch.cuda.synchronize()
    return a, C


def test_config_c3_full():
    a, C = _run("c3")
    _check(a, C, 1e-10)


def test_config_c4_full():
    a, C = _run("c4")
    _check(a, C, 1e-10, blocks=6)


def test_config_c5_full_tf32():
    a, C = _run("c5", precision="tf32")
    _check(a, C, 1e-4, blocks=6, offdiag_tol=1e-3)
    # the diagonal blocks in full: they carry the stored triangle's norm
    n = C.shape[0]
    for i in range(0, n, 256):
        ai = a[:, i:i + 256].astype(np.float64)
        ref = np.tril(ai.T @ ai)
        got = np.tril(C[i:i + 256, i:i + 256].double().cpu().numpy())
        assert np.linalg.norm(got - ref) <= 1e-4 * np.linalg.norm(ref), i
