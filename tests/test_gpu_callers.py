"""GPU checks of the callers either side of the path: fast_strassen with the
auto plan, the reference's distributed task tree (simulated in one process
and over torch.distributed), and the atamul-compatible CLI in every mode."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import atamul_oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("m,n,k", [(3001, 1030, 770), (700, 2049, 1500), (64, 300, 901)])
def test_fast_strassen_auto(m, n, k, rng):
    import torch
    import paper_2110_13042_b200 as P
    from paper_2110_13042_b200.auto_plan import AutoParams
    a = rng.standard_normal((m, n))
    b = rng.standard_normal((m, k))
    c0 = rng.standard_normal((n, k))
    C = torch.from_numpy(c0.copy()).cuda()
    P.fast_strassen(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), C, -2.0, threshold="auto",
                    auto_params=AutoParams(min_dim=128, hbm_gbs=1e9, max_depth=3))
    ref = c0 - 2.0 * (a.T @ b)
    assert np.linalg.norm(C.cpu().numpy() - ref) / np.linalg.norm(ref) <= 1e-13


@pytest.mark.parametrize("procs", [1, 2, 3, 6, 7, 8, 12])
@pytest.mark.parametrize("threshold", ["auto", 4096])
def test_ata_tree_simulated(procs, threshold, rng):
    import torch
    from paper_2110_13042_b200 import MultCounter, dist
    m, n = 901, 530
    a = rng.uniform(-1, 1, (m, n))
    A = torch.from_numpy(a).cuda()
    C = torch.zeros(n, n, dtype=torch.float64, device="cuda")
    C[torch.triu_indices(n, n, 1, device="cuda").unbind()] = 3.0
    cnt = MultCounter()
    dist.ata_tree(lambda r: A[r.row_offset:r.row_offset + r.rows, r.col_offset:r.col_offset + r.cols],
                  m, n, C, 1.0, threshold, procs=procs, counter=cnt)
    got = C.cpu().numpy()
    assert np.all(got[np.triu_indices(n, 1)] == 3.0)
    assert O.rel_frobenius_lower(got, O.gram_blas(a)) <= 1e-12
    assert cnt.scalar_mults > 0


def test_ata_tree_over_torch_distributed():
    for world, thr in ((8, "auto"), (3, "4096")):
        env = dict(os.environ, TREE_THRESHOLD=thr)
        r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
                            str(world), "--master-addr", "127.0.0.1", "--master-port", str(29551 + world),
                            os.path.join(ROOT, "tools", "dist_tree_check.py")],
                           capture_output=True, text=True, env=env, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        assert "OK" in r.stdout, r.stdout[-2000:]


def _cli(*args):
    r = subprocess.run([sys.executable, "-m", "paper_2110_13042_b200.cli", *args], capture_output=True,
                       text=True, timeout=600, cwd=ROOT)
    return r


@pytest.mark.parametrize("argv", [
    ["--mode", "seq", "--n", "300", "--m", "410", "--threshold", "4096"],
    ["--mode", "auto", "--n", "700"],
    ["--mode", "oracle", "--n", "257"],
    ["--mode", "shared", "--procs", "4", "--n", "500", "--m", "333", "--threshold", "4096"],
    ["--mode", "shared", "--procs", "3", "--n", "600", "--threshold", "auto"],
    ["--mode", "dist", "--procs", "8", "--n", "400", "--m", "900", "--threshold", "4096"],
    ["--mode", "dist", "--procs", "5", "--n", "400", "--leaf-kernel", "naive"],
    ["--mode", "seq", "--n", "256", "--dtype", "f32", "--threshold", "4096"],
])
def test_cli_modes_check(argv, tmp_path):
    csvp = tmp_path / "r.csv"
    r = _cli(*argv, "--check", "--count-mults", "--reps", "2", "--csv", str(csvp))
    assert r.returncode == 0, r.stdout + r.stderr[-3000:]
    assert "CHECK FAILED" not in r.stderr
    assert "effective GFLOPs" in r.stdout and "max abs err" in r.stdout
    assert csvp.read_text().splitlines()[0].startswith("mode,m,n,procs,threshold")


def test_cli_seq_count_matches_reference_and_atam(tmp_path):
    """--mode seq credits the reference's exact multiplication count; --out /
    --in round-trip the input through an ATAM file."""
    path = tmp_path / "a.atam"
    r = _cli("--mode", "seq", "--n", "96", "--m", "130", "--threshold", "512", "--seed", "4",
             "--count-mults", "--reps", "1", "--out", str(path))
    assert r.returncode == 0, r.stderr[-2000:]
    from paper_2110_13042_b200 import gen_matrix, read_matrix
    a = read_matrix(path).a
    assert np.array_equal(a, gen_matrix(130, 96, 4).a)
    want = [0]
    O.ata_lower(a, np.zeros((96, 96)), 1.0, 512, want)
    assert f", {want[0]} scalar mults" in r.stdout
    r2 = _cli("--mode", "seq", "--in", str(path), "--threshold", "512", "--count-mults", "--reps", "1",
              "--check")
    assert r2.returncode == 0 and f", {want[0]} scalar mults" in r2.stdout


def test_autotune_rates_and_leaf_choice(rng):
    """autotune.calibrate measures the FP64 leaf-product and addition-pass
    rates on this GPU; tune picks the SYRK leaf width by timing candidate
    plans; ata(auto_params="tune") computes the same Gram matrix."""
    import torch
    import paper_2110_13042_b200 as P
    from paper_2110_13042_b200 import autotune
    tf, gbs = autotune.calibrate()
    assert 15.0 <= tf <= 40.0, tf            # DMMA peak 37.2 TF/s
    assert 1500.0 <= gbs <= 7000.0, gbs      # HBM copy 6.5 TB/s
    m, n = 3000, 2600
    p = autotune.tune(m, n)
    assert p.leaf_cols in autotune.LEAF_CANDIDATES and p.dmma_tflops == tf and p.hbm_gbs == gbs
    assert autotune.tune(m, n) is p          # cached per shape
    a = rng.uniform(-1, 1, (m, n))
    C = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    P.ata(torch.from_numpy(a).cuda(), C, 1.0, threshold="auto", auto_params="tune")
    assert O.rel_frobenius_lower(C.cpu().numpy(), O.gram_blas(a)) <= 1e-12
