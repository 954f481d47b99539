"""Multi-rank GPU paths, 2 and 3 ranks over gloo on cuda:0 (gpurun exposes
one GPU): row shards, the units partition and the distribute-compute-
retrieve executor ata_d, each checked on rank 0 against the CPU oracle's
classical Gram (tests/dist_worker.py), plus the units partition's plans of
all ranks run on one GPU against the oracle."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import atamul_oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("mode,world,m,n", [("rows", 2, 40000, 3000), ("units", 2, 9000, 3000),
                                            ("units", 3, 8193, 2049), ("ata_d", 2, 3001, 2000),
                                            ("ata_d", 3, 3001, 2000)])
def test_multi_rank_vs_oracle(mode, world, m, n):
    env = dict(os.environ)
    port = str(29541 + world + 7 * ("rows", "units", "ata_d").index(mode))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
                        str(world), "--master-addr", "127.0.0.1", "--master-port", port,
                        os.path.join(ROOT, "tests", "dist_worker.py"), mode, str(m), str(n)],
                       capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "OK" in r.stdout, r.stdout[-2000:]
    print(r.stdout.strip().splitlines()[-1])


def test_collectives_over_nccl_single_rank():
    """The rows / units collectives through a real NCCL communicator (one rank:
    the box has one GPU), result against the oracle."""
    env = dict(os.environ, ATA_DIST_BACKEND="nccl")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", "29577",
                        os.path.join(ROOT, "tests", "dist_worker.py"), "nccl1", "6000", "3000"],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "OK" in r.stdout and "backend=nccl" in r.stdout, r.stdout[-2000:]
    print(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("procs", [2, 4, 8])
def test_units_partition_all_ranks_one_gpu(procs):
    """Every rank's plan_units plan run on one GPU into one C: the segments
    add up to lower(A^T A) (c4's aspect ratio, scaled down)."""
    import torch
    from paper_2110_13042_b200 import auto_plan, engine, _native as nat
    m, n = 8192, 4096
    params = auto_plan.AutoParams(leaf_cols=512, min_dim=256, hbm_gbs=1e9)
    a = np.random.default_rng(procs).uniform(-1, 1, (m, n))
    A = torch.from_numpy(a).cuda()
    C = torch.zeros(n, n, dtype=torch.float64, device="cuda")
    for segs in auto_plan.partition_units(m, n, procs, params):
        plan = auto_plan.plan_units(segs, m, n, n, n, params)
        ws = torch.empty(max(1, plan.ws_scalars), dtype=torch.float64, device="cuda")
        engine.run_plan(plan, nat.ATA_F64, A.data_ptr(), A.numel(), C.data_ptr(), C.numel(), 1.0,
                        ws=ws.data_ptr(), ws_elems=ws.numel())
    torch.cuda.synchronize()
    assert O.rel_frobenius_lower(C.cpu().numpy(), O.gram_blas(a)) <= 1e-13


@pytest.mark.parametrize("dist,prefix,port", [("units", "units x2", 29611), ("rows", "row-shard x2", 29613),
                                               ("tree", "task-tree x2", 29615)])
def test_bench_two_ranks_shared_gpu(dist, prefix, port):
    """bench.py's N>1 paths (2 ranks, gloo, one GPU): units partition, row
    shards and the reference's task tree; the driver's JSON line names the
    partition."""
    import json
    import paper_2110_13042_b200 as P
    P.release_cached_buffers()       # the ranks are subprocesses sharing this GPU's memory
    env = dict(os.environ, ATA_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--config", "c3", "--dist", dist, "--steps", "2", "--warmup", "1",
                        "--no-autotune"], capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["parallelism"].startswith(prefix)
    assert line["value"] > 0 and line["gpu_launches"] > 0
