"""One rank of the multi-rank GPU checks (run by tests/test_gpu_dist.py under
torch.distributed.run with gloo, every rank on cuda:0 -- the kernels of one
rank never wait on another's).  Modes:

  rows   -- dist.ata_dist: row shards + packed-triangle reduce
  units  -- dist.ata_units: the top level's AtA sub-problems and Strassen
            products as row-range segments + per-region reduces
  ata_d  -- distsim.ata_d over the group: A only on rank 0, operand blocks
            sent down the reference's distributed task tree, partials back
  nccl1  -- ATA_DIST_BACKEND=nccl, one rank: the collectives of the rows and
            units paths (packed-triangle reduce, per-region reduces) issued
            through a real NCCL communicator on the B200 (gpurun exposes one
            GPU, so this is the part of the NCCL path that can execute here)

Rank 0 checks the lower triangle against the CPU oracle's classical Gram
(relative Frobenius 1e-12) and prints OK.  Test infrastructure only."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2110_13042_b200 as P  # noqa: E402
from oracle import atamul_oracle as O  # noqa: E402
from paper_2110_13042_b200 import auto_plan, dist as pdist  # noqa: E402

mode = sys.argv[1]
m, n, seed = int(sys.argv[2]), int(sys.argv[3]), 3
backend = os.environ.get("ATA_DIST_BACKEND", "gloo")
torch.cuda.set_device(0)
if backend == "nccl":
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
else:
    dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
full = pdist.uniform_rows(m, n, seed, 0, m)
C = torch.zeros(n, n, dtype=torch.float64, device="cuda")
extra = ""
if mode == "rows":
    r0, r1 = pdist.shard_rows(m, world, rank)
    pdist.ata_dist(torch.from_numpy(full[r0:r1]).cuda(), C, 1.0, "auto")
elif mode == "units":
    params = auto_plan.AutoParams(leaf_cols=256, min_dim=128, hbm_gbs=1e9)
    parts = auto_plan.partition_units(m, n, world, params)
    A = torch.zeros(m, n, dtype=torch.float64, device="cuda")
    for lo, hi in auto_plan.a_rows_needed(parts[rank], m, n):   # only the rows this rank reads
        A[lo:hi] = torch.from_numpy(full[lo:hi])
    pdist.ata_units(A, C, parts[rank], parts, params)
    extra = f" segments={parts[rank]}"
elif mode == "ata_d":
    res, st = P.ata_d(full if rank == 0 else None, world, threshold="auto")
    if rank == 0:
        C = res.a if isinstance(res.a, torch.Tensor) else torch.from_numpy(res.a)
    extra = f" sent_words={st.sent_words} recv_messages={st.recv_messages}"
elif mode == "nccl1":
    assert backend == "nccl" and world == 1
    from paper_2110_13042_b200.distsim import DeviceBlocks
    A = torch.from_numpy(full).cuda()
    P.ata(A, C, 1.0, "auto")
    packed = torch.empty(n * (n + 1) // 2, dtype=C.dtype, device="cuda")
    P.pack_lower(C, out=packed)
    pdist.reduce_packed(packed, 0)                       # ncclReduce on the packed triangle
    C2 = torch.zeros_like(C)
    P.unpack_lower(P.PackedLowerTriangular(n, packed), C2)
    groups = {r: dist.group.WORLD for r in pdist.REGIONS}
    members = {r: [0] for r in pdist.REGIONS}
    pdist.reduce_regions(C2, n, 0, groups, members, DeviceBlocks(C.device, C.dtype))   # one ncclReduce per region
    t = torch.ones(1 << 20, device="cuda")
    dist.all_reduce(t)
    assert float(t.sum().item()) == float(1 << 20)
    C = C2
    extra = f" backend={dist.get_backend()} nccl={'.'.join(map(str, torch.cuda.nccl.version()))}"
else:
    raise SystemExit(f"unknown mode {mode}")
torch.cuda.synchronize()
if rank == 0:
    got = C.cpu().numpy() if isinstance(C, torch.Tensor) else C
    err = O.rel_frobenius_lower(got, O.gram_blas(full))
    print(f"dist_worker {mode} world={world} rel_err={err:.3e}{extra}", "OK" if err < 1e-12 else "FAIL")
dist.barrier()
dist.destroy_process_group()
