"""Row-sharded ata_dist on 2 ranks (gloo, shared GPU) vs a single-rank ata."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
import paper_2110_13042_b200 as P
from paper_2110_13042_b200 import dist as pdist
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
m, n, seed = 40000, 3000, 3
r0, r1 = pdist.shard_rows(m, world, rank)
A = torch.from_numpy(pdist.uniform_rows(m, n, seed, r0, r1)).cuda()
C = torch.zeros(n, n, dtype=torch.float64, device="cuda")
pdist.ata_dist(A, C, 1.0, "auto")
torch.cuda.synchronize()
if rank == 0:
    full = torch.from_numpy(pdist.uniform_rows(m, n, seed, 0, m)).cuda()
    ref = torch.zeros(n, n, dtype=torch.float64, device="cuda")
    P.ata(full, ref, 1.0, "auto")
    il = torch.tril_indices(n, n, device="cuda")
    err = ((C - ref)[il[0], il[1]].norm() / ref[il[0], il[1]].norm()).item()
    print(f"dist_check world={world} rel_err={err:.3e}", "OK" if err < 1e-12 else "FAIL")
dist.barrier()
dist.destroy_process_group()
