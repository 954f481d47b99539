"""dist.ata_tree over torch.distributed (gloo, every rank on cuda:0) vs a
single-rank ata: each rank generates only the rows its leaf reads, computes
its leaf, and the blocks are retrieved up the reference's task tree."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import paper_2110_13042_b200 as P
from paper_2110_13042_b200 import dist as pdist
from paper_2110_13042_b200.tasktree import build_tree_distributed
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
m, n, seed = int(os.environ.get("TREE_M", "6000")), int(os.environ.get("TREE_N", "2050")), 3
thr = os.environ.get("TREE_THRESHOLD", "auto")
thr = thr if thr == "auto" else int(thr)
tree = build_tree_distributed(world, m, n)
r0, r1 = pdist.tree_rows(tree, rank)
rows = torch.from_numpy(pdist.uniform_rows(m, n, seed, r0, r1)).cuda()


def get_block(r):   # this rank's rows only
    return rows[r.row_offset - r0:r.row_offset - r0 + r.rows, r.col_offset:r.col_offset + r.cols]


C = torch.zeros(n, n, dtype=torch.float64, device="cuda")
C[torch.triu_indices(n, n, 1, device="cuda").unbind()] = 7.0
pdist.ata_tree(get_block, m, n, C, 1.5, thr)
torch.cuda.synchronize()
if rank == 0:
    full = torch.from_numpy(pdist.uniform_rows(m, n, seed, 0, m)).cuda()
    ref = torch.zeros(n, n, dtype=torch.float64, device="cuda")
    P.ata(full, ref, 1.5, "auto")
    il = torch.tril_indices(n, n, device="cuda")
    err = ((C - ref)[il[0], il[1]].norm() / ref[il[0], il[1]].norm()).item()
    upper_ok = bool((C[torch.triu_indices(n, n, 1, device="cuda").unbind()] == 7.0).all())
    ok = err < 1e-12 and upper_ok
    print(f"dist_tree_check world={world} rel_err={err:.3e} upper_ok={upper_ok}", "OK" if ok else "FAIL")
dist.barrier()
dist.destroy_process_group()
