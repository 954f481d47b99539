"""Multi-GPU AtA: one process per GPU, row-sharded partial Gram matrices
summed with NCCL over NVLink.

Partition (reference-native): ``_tile_ata_horizontal`` (scheduler.py:305-314)
cuts A into horizontal row tiles; every tile's full lower-triangle partial is
summed by the parent (distsim.py:253-267), with AtA results shipped as packed
lower triangles (distsim.py:192-199) and added into the parent's triangle
(distsim.py:208-216).  Here: each rank owns rows [r0, r1) of A in its HBM, runs
the single-GPU plan on them (no data-path collective during compute), packs
its lower triangle (n(n+1)/2 scalars) and one ``reduce(SUM)`` to the root
combines the partials; the root unpacks into C.
"""
from __future__ import annotations

import numpy as np


def shard_rows(m: int, world: int, rank: int):
    """Balanced contiguous row range of `rank` (floor/ceil split as
    scheduler._split_extent)."""
    base, extra = divmod(m, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def uniform_rows(m: int, n: int, seed: int, r0: int, r1: int, dtype=np.float64):
    """Rows [r0, r1) of ``default_rng(seed).uniform(-1, 1, (m, n))`` without
    drawing the prefix: PCG64 advances one 64-bit draw per uniform double."""
    bg = np.random.PCG64(seed)
    bg.advance(r0 * n)
    g = np.random.Generator(bg)
    return g.uniform(-1.0, 1.0, (r1 - r0, n)).astype(dtype, copy=False)


def reduce_packed(packed, root: int = 0, group=None):
    """Sum packed lower triangles of every rank into `packed` on `root`."""
    import torch.distributed as dist
    if packed.is_cuda and dist.get_backend(group) == "gloo":
        # host-staged reduction for the gloo backend (CPU tests, shared-GPU checks)
        host = packed.cpu()
        dist.reduce(host, dst=root, op=dist.ReduceOp.SUM, group=group)
        packed.copy_(host)
        return packed
    dist.reduce(packed, dst=root, op=dist.ReduceOp.SUM, group=group)
    return packed


def ata_dist(A_shard, C, alpha=1.0, threshold="auto", root: int = 0, packed=None, group=None,
             **kw):
    """lower(C) += alpha * A^T A where A is row-sharded over the ranks of the
    default process group; `A_shard` is this rank's rows (CUDA tensor).  On
    return the root's C holds the result; other ranks' C hold their partials.
    `packed` optionally provides the n(n+1)/2 communication buffer."""
    import torch
    import torch.distributed as dist
    from .ata import ata
    from .matrix import pack_lower, unpack_lower, PackedLowerTriangular
    n = int(C.shape[0])
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        ata(A_shard, C, alpha, threshold, **kw)
        return C
    rank = dist.get_rank(group)
    if rank != root:
        C.zero_()
    ata(A_shard, C, alpha, threshold, **kw)
    if packed is None:
        packed = torch.empty(n * (n + 1) // 2, dtype=C.dtype, device=C.device)
    pack_lower(C, out=packed)
    reduce_packed(packed, root, group)
    if rank == root:
        unpack_lower(PackedLowerTriangular(n, packed), C)
    return C


# --------------------------------------------------------------------------
# Task-tree partition (the reference's distribute-compute-retrieve layout)
#
# tasktree.build_tree_distributed(P, m, n) assigns one leaf task to every
# process: an AtA of an operand block into a diagonal C block, or an AtB of
# two operand blocks into a rectangular C block (scheduler.py:283-363; at
# P = 8 on c4: four quadrant AtA's and four AtB tiles of C21).  Each rank
# computes its leaf with the single-GPU plans (ata / fast_strassen), then the
# results travel up the tree as in the reference's retrieve phase
# (distsim.py:253-267): every process walks its ownership chain
# (path_to_root) leaf first, assembling each owned node's C block from its own
# child's block plus the blocks the other children's owners send it, and
# finally sends its chain top to the parent's owner.  AtA blocks travel as
# packed lower triangles (distsim.py:192-199), AtB blocks as rectangles.
# Over NCCL these are point-to-point sends; the tree has one message per
# non-root process and no cycles, so the blocking order cannot deadlock.

def _block_words(task) -> int:
    c = task.c_region
    if task.b_region is None:           # lower triangle of a diagonal block
        return c.rows * (c.rows + 1) // 2
    return c.rows * c.cols


def tree_comm_stats(tree):
    """Retrieve-phase traffic of the tree (words and messages per process):
    the CommStats counters of distsim.py:72-111 restricted to result blocks."""
    from .tasktree import path_to_root
    P = tree.procs
    st = {k: [0] * P for k in ("sent_messages", "sent_words", "recv_messages", "recv_words")}
    for q in range(1, P):
        top = path_to_root(tree, q)[-1]
        dst = tree.nodes[top.parent_id].task.owner
        w = _block_words(top.task)
        st["sent_messages"][q] += 1
        st["sent_words"][q] += w
        st["recv_messages"][dst] += 1
        st["recv_words"][dst] += w
    return st


def write_comm_csv(path, stats, procs: int) -> None:
    """The reference's --comm-csv layout (distsim.py:101-111)."""
    import csv
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["process", "sent_messages", "sent_words", "recv_messages", "recv_words"])
        for p in range(procs):
            w.writerow([p, stats["sent_messages"][p], stats["sent_words"][p],
                        stats["recv_messages"][p], stats["recv_words"][p]])
        w.writerow(["critical_path", stats["sent_messages"][0], stats["sent_words"][0],
                    stats["recv_messages"][0], stats["recv_words"][0]])


class _LocalLink:
    """In-process transport: all processes of the tree run on this GPU in
    decreasing label order (a non-first child's owner always has a larger
    label than its parent's), so every block is produced before it is read."""

    def __init__(self):
        self.box = {}

    def send(self, block, src: int, dst: int, node) -> None:
        self.box[(src, dst, node.id)] = block

    def recv(self, shape_like, src: int, dst: int, node):
        return self.box.pop((src, dst, node.id))


class _DistLink:
    """torch.distributed point-to-point (NCCL; gloo stages through the host)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.gloo = dist.get_backend(group) == "gloo"

    def _peer(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def send(self, block, src: int, dst: int, node) -> None:
        t = block.cpu() if (self.gloo and block.is_cuda) else block
        self.dist.send(t.contiguous(), dst=self._peer(dst), group=self.group)

    def recv(self, shape_like, src: int, dst: int, node):
        import torch
        buf = torch.empty(shape_like[0], dtype=shape_like[1], device="cpu" if self.gloo else shape_like[2])
        self.dist.recv(buf, src=self._peer(src), group=self.group)
        return buf.to(shape_like[2]) if self.gloo else buf


def _leaf_block(task, get_block, alpha, threshold, dtype, device, counter, precision):
    """This process's leaf: a fresh C block (zeros) += alpha * leaf product."""
    import torch
    from .ata import ata
    from .strassen import fast_strassen
    c = task.c_region
    out = torch.zeros((c.rows, c.cols), dtype=dtype, device=device)
    a = get_block(task.a_region)
    if task.b_region is None:
        ata(a, out, alpha, threshold, counter=counter, precision=precision)
    else:
        fast_strassen(a, get_block(task.b_region), out, alpha, threshold=threshold, counter=counter)
    return out


def _wire(task, block):
    """Block as sent: packed lower triangle for AtA, rectangle for AtB."""
    if task.b_region is None:
        from .matrix import pack_lower
        return pack_lower(block).data
    return block


def run_tree_process(tree, p: int, get_block, link, alpha=1.0, threshold="auto", dtype=None,
                     device=None, counter=None, precision: str = "fp32", leaf_block=None):
    """Process p's part of the tree: its leaf (or the caller's `leaf_block`,
    already computed), then every node it owns (assembling children's
    blocks), then the send of its chain top.  Returns the chain top's C block
    (the whole n x n result on process 0)."""
    from .tasktree import path_to_root
    chain = path_to_root(tree, p)
    block = leaf_block if leaf_block is not None else \
        _leaf_block(chain[0].task, get_block, alpha, threshold, dtype, device, counter, precision)
    from .matrix import PackedLowerTriangular, add_truncated, unpack_lower
    for prev, node in zip(chain, chain[1:]):
        import torch
        c = node.task.c_region
        out = torch.zeros((c.rows, c.cols), dtype=dtype, device=device)
        # children's blocks accumulate in child order with the native kernels:
        # packed AtA partials unpack-accumulate straight into their diagonal
        # block (distsim.py:208-216), rectangles through the truncated add
        for child in tree.children_of(node):
            cc = child.task.c_region
            r0, c0 = cc.row_offset - c.row_offset, cc.col_offset - c.col_offset
            view = out[r0:r0 + cc.rows, c0:c0 + cc.cols]
            if child.id == prev.id:
                add_truncated(view, block, 1.0)
                continue
            q = child.task.owner
            wire = link.recv((_block_words(child.task), dtype, device), q, p, child)
            if child.task.b_region is None:
                unpack_lower(PackedLowerTriangular(cc.rows, wire), view, accumulate=True)
            else:
                add_truncated(view, wire.view(cc.rows, cc.cols), 1.0)
        block = out
    top = chain[-1]
    if top.parent_id is not None:
        link.send(_wire(top.task, block), p, tree.nodes[top.parent_id].task.owner, top)
    return block


def add_lower_into(C, block):
    """lower(C) += lower(block), C's strict upper triangle untouched: the
    native pack / accumulate-unpack kernels (one pass each over the triangle)."""
    from .matrix import PackedLowerTriangular, pack_lower, unpack_lower
    n = int(C.shape[0])
    packed = pack_lower(block)
    unpack_lower(PackedLowerTriangular(n, packed.data), C, accumulate=True)


def tree_link(group=None):
    """The torch.distributed transport of run_tree_process."""
    return _DistLink(group)


def ata_tree(get_block, m: int, n: int, C, alpha=1.0, threshold="auto", procs: int | None = None,
             group=None, counter=None, precision: str = "fp32"):
    """lower(C) += alpha * A^T A over the reference's distributed task tree.

    With a torch.distributed group of P > 1 ranks, every rank runs its own
    leaf and chain (get_block only needs to serve that rank's regions) and
    rank 0's C receives the result.  Without one, ``procs`` processes are
    simulated on this GPU one after another (the reference's in-process
    distributed executor, ata_d).  get_block(Region) -> CUDA tensor view."""
    from .tasktree import build_tree_distributed
    import torch.distributed as dist
    dtype, device = C.dtype, C.device
    if procs is None and dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        P, rank = dist.get_world_size(group), dist.get_rank(group)
        tree = build_tree_distributed(P, m, n)
        top = run_tree_process(tree, rank, get_block, _DistLink(group), alpha, threshold, dtype, device,
                               counter, precision)
        if rank == 0:
            add_lower_into(C, top)
        return tree
    P = procs or 1
    tree = build_tree_distributed(P, m, n)
    link = _LocalLink()
    top = None
    for p in reversed(range(P)):
        top = run_tree_process(tree, p, get_block, link, alpha, threshold, dtype, device, counter,
                               precision)
    add_lower_into(C, top)
    return tree


def tree_rows(tree, rank: int):
    """Row range [r0, r1) of A that `rank`'s leaf reads (its a and b regions
    share their rows) -- what a rank must generate or receive."""
    from .tasktree import leaf_task
    t = leaf_task(tree, rank)
    return t.a_region.row_offset, t.a_region.row_offset + t.a_region.rows


# --------------------------------------------------------------------------
# Units partition (north star): the top level's two AtA sub-problems and the
# seven Strassen products of its C21 node as row-range segments on the ranks
# (auto_plan.partition_units / plan_units), combined region by region.
#
# A rank's segments write only some of the three regions of lower(C): C11
# (lower triangle of the left diagonal block; "ata_l" segments), C22 (the
# right diagonal block; "ata_r") and C21 (the rectangle; every product
# segment, each adding its signed P_i into its C21 quadrants).  Each region
# is summed to the root with one NCCL reduce over the group of ranks that
# wrote it (plus the root): packed triangles for C11/C22, the rectangle for
# C21.  Row shards reduce the whole packed triangle from every rank; here a
# rank ships only what it computed.

REGIONS = ("c11", "c22", "c21")


def unit_regions(segments):
    """The C regions a rank's segments write."""
    out = set()
    for (u, _, _) in segments:
        out.add("c11" if u == "ata_l" else "c22" if u == "ata_r" else "c21")
    return out


def region_members(all_segments, root: int = 0):
    """Per region, the sorted ranks that take part in its reduce."""
    mem = {r: {root} for r in REGIONS}
    for rank, segs in enumerate(all_segments):
        for r in unit_regions(segs):
            mem[r].add(rank)
    return {r: sorted(v) for r, v in mem.items()}


def region_windows(C, n: int):
    """(kind, block view) of each region of an n x n C."""
    n1 = n // 2
    return {"c11": ("packed", C[:n1, :n1]), "c22": ("packed", C[n1:, n1:]), "c21": ("rect", C[n1:, :n1])}


def make_region_groups(all_segments, root: int = 0):
    """torch.distributed groups of the region reduces (every rank must call
    this, in the same order: new_group is collective)."""
    import torch.distributed as dist
    mem = region_members(all_segments, root)
    world = dist.get_world_size()
    groups = {}
    for r in REGIONS:
        ranks = mem[r]
        groups[r] = (None if len(ranks) == world else dist.new_group(ranks)) if len(ranks) > 1 else "solo"
    return groups, mem


def reduce_regions(C, n: int, rank: int, groups, members, ops, root: int = 0, bufs=None):
    """Sum each region's contributions into the root's C: pack (triangles) or
    copy (rectangle) this rank's block, NCCL reduce(SUM) to the root over the
    region's group, and the root writes the sum back.  Regions in a fixed
    order on every rank (no cross-communicator deadlock)."""
    import torch.distributed as dist
    wins = region_windows(C, n)
    bufs = {} if bufs is None else bufs
    for r in REGIONS:
        if rank not in members[r] or groups[r] == "solo":
            continue
        kind, blk = wins[r]
        data = ops.pack(blk) if kind == "packed" else ops.copy_rect(blk)
        g = groups[r]
        if ops.device.type == "cuda" and dist.get_backend(g) == "gloo":
            host = data.cpu()
            dist.reduce(host, dst=root, op=dist.ReduceOp.SUM, group=g)
            data.copy_(host)
        else:
            dist.reduce(data, dst=root, op=dist.ReduceOp.SUM, group=g)
        if rank == root:
            ops.write(blk, kind, data)
        bufs[r] = data
    return C


def ata_units(A, C, segments, all_segments=None, params=None, alpha: float = 1.0, groups=None,
              root: int = 0, precision: str = "fp32"):
    """lower(C) += alpha * A^T A over the ranks of the default process group
    with the units partition.  `A` is the full m x n CUDA operand (only the
    rows this rank's segments read must hold data: auto_plan.a_rows_needed),
    `segments` this rank's (unit, r0, r1) list, `all_segments` every rank's
    (for the region groups; built by partition_units when None).  The root's
    C holds the result; other ranks' C hold their partial regions."""
    import torch
    import torch.distributed as dist
    from . import _native as nat, auto_plan, engine
    from .distsim import DeviceBlocks
    m, n = int(A.shape[0]), int(A.shape[1])
    params = params or auto_plan.AutoParams()
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    if all_segments is None:
        all_segments = auto_plan.partition_units(m, n, world, params)
    plan = engine.cached_plan(("units", m, n, A.stride(0), C.stride(0), tuple(segments), params),
                              lambda: auto_plan.plan_units(segments, m, n, A.stride(0), C.stride(0), params))
    ws = torch.empty(max(1, plan.ws_scalars), dtype=C.dtype, device=C.device)
    if rank != root:
        C.zero_()
    engine.run_plan(plan, nat.dtype_code(C.dtype, precision), int(A.data_ptr()), A.numel(), int(C.data_ptr()),
                    C.numel(), alpha, ws=int(ws.data_ptr()), ws_elems=ws.numel())
    if world > 1:
        if groups is None:
            groups, members = make_region_groups(all_segments, root)
        else:
            groups, members = groups
        reduce_regions(C, n, rank, groups, members, DeviceBlocks(C.device, C.dtype), root)
    return C
