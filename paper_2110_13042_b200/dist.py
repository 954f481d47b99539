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
