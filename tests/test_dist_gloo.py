"""Multi-process host logic of the row-sharded multi-GPU path, on CPU with
gloo (world size 2): shard ranges, per-rank seeded row streams, and the packed
lower-triangle sum to the root (distsim.py:192-216 semantics).  The device
compute itself is covered by the GPU tests; here each rank's partial Gram is
produced by the oracle (test infrastructure)."""
import os
import socket

import numpy as np
import pytest

from paper_2110_13042_b200 import dist as pdist


def test_shard_rows_cover_exactly():
    for m in (1, 7, 100, 65536, 1048577):
        for world in (1, 2, 3, 4, 8):
            spans = [pdist.shard_rows(m, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_uniform_rows_match_full_stream():
    m, n, seed = 37, 13, 3
    full = np.random.default_rng(seed).uniform(-1.0, 1.0, (m, n))
    for world in (1, 2, 4):
        parts = [pdist.uniform_rows(m, n, seed, *pdist.shard_rows(m, world, r))
                 for r in range(world)]
        assert np.array_equal(np.concatenate(parts), full)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, m, n, seed, out):
    import torch
    import torch.distributed as dist
    from oracle import atamul_oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r0, r1 = pdist.shard_rows(m, world, rank)
    a = pdist.uniform_rows(m, n, seed, r0, r1)
    c = np.zeros((n, n))
    O.syrk_lower(a, c)                       # this rank's partial (oracle stands in for the GPU)
    packed = torch.from_numpy(O.pack_lower(c))
    pdist.reduce_packed(packed, root=0)
    if rank == 0:
        out.put(packed.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def test_packed_reduce_two_ranks():
    import torch.multiprocessing as mp
    m, n, seed, world = 301, 17, 5, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import atamul_oracle as O
    a = np.random.default_rng(seed).uniform(-1.0, 1.0, (m, n))
    ref = O.pack_lower(O.gram(a))
    assert np.abs(got - ref).max() <= 1e-12 * m
