"""Distribute-compute-retrieve executor over GPUs (reference distsim.py:1-393).

The reference simulates P processes in one Python process: process 0 holds A,
operand blocks travel DOWN the distributed task tree (``build_tree_distributed``,
scheduler.py:283-363), every process computes its leaf, and result blocks travel
UP, each owner summing its children's partials in child order; one send is one
message whatever the number of blocks it carries, AtA results travel as
packed lower triangles, everything else as dense rectangles, and ``CommStats``
counts messages and words per process (distsim.py:25-111, :219-297).

Here the same per-process program drives B200s:

* one process per rank of a ``torch.distributed`` group (``procs`` == world
  size): messages are NCCL point-to-point transfers of device buffers over
  NVLink (one flat payload per message), every rank computes its leaf with the
  single-GPU plans (``execute.run_leaf``), parents accumulate packed partials
  with the native unpack-accumulate kernel and rectangles with the native
  truncated add -- no host staging on the data path;
* otherwise the ``procs`` processes are simulated on the current GPU, driven
  by a seeded scheduler like the reference's (``run_processes``); a message is
  a device-to-device copy of its payload.

Because every process consumes messages from explicitly named peers in a fixed
program order and all device work of the simulated processes is issued on one
stream, the result is identical under every interleaving (the reference's
ordering-independence property).  ``CommStats``, ``verify_comm_bounds`` and the
bounds of distsim.py:353-393 are restated for the accounting.
"""
from __future__ import annotations

import csv
import random
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from .errors import ProtocolError
from .tasktree import (ComputationType, Region, Task, TaskTree, build_tree_distributed,
                       levels_distributed, path_to_root)
from .workspace import DEFAULT_THRESHOLD


# --------------------------------------------------------------------------
# messages and counters (distsim.py:47-111)

def _part_words(kind: str, region: Region) -> int:
    return region.rows * region.cols if kind == "rect" else region.rows * (region.rows + 1) // 2


@dataclass
class MessagePart:
    kind: str            # "rect" | "packed"
    region: Region       # absolute coordinates in the global matrix
    data: object         # flat payload (device tensor), rows*cols or r*(r+1)/2 words

    def __post_init__(self):
        expect = _part_words(self.kind, self.region)
        got = int(self.data.numel()) if hasattr(self.data, "numel") else int(np.size(self.data))
        if got != expect:
            raise ProtocolError(f"protocol error: payload length {got} != {expect}")


@dataclass
class Message:
    src: int
    dst: int
    parts: list

    @property
    def words(self) -> int:
        return sum(_part_words(p.kind, p.region) for p in self.parts)


@dataclass
class CommStats:
    """Messages and words sent / received per process; the critical path is
    process 0's traffic (distsim.py:70-111)."""
    procs: int
    sent_messages: list = field(default_factory=list)
    sent_words: list = field(default_factory=list)
    recv_messages: list = field(default_factory=list)
    recv_words: list = field(default_factory=list)
    compute_seconds: float = 0.0

    def __post_init__(self):
        for name in ("sent_messages", "sent_words", "recv_messages", "recv_words"):
            if not getattr(self, name):
                setattr(self, name, [0] * self.procs)

    @property
    def critical_path_messages(self) -> int:
        return self.sent_messages[0] + self.recv_messages[0]

    @property
    def total_messages(self) -> int:
        return sum(self.sent_messages)

    @property
    def total_words(self) -> int:
        return sum(self.sent_words)

    def write_csv(self, path) -> None:
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["process", "sent_messages", "sent_words", "recv_messages", "recv_words"])
            for p in range(self.procs):
                w.writerow([p, self.sent_messages[p], self.sent_words[p], self.recv_messages[p],
                            self.recv_words[p]])
            w.writerow(["critical_path", self.sent_messages[0], self.sent_words[0],
                        self.recv_messages[0], self.recv_words[0]])


# --------------------------------------------------------------------------
# communication bounds (distsim.py:300-393)

@dataclass
class CommReport:
    procs: int
    n: int
    levels: int
    latency_observed: int
    latency_bound: float
    words_observed: int
    words_bound: float
    failures: list = field(default_factory=list)

    @property
    def ok(self) -> bool:
        return not self.failures

    def summary(self) -> str:
        status = "ok" if self.ok else "FAILED " + "; ".join(self.failures)
        return (f"P={self.procs} n={self.n} levels={self.levels}: critical-path messages "
                f"{self.latency_observed} (bound {self.latency_bound:g}), total words "
                f"{self.words_observed} (bound {self.words_bound:g}) -> {status}")


def comm_bound_latency(procs: int) -> float:
    """2 x (5 messages at the first level + 7 per deeper level), one factor
    per phase (distsim.py:343-351)."""
    levels = levels_distributed(procs)
    return 0.0 if levels == 0 else 2.0 * (5 + 7 * (levels - 1))


def comm_bound_words(n: int, procs: int) -> float:
    """Words moved by both phases (distsim.py:354-370): one level moves five
    half-size operand blocks down and one half rectangle plus four packed
    half triangles up; deeper trees add the geometric quarter-and-below term."""
    levels = levels_distributed(procs)
    if levels == 0:
        return 0.0
    half_sq = (n / 2.0) ** 2
    if levels == 1:
        return 6 * half_sq + 4 * (n * (n + 2) / 8.0)
    return 6 * half_sq + n * (n + 2) / 2.0 + (7.0 / 6.0) * n * n * (1 - 0.25 ** (levels - 2))


def verify_comm_bounds(stats: CommStats, n: int, procs: int) -> CommReport:
    """Recorded counters against the latency and bandwidth bounds (distsim.py:373-393)."""
    rep = CommReport(procs, n, levels_distributed(procs), stats.critical_path_messages,
                     comm_bound_latency(procs), stats.total_words, comm_bound_words(n, procs))
    if rep.latency_observed > rep.latency_bound:
        rep.failures.append(f"critical-path messages {rep.latency_observed} > bound {rep.latency_bound:g}")
    if rep.words_observed > rep.words_bound:
        rep.failures.append(f"total words {rep.words_observed} > bound {rep.words_bound:g}")
    return rep


# --------------------------------------------------------------------------
# device-side block operations of the program

class DeviceBlocks:
    """Block operations on CUDA tensors with the native kernels: packing a
    result triangle (ata_pack_lower), accumulating a packed partial into a
    lower triangle (ata_unpack_lower, accumulate) and a rectangle
    (ata_add_truncated)."""

    def __init__(self, device, dtype):
        self.device, self.dtype = device, dtype

    def zeros(self, rows, cols):
        import torch
        return torch.zeros((rows, cols), dtype=self.dtype, device=self.device)

    def empty(self, words):
        import torch
        return torch.empty(words, dtype=self.dtype, device=self.device)

    def copy_rect(self, block):
        return block.contiguous().clone().view(-1)

    def pack(self, block):
        from .matrix import pack_lower
        return pack_lower(block).data

    def add_packed(self, block, data):
        from .matrix import PackedLowerTriangular, unpack_lower
        unpack_lower(PackedLowerTriangular(int(block.shape[0]), data), block, accumulate=True)

    def add_rect(self, block, data):
        from .matrix import add_truncated
        add_truncated(block, data.view(int(block.shape[0]), int(block.shape[1])), 1.0)

    def write(self, block, kind, data):
        """Overwrite a block's lower triangle ("packed") or the whole block ("rect")."""
        from .matrix import PackedLowerTriangular, unpack_lower
        if kind == "packed":
            unpack_lower(PackedLowerTriangular(int(block.shape[0]), data), block)
        else:
            block.copy_(data.view(int(block.shape[0]), int(block.shape[1])))

    def timer(self):
        import torch
        return torch.cuda.Event(enable_timing=True)

    @staticmethod
    def elapsed(pairs):
        import torch
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in pairs) * 1e-3


class _Store:
    """The operand blocks a process holds (distsim.py:176-189 keeps a full
    m x n array; here only the received rectangles): a requested region is
    served as a view of the part that contains it."""

    def __init__(self):
        self.parts = []

    def put(self, region: Region, block):
        self.parts.append((region, block))

    def get(self, r: Region):
        for reg, blk in self.parts:
            if (reg.row_offset <= r.row_offset and r.row_offset + r.rows <= reg.row_offset + reg.rows
                    and reg.col_offset <= r.col_offset and r.col_offset + r.cols <= reg.col_offset + reg.cols):
                r0, c0 = r.row_offset - reg.row_offset, r.col_offset - reg.col_offset
                return blk[r0:r0 + r.rows, c0:c0 + r.cols]
        raise ProtocolError(f"protocol error: operand region {r} was never received")


def _operand_regions(task: Task):
    return [task.a_region] + ([task.b_region] if task.b_region is not None else [])


def _result_kind(task: Task) -> str:
    return "packed" if task.computation is ComputationType.ATA else "rect"


def process_program(p: int, tree: TaskTree, a_root, ops, leaf_fn):
    """Process p (distsim.py:219-269) as a generator yielding
    ("send", Message) and ("recv", src, [(kind, region)]) requests; returns
    its C block (process 0: the whole n x n lower triangle) and the (start,
    end) timer pairs of its compute."""
    chain = path_to_root(tree, p)
    top = chain[-1]
    store = _Store()
    if p == 0:
        store.put(Region(0, 0, tree.m, tree.n), a_root)
    else:
        spec = [("rect", r) for r in _operand_regions(top.task)]
        msg = yield ("recv", top.task.parent, spec)
        for part in msg.parts:
            store.put(part.region, part.data.view(part.region.rows, part.region.cols))
    # distribution: each non-owned child of the owned chain gets its operand
    # blocks, top of the chain first
    for node in reversed(chain):
        for child in tree.children_of(node):
            q = child.task.owner
            if q != p:
                parts = [MessagePart("rect", r, ops.copy_rect(store.get(r)))
                         for r in _operand_regions(child.task)]
                yield ("send", Message(p, q, parts))
    # compute: the leaf into a C block covering the chain top's region
    tc = top.task.c_region
    c_local = ops.zeros(tc.rows, tc.cols)

    def cview(r: Region):
        r0, c0 = r.row_offset - tc.row_offset, r.col_offset - tc.col_offset
        return c_local[r0:r0 + r.rows, c0:c0 + r.cols]

    timers = []
    t0, t1 = ops.timer(), ops.timer()
    t0.record()
    leaf_fn(chain[0].task, store.get, cview(chain[0].task.c_region))
    t1.record()
    timers.append((t0, t1))
    # retrieval: children's partials bottom-up, in child order
    for node in chain:
        for child in tree.children_of(node):
            q = child.task.owner
            if q == p:
                continue
            msg = yield ("recv", q, [(_result_kind(child.task), child.task.c_region)])
            t0, t1 = ops.timer(), ops.timer()
            t0.record()
            for part in msg.parts:
                blk = cview(part.region)
                if part.kind == "packed":
                    ops.add_packed(blk, part.data)
                else:
                    ops.add_rect(blk, part.data)
            t1.record()
            timers.append((t0, t1))
    if top.parent_id is not None:
        blk = cview(tc)
        kind = _result_kind(top.task)
        data = ops.pack(blk) if kind == "packed" else ops.copy_rect(blk)
        yield ("send", Message(p, top.task.parent, [MessagePart(kind, tc, data)]))
        return None, timers
    return c_local, timers


def _check_spec(msg: Message, spec) -> None:
    got = [(pt.kind, pt.region) for pt in msg.parts]
    if got != list(spec):
        raise ProtocolError(f"protocol error: expected {spec} from {msg.src}, got {got}")


def _count(stats: CommStats, trace, req, msg) -> None:
    if req == "send":
        stats.sent_messages[msg.src] += 1
        stats.sent_words[msg.src] += msg.words
        if trace is not None:
            trace.append((msg.src, msg.dst, [(pt.kind, pt.region, _part_words(pt.kind, pt.region))
                                             for pt in msg.parts]))
    else:
        stats.recv_messages[msg.dst] += 1
        stats.recv_words[msg.dst] += msg.words


def run_processes(gens: dict, stats: CommStats, trace=None, seed: int = 0) -> dict:
    """In-process scheduler (the reference's run_processes, distsim.py:118-170):
    FIFO mailboxes per (src, dst), runnable processes picked in a seeded
    random order; a receive that can never be satisfied, or undelivered mail
    at the end, is a ProtocolError."""
    rng = random.Random(seed)
    boxes: dict = {}
    blocked: dict = {}        # pid -> (src, spec) it waits for
    pending: dict = {}        # pid -> message to resume with
    done: dict = {}
    runnable = sorted(gens)

    def resume(p):
        value = pending.pop(p, None)
        try:
            req = gens[p].send(value)
            while True:
                if req[0] == "send":
                    msg = req[1]
                    _count(stats, trace, "send", msg)
                    boxes.setdefault((msg.src, msg.dst), deque()).append(msg)
                    w = blocked.get(msg.dst)
                    if w is not None and w[0] == msg.src:
                        del blocked[msg.dst]
                        got = boxes[(msg.src, msg.dst)].popleft()
                        _check_spec(got, w[1])
                        _count(stats, trace, "recv", got)
                        pending[msg.dst] = got
                        runnable.append(msg.dst)
                    req = gens[p].send(None)
                elif req[0] == "recv":
                    src, spec = req[1], req[2]
                    box = boxes.get((src, p))
                    if box:
                        got = box.popleft()
                        _check_spec(got, spec)
                        _count(stats, trace, "recv", got)
                        req = gens[p].send(got)
                    else:
                        blocked[p] = (src, spec)
                        return
                else:
                    raise ProtocolError(f"protocol error: bad request {req!r}")
        except StopIteration as stop:
            done[p] = stop.value

    while runnable:
        i = rng.randrange(len(runnable))
        runnable[i], runnable[-1] = runnable[-1], runnable[i]
        resume(runnable.pop())
    if len(done) != len(gens):
        stuck = sorted(set(gens) - set(done))
        raise ProtocolError(f"protocol error: deadlock, processes {stuck} still waiting on "
                            f"{ {p: blocked.get(p, (None,))[0] for p in stuck} }")
    for (src, dst), box in boxes.items():
        if box:
            raise ProtocolError(f"protocol error: {len(box)} undelivered messages {src}->{dst}")
    return done


class _GroupLink:
    """Messages between the ranks of a torch.distributed group: one flat
    payload per message (NCCL: device buffers over NVLink; gloo: host
    tensors, for the CPU tests of the protocol)."""

    def __init__(self, group, ops):
        import torch.distributed as dist
        self.dist, self.group, self.ops = dist, group, ops
        # gloo has no point-to-point on CUDA tensors: stage through the host
        # (CPU checks of the multi-rank path on one shared GPU)
        self.stage = dist.get_backend(group) == "gloo" and getattr(ops.device, "type", "cpu") == "cuda"

    def _peer(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def send(self, msg: Message) -> None:
        import torch
        flat = torch.cat([pt.data.reshape(-1) for pt in msg.parts]) if len(msg.parts) > 1 \
            else msg.parts[0].data.reshape(-1)
        flat = flat.contiguous()
        self.dist.send(flat.cpu() if self.stage else flat, dst=self._peer(msg.dst), group=self.group)

    def recv(self, src: int, dst: int, spec) -> Message:
        words = [_part_words(k, r) for k, r in spec]
        flat = self.ops.empty(sum(words))
        if self.stage:
            host = flat.cpu()
            self.dist.recv(host, src=self._peer(src), group=self.group)
            flat.copy_(host)
        else:
            self.dist.recv(flat, src=self._peer(src), group=self.group)
        parts, o = [], 0
        for (k, r), w in zip(spec, words):
            parts.append(MessagePart(k, r, flat[o:o + w]))
            o += w
        return Message(src, dst, parts)


def run_rank(p: int, gen, link: _GroupLink, stats: CommStats, trace=None):
    """Drive this rank's program over the group link."""
    value = None
    while True:
        try:
            req = gen.send(value)
        except StopIteration as stop:
            return stop.value
        value = None
        if req[0] == "send":
            _count(stats, trace, "send", req[1])
            link.send(req[1])
        else:
            msg = link.recv(req[1], p, req[2])
            _count(stats, trace, "recv", msg)
            value = msg


def _gather_stats(stats: CommStats, group, device) -> CommStats:
    """Every rank counted only its own traffic: all-gather the counters."""
    import torch
    import torch.distributed as dist
    P, r = stats.procs, dist.get_rank(group)
    if dist.get_backend(group) == "gloo":
        device = "cpu"
    mine = torch.tensor([stats.sent_messages[r], stats.sent_words[r], stats.recv_messages[r],
                         stats.recv_words[r]], dtype=torch.int64, device=device)
    out = [torch.zeros_like(mine) for _ in range(P)]
    dist.all_gather(out, mine, group=group)
    rows = [o.cpu().tolist() for o in out]
    return CommStats(P, [x[0] for x in rows], [x[1] for x in rows], [x[2] for x in rows],
                     [x[3] for x in rows], stats.compute_seconds)


def _leaf_runner(threshold, leaf_kernel, counter, ata_kw):
    from .execute import run_leaf

    def leaf(task, get_block, c_block):
        run_leaf(task, get_block, c_block, threshold, counter, leaf_kernel, None, **ata_kw)
    return leaf


def ata_d(A, procs: int, threshold=DEFAULT_THRESHOLD, leaf_kernel: str = "fast",
          scheduler_seed: int = 0, counter=None, trace: list | None = None, *, group=None,
          **ata_kw):
    """Full symmetric A^T A over `procs` processes with A initially held only
    by process 0; returns (DenseMatrix, CommStats) (distsim.py:272-297).

    With an initialised torch.distributed group of exactly `procs` ranks,
    process r is rank r (A is read on rank 0 only; other ranks may pass
    None) and rank 0 returns the result (other ranks: None).  Otherwise the
    processes are simulated on the current GPU.  `trace` collects one
    (src, dst, [(kind, region, words)]) record per message (this rank's sends
    in the multi-rank mode)."""
    import torch
    from .matrix import DenseMatrix, as_array, mirror_lower_to_upper
    if leaf_kernel not in ("fast", "naive"):
        raise ValueError(f"unknown leaf kernel {leaf_kernel!r}")
    dist = torch.distributed
    multi = (dist.is_available() and dist.is_initialized() and procs > 1
             and dist.get_world_size(group) == procs)
    rank = dist.get_rank(group) if multi else 0
    dev = torch.device("cuda", torch.cuda.current_device())
    host_input = True
    if rank == 0:
        a = as_array(A)
        host_input = not (isinstance(a, torch.Tensor) and a.is_cuda)
        if host_input:
            h = a.numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
            if h.dtype not in (np.float32, np.float64):
                h = h.astype(np.float64)
            a = torch.from_numpy(np.ascontiguousarray(h)).to(dev)
        meta = torch.tensor([a.shape[0], a.shape[1], 8 if a.dtype == torch.float64 else 4],
                            dtype=torch.int64, device=dev)
    else:
        a, meta = None, torch.zeros(3, dtype=torch.int64, device=dev)
    if multi:
        if dist.get_backend(group) == "gloo":
            meta = meta.cpu()
        dist.broadcast(meta, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    m, n, w = (int(x) for x in meta.tolist())
    dtype = torch.float64 if w == 8 else torch.float32
    tree = build_tree_distributed(procs, m, n)
    ops = DeviceBlocks(dev, dtype)
    leaf = _leaf_runner(threshold, leaf_kernel, counter, ata_kw)
    stats = CommStats(procs)
    if multi:
        result, timers = run_rank(rank, process_program(rank, tree, a, ops, leaf),
                                  _GroupLink(group, ops), stats, trace)
        stats.compute_seconds = ops.elapsed(timers)
        stats = _gather_stats(stats, group, dev)
        if rank != 0:
            return None, stats
    else:
        gens = {p: process_program(p, tree, a if p == 0 else None, ops, leaf) for p in range(procs)}
        done = run_processes(gens, stats, trace, scheduler_seed)
        stats.compute_seconds = ops.elapsed([t for p in done for t in done[p][1]])
        result = done[0][0]
    mirror_lower_to_upper(result)
    return DenseMatrix(result.cpu().numpy() if host_input else result), stats
