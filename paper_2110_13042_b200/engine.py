"""Plan execution: plan cache + one native call per plan.

The executor itself is native (``ata_run_plan`` in csrc/abi.cu); this module
keeps plans keyed by shape/layout/threshold so repeated calls skip planning,
and owns the per-device int32 "sync" buffer the persistent kernels use for
their work counter and destination turn counters.
"""
from __future__ import annotations

import os

import ctypes
from collections import OrderedDict

import numpy as np

from . import _native as nat

_PLAN_CACHE: "OrderedDict[tuple, object]" = OrderedDict()
_PLAN_CACHE_MAX = 64
_SYNC: dict = {}


def cached_plan(key, builder):
    p = _PLAN_CACHE.get(key)
    if p is None:
        p = builder()
        _PLAN_CACHE[key] = p
        if len(_PLAN_CACHE) > _PLAN_CACHE_MAX:
            _PLAN_CACHE.popitem(last=False)
    else:
        _PLAN_CACHE.move_to_end(key)
    return p


def reference_dfs() -> bool:
    """ATA_REF_DFS=1: run integer-threshold recursions with the depth-first
    executor (planner._ReferencePlanner, the reference's per-depth scratch)
    instead of the breadth-first one (ref_bfs.py)."""
    return os.environ.get("ATA_REF_DFS", "0") == "1"


def sync_ints_needed(plan, dtype_code) -> int:
    need = getattr(plan, "_sync_need", {}).get(dtype_code)
    if need is None:
        ops = np.ascontiguousarray(plan.ops)
        need = int(nat.load().ata_sync_ints_needed(dtype_code, ops.ctypes.data_as(ctypes.c_void_p),
                                                   len(ops)))
        try:
            plan._sync_need = {**getattr(plan, "_sync_need", {}), dtype_code: need}
        except AttributeError:
            pass
    return need


def sync_buffer(device, ints: int):
    """Per-(device, stream) int32 scratch, grown on demand.  Keyed by stream so
    concurrent plans on different streams never share counters."""
    import torch
    stream = torch.cuda.current_stream(device)
    key = (device.index if device.index is not None else torch.cuda.current_device(),
           int(stream.cuda_stream))
    buf = _SYNC.get(key)
    if buf is None or buf.numel() < ints:
        buf = torch.zeros(max(ints, 1 << 16), dtype=torch.int32, device=device)
        _SYNC[key] = buf
    return buf


def run_plan(plan, dtype_code, A, a_elems, C, c_elems, alpha, ws=None, ws_elems=0, B=None,
             b_elems=0, stream=None, device=None, sync=None):
    """Issue every op of `plan` on `stream` (default: torch's current stream).
    A/B/C/ws are device pointers (ints)."""
    import torch
    lib = nat.load()
    if stream is None:
        stream = int(torch.cuda.current_stream().cuda_stream)
    ops = plan.ops
    if not ops.flags.c_contiguous:
        ops = np.ascontiguousarray(ops)
    if sync is None:
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        sync = sync_buffer(dev, sync_ints_needed(plan, dtype_code))
    rc = lib.ata_run_plan(dtype_code, ops.ctypes.data_as(ctypes.c_void_p), len(ops),
                          A, a_elems, B if B is not None else A, b_elems if B is not None else a_elems,
                          C, c_elems, ws or 0, ws_elems, int(sync.data_ptr()), int(sync.numel()),
                          float(alpha), stream)
    nat.check(rc)


_CAPTURE_STREAMS: dict = {}


def _capture_stream():
    """One capture stream per device (the executor keeps fork/join resources
    per calling stream)."""
    import torch
    dev = torch.cuda.current_device()
    st = _CAPTURE_STREAMS.get(dev)
    if st is None:
        st = _CAPTURE_STREAMS[dev] = torch.cuda.Stream()
    return st


class PlanGraph:
    """One plan execution with fixed pointers captured as a CUDA graph.

    Reference-faithful plans with small leaves issue thousands of launches
    (config c2 at t = 256^2: ~8000); replaying a captured graph removes the
    host-side launch cost.  The caller must have run the plan once eagerly
    (function attributes, sync buffer) before constructing the graph."""

    def __init__(self, plan, dtype_code, A, a_elems, C, c_elems, alpha, ws=None, ws_elems=0,
                 B=None, b_elems=0):
        import torch
        self.graph = torch.cuda.CUDAGraph()
        side = _capture_stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(self.graph, stream=side):
            run_plan(plan, dtype_code, A, a_elems, C, c_elems, alpha, ws=ws, ws_elems=ws_elems,
                     B=B, b_elems=b_elems, stream=int(side.cuda_stream))
        torch.cuda.current_stream().wait_stream(side)

    def replay(self):
        self.graph.replay()


_GRAPHS: "OrderedDict" = OrderedDict()
_GRAPH_SEEN: dict = {}
_GRAPHS_MAX = 8


def run_plan_graphed(key, plan, dtype_code, A, a_elems, C, c_elems, alpha, ws=None, ws_elems=0,
                     B=None, b_elems=0):
    """run_plan for launch-bound plans (breadth-first reference recursions:
    ~1000 small launches): the second call with identical plan, pointers and
    alpha captures a CUDA graph, later calls replay it on the current stream.
    `key` identifies the plan (its cache key)."""
    import torch
    dev = torch.cuda.current_device()
    gkey = (key, dtype_code, dev, int(torch.cuda.current_stream().cuda_stream), A, a_elems, C, c_elems,
            float(alpha), ws or 0, ws_elems, B or 0, b_elems)
    g = _GRAPHS.get(gkey)
    if g is None:
        seen = _GRAPH_SEEN.get(gkey, 0) + 1
        _GRAPH_SEEN[gkey] = seen
        if len(_GRAPH_SEEN) > 64:
            _GRAPH_SEEN.clear()
        if seen < 2:
            run_plan(plan, dtype_code, A, a_elems, C, c_elems, alpha, ws=ws, ws_elems=ws_elems,
                     B=B, b_elems=b_elems)
            return
        g = PlanGraph(plan, dtype_code, A, a_elems, C, c_elems, alpha, ws=ws, ws_elems=ws_elems,
                      B=B, b_elems=b_elems)
        _GRAPHS[gkey] = g
        if len(_GRAPHS) > _GRAPHS_MAX:
            _GRAPHS.popitem(last=False)
    else:
        _GRAPHS.move_to_end(gkey)
    g.replay()

