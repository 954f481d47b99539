"""Plan execution: plan cache + one native call per plan (+ optional CUDA graph).

The executor itself is native (``ata_run_plan`` in csrc/abi.cu); this module
keeps plans keyed by shape/layout/threshold so repeated calls skip planning,
and can capture a plan into a ``torch.cuda.CUDAGraph`` for launch-bound
(reference-faithful, small-leaf) plans.
"""
from __future__ import annotations

import ctypes
from collections import OrderedDict

import numpy as np

from . import _native as nat

_PLAN_CACHE: "OrderedDict[tuple, object]" = OrderedDict()
_PLAN_CACHE_MAX = 64


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


def run_plan(plan, dtype_code, A, a_elems, C, c_elems, alpha, ws=None, ws_elems=0, B=None,
             b_elems=0, stream=None):
    """Issue every op of `plan` on `stream` (default: torch's current stream).
    A/B/C/ws are device pointers (ints)."""
    import torch
    lib = nat.load()
    if stream is None:
        stream = int(torch.cuda.current_stream().cuda_stream)
    ops = plan.ops
    if not ops.flags.c_contiguous:
        ops = np.ascontiguousarray(ops)
    rc = lib.ata_run_plan(dtype_code, ops.ctypes.data_as(ctypes.c_void_p), len(ops),
                          A, a_elems, B if B is not None else A, b_elems if B is not None else a_elems,
                          C, c_elems, ws or 0, ws_elems, float(alpha), stream)
    nat.check(rc)
