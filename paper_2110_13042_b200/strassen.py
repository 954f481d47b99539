"""Drop-in Strassen entry points (reference pkg/src/atamul/strassen.py:187-307).

``fast_strassen(A, B, C, alpha, ws, threshold, counter)`` computes
C += alpha * A^T B through the reference's Strassen recursion on the GPU
(planner.plan_strassen_reference): same products, same odd-size semantics,
same per-depth workspace, alpha applied only where leaf products accumulate
(so scaling is exactly linear, strassen.py:284-285).
"""
from __future__ import annotations

import numpy as np

from . import ref_bfs, _native as nat
from . import engine, planner
from .errors import ShapeMismatchError, UnsupportedSizeError, WorkspaceUndersizedError
from .matrix import DeviceOperand, MultCounter, as_array
from .workspace import (DEFAULT_THRESHOLD, StrassenWorkspace, is_base_case,  # noqa: F401
                        workspace_for_calls)


def workspace_for(m: int, n: int, k: int, threshold: int = DEFAULT_THRESHOLD,
                  dtype=np.float64) -> StrassenWorkspace:
    """Workspace for one fast_strassen call on A (m x n), B (m x k) (strassen.py:187-192)."""
    if min(m, n, k) < 1 or threshold < 1:
        raise ShapeMismatchError("shape mismatch: dimensions must be >= 1")
    return workspace_for_calls([(m, n, k)], threshold, dtype=dtype)


def fast_strassen(A, B, C, alpha=1.0, ws: StrassenWorkspace | None = None,
                  threshold: int = DEFAULT_THRESHOLD, counter: MultCounter | None = None, *,
                  auto_params=None) -> None:
    """C += alpha * A^T B with A (m x n), B (m x k), C (n x k).  threshold
    "auto": the GPU plan (auto_plan.plan_gemm_auto) instead of the reference
    recursion."""
    a, b, c = as_array(A), as_array(B), as_array(C)
    m, n = int(a.shape[0]), int(a.shape[1])
    if b.shape[0] != m:
        raise ShapeMismatchError(f"shape mismatch: A {tuple(a.shape)} vs B {tuple(b.shape)}")
    k = int(b.shape[1])
    if tuple(c.shape) != (n, k):
        raise ShapeMismatchError(f"shape mismatch: C {tuple(c.shape)} != {(n, k)}")
    C_ = DeviceOperand(c, writable=True)
    from .ata import even_pitch
    A_ = even_pitch(DeviceOperand(a, dtype=C_.t.dtype, device=C_.t.device), slot=0)
    B_ = even_pitch(DeviceOperand(b, dtype=C_.t.dtype, device=C_.t.device), slot=1)
    if threshold == "auto":
        _fast_strassen_auto(A_, B_, C_, m, n, k, alpha, counter, auto_params, ws)
        return
    threshold = int(threshold)
    if ws is None:
        ws = workspace_for(m, n, k, threshold, dtype=C_.t.dtype)
    elif not ws.covers(m, n, k, threshold):
        raise WorkspaceUndersizedError(
            f"workspace undersized for ({m},{n},{k}) at threshold {threshold}")
    if engine.reference_dfs():
        offs = tuple(ws.level_offsets())
        key = ("strassen-ref", m, n, k, A_.ld, B_.ld, C_.ld, threshold, offs)
        plan = engine.cached_plan(key, lambda: planner.plan_strassen_reference(
            m, n, k, A_.ld, B_.ld, C_.ld, threshold, list(offs)))
        extra = 0
    else:   # same recursion tree, executed breadth first (ref_bfs.py)
        key = ("strassen-ref-bfs", m, n, k, A_.ld, B_.ld, C_.ld, threshold)
        plan = engine.cached_plan(key, lambda: ref_bfs.plan_strassen_reference_bfs(
            m, n, k, A_.ld, B_.ld, C_.ld, threshold))
        extra = plan.ws_scalars
    wbuf = ws.ensure(C_.t.device, extra=extra, dtype=C_.t.dtype) if plan.ws_scalars > 0 else None
    args = (plan, nat.dtype_code(C_.t.dtype), A_.ptr, A_.elems, C_.ptr, C_.elems, alpha)
    kw = dict(ws=int(wbuf.data_ptr()) if wbuf is not None else 0,
              ws_elems=int(wbuf.numel()) if wbuf is not None else 0, B=B_.ptr, b_elems=B_.elems)
    if engine.reference_dfs():
        engine.run_plan(*args, **kw)
    else:   # launch-bound breadth-first plan: graph replay on repeat calls
        engine.run_plan_graphed(key, *args, **kw)
    C_.commit()
    if counter is not None:
        counter.add(plan.mults)


def _fast_strassen_auto(A_, B_, C_, m, n, k, alpha, counter, auto_params, ws=None):
    """threshold="auto": the GPU plan; scratch from `ws` (a StrassenWorkspace,
    e.g. one per concurrent stream) or a per-(device, dtype) arena."""
    from . import auto_plan
    params = auto_params or auto_plan.AutoParams()
    key = ("gemm-auto", m, n, k, A_.ld, B_.ld, C_.ld, params)
    plan = engine.cached_plan(key, lambda: auto_plan.plan_gemm_auto(m, n, k, A_.ld, B_.ld, C_.ld, params))
    wbuf = None
    if plan.ws_scalars > 0 and ws is not None:
        wbuf = ws.ensure(C_.t.device, extra=plan.ws_scalars, dtype=C_.t.dtype)
    elif plan.ws_scalars > 0:
        wbuf = _AUTO_WS.get((str(C_.t.device), str(C_.t.dtype)))
        if wbuf is None or wbuf.numel() < plan.ws_scalars:
            import torch
            wbuf = torch.empty(plan.ws_scalars, dtype=C_.t.dtype, device=C_.t.device)
            _AUTO_WS[(str(C_.t.device), str(C_.t.dtype))] = wbuf
    engine.run_plan(plan, nat.dtype_code(C_.t.dtype), A_.ptr, A_.elems, C_.ptr, C_.elems, alpha,
                    ws=int(wbuf.data_ptr()) if wbuf is not None else 0,
                    ws_elems=int(wbuf.numel()) if wbuf is not None else 0, B=B_.ptr, b_elems=B_.elems)
    C_.commit()
    if counter is not None:
        counter.add(plan.mults)


_AUTO_WS: dict = {}   # scratch of auto GEMM plans, one per (device, dtype), grown on demand


def strassen_mult_count(n: int) -> int:
    """7**log2(n) (strassen.py:302-307)."""
    if n < 1 or n & (n - 1):
        raise UnsupportedSizeError(f"unsupported size: {n} is not a power of two")
    return 7 ** (n.bit_length() - 1)
