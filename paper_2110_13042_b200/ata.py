"""Drop-in AtA entry points (reference pkg/src/atamul/ata.py:118-154).

``ata(A, C, alpha, threshold, ws, counter)`` computes the lower triangle
(including the diagonal) of C += alpha * A^T A on the B200; the strict upper
triangle of C is never read or written by any kernel (ata.py:121-123).

``threshold`` keeps the reference's element-count meaning (ata.py:23-26,
strassen.py:38-41) and then reproduces the reference recursion tree exactly
(same leaves, same exact multiplication count), executed breadth first
(ref_bfs.py; ATA_REF_DFS=1 selects the depth-first executor).  ``threshold="auto"`` selects the
GPU plan (auto_plan.plan_ata_auto).  Inputs are torch CUDA tensors (zero copy)
or anything the reference accepts (staged through the device).
"""
from __future__ import annotations

import numpy as np

from . import _native as nat
from . import auto_plan, engine, planner, ref_bfs
from .errors import ShapeMismatchError, UnsupportedSizeError
from .matrix import (DenseMatrix, DeviceOperand, MultCounter, as_array, mirror_lower_to_upper)
from .workspace import (DEFAULT_THRESHOLD, StrassenWorkspace, ata_calls, check_ata_workspace,
                        workspace_for_calls)

AUTO = "auto"


def workspace_for_ata(m: int, n: int, threshold=DEFAULT_THRESHOLD, dtype=np.float64) -> StrassenWorkspace:
    """Workspace covering every Strassen call and leaf of an AtA recursion on an
    m x n input (ata.py:75-81).  For threshold="auto" the auto plan needs no
    scratch and an empty workspace is returned."""
    if threshold == AUTO:
        return StrassenWorkspace([], (1, 1, 1), AUTO, dtype)
    calls, base = ata_calls(m, n, int(threshold))
    return workspace_for_calls(calls, int(threshold), extra_base=base, dtype=dtype)


def _plan_for(m, n, lda, ldc, threshold, ws, auto_params=None, round_tf32=False):
    if threshold == AUTO:
        params = auto_params or auto_plan.AutoParams()
        key = ("ata-auto", m, n, lda, ldc, params, round_tf32)
        return engine.cached_plan(
            key, lambda: auto_plan.plan_ata_auto(m, n, lda, ldc, params, round_tf32=round_tf32))
    if engine.reference_dfs():
        offs = tuple(ws.level_offsets())
        key = ("ata-ref", m, n, lda, ldc, int(threshold), offs)
        return engine.cached_plan(
            key, lambda: planner.plan_ata_reference(m, n, lda, ldc, int(threshold), list(offs)))
    # the reference recursion tree, executed breadth first (ref_bfs.py)
    key = ("ata-ref-bfs", m, n, lda, ldc, int(threshold))
    return engine.cached_plan(key, lambda: ref_bfs.plan_ata_reference_bfs(m, n, lda, ldc, int(threshold)))


def ata(A, C, alpha=1.0, threshold=DEFAULT_THRESHOLD, ws: StrassenWorkspace | None = None,
        counter: MultCounter | None = None, *, auto_params=None, precision: str = "fp32") -> None:
    """Lower triangle of C += alpha * A^T A for A (m x n), C (n x n).

    ``precision`` only matters for f32: "fp32" (3xTF32 products, fp32-level
    accuracy like the reference's f32 einsum) or "tf32" (single-pass TF32)."""
    a, c = as_array(A), as_array(C)
    m, n = int(a.shape[0]), int(a.shape[1])
    if tuple(c.shape) != (n, n):
        raise ShapeMismatchError(f"shape mismatch: C {tuple(c.shape)} != {(n, n)}")
    if threshold != AUTO:
        threshold = int(threshold)
        if threshold < 1:
            raise ShapeMismatchError("shape mismatch: threshold must be >= 1")
    C_ = DeviceOperand(c, writable=True, lower=True)   # kernels touch only lower(C)
    A_ = DeviceOperand(a, dtype=C_.t.dtype, device=C_.t.device)
    if ws is None:
        ws = workspace_for_ata(m, n, threshold, dtype=C_.t.dtype)
    elif threshold != AUTO:
        check_ata_workspace(ws, m, n, threshold)
    import torch
    plan = _plan_for(m, n, A_.ld, C_.ld, threshold, ws, auto_params,
                     round_tf32=(precision == "tf32" and C_.t.dtype == torch.float32))
    extra = plan.ws_scalars if (threshold == AUTO or not engine.reference_dfs()) else 0
    wbuf = ws.ensure(C_.t.device, extra=extra) if plan.ws_scalars > 0 else None
    engine.run_plan(plan, nat.dtype_code(C_.t.dtype, precision), A_.ptr, A_.elems, C_.ptr, C_.elems, alpha,
                    ws=int(wbuf.data_ptr()) if wbuf is not None else 0,
                    ws_elems=int(wbuf.numel()) if wbuf is not None else 0)
    C_.commit()
    if counter is not None:
        counter.add(plan.mults)


def ata_full(A, threshold=DEFAULT_THRESHOLD, counter: MultCounter | None = None) -> DenseMatrix:
    """Full symmetric A^T A as a fresh matrix: recursion, then mirror
    (ata.py:136-145).  Host input -> host result; device input -> device."""
    import torch
    a = as_array(A)
    n = int(a.shape[1])
    if isinstance(a, torch.Tensor) and a.is_cuda:
        out = torch.zeros((n, n), dtype=a.dtype if a.dtype in (torch.float32, torch.float64)
                          else torch.float64, device=a.device)
        ata(a, out, 1.0, threshold, None, counter)
        mirror_lower_to_upper(out)
        return DenseMatrix(out)
    dt = a.dtype if getattr(a, "dtype", None) in (np.float32, np.float64) else np.float64
    host = np.asarray(a.cpu().numpy() if isinstance(a, torch.Tensor) else a)
    dev_a = torch.from_numpy(np.ascontiguousarray(host, dtype=dt)).cuda()
    out = torch.zeros((n, n), dtype=dev_a.dtype, device=dev_a.device)
    ata(dev_a, out, 1.0, threshold, None, counter)
    mirror_lower_to_upper(out)
    return DenseMatrix(out.cpu().numpy())


def ata_mult_count(n: int) -> int:
    """(2*7**j + 4**j) / 3 for n = 2**j (ata.py:148-154)."""
    if n < 1 or n & (n - 1):
        raise UnsupportedSizeError(f"unsupported size: {n} is not a power of two")
    j = n.bit_length() - 1
    return (2 * 7 ** j + 4 ** j) // 3
