"""Leaf-task execution for the parallel executors (reference execute.py:1-83).

A leaf task of a task tree (``tasktree.Task``) names absolute regions of the
global operand A and of the global result C.  ``execute_leaf`` runs it with the
single-GPU entry points -- ``fast_strassen`` for an AtB task, ``ata`` for the
diagonal part of an AtA task -- so the recursion, the leaf kernels and the
exact multiplication counts are the ones of the sequential path.  Operands
are views of ``a_global`` / ``c_global`` (torch CUDA tensors: zero copy;
host arrays: staged through the device and written back in place, exactly
like a direct ``ata`` call on those views).

AtA tasks of the shared tree are *stripes* (scheduler.py:365-405): their C
region is rows [s, e) of the Gram of the column prefix A[:, :e], i.e. a
rectangle left of the diagonal block (an AtB of A[:, s:e] against A[:, :s])
plus the diagonal block's lower triangle (an AtA of A[:, s:e]).  A plain AtA
task is the special case s == col_offset (no rectangle).
"""
from __future__ import annotations

import numpy as np

from .errors import ShapeMismatchError
from .tasktree import ComputationType, Region, Task
from .workspace import StrassenWorkspace, ata_calls, workspace_for_calls

LEAF_KERNELS = ("fast", "naive")


def _view(x, r: Region):
    return x[r.row_offset:r.row_offset + r.rows, r.col_offset:r.col_offset + r.cols]


def stripe_split(task: Task) -> int:
    """Width of the rectangle left of a stripe task's diagonal block
    (execute.py:23-27): C region columns minus rows; 0 for square AtA tasks."""
    return task.c_region.cols - task.c_region.rows


def workspace_for_leaf(task: Task, threshold, dtype=np.float64) -> StrassenWorkspace:
    """One workspace covering every call the leaf runs (execute.py:30-41):
    the AtB task's Strassen call, or the stripe's AtA recursion plus its
    rectangle's Strassen call.  threshold="auto": the GPU plans size their own
    scratch, an empty workspace is returned."""
    from .ata import AUTO, workspace_for_ata
    from .strassen import workspace_for
    a = task.a_region
    if threshold == AUTO:
        return workspace_for_ata(1, 1, AUTO, dtype=dtype)
    threshold = int(threshold)
    if task.computation is ComputationType.ATB:
        return workspace_for(a.rows, a.cols, task.b_region.cols, threshold, dtype=dtype)
    split = stripe_split(task)
    width = a.cols - split
    calls, base = ata_calls(a.rows, width, threshold)
    if split > 0:
        calls = list(calls) + [(a.rows, width, split)]
    return workspace_for_calls(calls, threshold, extra_base=base, dtype=dtype)


def execute_leaf(task: Task, a_global, c_global, threshold, counter=None, kernel: str = "fast",
                 ws: StrassenWorkspace | None = None, **kw) -> None:
    """Accumulate one leaf task into c_global (execute.py:44-83).

    kernel "fast": the recursive entry points (``ata`` / ``fast_strassen``,
    a workspace is built when none is passed); "naive": the classical
    single-kernel leaves (``naive_syrk_lower`` / ``naive_gemm_atb``).  Extra
    keyword arguments (``precision``, ``auto_params``) reach ``ata``."""
    run_leaf(task, lambda r: _view(a_global, r), _view(c_global, task.c_region), threshold, counter,
             kernel, ws, **kw)


def run_leaf(task: Task, get_block, c, threshold, counter=None, kernel: str = "fast",
             ws: StrassenWorkspace | None = None, **kw) -> None:
    """execute_leaf on explicit blocks: ``get_block(Region)`` serves operand
    views in global coordinates (a process of the distributed executor holds
    only the blocks it received), ``c`` is the task's C block."""
    from .ata import ata
    from .matrix import naive_gemm_atb, naive_syrk_lower
    from .strassen import fast_strassen
    if kernel not in LEAF_KERNELS:
        raise ValueError(f"unknown leaf kernel {kernel!r}")
    gemm_kw = {"auto_params": kw["auto_params"]} if "auto_params" in kw else {}
    if task.computation is ComputationType.ATB:
        if task.b_region is None:
            raise ShapeMismatchError("shape mismatch: AtB task without a B region")
        a, b = get_block(task.a_region), get_block(task.b_region)
        if kernel == "naive":
            naive_gemm_atb(a, b, c, 1.0, counter)
        else:
            fast_strassen(a, b, c, 1.0, ws, threshold, counter, **gemm_kw)
        return
    prefix = get_block(task.a_region)
    split = stripe_split(task)
    diag_cols = prefix[:, split:]
    if split > 0:
        if kernel == "naive":
            naive_gemm_atb(diag_cols, prefix[:, :split], c[:, :split], 1.0, counter)
        else:
            if ws is None:
                ws = workspace_for_leaf(task, threshold, dtype=getattr(c, "dtype", np.float64))
            fast_strassen(diag_cols, prefix[:, :split], c[:, :split], 1.0, ws, threshold, counter,
                          **gemm_kw)
    diag = c[:, split:]
    if kernel == "naive":
        naive_syrk_lower(diag_cols, diag, 1.0, counter)
        return
    if ws is None:
        ws = workspace_for_leaf(task, threshold, dtype=getattr(c, "dtype", np.float64))
    ata(diag_cols, diag, 1.0, threshold, ws, counter, **kw)
