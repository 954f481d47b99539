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

import dataclasses
import os

import numpy as np

from . import _native as nat
from . import auto_plan, engine, planner, ref_bfs
from .errors import ShapeMismatchError, UnsupportedSizeError
from .matrix import (DenseMatrix, DeviceOperand, MultCounter, _copy_lower, as_array,
                     mirror_lower_to_upper)
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
    accuracy like the reference's f32 einsum) or "tf32" (single-pass TF32).
    ``auto_params`` (threshold "auto"): AutoParams, or "tune" to measure the
    leaf-product and addition rates and pick the leaf width on this device
    (autotune.py; the first call per shape pays the measurement)."""
    a, c = as_array(A), as_array(C)
    m, n = int(a.shape[0]), int(a.shape[1])
    if tuple(c.shape) != (n, n):
        raise ShapeMismatchError(f"shape mismatch: C {tuple(c.shape)} != {(n, n)}")
    if threshold != AUTO:
        threshold = int(threshold)
        if threshold < 1:
            raise ShapeMismatchError("shape mismatch: threshold must be >= 1")
    if threshold == AUTO and isinstance(auto_params, str):
        if auto_params != "tune":
            raise ValueError(f"auto_params must be AutoParams, None or 'tune', not {auto_params!r}")
        auto_params = _tuned_params(a, c, m, n)
    if threshold == AUTO:
        es = 4 if str(getattr(c, "dtype", "")).endswith("float32") else 8
        auto_params = fit_workspace_budget(auto_params or auto_plan.AutoParams(),
                                           resident_bytes=(m * n + 2 * n * n) * es)
    if threshold == AUTO and _pipelined_host_ata(a, c, m, n, alpha, ws, counter, auto_params, precision):
        return
    if threshold != AUTO and _pipelined_host_ref(a, c, m, n, threshold, alpha, ws, counter):
        return
    C_ = DeviceOperand(c, writable=True, lower=True)   # kernels touch only lower(C)
    A_ = even_pitch(DeviceOperand(a, dtype=C_.t.dtype, device=C_.t.device))
    if ws is None:
        ws = _default_workspace(m, n, threshold, C_.t.dtype)
    elif threshold != AUTO:
        check_ata_workspace(ws, m, n, threshold)
    import torch
    plan = _plan_for(m, n, A_.ld, C_.ld, threshold, ws, auto_params,
                     round_tf32=(precision == "tf32" and C_.t.dtype == torch.float32))
    extra = plan.ws_scalars if (threshold == AUTO or not engine.reference_dfs()) else 0
    wbuf = ws.ensure(C_.t.device, extra=extra, dtype=C_.t.dtype) if plan.ws_scalars > 0 else None
    args = (plan, nat.dtype_code(C_.t.dtype, precision), A_.ptr, A_.elems, C_.ptr, C_.elems, alpha)
    kw = dict(ws=int(wbuf.data_ptr()) if wbuf is not None else 0,
              ws_elems=int(wbuf.numel()) if wbuf is not None else 0)
    if threshold != AUTO and not engine.reference_dfs():
        # launch-bound breadth-first reference plans: replay a CUDA graph on repeat calls
        engine.run_plan_graphed(("ata-ref-bfs", m, n, A_.ld, C_.ld, threshold), *args, **kw)
    else:
        engine.run_plan(*args, **kw)
    C_.commit()
    if counter is not None:
        counter.add(plan.mults)


_WS_CACHE: dict = {}
_PITCH_CACHE: dict = {}
EVEN_PITCH_MIN_ELEMS = 1 << 20


def even_pitch(op, slot: int = 0):
    """An fp64 device operand with an odd row pitch, re-laid out with an even
    one (one device copy, into a buffer kept per shape so repeated calls --
    and captured graphs -- see the same pointer): the TMA-fed FP64 leaf kernel
    needs 16-byte row pitches (config c2's 4097 columns).  Small operands, f32
    and even pitches pass through."""
    import torch
    t = op.t
    if t.dtype != torch.float64 or op.ld % 2 == 0 or op.rows < 2 or op.rows * op.cols < EVEN_PITCH_MIN_ELEMS:
        return op
    if os.environ.get("ATA_F64_TMA", "1") == "0":
        return op
    ld = op.cols + (op.cols & 1)
    key = (str(t.device), op.rows, ld, slot)   # slot: distinct buffers for the operands of one call
    buf = _PITCH_CACHE.get(key)
    if buf is None:
        if len(_PITCH_CACHE) >= 4:
            _PITCH_CACHE.pop(next(iter(_PITCH_CACHE)))
        buf = _PITCH_CACHE[key] = torch.empty((op.rows, ld), dtype=t.dtype, device=t.device)
    view = buf[:, :op.cols]
    view.copy_(t)
    op.t, op.ld = view, ld
    op.keep = buf
    return op


def fit_workspace_budget(params, device=None, headroom: float = 0.8, resident_bytes: int = 0):
    """AutoParams whose breadth-first workspace budget (default 40 GB) fits the
    HBM this process can still get: free device memory plus what torch's
    caching allocator holds unused, times `headroom`.  Unchanged (same plans,
    same cache keys) whenever the default budget fits -- e.g. c4 on a 180 GB
    B200 -- and a smaller budget (depth-first Strassen subtrees, less scratch)
    when the device is shared or nearly full.  The second scratch arena of
    riding plans (AutoParams.ride_arenas, up to twice the workspace) is kept
    only when the operands (`resident_bytes`) plus that workspace fit the
    device's TOTAL memory -- a figure that does not move between calls, so
    repeated calls plan alike while their buffers are alive."""
    import dataclasses
    import torch
    if not torch.cuda.is_available():
        return params
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    free, total = torch.cuda.mem_get_info(dev)
    avail = free + torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev)
    cap_gb = avail * headroom / 1e9
    if cap_gb < params.ws_budget_gb:
        return dataclasses.replace(params, ws_budget_gb=max(0.5, round(cap_gb, 1)), ride_arenas=False)
    if params.ride_arenas and resident_bytes + 2.2e9 * params.ws_budget_gb > headroom * total:
        return dataclasses.replace(params, ride_arenas=False)
    return params


def _tuned_params(a, c, m, n):
    """auto_params="tune": rates and SYRK leaf width measured on the device
    that runs the plan (autotune.tune, cached per shape); fp64 only -- other
    dtypes keep the default parameters."""
    import torch
    from . import autotune
    dt = getattr(c, "dtype", None)
    if dt not in (torch.float64, np.float64):
        return None
    dev = c.device if isinstance(c, torch.Tensor) and c.is_cuda else None
    return autotune.tune(m, n, dev)


def release_cached_buffers() -> None:
    """Drop the device buffers ata() keeps between calls (the two most recent
    per-shape workspace arenas, the host pipeline's staged C, even-pitch operand
    copies) and return torch's unused cached blocks to the device -- e.g. after a
    c4-sized call (110 GB of workspace) when other work needs the HBM."""
    _WS_CACHE.clear()
    _PIPE_CIN.clear()
    _PITCH_CACHE.clear()
    try:
        import torch
        if torch.cuda.is_available():
            torch.cuda.empty_cache()
    except ImportError:      # pragma: no cover
        pass


def _default_workspace(m, n, threshold, dtype):
    """ws=None: one arena per (shape, threshold, dtype), kept for the next call
    (the two most recent) -- repeated calls allocate nothing and keep their
    pointers, which lets launch-bound plans replay a captured graph."""
    key = (m, n, threshold, str(dtype))
    ws = _WS_CACHE.pop(key, None)
    if ws is None:
        ws = workspace_for_ata(m, n, threshold, dtype=dtype)
    _WS_CACHE[key] = ws
    while len(_WS_CACHE) > 2:
        _WS_CACHE.pop(next(iter(_WS_CACHE)))
    return ws


PIPELINE_MIN_BYTES = 1 << 30      # host A at least this large: copy/compute pipeline
PIPELINE_BLOCK_BYTES = 4 << 30    # ~ bytes of A per row block (PCIe-bound TF32 plans)
PIPELINE_GEOMETRIC = True         # compute-bound plans: geometric row blocks (_row_blocks)
PIPELINE_ZERO_C = bool(int(os.environ.get("ATA_PIPE_ZERO_C", "1")))   # device C starts at zero (_pipelined_host_ata)
# zero-start C: add the caller's C tile group by tile group right before each
# group's download (its upload then overlaps the last block's compute) instead
# of one whole-square add before the last block
PIPELINE_LATE_C_ADD = bool(int(os.environ.get("ATA_PIPE_LATE_C_ADD", "1")))
_PIPE_CIN: dict = {}   # the staged host-C buffer of the pipeline, one per (device, n, dtype)
PIPE_TRACE = None      # a list: the pipeline appends (label, stream, event) marks (tools/e2e_timeline.py)


def _mark(label, stream):
    if PIPE_TRACE is not None:
        import torch
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        PIPE_TRACE.append((label, ev))
PIPELINE_GEOMETRIC_MIN_RATIO = 1.5    # geometric blocks from this compute / upload ratio (c3: 1.9, c4: 3.8)
PIPELINE_GEOMETRIC_BLOCKS = 3     # (4 blocks: no gain, each block repeats the plan's C-sized work)
PIPELINE_GEOMETRIC_GROWTH = 2.5   # rows of block i+1 / rows of block i (_row_blocks)
PIPELINE_PCIE_GBS = 50.0          # measured pinned H2D on the box (e2e h2d bytes / time)
PIPELINE_FP64_TFLOPS = 54.0       # effective AtA rate of the fp64 auto plans (bench c4)
PIPELINE_TF32_TFLOPS = 460.0


def _first_c_writer(ops) -> int:
    """Index of the first op with a destination in C (ops before it only touch A / scratch)."""
    d = ops["d"]
    hits = np.nonzero(((d["base"] == nat.BASE_C) & (d["rows"] > 0)).any(axis=1))[0]
    return int(hits[0]) if len(hits) else len(ops)


_TILES = 64   # at most this many C download tiles per side ...
_TILE_MIN = 512   # ... of at least this many rows (each tile row is one 2-D copy: a 65-row tile of
                  # config c2 moved 30 KB per call and the calls' fixed cost dominated its e2e time)


def _dl_step(n: int) -> int:
    """Rows per C tile of the pipelines (uploads by _copy_lower and the early
    downloads use the same row bands: a diagonal tile goes home as a whole square
    whose upper part holds what the upload put there)."""
    return max(1, -(-n // _TILES), min(n, _TILE_MIN))


def _download_schedule(plan, n, remaining: bool = False, parts: int = 6):
    """C tiles (block row, block col) of the lower triangle grouped by the op
    after which their last writer in `plan` has run: [(cut, tiles)] with cut <
    len(plan.ops), a few groups of similar size.  remaining=True: the tiles
    written by the plan's last group of ops (or never written)."""
    cache = plan.__dict__.setdefault("_dl", {})
    if n not in cache:
        step = _dl_step(n)
        nb = -(-n // step)
        last = np.full((nb, nb), -1, dtype=np.int64)
        d = plan.ops["d"]
        ii, jj = np.nonzero((d["base"] == nat.BASE_C) & (d["rows"] > 0) & (d["cols"] > 0))
        for i, j in zip(ii.tolist(), jj.tolist()):
            w = d[i, j]
            r0, c0 = divmod(int(w["off"]), int(w["ld"]))
            r1, c1 = r0 + int(w["rows"]), c0 + int(w["cols"])
            last[r0 // step:(r1 - 1) // step + 1, c0 // step:(c1 - 1) // step + 1] = i
        low = [(bi, bj) for bi in range(nb) for bj in range(bi + 1)]
        order = sorted((int(last[t]), t) for t in low if last[t] >= 0)
        groups, cur, target = [], [], len(order) / parts
        for k, (li, t) in enumerate(order):
            cur.append(t)
            if (k + 1 == len(order) or order[k + 1][0] != li) and len(cur) >= target:
                groups.append((li + 1, cur))
                cur = []
        if cur:
            groups.append((order[-1][0] + 1, cur))
        n_ops = len(plan.ops)
        early = [(cut, ts) for (cut, ts) in groups if cut < n_ops]
        rest = [t for (cut, ts) in groups if cut >= n_ops for t in ts] + [t for t in low if last[t] < 0]
        cache[n] = (early, rest, step)
    early, rest, step = cache[n]
    if remaining:
        return [(bi, bj, step) for (bi, bj) in rest]
    return [(cut, [(bi, bj, step) for (bi, bj) in tiles]) for (cut, tiles) in early]


def _copy_tiles(host, dev, tiles):
    """D2H of C tiles (block row, block col, step) on the current stream; runs
    of adjacent tiles in one block row are one 2D copy.  Diagonal tiles are
    whole squares: their upper part holds the values uploaded by _copy_lower."""
    from .matrix import _cudart, _stream_ptr
    lib = _cudart()
    stream = _stream_ptr()
    n = int(dev.shape[0])
    es = dev.element_size()
    rows = {}
    for (bi, bj, step) in tiles:
        rows.setdefault((bi, step), []).append(bj)
    for (bi, step), cols in rows.items():
        cols.sort()
        r0, r1 = bi * step, min(n, (bi + 1) * step)
        k = 0
        while k < len(cols):
            j0 = cols[k]
            while k + 1 < len(cols) and cols[k + 1] == cols[k] + 1:
                k += 1
            c0, c1 = j0 * step, min(n, (cols[k] + 1) * step)
            k += 1
            d = host.data_ptr() + (r0 * host.stride(0) + c0) * es
            s = dev.data_ptr() + (r0 * dev.stride(0) + c0) * es
            rc = lib.cudaMemcpy2DAsync(d, host.stride(0) * es, s, dev.stride(0) * es, (c1 - c0) * es, r1 - r0,
                                       2, stream)
            if rc != 0:
                raise RuntimeError(f"cudaMemcpy2DAsync failed ({rc})")


class _SubPlan:
    def __init__(self, ops):
        self.ops = np.ascontiguousarray(ops)


def _pipelined_host_ata(a, c, m, n, alpha, ws, counter, auto_params, precision) -> bool:
    """Host A and C (pinned torch tensors): A^T A = sum over row blocks A_r^T A_r,
    so A crosses PCIe in R row blocks on a copy stream while the GPU runs the
    auto plan of the blocks already resident; C's lower block-trapezoids are
    uploaded behind the first block and awaited only by the first op that
    writes C.  Returns False (caller takes the plain path) when not applicable."""
    import torch
    if not (isinstance(a, torch.Tensor) and isinstance(c, torch.Tensor)) or a.is_cuda or c.is_cuda:
        return False
    if a.dtype != c.dtype or a.dtype not in (torch.float32, torch.float64):
        return False
    if not (a.is_contiguous() and c.is_contiguous() and a.is_pinned() and c.is_pinned()):
        return False
    es = a.element_size()
    if m * n * es < PIPELINE_MIN_BYTES or m < 2:
        return False
    dev = torch.device("cuda", torch.cuda.current_device())
    main = torch.cuda.current_stream(dev)
    copy = _copy_stream(dev)
    dA = torch.empty((m, n), dtype=a.dtype, device=dev)
    dC = torch.empty((n, n), dtype=c.dtype, device=dev)
    code = nat.dtype_code(c.dtype, precision)
    round_tf32 = precision == "tf32" and c.dtype == torch.float32
    params = auto_params or auto_plan.AutoParams()
    blocks = []
    rb = _row_blocks(m, n, es, round_tf32 or es == 4)
    if not (PIPELINE_ZERO_C and len(rb) >= 3 and rb[0][1] * 2 < rb[1][1]) and params.diag_first:
        # C is uploaded behind block 0 and awaited by its first C writer: keep the
        # diagonal SYRK leaves (C writers) out of the front of the plan
        params = dataclasses.replace(params, diag_first=False)
    for (r0, rows) in rb:
        # each block's plan takes the Strassen tree of the whole A (cost model at m
        # rows): the blocks together execute the single plan's multiplications
        bp = dataclasses.replace(params, cost_row_scale=params.cost_row_scale * m / rows)
        key = ("ata-auto", rows, n, n, n, bp, round_tf32)
        blocks.append((r0, rows, engine.cached_plan(
            key, lambda rows=rows, bp=bp: auto_plan.plan_ata_auto(rows, n, n, n, bp, round_tf32=round_tf32))))
    need = max(p.ws_scalars for (_, _, p) in blocks)
    if ws is None:
        # the cached arena of this shape (shared with the device-operand path: one
        # workspace per shape, grown to the larger of the two plans' needs)
        ws = _default_workspace(m, n, AUTO, c.dtype)
    wbuf = ws.ensure(dev, extra=need, dtype=c.dtype) if need > 0 else None
    wptr = int(wbuf.data_ptr()) if wbuf is not None else 0
    wel = int(wbuf.numel()) if wbuf is not None else 0
    # zero-start C pays one extra add pass but lets block 0 run without C; it
    # wins with the small first block of geometric row blocks (c4: 1680 -> 1642
    # ms e2e), not with two equal blocks (c3: 138.1 vs 139.2 ms)
    zero_start = PIPELINE_ZERO_C and len(blocks) >= 3 and blocks[0][1] * 2 < blocks[1][1]
    events = []
    c_ready = torch.cuda.Event()
    if zero_start:
        # C starts at zero on the device, so no block waits for C's upload; the
        # host C's lower trapezoids cross PCIe after all of A into a zeroed
        # buffer and are added in (whole square: the diagonal tiles' upper parts
        # come back as uploaded) just before the last block
        dC.zero_()
        key = (str(dev), n, str(c.dtype))
        dCin = _PIPE_CIN.get(key)
        if dCin is None:
            _PIPE_CIN.clear()
            dCin = _PIPE_CIN[key] = torch.empty((n, n), dtype=c.dtype, device=dev)
        dCin.zero_()
    # dA / dC / scratch are free to overwrite, and the zero fills above are
    # ordered before the copy stream's uploads into dCin
    copy.wait_stream(main)
    with torch.cuda.stream(copy):
        for i, (r0, rows, _) in enumerate(blocks):
            dA[r0:r0 + rows].copy_(a[r0:r0 + rows], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy)
            events.append(ev)
            _mark(f"A block {i} uploaded", copy)
            if i == 0 and not zero_start:
                _copy_lower(dC, c, to_device=True, step=_dl_step(n))
                c_ready.record(copy)
        if zero_start:
            _copy_lower(dCin, c, to_device=True, step=_dl_step(n))
            c_ready.record(copy)
            _mark("C uploaded", copy)
    mults = 0
    last = len(blocks) - 1
    _mark("start", main)
    for i, (r0, rows, plan) in enumerate(blocks):
        main.wait_event(events[i])
        _mark(f"block {i} starts", main)
        ops = plan.ops
        A_ptr = int(dA.data_ptr()) + r0 * n * es
        # segment boundaries: the first C writer of block 0 waits for C's upload
        # (unless C starts at zero); in the last block, C tiles whose last writer
        # has run go home early
        cuts, downloads = [], {}
        if i == 0 and not zero_start:
            cuts.append(_first_c_writer(ops))
        if i == last:
            if zero_start and not PIPELINE_LATE_C_ADD:
                main.wait_event(c_ready)
                engine.run_plan(_add_plan(n), code, int(dCin.data_ptr()), dCin.numel(), int(dC.data_ptr()),
                                dC.numel(), 1.0)
            sched = _download_schedule(plan, n)
            for cut, tiles in sched:
                cuts.append(cut)
                downloads[cut] = tiles
        prev = 0
        for cut in sorted(set(cuts)) + [len(ops)]:
            if cut > prev:
                engine.run_plan(_SubPlan(ops[prev:cut]), code, A_ptr, rows * n, int(dC.data_ptr()), dC.numel(),
                                alpha, ws=wptr, ws_elems=wel)
                prev = cut
            if i == 0 and not zero_start and cut == cuts[0]:
                main.wait_event(c_ready)
            if cut in downloads:
                if zero_start and PIPELINE_LATE_C_ADD:
                    # the caller's C joins these final tiles just before they go home
                    # (its upload ran behind the last block's compute, not before it)
                    main.wait_event(c_ready)
                    engine.run_plan(_add_tiles_plan(n, downloads[cut]), code, int(dCin.data_ptr()), dCin.numel(),
                                    int(dC.data_ptr()), dC.numel(), 1.0)
                ev = torch.cuda.Event()
                ev.record(main)
                copy.wait_event(ev)
                with torch.cuda.stream(copy):
                    _copy_tiles(c, dC, downloads[cut])
                    _mark(f"download group at op {cut} done ({len(downloads[cut])} tiles)", copy)
        mults += plan.mults
    main.wait_event(c_ready)               # (a plan with no C writer: download after the upload)
    rest = _download_schedule(blocks[last][2], n, remaining=True)
    if zero_start and PIPELINE_LATE_C_ADD:
        engine.run_plan(_add_tiles_plan(n, rest), code, int(dCin.data_ptr()), dCin.numel(), int(dC.data_ptr()),
                        dC.numel(), 1.0)
    _mark("last block done", main)
    _copy_tiles(c, dC, rest)
    _mark(f"remaining {len(rest)} tiles downloaded", main)
    main.wait_stream(copy)                 # the early downloads
    main.synchronize()
    if counter is not None:
        counter.add(mults)
    return True


PIPELINE_REF_MIN_BYTES = 64 << 20    # integer-threshold pipeline: host A at least this large
_PIPE_BUFS: dict = {}


def _pipe_buffer(dev, shape, tag):
    import torch
    key = (str(dev), tuple(shape), tag)
    buf = _PIPE_BUFS.get(key)
    if buf is None:
        for k in [k for k in _PIPE_BUFS if k[2] == tag]:
            _PIPE_BUFS.pop(k)
        buf = _PIPE_BUFS[key] = torch.empty(shape, dtype=torch.float64, device=dev)
    return buf


def _pipelined_host_ref(a, c, m, n, threshold, alpha, ws, counter) -> bool:
    """Integer-threshold plans (the reference recursion tree, breadth first)
    on pinned host fp64 A and C: A crosses PCIe first (straight into an
    even-pitch device buffer), C's lower block-trapezoids follow on the copy
    stream while the plan's operand-sum phase runs (the first op that writes C
    waits for them), and C tiles go home as soon as their last writer has run.
    The plan runs as a few CUDA-graph segments split at those points.  Returns
    False when not applicable (the caller stages A and C itself)."""
    import torch
    if engine.reference_dfs() or os.environ.get("ATA_PIPE_REF", "0") != "1":
        return False
    if not (isinstance(a, torch.Tensor) and isinstance(c, torch.Tensor)) or a.is_cuda or c.is_cuda:
        return False
    if a.dtype != torch.float64 or c.dtype != torch.float64 or m < 2:
        return False
    if not (a.is_contiguous() and c.is_contiguous() and a.is_pinned() and c.is_pinned()):
        return False
    if m * n * 8 < PIPELINE_REF_MIN_BYTES:
        return False
    from .matrix import _cudart, _stream_ptr
    dev = torch.device("cuda", torch.cuda.current_device())
    main = torch.cuda.current_stream(dev)
    copy = _copy_stream(dev)
    ld = n + (n & 1)
    dA = _pipe_buffer(dev, (m, ld), "ref-A")
    dC = _pipe_buffer(dev, (n, n), "ref-C")
    if ws is None:
        ws = _default_workspace(m, n, threshold, torch.float64)
    else:
        check_ata_workspace(ws, m, n, threshold)
    plan = _plan_for(m, n, ld, n, threshold, ws)
    wbuf = ws.ensure(dev, extra=plan.ws_scalars, dtype=torch.float64) if plan.ws_scalars > 0 else None
    wkw = dict(ws=int(wbuf.data_ptr()) if wbuf is not None else 0,
               ws_elems=int(wbuf.numel()) if wbuf is not None else 0)
    a_ready, c_ready = torch.cuda.Event(), torch.cuda.Event()
    copy.wait_stream(main)                 # the buffers are free to overwrite
    with torch.cuda.stream(copy):
        rc = _cudart().cudaMemcpy2DAsync(dA.data_ptr(), ld * 8, a.data_ptr(), n * 8, n * 8, m, 1, _stream_ptr())
        if rc != 0:
            raise RuntimeError(f"cudaMemcpy2DAsync failed ({rc})")
        a_ready.record(copy)
        _copy_lower(dC, c, to_device=True, step=_dl_step(n))
        c_ready.record(copy)
    ops = plan.ops
    first_c = _first_c_writer(ops)
    downloads = dict(_download_schedule(plan, n))
    cuts = sorted({first_c} | set(downloads))
    code = nat.ATA_F64
    A_ptr, a_elems = int(dA.data_ptr()), (m - 1) * ld + n
    main.wait_event(a_ready)
    prev, c_waited = 0, False
    for cut in cuts + [len(ops)]:
        if cut > prev:
            key = ("ata-ref-pipe", m, n, ld, threshold, prev, cut)
            engine.run_plan_graphed(key, _SubPlan(ops[prev:cut]), code, A_ptr, a_elems, int(dC.data_ptr()),
                                    dC.numel(), alpha, **wkw)
            prev = cut
        if cut == first_c and not c_waited:
            main.wait_event(c_ready)
            c_waited = True
        if cut in downloads:
            ev = torch.cuda.Event()
            ev.record(main)
            copy.wait_event(ev)
            with torch.cuda.stream(copy):
                _copy_tiles(c, dC, downloads[cut])
    main.wait_event(c_ready)
    _copy_tiles(c, dC, _download_schedule(plan, n, remaining=True))
    main.wait_stream(copy)
    main.synchronize()
    if counter is not None:
        counter.add(plan.mults)
    return True


def _add_tiles_plan(n: int, tiles):
    """combo4 passes C += A over the given (block row, block col, step) tiles
    (square tiles of the download grid; one multi-node launch per <= 104)."""
    tiles = tuple(tiles)

    def build():
        pb = planner.PlanBuilder("add-tiles")
        g = pb.new_group()
        for (bi, bj, step) in tiles:
            r0, c0 = bi * step, bj * step
            rows, cols = min(step, n - r0), min(step, n - c0)
            if rows <= 0 or cols <= 0:
                continue
            c = planner.Win(nat.BASE_C, r0 * n + c0, n, rows, cols)
            pb.combo4([c, planner.Win(nat.BASE_A, r0 * n + c0, n, rows, cols)], [(c, (1, 1))], group=g)
        return pb.finish()
    return engine.cached_plan(("add-tiles", n, hash(tiles), len(tiles)), build)


def _add_plan(n: int):
    """One combo4 pass: C = C + A over the whole n x n square."""
    def build():
        pb = planner.PlanBuilder("add-square")
        c = planner.Win(nat.BASE_C, 0, n, n, n)
        pb.combo4([c, planner.Win(nat.BASE_A, 0, n, n, n)], [(c, (1, 1))])
        return pb.finish()
    return engine.cached_plan(("add-square", n), build)


def _row_blocks(m: int, n: int, es: int, tensor_rate: bool):
    """Row blocks of the host pipeline.  Each block after the first crosses PCIe
    while the GPU computes the previous ones, and every block repeats the C-sized
    work of a plan (post-additions, C updates), so compute-bound plans -- per-row
    compute time over per-row upload time `ratio` >= 1.5 (fp64: ~n / 8600) -- use
    PIPELINE_GEOMETRIC_BLOCKS blocks growing by PIPELINE_GEOMETRIC_GROWTH: a small
    first block (short exposed upload; less than half the second, so C can start
    at zero on the device), few blocks in total.  Measured with the round's final
    device plans (tools/e2e_blocks.py, profiles/r02n_e2e_blocks.log): c4 1436 ms
    at growth 3.84 -> 1368-1370 ms at 2.3-2.7, 1399-1440 with four blocks,
    1402-1616 with two; c3 130 ms with two blocks -> 114-115 ms with three at
    growth 2.5-3.  Otherwise (TF32: PCIe bound) up to 8 equal blocks of
    ~PIPELINE_BLOCK_BYTES."""
    rate = (PIPELINE_TF32_TFLOPS if tensor_rate else PIPELINE_FP64_TFLOPS) * 1e12
    ratio = n * PIPELINE_PCIE_GBS * 1e9 / (rate * es)
    if PIPELINE_GEOMETRIC and ratio >= PIPELINE_GEOMETRIC_MIN_RATIO:
        g, R = PIPELINE_GEOMETRIC_GROWTH, PIPELINE_GEOMETRIC_BLOCKS
        w = [g ** i for i in range(R)]
        cuts = [0]
        for i in range(R - 1):
            cuts.append(max(cuts[-1] + 1, int(round(m * sum(w[:i + 1]) / sum(w)))))
        cuts = [c for c in cuts if c < m] + [m]
        return [(a, b - a) for a, b in zip(cuts, cuts[1:])]
    R = max(2, min(8, -(-m * n * es // PIPELINE_BLOCK_BYTES)))
    rb = -(-m // R)
    return [(r0, min(rb, m - r0)) for r0 in range(0, m, rb)]


_COPY_STREAMS = {}


def _copy_stream(dev):
    import torch
    s = _COPY_STREAMS.get(dev.index)
    if s is None:
        s = _COPY_STREAMS[dev.index] = torch.cuda.Stream(dev)
    return s


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
