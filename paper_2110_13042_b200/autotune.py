"""Measured-throughput tuning of the auto plan (``threshold="auto"``).

The auto planner decides each Strassen split from two rates -- the leaf
product kernel's FP64 rate and the one-pass addition kernels' HBM rate
(``AutoParams.dmma_tflops`` / ``hbm_gbs``) -- and cuts the AtA column
recursion at ``leaf_cols``.  This module measures those on the device that
will run the plan instead of trusting the constants:

* ``calibrate(device)``: one FP64 product group (16 products of
  4096 x 1024 x 1024 through the native executor) and one ``combo4`` pass
  over 2 x 1 GiB, each timed with CUDA events after a warm-up; rates are
  rounded to two significant digits so that the plans they produce are
  reproducible run to run.  Cached per device.
* ``tune(m, n, device)``: the calibrated rates, then the SYRK leaf width
  picked by timing the auto plan of the actual shape once per candidate
  (``leaf_cols`` in 512 / 1024 / 2048, each with its own Strassen depths from
  the cost model) and keeping the fastest; then, for a plan that has no
  successive leaf groups for its operand sums to ride on (all trees breadth
  first), the breadth-first workspace budget among {as planned, 1/2, 1/4 of
  the plan's scratch}, also timed.  Cached per (shape, device).

Used by ``ata(..., threshold="auto", auto_params="tune")`` and
``bench.py --autotune`` (config c3: "cutoff auto-tuned").  The measurement
runs before the caller's timed region; it allocates its own scratch.
"""
from __future__ import annotations

import dataclasses
import math

from . import _native as nat
from . import auto_plan, engine, planner

_RATES: dict = {}
_TUNED: dict = {}
LEAF_CANDIDATES = (512, 1024, 2048)


def _round2(x: float) -> float:
    if x <= 0:
        return x
    e = math.floor(math.log10(x)) - 1
    return round(x / 10 ** e) * 10 ** e


def _time(fn, reps: int = 3) -> float:
    import torch
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return best


def calibrate(device=None) -> tuple[float, float]:
    """(FP64 leaf-product TFLOP/s, addition-pass GB/s) measured on `device`."""
    import torch
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    key = str(dev)
    if key in _RATES:
        return _RATES[key]
    with torch.cuda.device(dev):
        m, n, cnt = 4096, 1024, 16
        A = torch.rand((m, cnt * n), dtype=torch.float64, device=dev)
        W = torch.empty(cnt * n * n, dtype=torch.float64, device=dev)
        pb = planner.PlanBuilder("calibrate")
        g = pb.new_group()
        for i in range(cnt):
            a = planner.Win(nat.BASE_A, i * n, cnt * n, m, n)
            b = planner.Win(nat.BASE_A, ((i + 1) % cnt) * n, cnt * n, m, n)
            pb.product("gemm", m, n, n, [(a, 1.0)], [(b, 1.0)], [(planner.Win(nat.BASE_WS, i * n * n, n, n, n), 1.0)],
                       accumulate=0, group=g)
        prod = pb.finish()
        C = torch.zeros((1, 1), dtype=torch.float64, device=dev)
        t_prod = _time(lambda: engine.run_plan(prod, nat.ATA_F64, A.data_ptr(), A.numel(), C.data_ptr(),
                                               C.numel(), 1.0, ws=W.data_ptr(), ws_elems=W.numel()))
        tflops = 2.0 * m * n * n * cnt / t_prod / 1e12
        # one combo4 pass: four 8192 x 8192 quadrants -> two sums (the planner's operand-sum shape)
        q = 8192
        X = torch.rand((2 * q, 2 * q), dtype=torch.float64, device=dev)
        O = torch.empty(2 * q * q, dtype=torch.float64, device=dev)
        pb = planner.PlanBuilder("calibrate-hbm")
        quads = [planner.Win(nat.BASE_A, r * q * 2 * q + c * q, 2 * q, q, q) for r in (0, 1) for c in (0, 1)]
        pb.combo4(quads, [(planner.Win(nat.BASE_WS, 0, q, q, q), (1, 0, 0, 1)),
                          (planner.Win(nat.BASE_WS, q * q, q, q, q), (0, 1, 0, 1))])
        ew = pb.finish()
        t_ew = _time(lambda: engine.run_plan(ew, nat.ATA_F64, X.data_ptr(), X.numel(), C.data_ptr(), C.numel(),
                                             1.0, ws=O.data_ptr(), ws_elems=O.numel()))
        gbs = (4 * q * q + 2 * q * q) * 8 / t_ew / 1e9
        del A, W, X, O
    rates = (_round2(tflops), _round2(gbs))
    _RATES[key] = rates
    return rates


def tune(m: int, n: int, device=None, lda: int | None = None, ldc: int | None = None,
         base: auto_plan.AutoParams | None = None) -> auto_plan.AutoParams:
    """AutoParams for an m x n fp64 AtA on `device`: calibrated rates and the
    fastest SYRK leaf width among LEAF_CANDIDATES (timed, each plan once after
    a warm-up run)."""
    import torch
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    lda, ldc = lda or n, ldc or n
    key = (m, n, lda, ldc, str(dev), base)
    if key in _TUNED:
        return _TUNED[key]
    tflops, gbs = calibrate(dev)
    params = dataclasses.replace(base or auto_plan.AutoParams(), dmma_tflops=tflops, hbm_gbs=gbs)
    cands = [c for c in LEAF_CANDIDATES if c < n] or [params.leaf_cols]
    if len(cands) > 1:
        with torch.cuda.device(dev):
            A = torch.rand((m, lda), dtype=torch.float64, device=dev)
            C = torch.zeros((n, ldc), dtype=torch.float64, device=dev)
            best, best_t = None, float("inf")
            for leaf in cands:
                p = dataclasses.replace(params, leaf_cols=leaf)
                plan = auto_plan.plan_ata_auto(m, n, lda, ldc, p)
                W = torch.empty(max(1, plan.ws_scalars), dtype=torch.float64, device=dev)
                t = _time(lambda: engine.run_plan(plan, nat.ATA_F64, A.data_ptr(), A.numel(), C.data_ptr(),
                                                  C.numel(), 1.0, ws=W.data_ptr(), ws_elems=W.numel()), reps=1)
                del W
                if t < best_t:
                    best, best_t = p, t
            params = best
            del A, C
        torch.cuda.empty_cache()
    params = _tune_budget(m, n, lda, ldc, dev, params)
    _TUNED[key] = params
    return params


def _tune_budget(m, n, lda, ldc, dev, params):
    """Riding operand sums need successive leaf groups: a plan whose Strassen
    trees are all breadth first (one leaf group per tree: config c3) hides
    nothing.  Time the plan at 1/2 and 1/4 of its own scratch size as the
    breadth-first budget (depth-first top levels: the next subtree's sums ride on
    the previous subtree's products) and keep the fastest."""
    import torch
    if not params.ride_sums:
        return params
    plan0 = auto_plan.plan_ata_auto(m, n, lda, ldc, params)
    combos = plan0.ops["type"] == nat.OP_COMBO4
    if not combos.any() or ((plan0.ops["flags"] & nat.OPF_RIDE) != 0).sum() * 2 > combos.sum():
        return params
    ws_gb = plan0.ws_scalars * 8 / 1e9
    cands = [params] + [dataclasses.replace(params, ws_budget_gb=round(ws_gb * f, 2)) for f in (0.5, 0.25)]
    with torch.cuda.device(dev):
        A = torch.rand((m, lda), dtype=torch.float64, device=dev)
        C = torch.zeros((n, ldc), dtype=torch.float64, device=dev)
        best, best_t = params, float("inf")
        for p in cands:
            plan = plan0 if p is params else auto_plan.plan_ata_auto(m, n, lda, ldc, p)
            W = torch.empty(max(1, plan.ws_scalars), dtype=torch.float64, device=dev)
            t = _time(lambda: engine.run_plan(plan, nat.ATA_F64, A.data_ptr(), A.numel(), C.data_ptr(),
                                              C.numel(), 1.0, ws=W.data_ptr(), ws_elems=W.numel()), reps=2)
            del W
            if t < best_t * 0.995:      # a smaller budget must win by a margin (reproducible plans)
                best, best_t = p, t
        del A, C
    torch.cuda.empty_cache()
    return best
