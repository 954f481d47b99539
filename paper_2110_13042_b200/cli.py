"""``atamul``-compatible command line on the GPU path.

Same flags, validation, printed summary and CSV schema as the reference CLI
(``pkg/src/atamul/bench.py:30-31``, ``:50-54``, ``:91-137``, ``:236-270``), so
scripts that drive ``atamul`` keep working with

    python -m paper_2110_13042_b200.cli [--mode ...] [--n ...] ...

Modes (all compute on cuda:0 through the native library; A is uploaded once,
each timed run allocates a zero C, computes, and mirrors, as the reference's
``once()`` does):

* ``seq``    -- ``ata`` with the integer threshold: the reference recursion tree
  (exact multiplication counts), executed breadth first on the GPU;
* ``auto``   -- ``ata`` with ``threshold="auto"`` (the GPU plan; extension);
* ``oracle`` -- one classical SYRK leaf kernel over the whole matrix;
* ``shared`` -- the reference's shared task tree (build_tree_shared): the
  write-disjoint leaf tasks run concurrently on separate CUDA streams;
* ``dist``   -- the reference's distributed task tree (build_tree_distributed),
  simulated in one process like the reference's ``ata_d``: the P processes'
  leaves run on this GPU one after another and their result blocks are
  retrieved up the tree in memory (``dist.ata_tree``; with a torch.distributed
  group the same function runs one leaf per GPU and retrieves over NCCL).

``--threshold`` also accepts ``auto``.  ``--check`` compares against the
classical SYRK kernel on the GPU with the reference's tolerance
(``bench.py:85-88``).  ``--comm-csv`` writes the retrieve-phase counters of
the distributed tree (result blocks only; there is no operand distribution
phase on a box where every GPU reads its own rows).
"""
from __future__ import annotations

import argparse
import csv
import os
import statistics
import sys
import time
from dataclasses import dataclass

import numpy as np

CSV_HEADER = ["mode", "m", "n", "procs", "threshold", "reps", "median_s",
              "eff_gflops", "max_abs_err", "mult_count"]
DEFAULT_THRESHOLD = 1 << 15


@dataclass
class BenchRecord:
    mode: str
    m: int
    n: int
    procs: int
    threshold: object
    reps: int
    median_s: float
    eff_gflops: float
    max_abs_err: float | None = None
    mult_count: int | None = None
    check_failed: bool = False

    def csv_row(self) -> list:
        """The reference's CSV row formatting (bench.py:50-54)."""
        return [self.mode, self.m, self.n, self.procs, self.threshold, self.reps,
                f"{self.median_s:.6g}", f"{self.eff_gflops:.6g}",
                "" if self.max_abs_err is None else f"{self.max_abs_err:.6g}",
                "" if self.mult_count is None else self.mult_count]


def _threshold(text: str):
    return "auto" if text == "auto" else int(text)


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="atamul", description="Benchmark the recursive A^T A kernels (B200).")
    p.add_argument("--mode", choices=["seq", "shared", "dist", "oracle", "auto"], default="seq")
    p.add_argument("--m", type=int, default=None, help="row count of A; --n when omitted")
    p.add_argument("--n", type=int, default=1024, help="column count of A (and order of C)")
    p.add_argument("--procs", type=int, default=None, help="task-tree processes; shared/dist modes only")
    p.add_argument("--threshold", type=_threshold, default=None,
                   help="leaf threshold in elements (32768 unless ATA_THRESHOLD is set) or 'auto'")
    p.add_argument("--dtype", choices=["f32", "f64"], default="f64")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--reps", type=int, default=5, help="timed runs after one warm-up; prints the median")
    p.add_argument("--check", action="store_true", help="check every run against one classical SYRK kernel")
    p.add_argument("--csv", metavar="PATH", help="append the result row to this CSV file")
    p.add_argument("--comm-csv", metavar="PATH", help="dist mode: write the retrieve-phase message/word counters")
    p.add_argument("--count-mults", action="store_true", help="print the exact number of scalar multiplications")
    p.add_argument("--in", dest="in_path", metavar="PATH", help="load A from this ATAM file (no generation)")
    p.add_argument("--out", dest="out_path", metavar="PATH", help="save the input matrix as an ATAM file")
    p.add_argument("--leaf-kernel", choices=["fast", "naive"], default="fast",
                   help="kernel used by dist-mode leaves (naive: one classical product per leaf)")
    p.add_argument("--dump-tree", action="store_true", help="render the task tree of the mode and stop")
    return p


def validate(args) -> None:
    """The reference's argument rules (bench.py:125-137)."""
    if args.mode in ("seq", "oracle", "auto") and args.procs is not None:
        raise SystemExit(f"--procs is not valid with --mode {args.mode}")
    if args.mode in ("shared", "dist") and args.procs is None:
        args.procs = 1
    if args.comm_csv and args.mode != "dist":
        raise SystemExit("--comm-csv is only valid with --mode dist")
    if args.threshold is None:
        env = os.environ.get("ATA_THRESHOLD")
        args.threshold = _threshold(env) if env else DEFAULT_THRESHOLD
    if args.mode == "auto":
        args.threshold = "auto"
    if args.m is None:
        args.m = args.n


def run_bench(args) -> list[BenchRecord]:
    import torch
    from . import dist as pdist
    from .ata import ata
    from .matrix import MultCounter, mirror_lower_to_upper, naive_syrk_lower, read_matrix, write_matrix
    from .measure import check_tolerance, effective_gflops, gen_matrix

    dtype = np.float64 if args.dtype == "f64" else np.float32
    if args.in_path:
        A = read_matrix(args.in_path)
        args.m, args.n = A.rows, A.cols
    else:
        A = gen_matrix(args.m, args.n, args.seed, dtype=dtype)
    if args.out_path:
        write_matrix(args.out_path, A)
    host = np.asarray(A.a)
    dev = torch.device("cuda", torch.cuda.current_device())
    a = torch.from_numpy(host).to(dev)
    tdt = a.dtype
    procs = args.procs or 1
    thr = args.threshold
    counter = MultCounter() if args.count_mults else None
    n = args.n

    if args.mode in ("seq", "auto"):
        def compute(C):
            ata(a, C, 1.0, thr, counter=counter)
    elif args.mode == "oracle":
        def compute(C):
            naive_syrk_lower(a, C, 1.0, counter)
    elif args.mode == "shared":
        # the reference's bench drives SharedRunner (bench.py:170-176): leaves
        # of the shared tree on concurrent CUDA streams (shared.py)
        from .shared import SharedRunner
        runner = SharedRunner(a, procs, thr)
        runner.counters = [counter] * procs
        runner.prepare()

        def compute(C):
            runner.run_into(C, mirror=False)
    else:   # dist
        leaf_thr = (1 << 62) if args.leaf_kernel == "naive" else thr

        def get_block(r):
            return a[r.row_offset:r.row_offset + r.rows, r.col_offset:r.col_offset + r.cols]

        def compute(C):
            pdist.ata_tree(get_block, args.m, n, C, 1.0, leaf_thr, procs=procs, counter=counter)

    def once():
        C = torch.zeros((n, n), dtype=tdt, device=dev)
        compute(C)
        mirror_lower_to_upper(C)
        return C

    oracle = tol = None
    if args.check:
        oracle = torch.zeros((n, n), dtype=tdt, device=dev)
        naive_syrk_lower(a, oracle, 1.0)
        mirror_lower_to_upper(oracle)
        tol = check_tolerance(host)
    if counter is not None:
        counter.reset()
    once()                                   # warm-up; also the counted run
    torch.cuda.synchronize()
    mult_count = None
    if counter is not None:
        mult_count = counter.scalar_mults
        counter.enabled = False
    times, max_err = [], None
    for _ in range(args.reps):
        t0 = time.perf_counter()
        res = once()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        if args.check:
            err = float((res - oracle).abs().max())
            max_err = err if max_err is None else max(max_err, err)
    median_s = statistics.median(times)
    rec = BenchRecord(mode=args.mode, m=args.m, n=n, procs=procs, threshold=thr, reps=args.reps,
                      median_s=median_s, eff_gflops=effective_gflops(args.m, n, median_s, r=1),
                      max_abs_err=max_err, mult_count=mult_count)
    if args.comm_csv:
        from .tasktree import build_tree_distributed
        t = build_tree_distributed(procs, args.m, n)
        pdist.write_comm_csv(args.comm_csv, pdist.tree_comm_stats(t), procs)
    if args.check and max_err is not None and max_err > tol:
        print(f"CHECK FAILED: max abs error {max_err:g} > tolerance {tol:g}", file=sys.stderr)
        rec.check_failed = True
    return [rec]


def write_csv(path: str, records: list[BenchRecord]) -> None:
    fresh = not os.path.exists(path)
    with open(path, "a", newline="") as fh:
        w = csv.writer(fh)
        if fresh:
            w.writerow(CSV_HEADER)
        for rec in records:
            w.writerow(rec.csv_row())


def summary_line(rec: BenchRecord) -> str:
    line = (f"{rec.mode} m={rec.m} n={rec.n} procs={rec.procs} threshold={rec.threshold}: "
            f"median {rec.median_s:.4g} s, {rec.eff_gflops:.3f} effective GFLOPs")
    if rec.max_abs_err is not None:
        line += f", max abs err {rec.max_abs_err:.3g}"
    if rec.mult_count is not None:
        line += f", {rec.mult_count} scalar mults"
    return line


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    validate(args)
    if args.dump_tree:
        from .tasktree import build_tree_distributed, build_tree_shared, render_tree
        build = build_tree_distributed if args.mode == "dist" else build_tree_shared
        print(render_tree(build(args.procs or 1, args.m, args.n)))
        return 0
    records = run_bench(args)
    for rec in records:
        print(summary_line(rec))
    if args.csv:
        write_csv(args.csv, records)
    return 1 if any(r.check_failed for r in records) else 0


if __name__ == "__main__":
    raise SystemExit(main())
