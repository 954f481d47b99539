"""The GPU plan for ``threshold="auto"`` (config c3/c4/c5 style workloads).

Shape of the plan (all windows into A, C and one HBM workspace):

1. AtA column recursion (ata.py:110-115): C11 <- A_l^T A_l, C22 <- A_r^T A_r,
   C21 <- A_r^T A_l, recursing on the diagonal blocks down to ``leaf_cols``.
   The reference also halves the rows (the contraction) at every level; on
   the GPU the contraction stays whole inside each product's K loop, so the
   two C21 addends of ata.py:114-115 are one product over all m rows.
2. Every C21 block is a Strassen tree (strassen.py:234-275) whose depth is
   chosen per node by a cost model (flops saved at the measured product
   rate vs. bytes moved by the operand sums and post-additions at the measured
   HBM rate), evaluated with three HBM-bound one-pass kernels around the
   tensor-core leaves:
     * pre-addition: ONE multi-output pass per operand and node (``combo4``:
       reads the four quadrants once, writes the five operand sums; the other
       two operands of the seven products are plain quadrant views);
     * leaves: plain products (one term per operand) writing private product
       buffers -- no shared destinations, no read-modify-write, one
       persistent launch per leaf group;
     * post-addition: ONE pass per node (``postadd7``: reads the seven child
       products once, writes the node's four output quadrants, accumulating
       into C at the root).  This replaces the reference's 12 read-modify-
       write updates per node (strassen.py:238-275) and is executed bottom-up.
   Quadrant splits are ceil-first (first half = ceil, the trailing half is
   the zero-extended one), so every node of a level has identical shapes.
3. Diagonal leaves are SYRK-lower products; they join the first breadth-
   first leaf group (they read only A), else form the last group.
The Strassen trees of one AtA level are planned breadth-first (one leaf group)
when their workspace fits ``ws_budget_gb``; otherwise depth-first over each
block's top-level children (one leaf group per subtree).

Arithmetic is the reference's (zero-extended Strassen, classical leaves); only
the recursion shape differs from an integer-threshold run, hence the
multiplication count differs (reported as plan.mults).
"""
from __future__ import annotations

import dataclasses
import os
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import ShapeMismatchError
from .planner import Plan, PlanBuilder, Win

# Strassen in the transposed orientation (strassen.py:234-275) for
# c = a^T b, quadrants X11 X12 / X21 X22 (rows = contraction):
#   P1 = (A11+A22)^T (B11+B22)     P5 = (A11+A21)^T  B22
#   P2 = (A12+A22)^T  B11          P6 = (A12-A11)^T (B11+B12)
#   P3 =  A11^T (B12-B22)          P7 = (A21-A22)^T (B21+B22)
#   P4 =  A22^T (B21-B11)
#   C11 = P1+P4-P5+P7  C12 = P3+P5  C21 = P2+P4  C22 = P1-P2+P3+P6
# Operand coefficient vectors over (X11, X12, X21, X22):
_S = [(1, 0, 0, 1), (0, 1, 0, 1), (1, 0, 0, 0), (0, 0, 0, 1), (1, 0, 1, 0), (-1, 1, 0, 0),
      (0, 0, 1, -1)]
_T = [(1, 0, 0, 1), (1, 0, 0, 0), (0, 1, 0, -1), (-1, 0, 1, 0), (0, 0, 0, 1), (1, 1, 0, 0),
      (0, 0, 1, 1)]


@dataclass(frozen=True)
class AutoParams:
    leaf_cols: int = 1024          # SYRK leaf width of the column recursion
    max_depth: int = 4             # Strassen levels per C21 block
    min_dim: int = 512             # never split a Strassen node below this output side
    dmma_tflops: float = 33.5      # measured leaf-product rate (profiles/)
    hbm_gbs: float = 5800.0        # achieved one-pass kernel bandwidth (profiles/)
    gain: float = 1.25             # split only when saved time > gain * added time
    ws_budget_gb: float = 40.0     # workspace for breadth-first planning of one AtA level
    fill_waves: int = 2            # split the contraction of groups with fewer tiles than this
    min_chunk: int = 8192          # ... into chunks of at least this many rows
    tf32_tflops: float = 400.0     # single-pass TF32 leaf-product rate (tcgen05, profiles/)
    tf32_fill_waves: int = 8       # 128x256 tcgen05 tiles: more chunks to fill 148 SMs
    tf32_ring: bool = True         # single-pass TF32: round through the product kernel's L2 ring
                                   # instead of an HBM rounding pass when the plan allows (_ringify)
    fuse_leaf_sums: bool = False   # FP64: leaf products read their Strassen operand sums as two
                                   # zero-extended terms summed in the kernel's load path (no
                                   # combo4 pass for the last Strassen level).  Off: measured
                                   # 2.1-2.2x slower on c3/c4 (the two-term kernel configuration
                                   # runs at 14 TF/s vs 34 for plain operands)
    min_leaf_rows: int = 0         # never split a node whose children would contract fewer rows than this
                                   # (the units partition plans row pieces with their unit's tree: 1024)
    cost_row_scale: float = 1.0    # the cost model sees m * this many contraction rows: a row
                                   # block of a larger A (the pinned-host pipeline) gets the
                                   # Strassen tree of the whole A, so the blocks' executed
                                   # multiplications add up to the single plan's
    ride_sums: bool = True         # FP64: the operand sums of the NEXT leaf group ride on the current
                                   # group's product launch (ATA_OPF_RIDE, executed by the leaf kernel's
                                   # spare warps while the DMMAs run): scratch of successive leaf groups
                                   # alternates between two regions and _hoist_sums reorders / flags the ops
    ride_gbs: float = 1500.0       # additions a product launch hides per second of its own duration
                                   # (measured, tools/ride_ab.py: with no FP64-pipe instruction left in
                                   # the ride 2.0 TB/s cost +2 % of the launch, 2.5 TB/s +8 %, bound near
                                   # 2.9 TB/s; c4: 1294 ms at 1200-1600, 1299 unlimited); _hoist_sums moves no more
    gain_ride: float = 1.0         # the split threshold `gain` of plans with riding sums (their operand
                                   # sums are nearly free): c4 executes 0.630 of the classical
                                   # multiplications instead of 0.6735, 1348 -> 1294 ms (deeper still --
                                   # gain 0.8, max_depth 5, 0.593 -- is slower: 1333 ms, 2048 x 512 x 512
                                   # leaves run at 0.86-0.88 of the DMMA peak)
    ride_lookback: int = 64        # a sum may ride up to this many product groups before the one it precedes
    ride_band_gb: float = 1.25     # ... and sums above this size are cut into row bands first (_hoist_sums);
                                   # c4: exposed operand sums 146.8 -> 94.2 GB, 1367 -> 1360 ms
    ride_arenas: bool = True       # successive top-level frames alternate between two scratch arenas
                                   # (_enter_frame): the later frames' first sums ride too (c4: exposed
                                   # 94.2 -> 2.4 GB, 1360 -> 1351 ms; workspace 45.6 -> 76.4 GB;
                                   # ata.fit_workspace_budget turns it off when HBM is short)
    diag_first: bool = True        # riding sums + a depth-first top tree: the diagonal SYRK leaves (they
                                   # read only A) run as the FIRST product group, so the top tree's first
                                   # operand sums ride on them instead of running exposed.  The host
                                   # pipeline turns it off when C is uploaded behind block 0 (the SYRKs
                                   # write C)
    tail_split: bool = True        # FP64: K-split a group's trailing products (partial last wave)
    tail_private: bool = True      # ... groups too large for shared-destination launches: private partials
    min_tail_rows: int = 1024      # ... only when every chunk keeps this many rows


TILE = 128        # output tile of the product kernels
NUM_SMS = 148     # B200
MAX_BATCH = 48    # products per persistent launch (kMaxBatch, ata_common.cuh)
MAX_BATCH_NARROW = 104   # FP64 products with <= 2 destinations (kMaxBatchNarrow)
TAIL_CHUNKS = 4          # K split of a leaf group's trailing products
UNIT_MIN_LEAF_ROWS = 1024   # units partition: leaf products of a row piece contract at least this many rows


def _ceil2(d: int) -> int:
    return (d + 1) // 2


def _clip(w: Win, r0: int, c0: int, h: int, wd: int) -> Win:
    h = max(0, min(h, w.rows - r0))
    wd = max(0, min(wd, w.cols - c0))
    if h == 0 or wd == 0:
        return Win(w.base, w.off, w.ld, 0, 0)
    return w.sub(r0, c0, h, wd)


def _quads(w: Win, r1: int, c1: int):
    """Ceil-first quadrants of a window whose logical extent is (2*r1) x (2*c1);
    quadrants beyond the actual extent are empty windows (zero-extended)."""
    return [_clip(w, 0, 0, r1, c1), _clip(w, 0, c1, r1, c1), _clip(w, r1, 0, r1, c1),
            _clip(w, r1, c1, r1, c1)]


def _terms(x):
    """A leaf operand as [(Win, coef)]: a plain window, or the <= 2 signed
    quadrant terms of a fused Strassen operand sum."""
    return [(x, 1.0)] if isinstance(x, Win) else list(x)


def _clip_terms(x, r0: int, h: int):
    """Rows [r0, r0 + h) of every term (contraction chunk); empty terms dropped
    (an all-empty operand keeps one empty window: it reads as zero)."""
    terms = [(_clip(w, r0, 0, h, w.cols), c) for w, c in _terms(x)]
    out = [(w, c) for w, c in terms if w.rows and w.cols]
    return out or terms[:1]


def _empty(x) -> bool:
    return all(w.rows == 0 or w.cols == 0 for w, _ in _terms(x))


class _AutoPlanner:
    def __init__(self, params: AutoParams):
        self.p = params
        self.pb = PlanBuilder("auto")
        self.ws_top = 0          # bump allocator over the workspace (elements)
        self.ws_peak = 0
        self.ws_floor = 0        # persistent prefix (the rounded operand copy)
        self.rate = params.dmma_tflops
        self.esize = 8
        self.fill_waves = params.fill_waves
        self.tile = (TILE, TILE)
        self.defer_sums = None   # breadth-first trees: [(depth_left, quadrants, outputs)] emitted by emit()
        self.flip_tree = 0       # ride_sums: successive breadth-first subtrees / depth-first operand
        self.flip_sums = 0       # sums alternate between two scratch regions
        self.flip_extra = 0      # elements below ws_top that are second copies of alternating regions
        self.frames = 0          # ride_arenas: top-level frames planned so far,
        self.arena1 = None       # where the odd ones start (above everything planned before the first),
        self.frame_off = 0       # and the current frame's offset above ws_floor

    # ---------------------------------------------------------------- workspace
    def alloc(self, rows: int, cols: int) -> Win:
        w = Win(nat.BASE_WS, self.ws_top, cols, rows, cols)
        self.ws_top += rows * cols
        self.ws_peak = max(self.ws_peak, self.ws_top)
        return w

    # ------------------------------------------------------------- cost model
    def worth_split(self, m: int, n: int, k: int, depth_left: int) -> bool:
        if depth_left <= 0 or min(n, k) < 2 * self.p.min_dim or m < 2 or m < 2 * self.p.min_leaf_rows:
            return False
        m = m * self.p.cost_row_scale
        gain = min(self.p.gain, self.p.gain_ride) if self._riding() else self.p.gain
        saved_s = 2.0 * m * n * k / 8 / (self.rate * 1e12)
        # pre: read both operands, write 5 + 5 quarter sums; post: write 7 child
        # products (leaf epilogue), read them back, write (or RMW) 4 quadrants
        moved = self.esize * (m * n * (1 + 5 / 4) + m * k * (1 + 5 / 4) + n * k * (7 / 4 + 7 / 4 + 2))
        added_s = moved / (self.p.hbm_gbs * 1e9)
        return saved_s > gain * added_s

    # --------------------------------------------------------------- Strassen
    def _sums(self, a: Win, b: Win, m: int, n: int, k: int, depth: int = 0):
        """Emit (or, inside a breadth-first tree, defer) one node's operand
        sums; return (S[7], T[7], m1, n1, k1)."""
        m1, n1, k1 = _ceil2(m), _ceil2(n), _ceil2(k)
        S, T = [None] * 7, [None] * 7
        for X, coefs, out, cols in ((_quads(a, m1, n1), _S, S, n1), (_quads(b, m1, k1), _T, T, k1)):
            outs = []
            for i, coef in enumerate(coefs):
                if sorted(coef) == [0, 0, 0, 1]:
                    out[i] = X[coef.index(1)]            # plain quadrant view
                else:
                    out[i] = self.alloc(m1, cols)
                    outs.append((out[i], coef))
            if self.defer_sums is not None:
                self.defer_sums.append((depth, X, outs))
            else:
                self.pb.combo4(X, outs)                  # one pass over the quadrants
        return S, T, m1, n1, k1

    def _post(self, kids, out: Win, sign: float, n1: int, k1: int, accumulate: bool, group: int = -1):
        q = [_clip(out, 0, 0, n1, k1), _clip(out, 0, k1, n1, k1), _clip(out, n1, 0, n1, k1),
             _clip(out, n1, k1, n1, k1)]
        self.pb.postadd7(kids, [(w, sign) for w in q], accumulate, group=group)

    def tree(self, a, b, m, n, k, out, sign, accumulate, depth, leaves, posts):
        """Breadth-first: emit sums now (pre-order), collect leaves and post-adds."""
        if not self.worth_split(m, n, k, depth):
            leaves.append((m, n, k, a, b, out, sign, accumulate))
            return
        m1, n1, k1 = _ceil2(m), _ceil2(n), _ceil2(k)
        if (self.p.fuse_leaf_sums and self.esize == 8 and isinstance(a, Win) and isinstance(b, Win)
                and not self.worth_split(m1, n1, k1, depth - 1)):
            # the children are leaves: hand them their operand sums as two
            # quadrant terms each (summed in the product kernel's load path)
            # (positive term first: the kernel applies the sign to the second term)
            S = [sorted([(w, float(c)) for w, c in zip(_quads(a, m1, n1), co) if c and w.rows and w.cols],
                        key=lambda t: -t[1]) for co in _S]
            T = [sorted([(w, float(c)) for w, c in zip(_quads(b, m1, k1), co) if c and w.rows and w.cols],
                        key=lambda t: -t[1]) for co in _T]
            if any(x and x[0][1] < 0 for x in S + T):   # a lone negative term: materialise instead
                S, T, m1, n1, k1 = self._sums(a, b, m, n, k, depth)
        else:
            S, T, m1, n1, k1 = self._sums(a, b, m, n, k, depth)
        kids = [self.alloc(n1, k1) for _ in range(7)]
        for i in range(7):
            self.tree(S[i], T[i], m1, n1, k1, kids[i], 1.0, False, depth - 1, leaves, posts)
        posts.append((kids, out, sign, n1, k1, accumulate, depth))

    def emit(self, leaves, posts, extra=()):
        # deferred operand sums, shallowest level first; the nodes of one level
        # are independent and run as one multi-node combo4 launch
        sums, self.defer_sums = self.defer_sums or [], None
        for d in sorted({d for d, _, _ in sums}, reverse=True):
            level = [(X, outs) for dd, X, outs in sums if dd == d]
            g = self.pb.new_group() if len(level) > 1 else -1
            for X, outs in level:
                self.pb.combo4(X, outs, group=g)
        prods = []
        for (m, n, k, a, b, out, sign, accumulate) in leaves:
            if _empty(a) or _empty(b):
                if not accumulate:            # an all-zero operand: the product buffer is zero
                    self.pb.fill(out)
                continue
            prods.append(("gemm", m, n, k, a, b, out, sign, accumulate))
        # products writing C go last in the group: everything before the first
        # C writer only needs A and scratch (ata._pipelined_host_ata uploads C
        # behind the first block of A and waits for it at the first C writer)
        prods = [p for p in prods if p[6].base != nat.BASE_C] + list(extra) + \
            [p for p in prods if p[6].base == nat.BASE_C]
        self.emit_products(prods)
        # post-additions deepest level first, one multi-node launch per level
        for d in sorted({p[6] for p in posts}):
            level = [p for p in posts if p[6] == d]
            g = self.pb.new_group() if len(level) > 1 else -1
            for (kids, out, sign, n1, k1, accumulate, _) in level:
                self._post(kids, out, sign, n1, k1, accumulate, group=g)

    def _tiles(self, kind, n, k):
        """Output tiles of one product on the leaf kernel this plan runs on
        (FP64: 128x128 tiles; single-pass TF32: 128x256 tcgen05 tiles, SYRK
        strips enumerate only the column tiles touching the lower triangle)."""
        bm, bn = self.tile
        tn, tk = -(-n // bm), -(-k // bn)
        if kind != "syrk":
            return tn * tk
        return sum(min(tk, (ti * bm + bm - 1) // bn + 1) for ti in range(tn))

    def _tail_split(self, prods) -> int:
        """Index of the first product whose contraction is split for the tail
        (FP64 groups only: ordered accumulation needs the FP64 kernel's turn
        counters).  The trailing products covering one wave of tiles are split
        when the group ends in a partial wave and stays within one launch."""
        self.tail_private = False
        if self.esize != 8 or not self.p.tail_split:
            return len(prods)
        tl = [self._tiles(p[0], p[2], p[3]) for p in prods]
        total = sum(tl)
        if total <= NUM_SMS or total % NUM_SMS == 0:
            return len(prods)
        j, acc = len(prods), 0
        while j > 0 and acc < NUM_SMS:
            j -= 1
            acc += tl[j]
        if any(prods[q][1] < TAIL_CHUNKS * self.p.min_tail_rows for q in range(j, len(prods))):
            return len(prods)
        if j + (len(prods) - j) * TAIL_CHUNKS > MAX_BATCH_NARROW:
            # launches with shared destination regions hold at most MAX_BATCH_NARROW products:
            # the chunks of a larger group's tail write private partials instead (summed by
            # one small combo4 launch behind the group), which keeps the group one launch
            self.tail_private = self.p.tail_private
            return j if self.tail_private else len(prods)
        return j

    def _chunks(self, tiles: int, rows: int, nprods: int = 1) -> int:
        """Contraction split S for a group of `tiles` output tiles: at least
        fill_waves waves, then the smallest S (up to 3x that) whose tile count fills >= 97% of
        whole waves of the persistent grid, else the best-filling one (rows/S >= min_chunk)."""
        target = self.fill_waves * NUM_SMS
        if tiles >= target:
            return 1
        # one persistent launch per group: at most MAX_BATCH products
        s_hi = min(rows // self.p.min_chunk, max(1, MAX_BATCH // nprods))
        s_lo = -(-target // tiles)
        if s_hi <= 1:
            return 1
        if s_lo >= s_hi:
            return s_hi
        best, best_eff = s_lo, -1.0
        for S in range(s_lo, min(3 * s_lo, s_hi) + 1):
            t = tiles * S
            eff = t / (NUM_SMS * -(-t // NUM_SMS))
            if eff >= 0.97:
                return S
            if eff > best_eff + 1e-9:
                best, best_eff = S, eff
        return best

    def emit_products(self, prods):
        """One launch group.  When the group's output tiles cannot fill the GPU
        (tall-skinny operands, config c5) the contraction is split into S
        chunks: chunk products write private partial buffers, then one-pass
        combo4 sums add them into the destination (lower triangle only for
        SYRK), so no atomics and a fixed summation order."""
        if not prods:
            return
        tiles = sum(self._tiles(p[0], p[2], p[3]) for p in prods)
        S = self._chunks(tiles, min(p[1] for p in prods), len(prods))
        group = self.pb.new_group()
        if S <= 1:
            split_from = self._tail_split(prods)
            for (kind, m, n, k, a, b, out, sign, accumulate) in prods[:split_from]:
                T = [] if kind == "syrk" else _terms(b)
                self.pb.product(kind, m, n, k, _terms(a), T, [(out, sign)],
                                accumulate=int(accumulate), group=group)
            # tail products: K split into TAIL_CHUNKS ordered partial products
            # (chunk 0 writes, the rest accumulate in turn through the FP64
            # kernel's per-tile turn counters), issued last so the dynamic tile
            # queue ends with short tiles instead of a partial wave of full ones
            reductions = []
            for (kind, m, n, k, a, b, out, sign, accumulate) in prods[split_from:]:
                region = 0 if self.tail_private else self.pb.new_region()
                mc = -(-m // TAIL_CHUNKS)
                parts = []
                for c in range(TAIL_CHUNKS):
                    r0 = c * mc
                    rows = min(mc, m - r0)
                    if rows <= 0:
                        break
                    ac = _clip_terms(a, r0, rows)
                    T = [] if kind == "syrk" else _clip_terms(b, r0, rows)
                    if self.tail_private:
                        P = self.alloc(n, k)
                        self.pb.product(kind, rows, n, k, ac, T, [(P, 1.0)], accumulate=0, group=group)
                        parts.append(P)
                    else:
                        self.pb.product(kind, rows, n, k, ac, T, [(out, sign, region)],
                                        accumulate=int(accumulate or c > 0), group=group)
                if parts:
                    reductions.append((kind, out, sign, accumulate, parts))
            self._reduce_partials(reductions)
            return
        # chunk-major order: the products of one row chunk are adjacent, so a
        # wave of the persistent grid runs whole chunks (periodic_workers)
        parts = [[] for _ in prods]
        for c in range(S):
            for pi, (kind, m, n, k, a, b, out, sign, accumulate) in enumerate(prods):
                mc = -(-m // S)
                r0 = c * mc
                rows = min(mc, m - r0)
                if rows <= 0:
                    continue
                ac = _clip_terms(a, r0, rows)
                bc = ac if b is None else _clip_terms(b, r0, rows)
                if _empty(ac) or _empty(bc):
                    continue
                P = self.alloc(n, k)
                T = [] if kind == "syrk" else bc
                self.pb.product(kind, rows, n, k, ac, T, [(P, 1.0)], accumulate=0,
                                group=group)
                parts[pi].append(P)
        self._reduce_partials([(kind, out, sign, accumulate, parts[pi])
                               for pi, (kind, m, n, k, a, b, out, sign, accumulate) in enumerate(prods)])

    def _reduce_partials(self, reductions):
        """out (+)= sign * sum(parts) for [(kind, out, sign, accumulate, parts)]."""
        # each product's partials are summed by a chain of combo4 passes; the
        # chains are independent, so passes of equal depth form one multi-node
        # launch (depth-major emission, one group per depth)
        chains = []
        for (kind, out, sign, accumulate, parts) in reductions:
            srcs, first, chain = list(parts), True, []
            while srcs or first:
                head = [] if (first and not accumulate) else [out]
                take = srcs[:4 - len(head)]
                srcs = srcs[len(take):]
                coefs = tuple([1] * len(head) + [int(sign)] * len(take))
                chain.append((head + take, [(out, coefs)], kind == "syrk"))
                first = False
            chains.append(chain)
        for d in range(max((len(c) for c in chains), default=0)):
            level = [c[d] for c in chains if d < len(c)]
            g = self.pb.new_group() if len(level) > 1 else -1
            for (srcs, outs, lower) in level:
                self.pb.combo4(srcs, outs, lower=lower, group=g)

    def _riding(self) -> bool:
        return self.p.ride_sums and self.esize == 8

    def _arenas(self) -> bool:
        return self._riding() and self.p.ride_arenas

    def _enter_frame(self):
        """ride_arenas: successive top-level frames (a depth-first C21 tree, or one
        breadth-first AtA level) alternate between two arenas, so the whole
        scratch of the next frame is free while the current one runs and its first
        operand sums can ride on the current frame's product launches
        (_hoist_sums looks back across groups).  The odd arena starts above
        everything planned before its first use; overlap between later frames
        would only block rides (the hoist tests the windows), never correctness."""
        if self.frames % 2 == 1:
            if self.arena1 is None:
                self.arena1 = self.ws_peak
            self.frame_off = self.arena1 - self.ws_floor
        else:
            self.frame_off = 0
        self.ws_top = self.ws_floor + self.frame_off
        self.frames += 1

    def node(self, a, b, m, n, k, out, sign, accumulate, depth, level=0):
        """Depth-first at this node when its breadth-first workspace exceeds the budget."""
        need = self._dry_ws(a, b, m, n, k, depth)
        # (the budget decides breadth- vs depth-first as without riding sums: the
        # second copies of alternating regions do not count against it)
        if (self.ws_top - self.frame_off - self.flip_extra + need <= self.budget
                or not self.worth_split(m, n, k, depth)):
            leaves, posts = [], []
            mark = self.ws_top
            if self._riding() and need > 0:
                # the next subtree's operand sums are computed while this one's
                # products run: successive subtrees use alternate scratch regions
                self.ws_top = mark + self.flip_tree * need
                self.ws_peak = max(self.ws_peak, mark + 2 * need)
                self.flip_tree ^= 1
            self.defer_sums = []
            self.tree(a, b, m, n, k, out, sign, accumulate, depth, leaves, posts)
            self.emit(leaves, posts)
            self.ws_top = mark
            return
        mark = self.ws_top
        if self._riding() and level >= 1:
            # likewise the operand sums of successive depth-first nodes below the top
            # (the products still running may read the previous node's sums through views)
            ext = 5 * _ceil2(m) * (_ceil2(n) + _ceil2(k))
            self.ws_top = mark + self.flip_sums * ext
            self.flip_sums ^= 1
            S, T, m1, n1, k1 = self._sums(a, b, m, n, k)
            self.ws_top = mark + 2 * ext
            self.ws_peak = max(self.ws_peak, self.ws_top)
            self.flip_extra += ext
        else:
            ext = 0
            S, T, m1, n1, k1 = self._sums(a, b, m, n, k)
        kids = [self.alloc(n1, k1) for _ in range(7)]
        for i in range(7):
            self.node(S[i], T[i], m1, n1, k1, kids[i], 1.0, False, depth - 1, level + 1)
        self._post(kids, out, sign, n1, k1, accumulate)
        self.ws_top = mark
        self.flip_extra -= ext

    def _dry_ws(self, a, b, m, n, k, depth) -> int:
        probe = _AutoPlanner(self.p)
        probe.rate, probe.esize = self.rate, self.esize
        leaves = []
        probe.tree(a, b, m, n, k, Win(nat.BASE_C, 0, max(k, 1), n, k), 1.0, True, depth, leaves, [])
        extra = 0
        if self.esize == 8 and self.p.tail_split and self.p.tail_private and len(leaves) > 1:
            # room for the private partials of a large group's K-split tail (emit_products:
            # the trailing products covering one wave of tiles, TAIL_CHUNKS partials each)
            nk = max(lf[1] * lf[2] for lf in leaves)
            extra = TAIL_CHUNKS * (NUM_SMS * TILE * TILE + 2 * nk)
        return probe.ws_peak + extra

    def ata(self, m: int, n: int, lda: int, ldc: int, round_tf32: bool = False):
        A = Win(nat.BASE_A, 0, lda, m, n)
        C = Win(nat.BASE_C, 0, ldc, n, n)
        if round_tf32:
            self.rate, self.esize, self.fill_waves = self.p.tf32_tflops, 4, self.p.tf32_fill_waves
            self.tile = (128, 256)
            # single-pass TF32: products read a TF32-rounded copy of A with a
            # 128-byte-aligned pitch (TMA-legal), written once by ATA_OP_ROUND
            ld = -(-n // 32) * 32
            R = Win(nat.BASE_WS, self.ws_top, ld, m, n)
            self.ws_top += m * ld
            self.ws_peak = max(self.ws_peak, self.ws_top)
            self.pb.round_tf32(A, R)
            A = R
            self.ws_floor = self.ws_top
        self.budget = int(self.p.ws_budget_gb * 1e9 / 8)
        self.ata_win(A, C)

    def ata_win(self, A: Win, C: Win):
        """lower(C) += A^T A for an A window (m x n) and the n x n C window at
        its diagonal position: the column recursion of ata() on windows (the
        multi-GPU unit planner runs it on row chunks and column halves)."""
        m, n = A.rows, A.cols
        # the diagonal SYRK leaves depend only on A: they join the first
        # breadth-first leaf group (more tiles per launch), else run last
        diag, level = [], [(0, n)]
        while level:
            nxt = []
            for (c0, w) in level:
                if w <= self.p.leaf_cols or w < 2:
                    diag.append((c0, w))
                else:
                    nxt += [(c0, w // 2), (c0 + w // 2, w - w // 2)]
            level = nxt
        diag_prods = [("syrk", m, w, w, A.sub(0, c0, m, w), None, C.sub(c0, c0, w, w), 1.0, True)
                      for (c0, w) in sorted(diag)]
        level = [(0, n)]
        while level:
            blocks, nxt = [], []
            for (c0, w) in level:
                if w <= self.p.leaf_cols or w < 2:
                    continue
                n1 = w // 2
                n2 = w - n1
                blocks.append((A.sub(0, c0 + n1, m, n2), A.sub(0, c0, m, n1),
                               C.sub(c0 + n1, c0, n2, n1)))
                nxt += [(c0, n1), (c0 + n1, n2)]
            if blocks:
                # the C21 blocks of one AtA level are disjoint: one breadth-first
                # leaf group for the whole level when it fits the budget
                need = sum(self._dry_ws(a, b, a.rows, a.cols, b.cols, self.p.max_depth)
                           for (a, b, _) in blocks)
                if need <= self.budget:
                    leaves, posts = [], []
                    if self._arenas():
                        self._enter_frame()
                    elif self._riding() and 0 < need <= self.budget // 4:
                        # alternate scratch regions for successive levels (see node())
                        self.ws_top = self.ws_floor + self.flip_tree * need
                        self.ws_peak = max(self.ws_peak, self.ws_floor + 2 * need)
                        self.flip_tree ^= 1
                    self.defer_sums = []
                    for (a, b, c) in blocks:
                        self.tree(a, b, a.rows, a.cols, b.cols, c, 1.0, True, self.p.max_depth,
                                  leaves, posts)
                    self.emit(leaves, posts, diag_prods)
                    diag_prods = []
                    self.ws_top, self.frame_off = self.ws_floor, 0
                else:
                    if diag_prods and self._riding() and self.p.diag_first and not self.pb.rows:
                        self.emit_products(diag_prods)     # nothing before it: the first launch
                        diag_prods = []
                    for (a, b, c) in blocks:
                        if self._arenas():
                            self._enter_frame()
                        self.node(a, b, a.rows, a.cols, b.cols, c, 1.0, True, self.p.max_depth)
                        self.ws_top, self.frame_off = self.ws_floor, 0
            level = nxt
        self.emit_products(diag_prods)


def _op_spans(ops, idx):
    """(read intervals, write intervals) of ops[idx] as int64 arrays [k, 3] of
    (base, first element, one past the last element): bounding intervals of the
    windows (exact for dense blocks, conservative for strided views)."""
    def spans(refs):
        refs = refs[(refs["rows"] > 0) & (refs["cols"] > 0)]
        lo = refs["off"].astype(np.int64)
        hi = lo + (refs["rows"].astype(np.int64) - 1) * refs["ld"].astype(np.int64) + refs["cols"]
        return np.stack([refs["base"].astype(np.int64), lo, hi], axis=1) if len(refs) else np.zeros((0, 3), np.int64)
    op = ops[idx]
    ns, nt, nd = int(op["ns"]), int(op["nt"]), int(op["nd"])
    reads = [spans(op["s"][:ns])]
    if int(op["type"]) in (nat.OP_GEMM, nat.OP_POSTADD7):
        reads.append(spans(op["t"][:nt]))
    return np.concatenate(reads), spans(op["d"][:nd])


def _hit(a, b) -> bool:
    """Any interval of a overlaps any interval of b (same base)."""
    if not len(a) or not len(b):
        return False
    return bool(((a[:, None, 0] == b[None, :, 0]) & (a[:, None, 1] < b[None, :, 2]) &
                 (b[None, :, 1] < a[:, None, 2])).any())


def _op_bytes(op, esize: int = 8) -> int:
    refs = list(op["s"][:int(op["ns"])]) + list(op["d"][:int(op["nd"])])
    return esize * sum(int(r["rows"]) * int(r["cols"]) for r in refs)


def _split_bands(op, band_rows: int, group: int):
    """Row bands of one full-extent COMBO4 op (sources zero-extended below their
    own extents, as in the whole op): independent ops writing disjoint row ranges."""
    rows = max(int(d["rows"]) for d in op["d"][:int(op["nd"])])
    out = []
    for r0 in range(0, rows, band_rows):
        h = min(band_rows, rows - r0)
        b = op.copy()
        b["group"] = group
        for key, cnt in (("s", int(op["ns"])), ("d", int(op["nd"]))):
            for j in range(cnt):
                ref = b[key][j]
                keep = max(0, min(h, int(ref["rows"]) - r0))
                if keep == 0:
                    ref["rows"], ref["cols"] = 0, 0
                else:
                    ref["off"] = int(ref["off"]) + r0 * int(ref["ld"])
                    ref["rows"] = keep
        out.append(b)
    return out


def _hoist_sums(ops, ride_gbs: float = 800.0, tflops: float = 35.0, lookback: int = 0,
                band_gb: float = 0.0):
    """Reorder a plan for riding operand sums (AutoParams.ride_sums).

    Between the end of a product group G and the start of the next one lie G's
    post-additions and the operand sums (COMBO4) of the next group.  Every such
    COMBO4 that is independent of G and of the ops between G and itself -- it
    writes nothing they read or write and reads nothing they write -- is moved
    directly in front of G and flagged ATA_OPF_RIDE: the executor then runs it
    inside G's launch, on the FP64 leaf kernel's spare warps, instead of as an HBM
    pass of its own between the two product launches.  The sequential meaning of
    the op list is unchanged (only independent ops are reordered).  A group carries
    at most ride_gbs x its own duration (flops / tflops) of additions: beyond
    that the ride outlasts the products and separate passes are faster.

    lookback > 0: a sum may also ride on one of the `lookback` groups before G, as
    far back as it stays independent of everything it jumps over; it takes the
    EARLIEST such group with room (sums that can only ride on G itself -- the next
    subtree's, whose scratch region the group before G still uses -- then find G's
    room free).  band_gb > 0: sums larger than that are first cut into row bands
    (independent ops of one launch group), so the sums of the upper tree levels,
    larger than any one group's room, spread over the groups before them."""
    n = len(ops)
    types, groups = ops["type"], ops["group"]
    prod = (types == nat.OP_GEMM) | (types == nat.OP_SYRK)

    def find_spans():
        spans, i = [], 0
        while i < n:
            if prod[i] and groups[i] >= 0:
                j = i + 1
                while j < n and prod[j] and groups[j] == groups[i]:
                    j += 1
                spans.append((i, j))
                i = j
            else:
                i += 1
        return spans
    spans = find_spans()
    if len(spans) < 2:
        return ops
    if band_gb > 0:
        # cut the big candidates (after the first group, before the last) into row bands
        rows_out, next_group = [], int(groups.max()) + 1
        first, last = spans[0][1], spans[-1][0]
        for q in range(n):
            op = ops[q]
            if (first <= q < last and int(types[q]) == nat.OP_COMBO4 and int(op["accumulate"]) == 0
                    and _op_bytes(op) > band_gb * 1e9):
                nd = int(op["nd"])
                rows = max(int(d["rows"]) for d in op["d"][:nd])
                full = all(int(d["rows"]) == rows for d in op["d"][:nd])
                band_rows = max(64, int(rows * band_gb * 1e9 / _op_bytes(op)) // 64 * 64)
                if full and band_rows < rows:
                    g = int(op["group"])
                    if g < 0:
                        g, next_group = next_group, next_group + 1
                    rows_out += _split_bands(op, band_rows, g)
                    continue
            rows_out.append(op)
        ops = np.array(rows_out, dtype=ops.dtype)
        n = len(ops)
        types, groups = ops["type"], ops["group"]
        prod = (types == nat.OP_GEMM) | (types == nat.OP_SYRK)
        spans = find_spans()
    empty = np.zeros((0, 3), np.int64)

    class Seg:       # one product group, the sums riding on it and the ops that stay behind it
        def __init__(self, g0, g1):
            rw = [_op_spans(ops, q) for q in range(g0, g1)]
            self.g0, self.g1 = g0, g1
            self.reads = np.concatenate([r for r, _ in rw])      # group + stays
            self.writes = np.concatenate([w for _, w in rw])
            self.r_reads, self.r_writes = empty, empty           # riders
            self.riders, self.stays = [], []
            flops = sum(2.0 * int(o["m"]) * int(o["n"]) * int(o["k"]) if int(o["type"]) == nat.OP_GEMM
                        else 1.0 * int(o["m"]) * int(o["n"]) * (int(o["n"]) + 1) for o in ops[g0:g1])
            self.room = ride_gbs * 1e9 * flops / (tflops * 1e12)  # bytes this group can hide

    def clear(r, w, reads, writes):
        return not _hit(w, reads) and not _hit(w, writes) and not _hit(r, writes)
    segs = [Seg(g0, g1) for (g0, g1) in spans]
    for si, seg in enumerate(segs):
        nxt = spans[si + 1][0] if si + 1 < len(spans) else n
        for q in range(seg.g1, nxt):
            r, w = _op_spans(ops, q)
            best = None
            if int(types[q]) == nat.OP_COMBO4 and int(ops[q]["accumulate"]) == 0:
                size, sj = _op_bytes(ops[q]), si
                ok = clear(r, w, seg.reads, seg.writes)
                while ok:
                    if size <= segs[sj].room:
                        best = sj
                    if sj == 0 or si - sj >= lookback:
                        break
                    # one group earlier: past the riders of sj and the group + stays of sj - 1
                    ok = (clear(r, w, segs[sj].r_reads, segs[sj].r_writes) and
                          clear(r, w, segs[sj - 1].reads, segs[sj - 1].writes))
                    sj -= 1
            if best is None:
                seg.stays.append(q)
                seg.reads = np.concatenate([seg.reads, r])
                seg.writes = np.concatenate([seg.writes, w])
            else:
                t = segs[best]
                t.room -= size
                t.riders.append(q)
                t.r_reads = np.concatenate([t.r_reads, r])
                t.r_writes = np.concatenate([t.r_writes, w])
    order, ride = list(range(spans[0][0])), set()
    for seg in segs:
        order += seg.riders + list(range(seg.g0, seg.g1)) + seg.stays
        ride.update(seg.riders)
    out = ops[np.asarray(order, dtype=np.int64)].copy()
    flag = np.asarray([q in ride for q in order])
    out["flags"][flag] |= nat.OPF_RIDE
    return out


def _finish(ap) -> Plan:
    plan = ap.pb.finish()
    plan.ws_scalars = max(plan.ws_scalars, ap.ws_peak)
    if ap.p.ride_sums and ap.esize == 8:
        plan.ops = _hoist_sums(plan.ops, ap.p.ride_gbs, ap.p.dmma_tflops, ap.p.ride_lookback, ap.p.ride_band_gb)
    return plan


RING_PIECE_ROWS = 192    # scratch sized for pieces of up to 192 rows (tc2::PR, gemm_tf32_2sm.cu)
RING_SLOTS = 64   # scratch for up to 64 slots per ring (the kernel uses TC2_RING_SLOTS)


def _tc2_tiles(kind: int, n: int, k: int) -> int:
    """256 x 256 CTA-pair tiles of one product (gemm_tf32_2sm.cu t2_decode)."""
    tn, tk = -(-n // 256), -(-k // 256)
    return tn * (tn + 1) // 2 if kind == nat.OP_SYRK else tn * tk


def _ringify(plan: Plan, m: int, n: int, lda: int) -> Plan:
    """Single-pass TF32 plan [ROUND A -> R, one product group over row chunks of
    R, partial sums]: when the product group is chunk-major with equal chunks,
    an even chunk count and two chunks per wave of the CTA-pair kernel's
    persistent grid (25..37 tiles per chunk on 74 pairs), the products read
    A's raw rows and the ROUND op becomes the kernel's L2 rounding ring
    (accumulate = 2, d[0] = a ~50 MB ring scratch in the rounded copy's
    former workspace region): no rounded copy of A is written to HBM.
    Otherwise the plan is returned unchanged."""
    ops = plan.ops
    if len(ops) < 2 or int(ops[0]["type"]) != nat.OP_ROUND or lda % 4 or n % 32:
        return plan
    if os.environ.get("ATA_TF32_TC", "2") != "2":   # only the CTA-pair kernel has the ring
        return plan
    src, dst = ops[0]["s"][0], ops[0]["d"][0]
    if int(dst["ld"]) != lda or int(src["base"]) != nat.BASE_A or int(src["off"]) != 0:
        return plan
    prods = [i for i in range(1, len(ops)) if int(ops[i]["type"]) in (nat.OP_GEMM, nat.OP_SYRK)]
    if not prods or prods != list(range(1, 1 + len(prods))) or len(prods) > MAX_BATCH:
        return plan
    if len({int(ops[i]["group"]) for i in prods}) != 1:
        return plan
    r_off, r_end = int(dst["off"]), int(dst["off"]) + m * lda
    chunk_rows, chunks, tiles = None, [], {}
    for i in prods:
        op = ops[i]
        if int(op["ns"]) != 1 or (int(op["type"]) == nat.OP_GEMM and int(op["nt"]) != 1):
            return plan
        terms = [op["s"][0]] + ([op["t"][0]] if int(op["type"]) == nat.OP_GEMM else [])
        rows0 = None
        for t in terms:
            if int(t["base"]) != nat.BASE_WS or not r_off <= int(t["off"]) < r_end or int(t["ld"]) != lda:
                return plan
            row = (int(t["off"]) - r_off) // lda
            chunk_rows = chunk_rows or int(t["rows"])
            if int(t["rows"]) != chunk_rows or row % chunk_rows or (rows0 is not None and row != rows0):
                return plan
            rows0 = row
        c = rows0 // chunk_rows
        if chunks and c not in (chunks[-1], chunks[-1] + 1):
            return plan
        chunks.append(c)
        tiles[c] = tiles.get(c, 0) + _tc2_tiles(int(op["type"]), int(op["n"]), int(op["k"]))
    tpc = set(tiles.values())
    nch = len(tiles)
    if len(tpc) != 1 or nch % 2 or chunk_rows * nch != m or not 25 <= next(iter(tpc)) <= 37:
        return plan
    out = ops.copy()
    ring_elems = 2 * RING_SLOTS * RING_PIECE_ROWS * n + 4 * RING_SLOTS
    out[0]["accumulate"] = 2
    if -(-ring_elems // n) * n > m * lda:
        return plan
    out[0]["d"][0]["off"] = r_off
    out[0]["d"][0]["ld"] = n
    out[0]["d"][0]["rows"] = -(-ring_elems // n)
    out[0]["d"][0]["cols"] = n
    for i in prods:
        for fld, cnt in (("s", int(out[i]["ns"])), ("t", int(out[i]["nt"]))):
            for j in range(cnt):
                t = out[i][fld][j]
                t["base"] = nat.BASE_A
                t["off"] = int(t["off"]) - r_off
    return Plan(out, plan.mults, plan.ws_scalars, plan.launches - 1, plan.kind)


def plan_ata_auto(m: int, n: int, lda: int, ldc: int, params: AutoParams = AutoParams(),
                  round_tf32: bool = False) -> Plan:
    """GPU plan for lower(C) += alpha A^T A (see module docstring).  round_tf32:
    single-pass TF32 plans (fp32 data, precision="tf32") first round A once."""
    if m < 1 or n < 1:
        raise ShapeMismatchError("shape mismatch: empty operand")
    ap = _AutoPlanner(params)
    ap.ata(m, n, lda, ldc, round_tf32)
    plan = _finish(ap)
    if round_tf32 and params.tf32_ring:
        plan = _ringify(plan, m, n, lda)
    return plan


def plan_gemm_auto(m: int, n: int, k: int, lda: int, ldb: int, ldc: int,
                   params: AutoParams = AutoParams()) -> Plan:
    """GPU plan for C (n x k) += alpha A^T B (fast_strassen with threshold
    "auto"; the A^T B leaves of the multi-GPU task tree): one Strassen tree
    chosen by the same cost model as the C21 blocks of plan_ata_auto, breadth
    first when its workspace fits the budget."""
    if min(m, n, k) < 1:
        raise ShapeMismatchError("shape mismatch: empty operand")
    ap = _AutoPlanner(params)
    ap.budget = int(params.ws_budget_gb * 1e9 / 8)
    A = Win(nat.BASE_A, 0, lda, m, n)
    B = Win(nat.BASE_B, 0, ldb, m, k)
    C = Win(nat.BASE_C, 0, ldc, n, k)
    ap.node(A, B, m, n, k, C, 1.0, True, params.max_depth)
    return _finish(ap)


# --------------------------------------------------------------------------
# Multi-GPU "units" partition (north star: the independent AtA sub-problems
# and the seven Strassen sub-products of the top level on different ranks).
#
# The top level of plan_ata_auto is: C11 += A_L^T A_L, C22 += A_R^T A_R (two
# AtA units, A_L / A_R the column halves) and C21 += A_R^T A_L, a Strassen
# node whose seven products P_i = S_i^T T_i (S_i, T_i signed sums of the
# quadrants of A_R and A_L, contraction = the top half's m1 rows) are
# combined into the four quadrants of C21 (strassen.py:234-275).  All nine
# units are sums over contraction rows, so any row range of a unit is an
# independent piece of work whose result simply adds into C: ranks receive
# contiguous row ranges of the unit sequence, balanced by the planner's own
# executed-multiplication counts, and a sum of the ranks' C triangles (one
# NCCL reduce) combines them -- each P_i is added with its sign into its C21
# quadrants on the rank that computes it.

UNITS = ("ata_l", "ata_r", "p1", "p2", "p3", "p4", "p5", "p6", "p7")
# destinations of P_i among the C21 quadrants (0 = C11, 1 = C12, 2 = C21,
# 3 = C22) with signs: C11 = P1+P4-P5+P7, C12 = P3+P5, C21 = P2+P4,
# C22 = P1-P2+P3+P6
_PDEST = [((0, 1.0), (3, 1.0)), ((2, 1.0), (3, -1.0)), ((1, 1.0), (3, 1.0)), ((0, 1.0), (2, 1.0)),
          ((0, -1.0), (1, 1.0)), ((3, 1.0),), ((0, 1.0),)]


def unit_geometry(m: int, n: int):
    """(n1, n2, m1): column halves of the top AtA level (floor first, as
    plan_ata_auto) and the ceil half of the contraction of the C21 node."""
    n1 = n // 2
    return n1, n - n1, _ceil2(m)


def unit_rows(unit: str, m: int, n: int) -> int:
    """Contraction rows of a unit: m for the AtA units, m1 for the products."""
    return m if unit in ("ata_l", "ata_r") else unit_geometry(m, n)[2]


def a_rows_needed(segments, m: int, n: int):
    """Row ranges of A a rank's segments read (a product's row r of the top
    half pairs with row m1 + r of the bottom half)."""
    m1 = unit_geometry(m, n)[2]
    out = []
    for (u, r0, r1) in segments:
        out.append((r0, r1))
        if u not in ("ata_l", "ata_r"):
            lo, hi = m1 + r0, min(m, m1 + r1)
            if lo < hi:
                out.append((lo, hi))
    out.sort()
    merged = []
    for lo, hi in out:
        if merged and lo <= merged[-1][1]:
            merged[-1] = (merged[-1][0], max(merged[-1][1], hi))
        else:
            merged.append((lo, hi))
    return merged


class _UnitPlanner(_AutoPlanner):
    def segment(self, unit: str, r0: int, r1: int, A: Win, C: Win, m: int, n: int):
        n1, n2, m1 = unit_geometry(m, n)
        rows = r1 - r0
        if rows <= 0:
            return
        # a piece keeps the Strassen tree of its whole unit (cost model at the unit's
        # rows, like the host pipeline's row blocks): the pieces of a unit together
        # execute the unit's multiplications, so equal rows are equal work
        keep = self.p
        self.p = dataclasses.replace(keep, cost_row_scale=keep.cost_row_scale * unit_rows(unit, m, n) / rows,
                                     min_leaf_rows=max(keep.min_leaf_rows, UNIT_MIN_LEAF_ROWS))
        try:
            self._segment(unit, r0, rows, A, C, m, n)
        finally:
            self.p = keep

    def _segment(self, unit: str, r0: int, rows: int, A: Win, C: Win, m: int, n: int):
        n1, n2, m1 = unit_geometry(m, n)
        mark = self.ws_top
        if unit == "ata_l":
            self.ata_win(A.sub(r0, 0, rows, n1), C.sub(0, 0, n1, n1))
        elif unit == "ata_r":
            self.ata_win(A.sub(r0, n1, rows, n2), C.sub(n1, n1, n2, n2))
        else:
            i = UNITS.index(unit) - 2
            a, b = A.sub(0, n1, m, n2), A.sub(0, 0, m, n1)          # C21 += A_R^T A_L
            out = C.sub(n1, 0, n2, n1)
            q1, k1 = _ceil2(n2), _ceil2(n1)
            X = [_clip(w, r0, 0, rows, w.cols) for w in _quads(a, m1, q1)]
            Y = [_clip(w, r0, 0, rows, w.cols) for w in _quads(b, m1, k1)]
            S = self._operand(X, _S[i], rows, q1)
            T = self._operand(Y, _T[i], rows, k1)
            outq = [_clip(out, 0, 0, q1, k1), _clip(out, 0, k1, q1, k1), _clip(out, q1, 0, q1, k1),
                    _clip(out, q1, k1, q1, k1)]
            dests = [(outq[d], sg) for (d, sg) in _PDEST[i] if outq[d].rows and outq[d].cols]
            if dests and not (_empty(S) or _empty(T)):
                depth = self.p.max_depth - 1
                if len(dests) == 1:
                    self.node(S, T, rows, q1, k1, dests[0][0], dests[0][1], True, depth)
                else:
                    P = self.alloc(q1, k1)
                    self.node(S, T, rows, q1, k1, P, 1.0, False, depth)
                    self.pb.update(P, dests)
        self.ws_top = mark

    def _operand(self, quads, coef, rows, cols):
        """S_i / T_i over the segment's rows: a quadrant view, or one combo4
        pass writing the signed sum into scratch."""
        if sorted(coef) == [0, 0, 0, 1]:
            return quads[coef.index(1)]
        buf = self.alloc(rows, cols)
        self.pb.combo4(quads, [(buf, coef)])
        return buf


def plan_units(segments, m: int, n: int, lda: int, ldc: int, params: AutoParams = AutoParams()) -> Plan:
    """One rank's plan of the units partition: lower(C) += the rank's
    segments [(unit, r0, r1)] (contraction rows [r0, r1) of a UNITS entry).
    Over all ranks' segments the sum is lower(A^T A)."""
    if m < 2 or n < 2:
        raise ShapeMismatchError("shape mismatch: the units partition needs m, n >= 2")
    up = _UnitPlanner(params)
    up.budget = int(params.ws_budget_gb * 1e9 / 8)
    A = Win(nat.BASE_A, 0, lda, m, n)
    C = Win(nat.BASE_C, 0, ldc, n, n)
    for (u, r0, r1) in segments:
        if u not in UNITS:
            raise ValueError(f"unknown unit {u!r}")
        up.segment(u, r0, r1, A, C, m, n)
    return _finish(up)


def unit_costs(m: int, n: int, params: AutoParams = AutoParams()):
    """Executed multiplications per contraction row of each unit (the
    planner's own count at the unit's full row extent)."""
    out = {}
    for u in UNITS:
        rows = unit_rows(u, m, n)
        p = plan_units([(u, 0, rows)], m, n, n, n, params)
        out[u] = p.mults / rows
    return out


def partition_units(m: int, n: int, procs: int, params: AutoParams = AutoParams(), align: int = 256,
                    costs=None):
    """Split the unit sequence (UNITS order, each unit's rows in order) into
    `procs` contiguous pieces of equal executed multiplications.  Each cut is
    rounded to `align` rows and snapped to the unit's edge when it would leave
    a piece shorter than `align` rows.  Returns per rank [(unit, r0, r1)]."""
    costs = costs or unit_costs(m, n, params)
    ext = [(u, unit_rows(u, m, n), costs[u]) for u in UNITS]
    total = sum(rows * c for (_, rows, c) in ext)

    def position(work):
        """(unit index, row) where the cumulative work reaches `work`."""
        before = 0.0
        for ui, (u, rows, c) in enumerate(ext):
            span = rows * c
            if work < before + span:
                r = int(round((work - before) / c / align)) * align
                if r < align:
                    return (ui, 0)
                if rows - r < align:
                    return (ui + 1, 0)
                return (ui, r)
            before += span
        return (len(ext), 0)

    cuts = [(0, 0)] + [position(total * j / procs) for j in range(1, procs)] + [(len(ext), 0)]
    for j in range(1, len(cuts)):                       # monotone after rounding
        cuts[j] = max(cuts[j], cuts[j - 1])
    ranks = []
    for (u0, r0), (u1, r1) in zip(cuts, cuts[1:]):
        segs = []
        ui, r = u0, r0
        while (ui, r) < (u1, r1):
            u, rows, _ = ext[ui]
            end = r1 if ui == u1 else rows
            if end > r:
                segs.append((u, r, end))
            ui, r = ui + 1, 0
        ranks.append(segs)
    return ranks
