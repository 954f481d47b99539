"""The GPU plan for ``threshold="auto"`` (config c3/c4/c5 style workloads).

Shape of the plan (all windows into A, C and one HBM workspace):

1. AtA column recursion (ata.py:110-115): C11 <- A_l^T A_l, C22 <- A_r^T A_r,
   C21 <- A_r^T A_l, recursing on the diagonal blocks down to ``leaf_cols``.
   The reference also halves the rows (the contraction) at every level; on
   the GPU the contraction stays whole inside each product's K loop, so the
   two C21 addends of ata.py:114-115 are one product over all m rows.
2. Every C21 product is a breadth-first Strassen tree (strassen.py:234-275)
   of depth up to ``max_depth``, chosen per node from a cost model (flops
   saved at the measured DMMA rate vs. bytes moved by the operand sums at HBM
   rate):
     * the operand sums of a node (5 S-sums, 5 T-sums; the other 4 operands
       are plain quadrant views) are written by ONE multi-output combo kernel
       per operand (reads each quadrant once) into the workspace;
     * leaf products read plain windows (1 term per operand) and their
       post-additions are fused into the epilogue: a depth-d leaf writes its
       signed contribution straight into up to 2^d C sub-blocks (no product
       buffers, no update kernels);
     * leaves of one subtree share launches of the persistent product kernel;
       C sub-blocks written by several leaves are ordered regions
       (deterministic accumulation in product order).
   Quadrant splits are ceil-first (first half = ceil, the second half is the
   zero-extended one), so every node of a level has identical product shapes
   and every C sub-block has a single origin shared by all its writers.
3. Diagonal leaves are SYRK-lower products, one group.

Exact arithmetic is the reference's (zero-extended Strassen, classical
leaves); only the recursion shape differs from an integer-threshold run,
hence the multiplication count differs (reported as plan.mults).
"""
from __future__ import annotations

from dataclasses import dataclass

from . import _native as nat
from .errors import ShapeMismatchError
from .planner import Plan, PlanBuilder, Win

# Strassen in the transposed orientation (strassen.py:234-275) for
# c = a^T b, quadrants X11 X12 / X21 X22 (rows = contraction):
#   P1 = (A11+A22)^T (B11+B22) -> +C11 +C22
#   P2 = (A12+A22)^T  B11      -> +C21 -C22
#   P3 =  A11^T (B12-B22)      -> +C12 +C22
#   P4 =  A22^T (B21-B11)      -> +C11 +C21
#   P5 = (A11+A21)^T  B22      -> -C11 +C12
#   P6 = (A12-A11)^T (B11+B12) -> +C22
#   P7 = (A21-A22)^T (B21+B22) -> +C11
# Operand coefficient vectors over (X11, X12, X21, X22):
_S = [(1, 0, 0, 1), (0, 1, 0, 1), (1, 0, 0, 0), (0, 0, 0, 1), (1, 0, 1, 0), (-1, 1, 0, 0),
      (0, 0, 1, -1)]
_T = [(1, 0, 0, 1), (1, 0, 0, 0), (0, 1, 0, -1), (-1, 0, 1, 0), (0, 0, 0, 1), (1, 1, 0, 0),
      (0, 0, 1, 1)]
# destinations: (quadrant index 0..3 = C11, C12, C21, C22, sign)
_D = [[(0, 1), (3, 1)], [(2, 1), (3, -1)], [(1, 1), (3, 1)], [(0, 1), (2, 1)],
      [(0, -1), (1, 1)], [(3, 1)], [(0, 1)]]


@dataclass(frozen=True)
class AutoParams:
    leaf_cols: int = 1024          # SYRK leaf width of the column recursion
    max_depth: int = 3             # Strassen levels per C21 product (dests <= 2^depth <= 8)
    min_dim: int = 512             # never split a Strassen node below this output side
    dmma_tflops: float = 33.5      # measured product-kernel rate (profiles/)
    hbm_gbs: float = 5500.0        # achieved combo-kernel bandwidth (profiles/)
    gain: float = 1.5              # split only when saved time > gain * added time
    ws_budget_gb: float = 40.0     # breadth-first operand sums of one AtA level up to this size


def _ceil2(d: int) -> int:
    return (d + 1) // 2


def _quads(w: Win, r1: int, c1: int):
    """Ceil-first quadrants of a window whose logical extent is (2*r1) x (2*c1);
    quadrants beyond the actual extent are empty windows (zero-extended)."""
    def clip(r0, c0, h, wd):
        h = max(0, min(h, w.rows - r0))
        wd = max(0, min(wd, w.cols - c0))
        if h == 0 or wd == 0:
            return Win(w.base, w.off, w.ld, 0, 0)
        return w.sub(r0, c0, h, wd)
    return [clip(0, 0, r1, c1), clip(0, c1, r1, c1), clip(r1, 0, r1, c1), clip(r1, c1, r1, c1)]


class _AutoPlanner:
    def __init__(self, params: AutoParams):
        self.p = params
        self.pb = PlanBuilder("auto")
        self.ws_top = 0          # bump allocator over the workspace (elements)
        self.ws_peak = 0
        self.region_of = {}      # (base, off) -> region id, per leaf group

    # ---------------------------------------------------------------- workspace
    def alloc(self, rows: int, cols: int) -> Win:
        w = Win(nat.BASE_WS, self.ws_top, cols, rows, cols)
        self.ws_top += rows * cols
        self.ws_peak = max(self.ws_peak, self.ws_top)
        return w

    # ------------------------------------------------------------- cost model
    def worth_split(self, m: int, n: int, k: int, depth_left: int) -> bool:
        if depth_left <= 0 or min(n, k) < 2 * self.p.min_dim or m < 2:
            return False
        saved_s = 2.0 * m * n * k / 8 / (self.p.dmma_tflops * 1e12)
        # one multi-output combo per operand: read the whole operand, write 5 quarter sums
        moved = 8.0 * (m * n * (1 + 5 / 4) + m * k * (1 + 5 / 4))
        added_s = moved / (self.p.hbm_gbs * 1e9)
        return saved_s > self.p.gain * added_s

    # --------------------------------------------------------------- Strassen
    def split(self, a: Win, b: Win, m: int, n: int, k: int, dests):
        """Emit one node's operand sums; return its 7 children as
        (a, b, m, n, k, dests) with composed destinations."""
        m1, n1, k1 = _ceil2(m), _ceil2(n), _ceil2(k)
        Aq = _quads(a, m1, n1)
        Bq = _quads(b, m1, k1)
        S = [None] * 7
        T = [None] * 7
        for X, coefs, out, rows, cols in ((Aq, _S, S, m1, n1), (Bq, _T, T, m1, k1)):
            outs = []
            for i, coef in enumerate(coefs):
                if sorted(coef) == [0, 0, 0, 1]:
                    out[i] = X[coef.index(1)]           # plain quadrant view
                else:
                    out[i] = self.alloc(rows, cols)
                    outs.append((out[i], coef))
            self.pb.combo4(X, outs)                     # one pass over the quadrants
        qoff = [(0, 0), (0, k1), (n1, 0), (n1, k1)]
        children = []
        for i in range(7):
            child = []
            for q, sg in _D[i]:
                r0, c0 = qoff[q]
                for (W, s) in dests:
                    h = min(n1, W.rows - r0)
                    wd = min(k1, W.cols - c0)
                    if h > 0 and wd > 0:
                        child.append((W.sub(r0, c0, h, wd), s * sg))
            if child:
                children.append((S[i], T[i], m1, n1, k1, child))
        return children

    def strassen(self, a: Win, b: Win, m: int, n: int, k: int, dests, depth_left: int, leaves):
        """Plan c (+)= a^T b for LOGICAL extents m x n (a), m x k (b): windows may be
        smaller (zero-extended).  dests = [(C window, sign)], origin = product (0,0)."""
        if not self.worth_split(m, n, k, depth_left):
            leaves.append((m, n, k, a, b, dests))
            return
        for ch in self.split(a, b, m, n, k, dests):
            self.strassen(*ch, depth_left - 1, leaves)

    def emit_leaves(self, leaves):
        group = self.pb.new_group()
        regions = {}
        for (m, n, k, a, b, dests) in leaves:
            D = []
            for (W, s) in dests:
                key = (W.base, W.off)
                if key not in regions:
                    regions[key] = self.pb.new_region()
                D.append((W, s, regions[key]))
            S = [(a, 1.0)] if a.rows > 0 and a.cols > 0 else []
            T = [(b, 1.0)] if b.rows > 0 and b.cols > 0 else []
            if not S or not T:
                continue  # an all-zero operand contributes nothing
            self.pb.product("gemm", m, n, k, S, T, D, group=group)

    def _dry_ws(self, a: Win, b: Win) -> int:
        """Workspace a breadth-first plan of this block's Strassen tree needs."""
        probe = _AutoPlanner(self.p)
        probe.strassen(a, b, a.rows, a.cols, b.cols, [(Win(nat.BASE_C, 0, b.cols, a.cols, b.cols), 1.0)],
                       self.p.max_depth, [])
        return probe.ws_peak

    def atb(self, a: Win, b: Win, c: Win):
        """c += a^T b for one C21 block (a, b: m x n2 / m x n1 windows of A).
        Depth-first over the top node's 7 products: only one subtree's sums are
        alive beside the top-level sums; each subtree's leaves share launches."""
        m, n, k = a.rows, a.cols, b.cols
        depth = self.p.max_depth
        if not self.worth_split(m, n, k, depth):
            self.emit_leaves([(m, n, k, a, b, [(c, 1.0)])])
            return
        mark = self.ws_top
        for ch in self.split(a, b, m, n, k, [(c, 1.0)]):
            sub = self.ws_top
            leaves = []
            self.strassen(*ch, depth - 1, leaves)
            self.emit_leaves(leaves)
            self.ws_top = sub
        self.ws_top = mark

    def ata(self, m: int, n: int, lda: int, ldc: int):
        A = Win(nat.BASE_A, 0, lda, m, n)
        C = Win(nat.BASE_C, 0, ldc, n, n)
        level = [(0, n)]
        leaves = []
        budget = int(self.p.ws_budget_gb * 1e9 / 8)
        while level:
            blocks, nxt = [], []
            for (c0, w) in level:
                if w <= self.p.leaf_cols or w < 2:
                    leaves.append((c0, w))
                    continue
                n1 = w // 2
                n2 = w - n1
                blocks.append((A.sub(0, c0 + n1, m, n2), A.sub(0, c0, m, n1),
                               C.sub(c0 + n1, c0, n2, n1)))
                nxt += [(c0, n1), (c0 + n1, n2)]
            if blocks:
                # the C21 blocks of one AtA level are disjoint: plan them breadth-first
                # into ONE leaf group when their operand sums fit the workspace budget
                need = sum(self._dry_ws(a, b) for (a, b, _) in blocks)
                if need <= budget:
                    lv_leaves = []
                    for (a, b, c) in blocks:
                        self.strassen(a, b, a.rows, a.cols, b.cols, [(c, 1.0)], self.p.max_depth,
                                      lv_leaves)
                    self.emit_leaves(lv_leaves)
                    self.ws_top = 0  # stream order: the next level may reuse the sums
                else:
                    # top-child-major: all blocks' top-level sums, then subtree i of
                    # every block as one leaf group (only one subtree per block alive)
                    tops = []
                    for (a, b, c) in blocks:
                        m_, n_, k_ = a.rows, a.cols, b.cols
                        if self.worth_split(m_, n_, k_, self.p.max_depth):
                            tops.append(self.split(a, b, m_, n_, k_, [(c, 1.0)]))
                        else:
                            self.emit_leaves([(m_, n_, k_, a, b, [(c, 1.0)])])
                    mark = self.ws_top
                    for i in range(7):
                        lv_leaves = []
                        for children in tops:
                            if i < len(children):
                                self.strassen(*children[i], self.p.max_depth - 1, lv_leaves)
                        self.emit_leaves(lv_leaves)
                        self.ws_top = mark
                    self.ws_top = 0
            level = nxt
        group = self.pb.new_group()
        for (c0, w) in sorted(leaves):
            self.pb.product("syrk", m, w, w, [(A.sub(0, c0, m, w), 1.0)], [],
                            [(C.sub(c0, c0, w, w), 1.0)], group=group)


def plan_ata_auto(m: int, n: int, lda: int, ldc: int, params: AutoParams = AutoParams()) -> Plan:
    """GPU plan for lower(C) += alpha A^T A (see module docstring)."""
    if m < 1 or n < 1:
        raise ShapeMismatchError("shape mismatch: empty operand")
    ap = _AutoPlanner(params)
    ap.ata(m, n, lda, ldc)
    plan = ap.pb.finish()
    plan.ws_scalars = max(plan.ws_scalars, ap.ws_peak)
    return plan
