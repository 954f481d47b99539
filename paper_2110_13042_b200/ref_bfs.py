"""Breadth-first execution of the reference recursion (integer threshold).

The recursion TREE is the reference's, node for node: the AtA recursion of
ata.py:97-115 (floor/ceil halves, four AtA calls and two Strassen calls per
node, leaf predicate ata.py:23-26) and the Strassen recursion of
strassen.py:206-275 (floor-first quadrants, the seven products with the
reference's operand shapes including the contraction cut A22[:m1], leaf
predicate strassen.py:38-41).  Hence the same leaves, the same classical leaf
products and the same exact multiplication count as the reference (and as the
depth-first `planner._ReferencePlanner`).

What changes is the ORDER of execution.  The reference walks the tree depth
first with one scratch buffer per depth, so on a GPU every tiny node becomes
its own launch (config c2: 16586 ops, 8006 launches).  Here all Strassen calls
are expanded breadth first with private buffers per node:

  1. operand sums, top-down, one multi-node ``combo4`` launch per level
     (strassen.py:195-203; ``fused_leaves=True`` instead lets leaf children
     take their two-term operands fused into the product's tile load);
  2. all leaf products into private product buffers in few persistent
     launches (up to 48 products each);
  3. post-additions bottom-up, one multi-node ``postadd7`` launch per level
     (strassen.py:238-275: the same +/- combinations, one pass per node).

Destinations shared by several calls (the two Strassen calls of an AtA node,
and the AtA nodes of different row blocks writing the same C block) are
accumulated in "rounds": the r-th contribution to each C block runs in the
r-th launch, so no launch has two writers of one element and the summation
order is fixed (bitwise reproducible).  The diagonal SYRK leaves
(ata.py:100-101) are issued the same way.

Breadth-first needs more scratch than the reference's per-depth buffers: calls
are packed into waves whose scratch fits ``budget_scalars``; a call too large
for the budget is expanded one level depth-first (its seven children become
calls of their own).  The caller provides the scratch (plan.ws_scalars).
"""
from __future__ import annotations

from collections import defaultdict

from . import _native as nat
from .auto_plan import _S, _T
from .planner import Plan, PlanBuilder, Win, _strassen_products
from .workspace import is_ata_base_case, is_base_case

DEFAULT_BUDGET = 2_000_000_000      # scratch scalars per wave (16 GB of fp64)


class _Node:
    __slots__ = ("S", "T", "m", "n", "k", "out", "acc", "sign", "level", "kids", "sums", "merged")

    def __init__(self, S, T, m, n, k, out, acc, sign, level):
        self.S, self.T = S, T            # operand terms [(Win, sign)] (internal nodes: one view)
        self.m, self.n, self.k = m, n, k
        self.out, self.acc, self.sign = out, acc, sign
        self.level = level
        self.kids = None
        self.sums = None                 # (A quadrants, [(Win, coefs)], B quadrants, [(Win, coefs)])
        self.merged = False              # merged reference leaves: a leaf whatever its size


def _quads(w: Win, r1: int, c1: int):
    r2, c2 = w.rows - r1, w.cols - c1
    return [w.sub(0, 0, r1, c1), w.sub(0, c1, r1, c2), w.sub(r1, 0, r2, c1), w.sub(r1, c1, r2, c2)]


class _RefBFS:
    def __init__(self, threshold: int, budget: int = DEFAULT_BUDGET, fused_leaves: bool = False):
        self.t = int(threshold)
        self.budget = int(budget)
        # False: leaf children read materialized operand sums (one multi-node
        # combo4 pass per level; 1-term products run ~1.6x faster than the
        # 2-term fused loads at these small sizes -- tools/prof_small.py)
        self.fused_leaves = fused_leaves
        self.extra = []          # C writers joining the next leaf group (diagonal SYRKs)
        self.pb = PlanBuilder("reference")
        self.ws_top = 0
        self.ws_peak = 0

    # ------------------------------------------------------------ scratch
    def alloc(self, rows: int, cols: int) -> Win:
        # even pitch (16-byte rows): the TMA-fed FP64 leaf kernel's 2-D tensor maps
        # need it; one padding column per odd-width buffer, never read
        ld = max(cols + (cols & 1), 2)
        w = Win(nat.BASE_WS, self.ws_top, ld, rows, cols)
        self.ws_top += rows * ld
        self.ws_peak = max(self.ws_peak, self.ws_top)
        return w

    # ------------------------------------------------------------ expansion
    def _leaf(self, node: _Node) -> bool:
        return node.merged or is_base_case(node.m, node.n, node.k, self.t)

    def split(self, node: _Node, materialize_all: bool = False):
        """Children of an internal node (its S and T are single windows)."""
        a, b = node.S[0][0], node.T[0][0]
        m, n, k = node.m, node.n, node.k
        m1, n1, k1 = m // 2, n // 2, k // 2
        qa, qb = _quads(a, m1, n1), _quads(b, m1, k1)
        sums_a, sums_b, kids = [], [], []
        for i, (s_shape, s_terms, t_shape, t_terms, _) in enumerate(_strassen_products(a, b, node.out)):
            ms, ns = s_shape if s_shape else (s_terms[0][0].rows, s_terms[0][0].cols)
            _, kt = t_shape if t_shape else (t_terms[0][0].rows, t_terms[0][0].cols)
            leaf = is_base_case(ms, ns, kt, self.t) and not materialize_all and self.fused_leaves
            if leaf or not s_shape:
                S = [(w, sg) for (w, sg) in s_terms]
            else:
                W = self.alloc(ms, ns)
                sums_a.append((W, _S[i]))
                S = [(W, 1.0)]
            if leaf or not t_shape:
                T = [(w, sg) for (w, sg) in t_terms]
            else:
                W = self.alloc(ms, kt)
                sums_b.append((W, _T[i]))
                T = [(W, 1.0)]
            kids.append(_Node(S, T, ms, ns, kt, self.alloc(ns, kt), False, 1.0, node.level + 1))
        node.kids = kids
        node.sums = (qa, sums_a, qb, sums_b)
        return kids

    def expand(self, node: _Node, levels, leaves):
        if self._leaf(node):
            leaves.append(node)
            return
        levels[node.level].append(node)
        for kid in self.split(node):
            self.expand(kid, levels, leaves)

    # ------------------------------------------------------------ emission
    @staticmethod
    def _rounds_rect(items, win_of, cell: int = 32):
        """Rounds for writers of possibly overlapping windows of one base: an
        item goes one round after the latest earlier item it overlaps (diagonal
        SYRK leaves of uneven splits nest: a 2x2 leaf block and a 1x1 block
        of a deeper row block can share elements)."""
        buckets = defaultdict(list)      # (base, cell row, cell col) -> [(r0, c0, r1, c1, round)]
        rounds = []
        for it in items:
            w = win_of(it)
            r0, c0 = divmod(w.off, w.ld)
            r1, c1 = r0 + w.rows, c0 + w.cols
            cells = [(w.base, i, j) for i in range(r0 // cell, (r1 - 1) // cell + 1)
                     for j in range(c0 // cell, (c1 - 1) // cell + 1)]
            r = 0
            for key in cells:
                for (a0, b0, a1, b1, rr) in buckets[key]:
                    if a0 < r1 and r0 < a1 and b0 < c1 and c0 < b1:
                        r = max(r, rr + 1)
            for key in cells:
                buckets[key].append((r0, c0, r1, c1, r))
            while len(rounds) <= r:
                rounds.append([])
            rounds[r].append(it)
        return rounds

    def _combo(self, nodes):
        g = self.pb.new_group()
        for nd in nodes:
            qa, sa, qb, sb = nd.sums
            if sa:
                self.pb.combo4(qa, sa, group=g)
            if sb:
                self.pb.combo4(qb, sb, group=g)

    def _post(self, nodes, accumulate):
        g = self.pb.new_group()
        for nd in nodes:
            n1, k1 = nd.n // 2, nd.k // 2
            q = _quads(nd.out, n1, k1)
            self.pb.postadd7([kid.out for kid in nd.kids], [(w, nd.sign) for w in q], accumulate, group=g)

    def _emit_item(self, it, group, private):
        if isinstance(it, tuple):                      # ("syrk", a, c): diagonal leaf
            _, a, c = it
            self.pb.product("syrk", a.rows, a.cols, a.cols, [(a, 1.0)], [], [(c, 1.0)],
                            accumulate=1, group=group)
        else:
            self.pb.product("gemm", it.m, it.n, it.k, it.S, it.T, [(it.out, it.sign)],
                            accumulate=0 if private else 1, group=group)

    def _products(self, leaves, extra=()):
        """Leaf products: one group holding every private leaf plus the first
        round of C writers (diagonal SYRKs, Strassen calls that are leaves --
        the long ones, issued first), then one group per further round."""
        private = [l for l in leaves if not l.acc]
        shared = list(extra) + [l for l in leaves if l.acc]
        rounds = self._rounds_rect(shared, lambda it: it[2] if isinstance(it, tuple) else it.out)
        first = rounds[0] if rounds else []
        if private or first:
            g = self.pb.new_group()
            for it in first:
                self._emit_item(it, g, False)
            for l in private:
                self._emit_item(l, g, True)
        for rnd in rounds[1:]:
            g = self.pb.new_group()
            for it in rnd:
                self._emit_item(it, g, False)

    def emit_wave(self, roots):
        """Breadth-first execution of independent Strassen calls."""
        levels, leaves = defaultdict(list), []
        for r in roots:
            self.expand(r, levels, leaves)
        for lv in sorted(levels):
            self._combo([nd for nd in levels[lv] if nd.sums[1] or nd.sums[3]])
        extra, self.extra = self.extra, []
        self._products(leaves, extra)
        for lv in sorted(levels, reverse=True):
            inner = [nd for nd in levels[lv] if not nd.acc]
            if inner:
                self._post(inner, False)
            for rnd in self._rounds_rect([nd for nd in levels[lv] if nd.acc], lambda nd: nd.out):
                self._post(rnd, True)

    def need(self, node: _Node) -> int:
        probe = _RefBFS(self.t, self.budget, self.fused_leaves)
        copy = _Node(node.S, node.T, node.m, node.n, node.k, node.out, node.acc, node.sign, 0)
        copy.merged = node.merged
        probe.expand(copy, defaultdict(list), [])
        return probe.ws_peak

    def _merge_leaf_roots(self, roots):
        """Strassen calls that are leaves themselves (strassen.py:38-41) and add
        into the same C block from vertically adjacent row blocks (the two
        calls of an AtA node, ata.py:114-115, and the nodes of every row block
        of one column block) are one classical product over the union of
        their rows: the same scalar multiplications, one launch slot."""
        out, runs, order = [], {}, []
        for r in roots:
            if not (r.acc and self._leaf(r) and len(r.S) == 1 and len(r.T) == 1):
                out.append(r)
                continue
            (x, sx), (y, sy) = r.S[0], r.T[0]
            key = (r.out, r.sign, sx, sy, x.base, x.ld, x.off % x.ld, x.cols, y.base, y.ld, y.off % y.ld, y.cols)
            if key not in runs:
                runs[key] = []
                order.append(key)
            runs[key].append(r)
        for key in order:
            rs = sorted(runs[key], key=lambda r: r.S[0][0].off)
            cur = rs[0]
            for r in rs[1:]:
                x, y = cur.S[0][0], cur.T[0][0]
                x2, y2 = r.S[0][0], r.T[0][0]
                if x2.off == x.off + x.rows * x.ld and y2.off == y.off + y.rows * y.ld and x2.rows == y2.rows:
                    X = Win(x.base, x.off, x.ld, x.rows + x2.rows, x.cols)
                    Y = Win(y.base, y.off, y.ld, y.rows + y2.rows, y.cols)
                    cur = _Node([(X, cur.S[0][1])], [(Y, cur.T[0][1])], X.rows, cur.n, cur.k, cur.out, True,
                                cur.sign, 0)
                    cur.merged = True
                else:
                    out.append(cur)
                    cur = r
            out.append(cur)
        return out

    def calls(self, roots):
        """Waves of calls whose breadth-first scratch fits the budget."""
        roots = self._merge_leaf_roots(roots)
        wave, wave_need = [], 0
        for r in roots:
            need = self.need(r)
            if need > self.budget - self.ws_top:
                if wave:
                    self._flush(wave)
                    wave, wave_need = [], 0
                self.depth_first(r)
                continue
            if wave_need + need > self.budget - self.ws_top:
                self._flush(wave)
                wave, wave_need = [], 0
            wave.append(r)
            wave_need += need
        if wave:
            self._flush(wave)

    def _flush(self, wave):
        mark = self.ws_top
        self.emit_wave(wave)
        self.ws_top = mark

    def depth_first(self, node: _Node):
        """One level of the node depth-first: sums, then each child as a call, then its post-addition."""
        if self._leaf(node) or self.need(node) <= self.budget - self.ws_top:
            self._flush([node])
            return
        mark = self.ws_top
        node.level = 0
        kids = self.split(node, materialize_all=True)
        self._combo([node])
        for kid in kids:
            kid.level = 0
            self.depth_first(kid)
        if node.acc:
            self._post([node], True)
        else:
            self._post([node], False)
        self.ws_top = mark

    # ------------------------------------------------------------ AtA
    def ata(self, A: Win, C: Win):
        syrk, roots = [], []

        def rec(a: Win, c: Win):
            m, n = a.rows, a.cols
            if is_ata_base_case(m, n, self.t):
                syrk.append((a, c))
                return
            m1, n1 = m // 2, n // 2
            m2, n2 = m - m1, n - n1
            a11, a12 = a.sub(0, 0, m1, n1), a.sub(0, n1, m1, n2)
            a21, a22 = a.sub(m1, 0, m2, n1), a.sub(m1, n1, m2, n2)
            c11, c21, c22 = c.sub(0, 0, n1, n1), c.sub(n1, 0, n2, n1), c.sub(n1, n1, n2, n2)
            rec(a11, c11)
            rec(a21, c11)
            rec(a12, c22)
            rec(a22, c22)
            for (x, y) in ((a12, a11), (a22, a21)):
                roots.append(_Node([(x, 1.0)], [(y, 1.0)], x.rows, x.cols, y.cols, c21, True, 1.0, 0))

        rec(A, C)
        self.extra = [("syrk", a, c) for (a, c) in self._merge_syrk(syrk)]
        self.calls(roots)
        if self.extra:                                 # no Strassen call took them
            extra, self.extra = self.extra, []
            self._products([], extra)

    @staticmethod
    def _merge_syrk(leaves):
        """Diagonal leaves that accumulate into the same C block from vertically
        adjacent row blocks of the same columns (ata.py:110-113 sends every row
        block of a column block to the same C block) are one SYRK over the
        union of their rows: the same scalar multiplications (sum over the row
        blocks of m_r * n(n+1)/2), one product instead of one per row block."""
        runs = {}
        order = []
        for (a, c) in leaves:
            key = (c, a.base, a.ld, a.off % a.ld, a.cols)
            if key not in runs:
                runs[key] = []
                order.append(key)
            runs[key].append(a)
        out = []
        for key in order:
            blocks = sorted(runs[key], key=lambda w: w.off)
            cur = blocks[0]
            for w in blocks[1:]:
                if w.off == cur.off + cur.rows * cur.ld:      # the next rows of the same columns
                    cur = Win(cur.base, cur.off, cur.ld, cur.rows + w.rows, cur.cols)
                else:
                    out.append((cur, key[0]))
                    cur = w
            out.append((cur, key[0]))
        return out

    def strassen(self, A: Win, B: Win, C: Win):
        self.calls([_Node([(A, 1.0)], [(B, 1.0)], A.rows, A.cols, B.cols, C, True, 1.0, 0)])

    def finish(self) -> Plan:
        plan = self.pb.finish()
        plan.ws_scalars = max(plan.ws_scalars, self.ws_peak)
        return plan


def plan_ata_reference_bfs(m, n, lda, ldc, threshold, budget: int = DEFAULT_BUDGET,
                           fused_leaves: bool = False) -> Plan:
    p = _RefBFS(threshold, budget, fused_leaves)
    p.ata(Win(nat.BASE_A, 0, lda, m, n), Win(nat.BASE_C, 0, ldc, n, n))
    return p.finish()


def plan_strassen_reference_bfs(m, n, k, lda, ldb, ldc, threshold, budget: int = DEFAULT_BUDGET,
                                fused_leaves: bool = False) -> Plan:
    p = _RefBFS(threshold, budget, fused_leaves)
    p.strassen(Win(nat.BASE_A, 0, lda, m, n), Win(nat.BASE_B, 0, ldb, m, k), Win(nat.BASE_C, 0, ldc, n, k))
    return p.finish()
