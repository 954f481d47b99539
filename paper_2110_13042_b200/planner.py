"""Recursion planners: turn an AtA / Strassen call into a flat list of
native plan ops (include/atamul_b200.h, ``ata_op``).

Two planners share one op vocabulary:

* ``plan_ata_reference`` / ``plan_strassen_reference`` — the reference
  recursion with an integer element-count ``threshold``: same leaf
  predicates (ata.py:23-26, strassen.py:38-41), same floor/ceil quadrants
  (ata.py:104-109, strassen.py:216-220), same seven products and
  destinations (strassen.py:234-275), same per-depth workspace use
  (strassen.py:74-85) — hence the same leaves and the same exact
  multiplication count as the reference's MultCounter.  One GPU-first
  change, numerically equivalent: a Strassen product whose recursive call is
  a leaf is emitted as ONE fused product op (pre-additions in the operand
  load, post-additions in the epilogue) instead of combo + fill + leaf +
  update (same operand sums, same single rounding of each C update).

* ``plan_ata_auto`` — ``threshold="auto"``: the GPU plan.  The contraction
  (rows of A) is never split -- a long contraction belongs in one kernel's K
  loop -- the column recursion of the AtA scheme (ata.py:110-115, with the
  two C21 addends merged into one product over all m rows) runs to a leaf
  width chosen from the B200 tile grid, every below-diagonal block uses one
  fused Strassen level (7 products, strassen.py:234-275), products of the
  same index across all blocks of one level share a launch (their C windows
  are disjoint), and every SYRK leaf shares one launch.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _native as nat
from .errors import ShapeMismatchError
from .workspace import is_ata_base_case, is_base_case

_EMPTY = (0, 0, 0, 0, 0, 0, 0.0)


class Win(NamedTuple):
    """Window (base, element offset, ld, rows, cols) into a base buffer."""
    base: int
    off: int
    ld: int
    rows: int
    cols: int

    def sub(self, r0: int, c0: int, rows: int, cols: int) -> "Win":
        return Win(self.base, self.off + r0 * self.ld + c0, self.ld, rows, cols)

    def top(self, rows: int) -> "Win":
        return Win(self.base, self.off, self.ld, min(rows, self.rows), self.cols)

    def clip(self, rows: int, cols: int) -> "Win":
        return Win(self.base, self.off, self.ld, min(rows, self.rows), min(cols, self.cols))


def _ref(w: Win, sign: float = 1.0, region: int = 0):
    return (w.base, w.rows, w.off, w.ld, w.cols, int(region), float(sign))


@dataclass
class Plan:
    ops: np.ndarray          # OP_DTYPE records
    mults: int               # exact scalar multiplications (MultCounter semantics)
    ws_scalars: int          # workspace scalars the plan touches (extent of WS refs)
    launches: int            # kernel launches the executor will issue
    kind: str

    def __len__(self):
        return len(self.ops)


class PlanBuilder:
    def __init__(self, kind: str):
        self.kind = kind
        self.rows = []
        self.mults = 0
        self.ws_hi = 0
        self._last_group = None
        self.launches = 0

    def _touch(self, w: Win):
        if w.base == nat.BASE_WS and w.rows > 0 and w.cols > 0:
            self.ws_hi = max(self.ws_hi, w.off + (w.rows - 1) * w.ld + w.cols)

    def new_group(self) -> int:
        self._groups = getattr(self, "_groups", 0) + 1
        return self._groups

    def new_region(self) -> int:
        self._regions = getattr(self, "_regions", 0) + 1
        return self._regions

    def product(self, kind, m, n, k, S, T, D, accumulate=1, group=-1, count=True):
        """S, T: [(Win, sign)] operand terms; D: [(Win, sign[, region])]
        destinations (region > 0: window shared with other products of the
        same group, accumulated in op order)."""
        if len(S) > nat.PROD_MAX_TERMS or len(T) > nat.PROD_MAX_TERMS or len(D) > nat.MAX_DESTS:
            raise ValueError("too many product terms")
        for w, *_ in list(S) + list(T) + list(D):
            self._touch(w)
        s = [_ref(w.clip(m, n), sg) for w, sg in S] + [_EMPTY] * (nat.MAX_TERMS - len(S))
        t = [_ref(w.clip(m, k), sg) for w, sg in T] + [_EMPTY] * (nat.MAX_TERMS - len(T))
        d = [_ref(dd[0].clip(n, k), dd[1], dd[2] if len(dd) > 2 else 0) for dd in D] \
            + [_EMPTY] * (nat.MAX_DESTS - len(D))
        op = nat.OP_SYRK if kind == "syrk" else nat.OP_GEMM
        self.rows.append((op, m, n, k, len(S), len(T), len(D), accumulate, group, 0, s, t, d))
        if group < 0 or group != self._last_group:
            self.launches += 1
        self._last_group = group if group >= 0 else None
        self._last_ew = None
        if count:
            self.mults += m * n * (n + 1) // 2 if kind == "syrk" else m * n * k

    def _ew(self, op, S, D):
        for w, _ in list(S) + list(D):
            self._touch(w)
        s = [_ref(w, sg) for w, sg in S] + [_EMPTY] * (nat.MAX_TERMS - len(S))
        d = [_ref(w, sg) for w, sg in D] + [_EMPTY] * (nat.MAX_DESTS - len(D))
        self.rows.append((op, 0, 0, 0, len(S), 0, len(D), 0, -1, 0, s, [_EMPTY] * nat.MAX_TERMS, d))
        self.launches += 1
        self._last_group = None
        self._last_ew = None

    def combo(self, dst: Win, terms):
        self._ew(nat.OP_COMBO, [(w.clip(dst.rows, dst.cols), sg) for w, sg in terms], [(dst, 1.0)])

    def update(self, src: Win, dests):
        self._ew(nat.OP_UPDATE, [(src, 1.0)],
                 [(w.clip(src.rows, src.cols), sg) for w, sg in dests])

    def fill(self, dst: Win):
        self._ew(nat.OP_FILL, [], [(dst, 1.0)])

    def _ew_launch(self, op, group):
        # consecutive COMBO4 / POSTADD7 ops of one group >= 0 share a launch
        key = (op, group)
        if group < 0 or key != getattr(self, "_last_ew", None):
            self.launches += 1
        self._last_ew = key if group >= 0 else None
        self._last_group = None

    def combo4(self, sources, outputs, lower: bool = False, group: int = -1):
        """One pass over up to 4 source windows writing up to 8 sums:
        outputs = [(dst Win, (c_0, .., c_{ns-1}))] with c_q in {0, +1, -1};
        lower=True writes only the lower triangle of each output window.
        group >= 0: consecutive combo4 ops of the group (independent nodes)
        run as one multi-node launch."""
        if len(sources) > nat.MAX_TERMS or len(outputs) > nat.MAX_DESTS:
            raise ValueError("combo4: too many sources/outputs")
        for w in list(sources) + [o[0] for o in outputs]:
            self._touch(w)
        s = [_ref(w) for w in sources] + [_EMPTY] * (nat.MAX_TERMS - len(sources))
        d = []
        for w, coefs in outputs:
            code = 0
            for q, cq in enumerate(coefs):
                code |= (1 if cq > 0 else 2 if cq < 0 else 0) << (2 * q)
            d.append(_ref(w, 1.0, code))
        d += [_EMPTY] * (nat.MAX_DESTS - len(outputs))
        self.rows.append((nat.OP_COMBO4, 0, 0, 0, len(sources), 0, len(outputs), int(lower), group, 0, s,
                          [_EMPTY] * nat.MAX_TERMS, d))
        self._ew_launch(nat.OP_COMBO4, group)

    def round_tf32(self, src: Win, dst: Win):
        """dst = round-to-nearest TF32(src) (ATA_OP_ROUND)."""
        self._ew(nat.OP_ROUND, [(src, 1.0)], [(dst, 1.0)])

    def postadd7(self, children, outputs, accumulate: bool, group: int = -1):
        """Strassen post-addition of one node: children = 7 product windows
        (P1..P7), outputs = [(C11 win, sign), (C12..), (C21..), (C22..)].
        group >= 0: consecutive postadd7 ops of the group share one launch."""
        for w in list(children) + [o[0] for o in outputs]:
            self._touch(w)
        s = [_ref(w) for w in children[:4]]
        t = [_ref(w) for w in children[4:]] + [_EMPTY]
        d = [_ref(w, sg) for (w, sg) in outputs] + [_EMPTY] * (nat.MAX_DESTS - 4)
        self.rows.append((nat.OP_POSTADD7, 0, 0, 0, 4, 3, 4, int(accumulate), group, 0, s, t, d))
        self._ew_launch(nat.OP_POSTADD7, group)

    def finish(self) -> Plan:
        ops = np.array(self.rows, dtype=nat.OP_DTYPE) if self.rows else np.zeros(0, nat.OP_DTYPE)
        return Plan(ops, self.mults, self.ws_hi, self.launches, self.kind)


# ------------------------------------------------------------------ Strassen

def _strassen_products(a: Win, b: Win, c: Win, regions=None):
    """The seven products of one node (strassen.py:234-275) as
    (S-shape, S-terms, T-shape, T-terms, dests); shape None = plain view.
    `regions` = region ids of (C11, C12, C21, C22) when the products are
    launched together (ordered accumulation into shared quadrants)."""
    if regions is not None:
        def tag(blocks):
            return [(w, sg, regions[q]) for (w, sg, q) in blocks]
    else:
        def tag(blocks):
            return [(w, sg) for (w, sg, q) in blocks]
    m, n = a.rows, a.cols
    k = b.cols
    m1, n1, k1 = m // 2, n // 2, k // 2
    m2, n2, k2 = m - m1, n - n1, k - k1
    A11, A12 = a.sub(0, 0, m1, n1), a.sub(0, n1, m1, n2)
    A21, A22 = a.sub(m1, 0, m2, n1), a.sub(m1, n1, m2, n2)
    B11, B12 = b.sub(0, 0, m1, k1), b.sub(0, k1, m1, k2)
    B21, B22 = b.sub(m1, 0, m2, k1), b.sub(m1, k1, m2, k2)
    C11, C12 = c.sub(0, 0, n1, k1), c.sub(0, k1, n1, k2)
    C21, C22 = c.sub(n1, 0, n2, k1), c.sub(n1, k1, n2, k2)
    Q11, Q12, Q21, Q22 = 0, 1, 2, 3
    return [
        ((m2, n2), [(A22, 1.0), (A11, 1.0)], (m2, k2), [(B22, 1.0), (B11, 1.0)],
         tag([(C11, 1.0, Q11), (C22, 1.0, Q22)])),
        ((m1, n2), [(A12, 1.0), (A22.top(m1), 1.0)], None, [(B11, 1.0)],
         tag([(C21, 1.0, Q21), (C22, -1.0, Q22)])),
        (None, [(A11, 1.0)], (m1, k2), [(B12, 1.0), (B22.top(m1), -1.0)],
         tag([(C12, 1.0, Q12), (C22, 1.0, Q22)])),
        (None, [(A22, 1.0)], (m2, k1), [(B21, 1.0), (B11, -1.0)],
         tag([(C11, 1.0, Q11), (C21, 1.0, Q21)])),
        ((m2, n1), [(A21, 1.0), (A11, 1.0)], None, [(B22, 1.0)],
         tag([(C11, -1.0, Q11), (C12, 1.0, Q12)])),
        ((m1, n2), [(A12, 1.0), (A11, -1.0)], (m1, k2), [(B12, 1.0), (B11, 1.0)],
         tag([(C22, 1.0, Q22)])),
        ((m2, n2), [(A21, 1.0), (A22, -1.0)], (m2, k2), [(B22, 1.0), (B21, 1.0)],
         tag([(C11, 1.0, Q11)])),
    ]


class _ReferencePlanner:
    def __init__(self, threshold: int, level_offsets, fuse: bool = True):
        self.t = threshold
        self.lv = level_offsets
        self.fuse = fuse
        self.pb = PlanBuilder("reference")

    def strassen(self, a: Win, b: Win, c: Win, depth: int):
        m, n, k = a.rows, a.cols, b.cols
        if is_base_case(m, n, k, self.t):
            self.pb.product("gemm", m, n, k, [(a, 1.0)], [(b, 1.0)], [(c, 1.0)])
            return
        if depth >= len(self.lv):
            from .errors import WorkspaceUndersizedError
            raise WorkspaceUndersizedError(f"workspace undersized: no level {depth} for ({m},{n},{k})")
        prod_off, lhs_off, rhs_off = self.lv[depth]
        # fused leaf products of this node share one launch; their C quadrants
        # are ordered regions (accumulated in the reference's product order)
        regions = tuple(self.pb.new_region() for _ in range(4)) if self.fuse else None
        group = self.pb.new_group()
        for s_shape, s_terms, t_shape, t_terms, dests in _strassen_products(a, b, c, regions):
            ms, ns = s_shape if s_shape else (s_terms[0][0].rows, s_terms[0][0].cols)
            mt, kt = t_shape if t_shape else (t_terms[0][0].rows, t_terms[0][0].cols)
            assert ms == mt
            if self.fuse and is_base_case(ms, ns, kt, self.t):
                self.pb.product("gemm", ms, ns, kt, s_terms, t_terms, dests, group=group)
                continue
            dests = [(w, sg) for (w, sg, *_) in dests]
            if s_shape:
                S = Win(nat.BASE_WS, lhs_off, ns, ms, ns)
                self.pb.combo(S, s_terms)
            else:
                S = s_terms[0][0]
            if t_shape:
                T = Win(nat.BASE_WS, rhs_off, kt, mt, kt)
                self.pb.combo(T, t_terms)
            else:
                T = t_terms[0][0]
            P = Win(nat.BASE_WS, prod_off, kt, ns, kt)
            self.pb.fill(P)
            self.strassen(S, T, P, depth + 1)
            self.pb.update(P, dests)

    def ata(self, a: Win, c: Win):
        m, n = a.rows, a.cols
        if is_ata_base_case(m, n, self.t):
            self.pb.product("syrk", m, n, n, [(a, 1.0)], [], [(c, 1.0)])
            return
        m1, n1 = m // 2, n // 2
        m2, n2 = m - m1, n - n1
        a11, a12 = a.sub(0, 0, m1, n1), a.sub(0, n1, m1, n2)
        a21, a22 = a.sub(m1, 0, m2, n1), a.sub(m1, n1, m2, n2)
        c11, c21, c22 = c.sub(0, 0, n1, n1), c.sub(n1, 0, n2, n1), c.sub(n1, n1, n2, n2)
        self.ata(a11, c11)
        self.ata(a21, c11)
        self.ata(a12, c22)
        self.ata(a22, c22)
        self.strassen(a12, a11, c21, 0)
        self.strassen(a22, a21, c21, 0)


def plan_ata_reference(m, n, lda, ldc, threshold, level_offsets, fuse=True) -> Plan:
    p = _ReferencePlanner(threshold, level_offsets, fuse)
    p.ata(Win(nat.BASE_A, 0, lda, m, n), Win(nat.BASE_C, 0, ldc, n, n))
    return p.pb.finish()


def plan_strassen_reference(m, n, k, lda, ldb, ldc, threshold, level_offsets, fuse=True) -> Plan:
    p = _ReferencePlanner(threshold, level_offsets, fuse)
    p.strassen(Win(nat.BASE_A, 0, lda, m, n), Win(nat.BASE_B, 0, ldb, m, k),
               Win(nat.BASE_C, 0, ldc, n, k), 0)
    return p.pb.finish()


# ---------------------------------------------------------------------- auto

TILE = 128


@dataclass(frozen=True)
class AutoParamsV1:
    leaf_cols: int = 1024        # stop the column recursion at this width
    strassen_min: int = 1024     # use a fused Strassen level when both C21 sides >= this


def plan_ata_auto_v1(m, n, lda, ldc, params: AutoParamsV1 = AutoParamsV1()) -> Plan:
    """GPU plan for lower(C) += alpha A^T A (see module docstring)."""
    if m < 1 or n < 1:
        raise ShapeMismatchError("shape mismatch: empty operand")
    pb = PlanBuilder("auto")
    A = Win(nat.BASE_A, 0, lda, m, n)
    C = Win(nat.BASE_C, 0, ldc, n, n)
    nodes = [(0, n)]
    group = 0
    while True:
        split = [(c0, w) for (c0, w) in nodes if w > params.leaf_cols and w >= 2]
        if not split:
            break
        keep = [(c0, w) for (c0, w) in nodes if not (w > params.leaf_cols and w >= 2)]
        nxt = list(keep)
        fused = []     # (a, b, c) blocks taking the Strassen path
        plain = []
        for (c0, w) in split:
            n1 = w // 2
            n2 = w - n1
            nxt += [(c0, n1), (c0 + n1, n2)]
            a = A.sub(0, c0 + n1, m, n2)      # A_right
            b = A.sub(0, c0, m, n1)           # A_left
            c = C.sub(c0 + n1, c0, n2, n1)    # C21
            if min(n1, n2) >= params.strassen_min and m >= 2:
                fused.append((a, b, c))
            else:
                plain.append((a, b, c))
        if plain:
            for (a, b, c) in plain:
                pb.product("gemm", m, a.cols, b.cols, [(a, 1.0)], [(b, 1.0)],
                           [(c, 1.0)], group=group)
            group += 1
        if fused:
            # all 7 products of every node of this level in one persistent launch;
            # each node's C quadrants are ordered regions
            per_node = [_strassen_products(a, b, c, tuple(pb.new_region() for _ in range(4)))
                        for (a, b, c) in fused]
            for pi in range(7):
                for prods in per_node:
                    s_shape, s_terms, t_shape, t_terms, dests = prods[pi]
                    ms, ns = s_shape if s_shape else (s_terms[0][0].rows, s_terms[0][0].cols)
                    _, kt = t_shape if t_shape else (t_terms[0][0].rows, t_terms[0][0].cols)
                    pb.product("gemm", ms, ns, kt, s_terms, t_terms, dests, group=group)
            group += 1
        nodes = nxt
    for (c0, w) in sorted(nodes):
        pb.product("syrk", m, w, w, [(A.sub(0, c0, m, w), 1.0)], [], [(C.sub(c0, c0, w, w), 1.0)],
                   group=group)
    return pb.finish()
