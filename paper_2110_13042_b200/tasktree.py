"""Task trees of the parallel executors (host logic, no GPU).

Restates the reference's tree construction (``pkg/src/atamul/scheduler.py``)
so callers keep its process layout: the CLI's ``--dump-tree`` and the
multi-GPU "tree" partition (``dist.ata_dist_tree``) use the same leaf tasks,
owners and ranks-to-regions map as the reference's distribute-compute-retrieve
executor.  Pinned against trees the reference itself built
(``tests/golden/trees.json``, ``tools/make_golden_cli.py``).

Rules (reference line numbers in parentheses):

* distributed AtA node, process budget p, level budget r (scheduler.py:283-314):
  a *bunch* of six children -- the four quadrant self-products
  A11, A21 -> C11 and A12, A22 -> C22, then A12^T A11 and A22^T A21 -> C21 --
  when p >= 6 (p == 6 on the last level); half the budget (rounded so that
  four remain) goes to the two products.  Otherwise the rows are cut into p
  horizontal tiles whose full partial triangles the parent sums.
* distributed AtB node (:316-363): a bunch of eight children (output row
  block i, output column block j, contraction block l) when p >= 8 (== 8 on
  the last level), else a u x v grid of disjoint output blocks.
* shared AtA node (:365-405): three column-half children (left -> C11,
  right -> C22, right^T left -> C21) when p >= 3 (== 3 last level), else
  column stripes of near-equal result area.
* shared AtB node (:407-432): four output quadrants when p >= 4, else a grid.
* labels (:222-241): children are created breadth first; the first child
  keeps its parent's owner, every other child takes the next fresh label.
"""
from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from .errors import UnknownProcessError, UnsplittableError


class ComputationType(Enum):
    ATA = "AtA"
    ATB = "AtB"


@dataclass(frozen=True)
class Region:
    row_offset: int
    col_offset: int
    rows: int
    cols: int

    @property
    def size(self) -> int:
        return self.rows * self.cols

    def sub(self, r0: int, c0: int, rows: int, cols: int) -> "Region":
        return Region(self.row_offset + r0, self.col_offset + c0, rows, cols)

    def __str__(self):
        r, c = self.row_offset, self.col_offset
        return f"[{r}:{r + self.rows},{c}:{c + self.cols}]"


@dataclass
class Task:
    computation: ComputationType
    a_region: Region
    b_region: Region | None
    c_region: Region
    parent: int   # owner label of the parent node
    owner: int

    @property
    def operand_words(self) -> int:
        return self.a_region.size + (self.b_region.size if self.b_region is not None else 0)


@dataclass
class TreeNode:
    id: int
    task: Task
    parent_id: int | None
    depth: int
    children: list[int] = field(default_factory=list)
    bunch: bool = False


@dataclass
class TaskTree:
    mode: str
    procs: int
    m: int
    n: int
    nodes: list[TreeNode]
    leaf_ids: list[int]

    @property
    def root(self) -> TreeNode:
        return self.nodes[0]

    @property
    def depth(self) -> int:
        return max(nd.depth for nd in self.nodes)

    def node(self, node_id: int) -> TreeNode:
        return self.nodes[node_id]

    def children_of(self, node: TreeNode) -> list[TreeNode]:
        return [self.nodes[i] for i in node.children]


# ------------------------------------------------------------------ counts

def _levels(procs: int, anchor: int, group: int, fanout: int) -> int:
    if procs < 1:
        raise ValueError("process count must be >= 1")
    if procs == 1:
        return 0
    if procs <= anchor:
        return 1
    q = procs // group
    k = 0
    while q >= fanout ** (k + 1):
        k += 1
    return 1 + k + (1 if q % fanout ** max(k, 1) else 0)


def levels_distributed(procs: int) -> int:
    """Parallel levels of the distributed tree (scheduler.py:129-145)."""
    return _levels(procs, anchor=6, group=4, fanout=8)


def levels_shared(procs: int) -> int:
    """Parallel levels of the shared tree (scheduler.py:148-163)."""
    return _levels(procs, anchor=3, group=2, fanout=4)


def _even(total: int, parts: int) -> list[int]:
    """`parts` integers summing to `total`, differing by <= 1, larger first."""
    q, r = divmod(total, parts)
    return [q + (1 if i < r else 0) for i in range(parts)]


def _spans(extent: int, parts: int) -> list[tuple[int, int]]:
    """[0, extent) cut into `parts` (offset, width) spans of near-equal width."""
    if parts > extent:
        raise UnsplittableError(f"unsplittable: {parts} tiles over extent {extent}")
    out, start = [], 0
    for w in _even(extent, parts):
        out.append((start, w))
        start += w
    return out


def _grid(q: int) -> tuple[int, int]:
    """q = u * v, v the largest divisor <= sqrt(q) (more row tiles)."""
    v = max(d for d in range(1, math.isqrt(q) + 1) if q % d == 0)
    return q // v, v


def _stripe_ends(cols: int, parts: int) -> list[int]:
    """Stripe end columns over a triangular output with near-equal areas
    (scheduler.py:193-210): end_i ~ cols * sqrt(i / parts), strictly increasing."""
    if parts > cols:
        raise UnsplittableError(f"unsplittable: {parts} stripes over {cols} columns")
    ends = [max(1, round(cols * math.sqrt(i / parts))) for i in range(1, parts + 1)]
    ends[-1] = cols
    for i in reversed(range(parts - 1)):
        ends[i] = min(ends[i], ends[i + 1] - 1)
    for i in range(1, parts):
        ends[i] = max(ends[i], ends[i - 1] + 1)
    if ends[-1] != cols:
        raise UnsplittableError("unsplittable: stripe repair failed")
    return ends


# ------------------------------------------------------------- expansion

_ATA, _ATB = ComputationType.ATA, ComputationType.ATB


def _halves(extent: int) -> tuple[int, int]:
    return extent // 2, extent - extent // 2


def _complete(budget: int, rem: int, size: int) -> bool:
    return budget == size if rem <= 1 else budget >= size


def _dist_ata(t: Task, p: int, rem: int):
    a, c = t.a_region, t.c_region
    if not _complete(p, rem, 6):
        return False, [(_ATA, a.sub(r0, 0, h, a.cols), None, c, 1) for r0, h in _spans(a.rows, p)]
    if a.rows < 2 or a.cols < 2:
        raise UnsplittableError(f"unsplittable: A^T A block {a.rows}x{a.cols} under budget")
    (m1, m2), (n1, n2) = _halves(a.rows), _halves(a.cols)
    q = {(0, 0): a.sub(0, 0, m1, n1), (0, 1): a.sub(0, n1, m1, n2),
         (1, 0): a.sub(m1, 0, m2, n1), (1, 1): a.sub(m1, n1, m2, n2)}
    c11, c21, c22 = c.sub(0, 0, n1, n1), c.sub(n1, 0, n2, n1), c.sub(n1, n1, n2, n2)
    n_atb = min((p + 1) // 2, p - 4)
    pa, pb = _even(p - n_atb, 4), _even(n_atb, 2)
    return True, [(_ATA, q[0, 0], None, c11, pa[0]), (_ATA, q[1, 0], None, c11, pa[1]),
                  (_ATA, q[0, 1], None, c22, pa[2]), (_ATA, q[1, 1], None, c22, pa[3]),
                  (_ATB, q[0, 1], q[0, 0], c21, pb[0]), (_ATB, q[1, 1], q[1, 0], c21, pb[1])]


def _atb_grid(t: Task, p: int):
    a, b, c = t.a_region, t.b_region, t.c_region
    u, v = _grid(p)
    return False, [(_ATB, a.sub(0, ao, a.rows, aw), b.sub(0, bo, b.rows, bw), c.sub(ao, bo, aw, bw), 1)
                   for ao, aw in _spans(a.cols, u) for bo, bw in _spans(b.cols, v)]


def _dist_atb(t: Task, p: int, rem: int):
    if not _complete(p, rem, 8):
        return _atb_grid(t, p)
    a, b, c = t.a_region, t.b_region, t.c_region
    if a.rows < 2 or a.cols < 2 or b.cols < 2:
        raise UnsplittableError(f"unsplittable: A^T B block {a.rows}x{a.cols} under budget")
    rows = list(zip((0, a.rows // 2), _halves(a.rows)))
    acols = list(zip((0, a.cols // 2), _halves(a.cols)))
    bcols = list(zip((0, b.cols // 2), _halves(b.cols)))
    budgets = iter(_even(p, 8))
    return True, [(_ATB, a.sub(r0, ao, h, aw), b.sub(r0 + a.row_offset - b.row_offset, bo, h, bw),
                   c.sub(ao, bo, aw, bw), next(budgets))
                  for ao, aw in acols for bo, bw in bcols for r0, h in rows]


def _shared_ata(t: Task, p: int, rem: int):
    a, c = t.a_region, t.c_region
    if not _complete(p, rem, 3):
        specs, start = [], 0
        for end in _stripe_ends(a.cols, p):
            specs.append((_ATA, a.sub(0, 0, a.rows, end), None, c.sub(start, 0, end - start, end), 1))
            start = end
        return False, specs
    if a.cols < 2:
        raise UnsplittableError(f"unsplittable: A^T A block {a.rows}x{a.cols} under budget")
    n1, n2 = _halves(a.cols)
    left, right = a.sub(0, 0, a.rows, n1), a.sub(0, n1, a.rows, n2)
    n_atb = min((p + 1) // 2, p - 2)
    pa = _even(p - n_atb, 2)
    return True, [(_ATA, left, None, c.sub(0, 0, n1, n1), pa[0]),
                  (_ATA, right, None, c.sub(n1, n1, n2, n2), pa[1]),
                  (_ATB, right, left, c.sub(n1, 0, n2, n1), n_atb)]


def _shared_atb(t: Task, p: int, rem: int):
    if not _complete(p, rem, 4):
        return _atb_grid(t, p)
    a, b, c = t.a_region, t.b_region, t.c_region
    if a.cols < 2 or b.cols < 2:
        raise UnsplittableError(f"unsplittable: A^T B block under budget {p}")
    acols = list(zip((0, a.cols // 2), _halves(a.cols)))
    bcols = list(zip((0, b.cols // 2), _halves(b.cols)))
    budgets = iter(_even(p, 4))
    return True, [(_ATB, a.sub(0, ao, a.rows, aw), b.sub(0, bo, b.rows, bw), c.sub(ao, bo, aw, bw), next(budgets))
                  for ao, aw in acols for bo, bw in bcols]


_RULES = {("distributed", _ATA): _dist_ata, ("distributed", _ATB): _dist_atb,
          ("shared", _ATA): _shared_ata, ("shared", _ATB): _shared_atb}


def _build(mode: str, procs: int, m: int, n: int) -> TaskTree:
    if procs < 1 or m < 1 or n < 1:
        raise ValueError("procs, m and n must all be >= 1")
    levels = levels_distributed(procs) if mode == "distributed" else levels_shared(procs)
    nodes = [TreeNode(0, Task(_ATA, Region(0, 0, m, n), None, Region(0, 0, n, n), 0, 0), None, 0)]
    fresh = 1
    work = deque([(0, procs, levels)])
    while work:
        nid, budget, rem = work.popleft()
        if budget == 1:
            continue
        node = nodes[nid]
        bunch, specs = _RULES[mode, node.task.computation](node.task, budget, rem)
        node.bunch = bunch
        for i, (kind, a, b, c, bud) in enumerate(specs):
            owner = node.task.owner if i == 0 else fresh
            fresh += 0 if i == 0 else 1
            child = TreeNode(len(nodes), Task(kind, a, b, c, node.task.owner, owner), nid, node.depth + 1)
            nodes.append(child)
            node.children.append(child.id)
            if bunch:
                work.append((child.id, bud, rem - 1))
    leaves = [nd for nd in nodes if not nd.children]
    if len(leaves) != procs:
        raise AssertionError(f"tree built {len(leaves)} leaves for {procs} processes")
    leaf_ids = [-1] * procs
    for nd in leaves:
        leaf_ids[nd.task.owner] = nd.id
    if min(leaf_ids) < 0:
        raise AssertionError("leaf labels are not a bijection")
    return TaskTree(mode, procs, m, n, nodes, leaf_ids)


def build_tree_distributed(procs: int, m: int, n: int) -> TaskTree:
    """Task tree of the distribute-compute-retrieve executor (scheduler.py:497-499)."""
    return _build("distributed", procs, m, n)


def build_tree_shared(procs: int, m: int, n: int) -> TaskTree:
    """Task tree of the worker-thread executor (scheduler.py:502-506)."""
    return _build("shared", procs, m, n)


def leaf_task(tree: TaskTree, p: int) -> Task:
    """The leaf task of process p (scheduler.py:514-518)."""
    if not 0 <= p < tree.procs:
        raise UnknownProcessError(f"unknown process {p}")
    return tree.nodes[tree.leaf_ids[p]].task


def path_to_root(tree: TaskTree, p: int) -> list[TreeNode]:
    """Nodes owned by process p, leaf first (scheduler.py:521-536)."""
    if not 0 <= p < tree.procs:
        raise UnknownProcessError(f"unknown process {p}")
    chain, nd = [], tree.nodes[tree.leaf_ids[p]]
    while nd is not None and nd.task.owner == p:
        chain.append(nd)
        nd = None if nd.parent_id is None else tree.nodes[nd.parent_id]
    return chain


def covered_mask(task: Task, n: int) -> np.ndarray:
    """Result cells a leaf task writes (AtA: at or below the diagonal)."""
    c = task.c_region
    mask = np.zeros((n, n), dtype=bool)
    mask[c.row_offset:c.row_offset + c.rows, c.col_offset:c.col_offset + c.cols] = True
    if task.computation is _ATA:
        mask &= np.tri(n, dtype=bool)
    return mask


def render_tree(tree: TaskTree) -> str:
    """One line per node, two spaces per level (the CLI's --dump-tree)."""
    out = [f"{tree.mode} tree: P={tree.procs} A={tree.m}x{tree.n} levels={tree.depth}"]
    stack = [(tree.root, 0)]
    while stack:
        nd, ind = stack.pop()
        t = nd.task
        line = f"{'  ' * ind}p{t.owner} {t.computation.value} A{t.a_region}"
        if t.b_region is not None:
            line += f" B{t.b_region}"
        line += f" -> C{t.c_region}"
        if nd.children:
            line += " (bunch)" if nd.bunch else " (tiles)"
        out.append(line)
        stack.extend((ch, ind + 1) for ch in reversed(tree.children_of(nd)))
    return "\n".join(out)
