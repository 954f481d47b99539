"""Workspace sizing for the reference-faithful recursion, and the HBM arena.

Sizing restates the reference planner so a drop-in ``workspace_for`` /
``workspace_for_ata`` hands back the same per-depth (prod, lhs, rhs) buffer
sizes the reference tests inspect (tests/test_strassen.py:262-289):

  * ``chain``        ceil-halved dims per Strassen depth     strassen.py:48-54
  * ``base_dims``    largest leaf call of a recursion        strassen.py:57-71
  * ``calls_sizes``  elementwise maxima over calls            strassen.py:150-184
  * ``ata_calls``    Strassen calls of an AtA recursion       ata.py:29-72

On the GPU the reference's three base-case staging blocks (strassen.py:92-132)
are not needed -- the leaf kernels read strided windows directly -- so they
are planned (for ``covers``) but never allocated.  The per-depth triples live
in ONE device allocation (an arena); levels are 1-D views into it.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .errors import ShapeMismatchError, WorkspaceUndersizedError

DEFAULT_THRESHOLD = 1 << 15  # strassen.py:35


def is_base_case(m: int, n: int, k: int, threshold: int) -> bool:
    """Strassen leaf predicate (strassen.py:38-41)."""
    return m * n + m * k <= threshold or min(m, n, k) == 1


def is_ata_base_case(m: int, n: int, threshold: int) -> bool:
    """AtA leaf predicate (ata.py:23-26)."""
    return m * n <= threshold or m == 1 or n == 1


def ceil_half(d: int) -> int:
    return (d + 1) // 2


def chain(m: int, n: int, k: int, threshold: int):
    """(m_i, n_i, k_i) of each Strassen depth i >= 1 along the ceil chain."""
    out = []
    cm, cn, ck = m, n, k
    while not is_base_case(cm, cn, ck, threshold):
        cm, cn, ck = ceil_half(cm), ceil_half(cn), ceil_half(ck)
        out.append((cm, cn, ck))
    return out


def base_dims(m: int, n: int, k: int, threshold: int):
    fm, fn, fk = m, n, k
    cm, cn, ck = m, n, k
    while not is_base_case(fm, fn, fk, threshold):
        fm, fn, fk = fm // 2, fn // 2, fk // 2
        cm, cn, ck = ceil_half(cm), ceil_half(cn), ceil_half(ck)
    return cm, cn, ck


def _strassen_base_need(lo, hi, threshold):
    flm, fln, flk = lo
    chm, chn, chk = hi
    while not is_base_case(flm, fln, flk, threshold):
        flm, fln, flk = max(1, flm // 2), max(1, fln // 2), max(1, flk // 2)
        chm, chn, chk = ceil_half(chm), ceil_half(chn), ceil_half(chk)
    return chn * chk, chm * chn, chm * chk


def ata_calls(m: int, n: int, threshold: int):
    """Strassen call shapes and base scratch of an AtA recursion (ata.py:43-72)."""
    calls = []
    acc = lhs = rhs = 0
    lo_m, lo_n, hi_m, hi_n = m, n, m, n
    while True:
        if is_ata_base_case(lo_m, lo_n, threshold):
            acc = max(acc, hi_n * hi_n)
            lhs = max(lhs, hi_m * hi_n)
        if is_ata_base_case(hi_m, hi_n, threshold):
            break
        lo_call = (max(1, lo_m // 2), max(1, lo_n // 2), max(1, lo_n // 2))
        hi_call = (hi_m - hi_m // 2, ceil_half(hi_n), ceil_half(hi_n))
        calls.append(hi_call)
        a, l, r = _strassen_base_need(lo_call, hi_call, threshold)
        acc, lhs, rhs = max(acc, a), max(lhs, l), max(rhs, r)
        lo_m, lo_n = max(1, lo_m // 2), max(1, lo_n // 2)
        hi_m, hi_n = ceil_half(hi_m), ceil_half(hi_n)
    return calls, (acc, lhs, rhs)


def calls_sizes(calls, threshold, extra_base=(0, 0, 0)):
    """Per-depth (prod, lhs, rhs) maxima and base needs over `calls`."""
    depth = []
    acc, lhs, rhs = extra_base
    for (m, n, k) in calls:
        for d, (cm, cn, ck) in enumerate(chain(m, n, k, threshold)):
            if d == len(depth):
                depth.append([0, 0, 0])
            s = depth[d]
            s[0], s[1], s[2] = max(s[0], cn * ck), max(s[1], cm * cn), max(s[2], cm * ck)
        bm, bn, bk = base_dims(m, n, k, threshold)
        acc, lhs, rhs = max(acc, bn * bk), max(lhs, bm * bn), max(rhs, bm * bk)
    return [tuple(s) for s in depth], (max(acc, 1), max(lhs, 1), max(rhs, 1))


@dataclass
class Buf:
    """A 1-D window of the arena; ``.size`` is an int like numpy's."""
    offset: int
    size: int
    arena: object = field(default=None, repr=False)

    @property
    def tensor(self):
        return self.arena.buffer[self.offset:self.offset + self.size]


@dataclass
class Level:
    prod: Buf
    lhs: Buf
    rhs: Buf


class StrassenWorkspace:
    """Device scratch for ``fast_strassen`` / ``ata`` (strassen.py:88-147).

    ``levels[i].{prod,lhs,rhs}`` carry the reference sizes; ``buffer`` is the
    single torch allocation behind them (allocated lazily on first use on a
    device, then reused: nothing allocates afterwards).  ``extra`` reserves
    additional scalars for planner-managed scratch (auto plans)."""

    def __init__(self, level_sizes, base_sizes, threshold, dtype, extra: int = 0, device=None):
        self.threshold = threshold
        self.dtype = dtype
        self._base_sizes = tuple(base_sizes)
        off = 0
        self.levels = []
        for (p, l, r) in level_sizes:
            lv = Level(Buf(off, p, self), Buf(off + p, l, self), Buf(off + p + l, r, self))
            off += p + l + r
            self.levels.append(lv)
        self.level_scalars = off
        self.extra = extra
        self.device = device
        self.buffer = None

    @property
    def total_scalars(self) -> int:
        """Scalars of device scratch this workspace owns."""
        return self.level_scalars + self.extra

    @property
    def base_sizes(self):
        """Reference base-block sizes (accumulator, lhs stage, rhs stage); on the
        GPU these are satisfied by strided reads and never allocated."""
        return self._base_sizes

    def level_offsets(self):
        return [(lv.prod.offset, lv.lhs.offset, lv.rhs.offset) for lv in self.levels]

    def covers(self, m: int, n: int, k: int, threshold: int) -> bool:
        """True when every buffer this call's recursion can touch fits
        (strassen.py:134-147)."""
        for d, (cm, cn, ck) in enumerate(chain(m, n, k, threshold)):
            if d >= len(self.levels):
                return False
            lv = self.levels[d]
            if cn * ck > lv.prod.size or cm * cn > lv.lhs.size or cm * ck > lv.rhs.size:
                return False
        bm, bn, bk = base_dims(m, n, k, threshold)
        a, l, r = self._base_sizes
        return bn * bk <= a and bm * bn <= l and bm * bk <= r

    def ensure(self, device, extra: int = 0, dtype=None):
        """Allocate (once) the arena on `device`; grow only if `extra` grows.

        The arena is always held in the dtype the call computes in (`dtype`,
        default the workspace's own): the native executor counts scratch in
        scalars of the plan's dtype, so a workspace built for f32 and handed
        to an f64 call gets an f64 arena of the same scalar count (the
        reference's NumPy buffers cast on assignment, so such a call is legal
        there) instead of being overrun."""
        from .matrix import _as_torch_dtype, _new_buffer
        tdt = _as_torch_dtype(self.dtype if dtype is None else dtype)
        need = self.level_scalars + max(self.extra, extra)
        if (self.buffer is not None and self.buffer.device == device and self.buffer.dtype == tdt
                and self.buffer.numel() >= max(need, 1)):
            return self.buffer
        self.extra = max(self.extra, extra)
        self.buffer = None      # release the smaller arena before allocating its replacement
        self.buffer = _new_buffer(max(need, 1), tdt, device)
        self.device = device
        return self.buffer


def workspace_for_calls(calls, threshold, extra_base=(0, 0, 0), dtype=None) -> StrassenWorkspace:
    levels, base = calls_sizes(calls, threshold, extra_base)
    return StrassenWorkspace(levels, base, threshold, dtype)


def check_ata_workspace(ws: StrassenWorkspace, m: int, n: int, threshold: int) -> None:
    """ata.py:84-94."""
    calls, (acc, lhs, rhs) = ata_calls(m, n, threshold)
    a, l, r = ws.base_sizes
    if acc > a or lhs > l or rhs > r:
        raise WorkspaceUndersizedError(
            f"workspace undersized: A^T A leaves need ({acc}, {lhs}, {rhs}) scratch scalars")
    for (cm, cn, ck) in calls:
        if not ws.covers(cm, cn, ck, threshold):
            raise WorkspaceUndersizedError(f"workspace undersized for inner call ({cm},{cn},{ck})")


def validate_dims(*dims):
    if min(dims) < 1:
        raise ShapeMismatchError("shape mismatch: dimensions must be >= 1")
