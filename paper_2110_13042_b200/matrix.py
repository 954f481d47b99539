"""Device-side mirror of the reference's matrix layer (pkg/src/atamul/matrix.py).

Same public names and argument meanings; the arithmetic runs on the B200
through the C ABI (``_native``).  Operands may be torch CUDA tensors
(zero-copy when rows have unit column stride), or anything the reference
accepts (numpy arrays, CPU tensors, ``DenseMatrix``/``MatrixView``): those are
staged to the current CUDA device, computed there, and written back in place.
Nothing is ever computed on the CPU.
"""
from __future__ import annotations

import contextlib
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .errors import ShapeMismatchError, UnsplittableError

_alloc_counter = {"count": 0}


def _torch():
    import torch
    return torch


def _new_buffer(numel, dtype, device):
    """Allocation chokepoint (matrix.py:35-42) for device scratch."""
    torch = _torch()
    _alloc_counter["count"] += 1
    tdt = _as_torch_dtype(dtype)
    return torch.empty(int(numel), dtype=tdt, device=device)


@contextlib.contextmanager
def count_allocations():
    """Count scratch allocations made while the context is open (matrix.py:45-54)."""
    start = _alloc_counter["count"]
    tracker = {"count": 0}
    try:
        yield tracker
    finally:
        tracker["count"] = _alloc_counter["count"] - start


def _as_torch_dtype(dtype):
    torch = _torch()
    if dtype is None:
        return torch.float64
    if isinstance(dtype, torch.dtype):
        return dtype
    d = np.dtype(dtype)
    if d == np.float32:
        return torch.float32
    if d == np.float64:
        return torch.float64
    raise ShapeMismatchError(f"shape mismatch: only f32/f64 supported, got {d}")


# ----------------------------------------------------------------- containers

class DenseMatrix:
    """Rows x cols matrix in one row-major buffer (matrix.py:62-104).  The
    buffer ``.a`` may be a numpy array or a torch tensor (host or device)."""

    __slots__ = ("a",)

    def __init__(self, array):
        torch = _torch()
        if isinstance(array, torch.Tensor):
            a = array
            if a.dim() != 2:
                raise ShapeMismatchError("shape mismatch: DenseMatrix needs a 2-D array")
            if a.dtype not in (torch.float32, torch.float64):
                a = a.to(torch.float64)
            if a.shape[0] < 1 or a.shape[1] < 1:
                raise ShapeMismatchError("shape mismatch: rows and cols must be >= 1")
            self.a = a.contiguous()
            return
        a = np.asarray(array)
        if a.ndim != 2:
            raise ShapeMismatchError("shape mismatch: DenseMatrix needs a 2-D array")
        if a.shape[0] < 1 or a.shape[1] < 1:
            raise ShapeMismatchError("shape mismatch: rows and cols must be >= 1")
        if a.dtype.type not in (np.float32, np.float64):
            a = a.astype(np.float64)
        self.a = np.ascontiguousarray(a)

    @classmethod
    def zeros(cls, rows, cols, dtype=np.float64, device=None):
        if device is None:
            return cls(np.zeros((rows, cols), dtype=dtype))
        torch = _torch()
        return cls(torch.zeros((rows, cols), dtype=_as_torch_dtype(dtype), device=device))

    @property
    def rows(self):
        return int(self.a.shape[0])

    @property
    def cols(self):
        return int(self.a.shape[1])

    @property
    def dtype(self):
        return self.a.dtype

    def view(self, row_offset=0, col_offset=0, rows=None, cols=None):
        rows = self.rows - row_offset if rows is None else rows
        cols = self.cols - col_offset if cols is None else cols
        return MatrixView(self, row_offset, col_offset, rows, cols)

    def copy(self):
        return DenseMatrix(self.a.clone() if hasattr(self.a, "clone") else self.a.copy())

    def __repr__(self):
        return f"DenseMatrix({self.rows}x{self.cols}, {self.a.dtype})"


class MatrixView:
    """Rectangular window of a DenseMatrix (matrix.py:107-150)."""

    __slots__ = ("base", "row_offset", "col_offset", "rows", "cols", "a")

    def __init__(self, base, row_offset, col_offset, rows, cols):
        if rows < 1 or cols < 1:
            raise ShapeMismatchError("shape mismatch: empty view")
        if row_offset < 0 or col_offset < 0 or row_offset + rows > base.rows \
                or col_offset + cols > base.cols:
            raise ShapeMismatchError("shape mismatch: view exceeds base matrix")
        self.base, self.row_offset, self.col_offset = base, row_offset, col_offset
        self.rows, self.cols = rows, cols
        self.a = base.a[row_offset:row_offset + rows, col_offset:col_offset + cols]

    @property
    def row_stride(self):
        s = self.a.stride(0) if hasattr(self.a, "stride") and callable(self.a.stride) \
            else self.a.strides[0] // self.a.itemsize
        return int(s)

    def subview(self, row_offset, col_offset, rows, cols):
        return MatrixView(self.base, self.row_offset + row_offset, self.col_offset + col_offset,
                          rows, cols)

    def overlaps(self, other):
        if self.base is not other.base:
            return False
        return not (self.row_offset + self.rows <= other.row_offset
                    or other.row_offset + other.rows <= self.row_offset
                    or self.col_offset + self.cols <= other.col_offset
                    or other.col_offset + other.cols <= self.col_offset)

    def __repr__(self):
        return f"MatrixView({self.rows}x{self.cols} at ({self.row_offset},{self.col_offset}))"


def as_array(x):
    """MatrixView / DenseMatrix / array-like -> the underlying 2-D array."""
    if isinstance(x, (MatrixView, DenseMatrix)):
        return x.a
    torch = _torch()
    if isinstance(x, torch.Tensor):
        if x.dim() != 2:
            raise ShapeMismatchError("shape mismatch: expected a 2-D operand")
        return x
    a = np.asarray(x)
    if a.ndim != 2:
        raise ShapeMismatchError("shape mismatch: expected a 2-D operand")
    return a


@dataclass
class MultCounter:
    """Scalar-multiplication counter (matrix.py:168-185); credited from the
    plan, exactly as the reference's leaves would credit it."""
    scalar_mults: int = 0
    enabled: bool = True

    def add(self, k: int) -> None:
        if self.enabled:
            self.scalar_mults += k

    def reset(self) -> None:
        self.scalar_mults = 0


def split4(A):
    """Floor/ceil quadrants (matrix.py:193-215)."""
    if isinstance(A, MatrixView):
        m, n = A.rows, A.cols
        if m < 2 or n < 2:
            raise UnsplittableError("unsplittable: block needs >= 2 rows and cols")
        m1, n1 = m // 2, n // 2
        return (A.subview(0, 0, m1, n1), A.subview(0, n1, m1, n - n1),
                A.subview(m1, 0, m - m1, n1), A.subview(m1, n1, m - m1, n - n1))
    a = as_array(A)
    m, n = a.shape
    if m < 2 or n < 2:
        raise UnsplittableError("unsplittable: block needs >= 2 rows and cols")
    m1, n1 = m // 2, n // 2
    return a[:m1, :n1], a[:m1, n1:], a[m1:, :n1], a[m1:, n1:]


# ------------------------------------------------------- device operand staging

class DeviceOperand:
    """A caller operand seen as a CUDA tensor with unit column stride.

    ``t`` is the tensor the kernels use; ``ld`` its row stride.  When the
    caller's buffer is on the host (or has an unusable layout) ``t`` is a
    staged copy and ``commit()`` writes the result back in place."""

    def __init__(self, x, dtype=None, device=None, writable=False, stream=None, lower=False):
        torch = _torch()
        self.src = as_array(x)
        self.writable = writable
        self.staged = False
        self.lower = False
        src = self.src
        if isinstance(src, torch.Tensor):
            t = src
        else:
            shares = isinstance(src, np.ndarray) and src.flags.c_contiguous
            t = torch.from_numpy(np.ascontiguousarray(src))
            lower = lower and shares
        want = _as_torch_dtype(dtype) if dtype is not None else (
            t.dtype if t.dtype in (torch.float32, torch.float64) else torch.float64)
        if device is None:
            device = t.device if t.is_cuda else torch.device("cuda", torch.cuda.current_device())
        rows, cols = int(t.shape[0]), int(t.shape[1])
        ok = (t.is_cuda and t.device == device and t.dtype == want
              and (cols == 1 or t.stride(1) == 1) and (rows == 1 or t.stride(0) >= cols))
        if ok:
            self.t = t
        elif (lower and not t.is_cuda and rows == cols and rows > 1 and t.dtype == want
              and t.stride(1) == 1 and t.stride(0) >= cols):
            # host C of an AtA call: only the lower triangle is read or written by
            # the kernels, so only lower block-trapezoids cross PCIe (~51% of C)
            self.t = torch.empty((rows, cols), dtype=want, device=device)
            self.host = t
            _copy_lower(self.t, t, to_device=True)
            self.lower = True
            self.staged = True
        elif (want == torch.float64 and t.dtype == want and not t.is_cuda and cols % 2 == 1 and rows > 1
              and rows * cols >= (1 << 20) and t.is_contiguous()):
            # odd-width fp64 host operand: staged straight into an even-pitch
            # buffer (16-byte rows for the TMA-fed leaf kernel, ata.even_pitch)
            buf = torch.empty((rows, cols + 1), dtype=want, device=device)
            rc = _cudart().cudaMemcpy2DAsync(buf.data_ptr(), (cols + 1) * 8, t.data_ptr(), cols * 8, cols * 8,
                                             rows, 1, _stream_ptr())
            if rc != 0:
                raise RuntimeError(f"cudaMemcpy2DAsync failed ({rc})")
            self.t = buf[:, :cols]
            self.keep = buf
            self.staged = True
        else:
            self.t = t.to(device=device, dtype=want).contiguous()
            self.staged = True
        self.rows, self.cols = rows, cols
        self.ld = int(self.t.stride(0)) if rows > 1 else cols

    @property
    def ptr(self) -> int:
        return int(self.t.data_ptr())

    @property
    def elems(self) -> int:
        return (self.rows - 1) * self.ld + self.cols

    def commit(self):
        """Write a staged result back into the caller's buffer."""
        if not (self.writable and self.staged):
            return
        torch = _torch()
        if self.lower:
            _copy_lower(self.host, self.t, to_device=False)
            return
        if isinstance(self.src, torch.Tensor):
            self.src.copy_(self.t)
        else:
            host = self.t.cpu().numpy()
            np.copyto(self.src, host.astype(self.src.dtype, copy=False))


_CUDART = None


def _cudart():
    global _CUDART
    if _CUDART is None:
        import ctypes
        lib = ctypes.CDLL("libcudart.so.12")
        lib.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                          ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t,
                                          ctypes.c_int, ctypes.c_void_p]
        lib.cudaStreamSynchronize.argtypes = [ctypes.c_void_p]
        _CUDART = lib
    return _CUDART


def _copy_lower(dst, src, to_device: bool, blocks: int = 64, step: int | None = None):
    """Copy the lower block-trapezoids of a square row-major matrix between host
    and device (rows [r0, r1) x columns [0, r1)); ~(1/2 + 1/(2*blocks)) of it.
    `step` (rows per band) overrides `blocks`."""
    torch = _torch()
    n = int(dst.shape[0])
    es = dst.element_size()
    lib = _cudart()
    stream = _stream_ptr()
    kind = 1 if to_device else 2   # cudaMemcpyHostToDevice / DeviceToHost
    step = max(1, -(-n // blocks)) if step is None else max(1, int(step))
    for r0 in range(0, n, step):
        r1 = min(n, r0 + step)
        d = dst.data_ptr() + r0 * dst.stride(0) * es
        s = src.data_ptr() + r0 * src.stride(0) * es
        rc = lib.cudaMemcpy2DAsync(d, dst.stride(0) * es, s, src.stride(0) * es, r1 * es, r1 - r0, kind,
                                   stream)
        if rc != 0:
            raise RuntimeError(f"cudaMemcpy2DAsync failed ({rc})")
    if not to_device:
        lib.cudaStreamSynchronize(stream)


def _stream_ptr():
    torch = _torch()
    return int(torch.cuda.current_stream().cuda_stream)


def _dtcode(t):
    return nat.dtype_code(t.dtype)


# -------------------------------------------------------------- leaf kernels

def naive_gemm_atb(A, B, C, alpha=1.0, counter: MultCounter | None = None, work=None) -> None:
    """C += alpha * A^T B, A m x n, B m x k, C n x k (matrix.py:269-289), on the GPU.
    ``work`` is accepted for signature compatibility; the kernel needs no scratch."""
    a, b, c = as_array(A), as_array(B), as_array(C)
    m, n = a.shape
    if b.shape[0] != m:
        raise ShapeMismatchError(f"shape mismatch: A is {tuple(a.shape)}, B is {tuple(b.shape)}")
    k = b.shape[1]
    if tuple(c.shape) != (n, k):
        raise ShapeMismatchError(f"shape mismatch: C is {tuple(c.shape)}, expected {(n, k)}")
    lib = nat.load()
    C_ = DeviceOperand(c, writable=True)
    A_ = DeviceOperand(a, dtype=C_.t.dtype, device=C_.t.device)
    B_ = DeviceOperand(b, dtype=C_.t.dtype, device=C_.t.device)
    nat.check(lib.ata_gemm_atb(_dtcode(C_.t), A_.ptr, A_.ld, B_.ptr, B_.ld, m, n, k, C_.ptr, C_.ld,
                               float(alpha), _stream_ptr()))
    C_.commit()
    if counter is not None:
        counter.add(m * n * k)


def naive_syrk_lower(A, C, alpha=1.0, counter: MultCounter | None = None, work=None) -> None:
    """Lower triangle of C += alpha * A^T A (matrix.py:292-311); the strict
    upper triangle is never read or written by the kernel."""
    a, c = as_array(A), as_array(C)
    m, n = a.shape
    if tuple(c.shape) != (n, n):
        raise ShapeMismatchError(f"shape mismatch: C is {tuple(c.shape)}, expected {(n, n)}")
    lib = nat.load()
    C_ = DeviceOperand(c, writable=True)
    A_ = DeviceOperand(a, dtype=C_.t.dtype, device=C_.t.device)
    nat.check(lib.ata_syrk_lower(_dtcode(C_.t), A_.ptr, A_.ld, m, n, C_.ptr, C_.ld, float(alpha),
                                 _stream_ptr()))
    C_.commit()
    if counter is not None:
        counter.add(m * n * (n + 1) // 2)


def add_truncated(dst, src, scale=1.0) -> None:
    """dst[:r,:c] += scale * src[:r,:c] (matrix.py:218-239)."""
    d, s = as_array(dst), as_array(src)
    if abs(d.shape[0] - s.shape[0]) > 1 or abs(d.shape[1] - s.shape[1]) > 1:
        raise ShapeMismatchError(
            f"shape mismatch: add_truncated {tuple(d.shape)} vs {tuple(s.shape)}")
    lib = nat.load()
    D_ = DeviceOperand(d, writable=True)
    S_ = DeviceOperand(s, dtype=D_.t.dtype, device=D_.t.device)
    nat.check(lib.ata_add_truncated(_dtcode(D_.t), D_.ptr, D_.ld, D_.rows, D_.cols, S_.ptr, S_.ld,
                                    S_.rows, S_.cols, float(scale), _stream_ptr()))
    D_.commit()


@dataclass
class PackedLowerTriangular:
    """n(n+1)/2 lower-triangle entries, rows concatenated (matrix.py:319-330).
    ``data`` is a 1-D tensor (device) or array."""
    n: int
    data: object = field(repr=False)

    def __post_init__(self):
        if tuple(self.data.shape) != (self.n * (self.n + 1) // 2,):
            raise ShapeMismatchError(
                f"shape mismatch: packed length {tuple(self.data.shape)} for n={self.n}")


def pack_lower(C, out=None) -> PackedLowerTriangular:
    """Packed copy of the lower triangle of square C (matrix.py:353-360)."""
    torch = _torch()
    c = as_array(C)
    n = c.shape[0]
    if c.shape[1] != n:
        raise ShapeMismatchError("shape mismatch: pack_lower needs a square block")
    C_ = DeviceOperand(c)
    if out is None:
        out = torch.empty(n * (n + 1) // 2, dtype=C_.t.dtype, device=C_.t.device)
    nat.check(nat.load().ata_pack_lower(_dtcode(C_.t), C_.ptr, C_.ld, n, int(out.data_ptr()),
                                        _stream_ptr()))
    if not isinstance(c, torch.Tensor):
        return PackedLowerTriangular(n, out.cpu().numpy())
    return PackedLowerTriangular(n, out)


def unpack_lower(p: PackedLowerTriangular, C, accumulate: bool = False) -> None:
    """Write (or add, for the parent sums of distsim.py:208-216) packed
    entries into the lower triangle of square C (matrix.py:363-370)."""
    torch = _torch()
    c = as_array(C)
    n = c.shape[0]
    if c.shape[1] != n or n != p.n:
        raise ShapeMismatchError("shape mismatch: unpack_lower target")
    C_ = DeviceOperand(c, writable=True)
    data = p.data if isinstance(p.data, torch.Tensor) else torch.from_numpy(np.asarray(p.data))
    data = data.to(device=C_.t.device, dtype=C_.t.dtype).contiguous()
    nat.check(nat.load().ata_unpack_lower(_dtcode(C_.t), int(data.data_ptr()), n, C_.ptr, C_.ld,
                                          int(bool(accumulate)), _stream_ptr()))
    C_.commit()


def mirror_lower_to_upper(C) -> None:
    """C[i, j] = C[j, i] for i < j (matrix.py:373-380)."""
    c = as_array(C)
    n = c.shape[0]
    if c.shape[1] != n:
        raise ShapeMismatchError("shape mismatch: mirror needs a square block")
    C_ = DeviceOperand(c, writable=True)
    nat.check(nat.load().ata_mirror_lower(_dtcode(C_.t), C_.ptr, C_.ld, n, _stream_ptr()))
    C_.commit()


# ------------------------------------------------------------ ATAM files
# The reference's binary matrix format (matrix.py:383-417): magic b"ATAM",
# three little-endian uint64 (rows, cols, scalar width 4 or 8), then the
# row-major little-endian scalars.  Device tensors are staged through the host.

_ATAM = b"ATAM"
_ATAM_HEAD = struct.Struct("<4sQQQ")


def write_matrix(path, M) -> None:
    """Write an f32/f64 matrix (numpy, torch host or device, DenseMatrix,
    MatrixView) as an ATAM file; other dtypes are ShapeMismatchError, as in
    the reference (matrix.py:392-402)."""
    a = as_array(M)
    torch = _torch()
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    width = a.dtype.itemsize if a.dtype.type in (np.float32, np.float64) else 0
    if width not in (4, 8):
        raise ShapeMismatchError("shape mismatch: only f32/f64 matrices supported")
    data = np.ascontiguousarray(a, dtype="<f4" if width == 4 else "<f8")
    with open(path, "wb") as fh:
        fh.write(_ATAM_HEAD.pack(_ATAM, data.shape[0], data.shape[1], width))
        fh.write(data.tobytes())


def read_matrix(path, device=None) -> DenseMatrix:
    """Read an ATAM file into a DenseMatrix (host numpy, or a torch tensor on
    `device`).  Bad magic / scalar width -> ValueError (matrix.py:405-417)."""
    with open(path, "rb") as fh:
        head = fh.read(_ATAM_HEAD.size)
        if len(head) < 4 or head[:4] != _ATAM:
            raise ValueError(f"not an ATAM file: bad magic {head[:4]!r}")
        if len(head) < _ATAM_HEAD.size:
            raise ValueError("truncated ATAM header")
        _, rows, cols, width = _ATAM_HEAD.unpack(head)
        if width not in (4, 8):
            raise ValueError(f"bad ATAM scalar width {width}")
        payload = fh.read(rows * cols * width)
    if len(payload) != rows * cols * width:
        raise ValueError("truncated ATAM payload")
    data = np.frombuffer(payload, dtype="<f4" if width == 4 else "<f8").reshape(rows, cols)
    data = data.astype(np.float32 if width == 4 else np.float64)
    if device is None:
        return DenseMatrix(data)
    return DenseMatrix(_torch().from_numpy(data).to(device))
