"""ctypes binding of the C ABI in include/atamul_b200.h.

The library is built in-tree (``build.py``) and loaded from
``paper_2110_13042_b200/_lib/libatamul_b200.so``.  There is no fallback: if
the library is missing the import of any compute entry point raises.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from . import errors

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libatamul_b200.so"
# developer knob for A/B kernel experiments: load another in-tree build instead
if os.environ.get("ATA_LIB_PATH"):
    LIB_PATH = Path(os.environ["ATA_LIB_PATH"]).resolve()

ATA_F64, ATA_F32, ATA_TF32 = 0, 1, 2
OP_GEMM, OP_SYRK, OP_COMBO, OP_UPDATE, OP_FILL, OP_COMBO4, OP_POSTADD7, OP_ROUND = \
    0, 1, 2, 3, 4, 5, 6, 7
BASE_A, BASE_C, BASE_WS, BASE_B = 0, 1, 2, 3
MAX_TERMS, MAX_DESTS = 4, 8
PROD_MAX_TERMS = 2
OPF_RIDE = 1

# numpy mirrors of ata_ref / ata_op (include/atamul_b200.h)
REF_DTYPE = np.dtype([("base", "<i4"), ("rows", "<i4"), ("off", "<i8"), ("ld", "<i8"),
                      ("cols", "<i4"), ("region", "<i4"), ("sign", "<f8")], align=True)
OP_DTYPE = np.dtype([("type", "<i4"), ("m", "<i4"), ("n", "<i4"), ("k", "<i4"),
                     ("ns", "<i4"), ("nt", "<i4"), ("nd", "<i4"), ("accumulate", "<i4"),
                     ("group", "<i4"), ("flags", "<i4"),
                     ("s", REF_DTYPE, (MAX_TERMS,)), ("t", REF_DTYPE, (MAX_TERMS,)),
                     ("d", REF_DTYPE, (MAX_DESTS,))], align=True)

EXPORTS = [
    "ata_last_error", "ata_strerror", "ata_version", "ata_abi_op_size",
    "ata_syrk_lower", "ata_gemm_atb", "ata_add_truncated", "ata_mirror_lower",
    "ata_pack_lower", "ata_unpack_lower", "ata_run_plan", "ata_sync_ints_needed", "ata_launch_count", "ata_ride_count",
]

_CODE_TO_EXC = {
    -1: errors.ShapeMismatchError,
    -2: errors.UnsplittableError,
    -3: errors.WorkspaceUndersizedError,
    -5: errors.UnsupportedSizeError,
    -6: errors.ProtocolError,
    -100: errors.NativeError,
    -101: ValueError,
}

_lib = None


def load() -> ctypes.CDLL:
    """Load (once) the native library; raise loudly when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise errors.NativeError(
            f"native library {LIB_PATH} not built: run `python -m paper_2110_13042_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(LIB_PATH))
    c_i32, c_i64, c_dbl, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
    lib.ata_last_error.restype = ctypes.c_char_p
    lib.ata_strerror.restype = ctypes.c_char_p
    lib.ata_strerror.argtypes = [ctypes.c_int]
    lib.ata_version.restype = ctypes.c_int
    lib.ata_abi_op_size.restype = ctypes.c_int
    lib.ata_syrk_lower.argtypes = [ctypes.c_int, c_vp, c_i64, c_i32, c_i32, c_vp, c_i64, c_dbl, c_vp]
    lib.ata_gemm_atb.argtypes = [ctypes.c_int, c_vp, c_i64, c_vp, c_i64, c_i32, c_i32, c_i32, c_vp,
                                 c_i64, c_dbl, c_vp]
    lib.ata_add_truncated.argtypes = [ctypes.c_int, c_vp, c_i64, c_i32, c_i32, c_vp, c_i64, c_i32,
                                      c_i32, c_dbl, c_vp]
    lib.ata_mirror_lower.argtypes = [ctypes.c_int, c_vp, c_i64, c_i32, c_vp]
    lib.ata_pack_lower.argtypes = [ctypes.c_int, c_vp, c_i64, c_i32, c_vp, c_vp]
    lib.ata_unpack_lower.argtypes = [ctypes.c_int, c_vp, c_i32, c_vp, c_i64, c_i32, c_vp]
    lib.ata_run_plan.argtypes = [ctypes.c_int, c_vp, c_i32, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64,
                                 c_vp, c_i64, c_vp, c_i64, c_dbl, c_vp]
    lib.ata_sync_ints_needed.argtypes = [ctypes.c_int, c_vp, c_i32]
    lib.ata_sync_ints_needed.restype = ctypes.c_int64
    lib.ata_launch_count.restype = ctypes.c_int64
    lib.ata_launch_count.argtypes = []
    lib.ata_ride_count.restype = ctypes.c_int64
    lib.ata_ride_count.argtypes = []
    for name in EXPORTS:
        getattr(lib, name).restype = getattr(lib, name).restype or ctypes.c_int
    if lib.ata_abi_op_size() != OP_DTYPE.itemsize:
        raise errors.NativeError(
            f"ABI mismatch: sizeof(ata_op)={lib.ata_abi_op_size()} vs {OP_DTYPE.itemsize}")
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = load().ata_last_error().decode(errors="replace")
    exc = _CODE_TO_EXC.get(rc, errors.NativeError)
    raise exc(msg or load().ata_strerror(rc).decode())


def dtype_code(torch_dtype, precision: str = "fp32") -> int:
    """f64 -> DMMA path; f32 -> 3xTF32 ("fp32", default, fp32-level accuracy)
    or single-pass TF32 ("tf32", the c5 configuration's leaves)."""
    import torch
    if torch_dtype == torch.float64:
        return ATA_F64
    if torch_dtype == torch.float32:
        if precision == "tf32":
            return ATA_TF32
        if precision != "fp32":
            raise ValueError(f"unknown precision {precision!r}")
        return ATA_F32
    raise errors.ShapeMismatchError(f"shape mismatch: only f32/f64 supported, got {torch_dtype}")


def loaded_path() -> str:
    return os.fspath(LIB_PATH)
