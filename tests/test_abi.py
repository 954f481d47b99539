"""The C-ABI library loads on a CPU-only host and exports every symbol
include/atamul_b200.h declares (no compute calls without a GPU)."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_2110_13042_b200 import _native as nat
from paper_2110_13042_b200.build import build

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    names = []
    for h in (ROOT / "include").glob("*.h"):
        text = h.read_text()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names += re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(ata_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_library_builds_and_exports_header_symbols():
    build()
    lib = ctypes.CDLL(str(nat.LIB_PATH))
    declared = _declared()
    assert len(declared) >= 11
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(nat.EXPORTS)


def test_abi_struct_layout_and_errors():
    lib = nat.load()
    assert lib.ata_abi_op_size() == nat.OP_DTYPE.itemsize == 680
    assert lib.ata_version() >= 100
    assert lib.ata_strerror(-3) == b"workspace undersized"


def test_plan_validation_without_gpu():
    """Validation happens before any launch: bad windows fail with the
    reference's exception classes even on a host without a device."""
    import numpy as np
    from paper_2110_13042_b200 import planner
    from paper_2110_13042_b200.errors import ShapeMismatchError, WorkspaceUndersizedError
    with pytest.raises(WorkspaceUndersizedError):
        planner.plan_ata_reference(8, 8, 8, 8, 1, [])
    # a workspace window beyond the arena is rejected by the native validator
    ws = __import__("paper_2110_13042_b200").workspace_for_ata(16, 16, 4)
    plan = planner.plan_ata_reference(16, 16, 16, 16, 4, ws.level_offsets())
    lib = nat.load()
    fake = ctypes.c_void_p(16)  # never dereferenced: validation fails first
    rc = lib.ata_run_plan(0, plan.ops.ctypes.data_as(ctypes.c_void_p), len(plan.ops), fake, 256,
                          fake, 256, fake, 256, fake, 8, None, 0, 1.0, None)
    assert rc == -3
    with pytest.raises(WorkspaceUndersizedError):
        nat.check(rc)
    bad = plan.ops.copy()
    bad[0]["s"][0]["rows"] = 999
    rc = lib.ata_run_plan(0, bad.ctypes.data_as(ctypes.c_void_p), len(bad), fake, 256,
                          fake, 256, fake, 256, fake, 10**6, None, 0, 1.0, None)
    assert rc == -1


def test_python_surface_covers_reference_exports():
    """Every name of the reference's atamul.__all__ (pkg/src/atamul/__init__.py:29-46)
    is exported under the same name (import swap)."""
    import paper_2110_13042_b200 as P
    reference_all = [
        "AtamulError", "CommStats", "ComputationType", "DEFAULT_THRESHOLD", "DenseMatrix",
        "InvalidMeasurementError", "MatrixView", "MultCounter", "PackedLowerTriangular", "ProtocolError",
        "Region", "ShapeMismatchError", "SharedRunner", "StrassenWorkspace", "Task", "TaskTree",
        "TooManyWorkersError", "UnknownProcessError", "UnsplittableError", "UnsupportedSizeError",
        "WorkspaceUndersizedError", "add_truncated", "ata", "ata_d", "ata_full", "ata_mult_count", "ata_s",
        "build_tree_distributed", "build_tree_shared", "effective_gflops", "fast_strassen", "gen_matrix",
        "leaf_task", "levels_distributed", "levels_shared", "mirror_lower_to_upper", "naive_gemm_atb",
        "naive_syrk_lower", "pack_lower", "path_to_root", "read_matrix", "render_tree", "split4",
        "strassen_mult_count", "unpack_lower", "verify_comm_bounds", "workspace_for", "workspace_for_ata",
        "write_matrix"]
    missing = [n for n in reference_all if not hasattr(P, n)]
    assert not missing, missing
    from paper_2110_13042_b200.execute import execute_leaf, workspace_for_leaf  # noqa: F401
    from paper_2110_13042_b200.shared import MAX_WORKERS
    assert MAX_WORKERS == 128
