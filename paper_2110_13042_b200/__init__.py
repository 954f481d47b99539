"""paper_2110_13042_b200 — B200-native AtA (C = alpha*A^T A + C, lower triangle,
Strassen sub-kernel) behind the reference ``atamul`` entry points.

Drop-in surface (reference pkg/src/atamul/__init__.py:9-27, hot path only):
``ata``, ``ata_full``, ``ata_mult_count``, ``workspace_for_ata``,
``fast_strassen``, ``workspace_for``, ``strassen_mult_count``,
``DEFAULT_THRESHOLD``, ``StrassenWorkspace``, ``naive_gemm_atb``,
``naive_syrk_lower``, ``add_truncated``, ``mirror_lower_to_upper``,
``pack_lower``/``unpack_lower``/``PackedLowerTriangular``, ``split4``,
``DenseMatrix``/``MatrixView``, ``MultCounter``, ``effective_gflops``,
``gen_matrix``, the exception classes, the executors ``ata_s`` /
``SharedRunner`` (leaves of the shared task tree on concurrent CUDA streams,
shared.py), ``ata_d`` / ``CommStats`` / ``verify_comm_bounds`` (the
distribute-compute-retrieve executor over NCCL ranks or simulated on one GPU,
distsim.py), ``execute_leaf`` / ``workspace_for_leaf`` (execute.py), the
multi-GPU entries ``dist.ata_dist`` (row shards) and ``dist.ata_tree``,
and the formats/callers either side of the path: ATAM ``read_matrix`` /
``write_matrix``, the task trees (``build_tree_*``, ``render_tree``) and the
``atamul`` command line (``python -m paper_2110_13042_b200.cli``).
"""
from .ata import AUTO, ata, ata_full, ata_mult_count, release_cached_buffers, workspace_for_ata
from .distsim import CommStats, ata_d, verify_comm_bounds
from .errors import (AtamulError, InvalidMeasurementError, NativeError, ProtocolError,
                     ShapeMismatchError, TooManyWorkersError, UnknownProcessError,
                     UnsplittableError, UnsupportedSizeError, WorkspaceUndersizedError)
from .matrix import (DenseMatrix, MatrixView, MultCounter, PackedLowerTriangular, add_truncated,
                     count_allocations, mirror_lower_to_upper, naive_gemm_atb, naive_syrk_lower,
                     pack_lower, read_matrix, split4, unpack_lower, write_matrix)
from .execute import execute_leaf, workspace_for_leaf
from .measure import check_tolerance, effective_gflops, gen_matrix
from .shared import SharedRunner, ata_s
from .strassen import fast_strassen, strassen_mult_count, workspace_for
from .tasktree import (ComputationType, Region, Task, TaskTree, build_tree_distributed,
                       build_tree_shared, leaf_task, levels_distributed, levels_shared, path_to_root,
                       render_tree)
from .workspace import DEFAULT_THRESHOLD, StrassenWorkspace

__version__ = "0.1.0"

__all__ = [
    "AUTO", "AtamulError", "CommStats", "SharedRunner", "ata_d", "ata_s", "execute_leaf",
    "verify_comm_bounds", "workspace_for_leaf", "DEFAULT_THRESHOLD", "DenseMatrix", "InvalidMeasurementError",
    "MatrixView", "MultCounter", "NativeError", "PackedLowerTriangular", "ProtocolError",
    "ShapeMismatchError", "StrassenWorkspace", "TooManyWorkersError", "UnknownProcessError",
    "UnsplittableError", "UnsupportedSizeError", "WorkspaceUndersizedError", "add_truncated",
    "ata", "ata_full", "ata_mult_count", "check_tolerance", "count_allocations",
    "effective_gflops", "fast_strassen", "gen_matrix", "mirror_lower_to_upper",
    "naive_gemm_atb", "naive_syrk_lower", "pack_lower", "split4", "strassen_mult_count",
    "unpack_lower", "workspace_for", "workspace_for_ata", "release_cached_buffers",
    # callers / formats either side of the path
    "ComputationType", "Region", "Task", "TaskTree", "build_tree_distributed",
    "build_tree_shared", "leaf_task", "levels_distributed", "levels_shared", "path_to_root",
    "read_matrix", "render_tree", "write_matrix",
]
