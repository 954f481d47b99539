"""Containers and quadrant geometry: DenseMatrix /
MatrixView / split4 (reference matrix.py:62-215) on host arrays and CPU
tensors -- no GPU needed.  The GPU tests feed MatrixView operands through
ata / fast_strassen (tests/test_gpu_executors.py)."""
import numpy as np
import pytest
import torch

import paper_2110_13042_b200 as P


@pytest.mark.parametrize("m,n", [(2, 2), (3, 3), (5, 2), (7, 9), (13, 2), (64, 63), (2, 101)])
def test_split4_floor_ceil_geometry(m, n):
    base = P.DenseMatrix(np.arange(m * n, dtype=np.float64).reshape(m, n))
    q = P.split4(base.view())
    m1, n1 = m // 2, n // 2
    assert [(b.rows, b.cols) for b in q] == [(m1, n1), (m1, n - n1), (m - m1, n1), (m - m1, n - n1)]
    assert [(b.row_offset, b.col_offset) for b in q] == [(0, 0), (0, n1), (m1, 0), (m1, n1)]
    # every element lands in exactly one quadrant, and views are zero-copy windows
    hit = np.zeros((m, n), dtype=int)
    for b in q:
        hit[b.row_offset:b.row_offset + b.rows, b.col_offset:b.col_offset + b.cols] += 1
        assert np.shares_memory(b.a, base.a)
        assert np.array_equal(b.a, base.a[b.row_offset:b.row_offset + b.rows,
                                           b.col_offset:b.col_offset + b.cols])
    assert np.all(hit == 1)
    # the array form gives the same blocks
    for b, x in zip(q, P.split4(base.a)):
        assert np.array_equal(b.a, x)


def test_split4_nested_views_and_tensors():
    base = P.DenseMatrix(torch.arange(90, dtype=torch.float64).reshape(9, 10))
    outer = base.view(1, 2, 7, 7)
    q = P.split4(outer)
    assert (q[3].row_offset, q[3].col_offset, q[3].rows, q[3].cols) == (4, 5, 4, 4)
    assert q[3].a.data_ptr() == base.a[4:, 5:].data_ptr()
    assert q[3].row_stride == 10
    qq = P.split4(q[3])
    assert (qq[0].row_offset, qq[0].col_offset) == (4, 5) and (qq[3].rows, qq[3].cols) == (2, 2)


def test_split4_unsplittable():
    for shape in ((1, 5), (5, 1), (1, 1)):
        with pytest.raises(P.UnsplittableError):
            P.split4(P.DenseMatrix.zeros(*shape).view())
        with pytest.raises(P.UnsplittableError):
            P.split4(np.zeros(shape))


def test_view_bounds_overlaps_and_casts():
    m = P.DenseMatrix.zeros(6, 6)
    a, b, c = m.view(0, 0, 3, 3), m.view(3, 3, 3, 3), m.view(2, 2, 2, 2)
    assert not a.overlaps(b) and a.overlaps(c) and c.overlaps(b)
    assert not a.overlaps(P.DenseMatrix.zeros(6, 6).view(0, 0, 3, 3))   # other base
    for bad in ((0, 0, 7, 1), (5, 0, 2, 1), (0, 4, 1, 3), (0, 0, 0, 2)):
        with pytest.raises(P.ShapeMismatchError):
            m.view(*bad)
    v = m.view(1, 1, 2, 2)
    v.a[0, 0] = 9.0
    assert m.a[1, 1] == 9.0
    assert P.DenseMatrix(np.ones((2, 3), dtype=np.int32)).a.dtype == np.float64   # matrix.py:73-74
    with pytest.raises(P.ShapeMismatchError):
        P.DenseMatrix(np.zeros((0, 3)))
    with pytest.raises(P.ShapeMismatchError):
        P.DenseMatrix(np.zeros(3))
