"""Task trees (host logic) pinned against trees the reference built
(tests/golden/trees.json, tools/make_golden_cli.py): rendering, per-process
leaf tasks, ownership chains, level formulas, unsplittable shapes; plus the
covering property every tree must have (the leaves' contributions sum to
the full lower triangle)."""
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2110_13042_b200 import tasktree as T
from paper_2110_13042_b200.errors import UnknownProcessError, UnsplittableError

GOLD = json.loads((Path(__file__).parent / "golden" / "trees.json").read_text())


def _reg(r):
    return None if r is None else [r.row_offset, r.col_offset, r.rows, r.cols]


@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: f"{c['mode'][0]}{c['p']}-{c['m']}x{c['n']}")
def test_tree_matches_reference(case):
    build = T.build_tree_distributed if case["mode"] == "distributed" else T.build_tree_shared
    if "error" in case:
        with pytest.raises(UnsplittableError):
            build(case["p"], case["m"], case["n"])
        return
    t = build(case["p"], case["m"], case["n"])
    assert T.render_tree(t) == case["render"]
    assert t.depth == case["depth"]
    for q, (kind, a, b, c, parent, owner) in enumerate(case["leaves"]):
        task = T.leaf_task(t, q)
        assert [task.computation.value, _reg(task.a_region), _reg(task.b_region), _reg(task.c_region),
                task.parent, task.owner] == [kind, a, b, c, parent, owner]
    assert [[nd.id for nd in T.path_to_root(t, q)] for q in range(case["p"])] == case["chains"]


def test_level_formulas_match_reference():
    assert [T.levels_distributed(p) for p in range(1, 131)] == GOLD["levels"]["distributed"]
    assert [T.levels_shared(p) for p in range(1, 131)] == GOLD["levels"]["shared"]
    with pytest.raises(ValueError):
        T.levels_distributed(0)
    with pytest.raises(UnknownProcessError):
        T.leaf_task(T.build_tree_distributed(2, 8, 8), 2)


@pytest.mark.parametrize("mode", ["distributed", "shared"])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 6, 7, 8, 12, 16])
def test_leaves_cover_the_gram_matrix(mode, p):
    """Sum of every leaf's contribution (AtA leaves: lower triangle of their
    diagonal block; AtB leaves: their rectangle) == lower(A^T A)."""
    m, n = 37, 29
    a = np.random.default_rng(p).standard_normal((m, n))
    t = (T.build_tree_distributed if mode == "distributed" else T.build_tree_shared)(p, m, n)
    c = np.zeros((n, n))
    for q in range(p):
        task = T.leaf_task(t, q)
        ar = task.a_region
        br = task.b_region or ar
        rows = slice(ar.row_offset, ar.row_offset + ar.rows)
        assert (br.row_offset, br.rows) == (ar.row_offset, ar.rows)
        ci = np.arange(ar.col_offset, ar.col_offset + ar.cols)
        cj = np.arange(br.col_offset, br.col_offset + br.cols)
        full = np.zeros((n, n))
        full[np.ix_(ci, cj)] = a[rows][:, ci].T @ a[rows][:, cj]
        c += np.where(T.covered_mask(task, n), full, 0.0)
    assert np.allclose(c, np.tril(a.T @ a), rtol=1e-12, atol=1e-12)
