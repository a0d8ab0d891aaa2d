"""2D cluster trees: build_cluster_tree's bisection and kmeans2 splits
(geometry.py:146-243) on 2D point sets, against trees the reference built on the same points
(tests/golden/make_golden_2d.py): the tree permutation and every node's index range equal."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_2d.npz")


def _ranges(ct):
    out = []

    def walk(nd):
        out.append((nd.start, nd.end))
        for c in nd.children:
            walk(c)
    walk(ct.root)
    return np.array(out, dtype=np.int64)


@pytest.mark.parametrize("name", ["lshape24", "grid20", "rand500"])
@pytest.mark.parametrize("strategy", ["kmeans2", "bisection"])
@pytest.mark.parametrize("leaf", [16, 32])
def test_tree_2d_matches_reference(name, strategy, leaf):
    import paper_1812_08324_b200 as P

    g = np.load(GOLD)
    ct = P.build_cluster_tree(g[f"pts_{name}"], leaf_size=leaf, strategy=strategy)
    assert np.array_equal(ct.perm.inverse, g[f"order_{name}_{strategy}_{leaf}"])
    assert np.array_equal(_ranges(ct), g[f"ranges_{name}_{strategy}_{leaf}"])


def test_tree_unknown_strategy():
    import paper_1812_08324_b200 as P

    with pytest.raises(ValueError):
        P.build_cluster_tree(np.zeros((4, 2)), strategy="quadtree")
