"""Point sets, cluster trees and admissibility -- API of levyh.geometry
(/root/reference/pkg/src/levyh/geometry.py:25-263).

The tree is built natively (csrc/tree.cpp, median bisection with the same
stable-argsort rule as geometry.py:146-154) and mirrored here as
``ClusterNode`` objects so callers see the reference's types.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib

__all__ = ["PointSet", "ClusterNode", "Permutation", "ClusterTree", "build_cluster_tree",
           "admissible", "bbox_distance"]


class PointSet:
    """Nonempty 1D or 2D finite points, stored (n, d) (geometry.py:37-63)."""

    def __init__(self, points):
        pts = np.asarray(points, dtype=float)
        if pts.ndim == 1:
            pts = pts[:, None]
        if pts.ndim != 2:
            raise ValueError("points must be an (n, d) array")
        if pts.shape[0] == 0:
            raise ValueError("point set must be nonempty")
        if pts.shape[1] not in (1, 2):
            raise ValueError("only 1D and 2D point sets are supported")
        if not np.all(np.isfinite(pts)):
            raise ValueError("points must have finite coordinates")
        self.points = np.ascontiguousarray(pts)

    def __len__(self):
        return self.points.shape[0]

    @property
    def dim(self):
        return self.points.shape[1]


@dataclass
class ClusterNode:
    """Contiguous tree-order range with its bounding box (geometry.py:66-107)."""

    start: int
    end: int
    bbox_lo: np.ndarray
    bbox_hi: np.ndarray
    children: tuple = field(default=())

    @property
    def size(self):
        return self.end - self.start

    @property
    def is_leaf(self):
        return not self.children

    @property
    def diameter(self):
        return float(np.linalg.norm(self.bbox_hi - self.bbox_lo))

    @property
    def center(self):
        return 0.5 * (self.bbox_lo + self.bbox_hi)

    def depth(self):
        d, stack = 0, [(self, 0)]
        while stack:
            n, k = stack.pop()
            d = max(d, k)
            stack.extend((c, k + 1) for c in n.children)
        return d

    def leaves(self):
        stack = [self]
        while stack:
            n = stack.pop()
            if n.is_leaf:
                yield n
            else:
                stack.extend(reversed(n.children))


@dataclass
class Permutation:
    """forward[i_orig] = i_tree, inverse[i_tree] = i_orig (geometry.py:110-127)."""

    forward: np.ndarray
    inverse: np.ndarray

    def to_tree(self, v):
        return np.asarray(v)[self.inverse]

    def from_tree(self, v):
        return np.asarray(v)[self.forward]


class ClusterTree:
    """Root node, permutation, points in tree order; owns the native tree."""

    def __init__(self, handle, points, dim):
        self._h = handle
        L = _lib.lib()
        n = points.shape[0]
        order = np.empty(n, dtype=np.int64)
        L.lh_tree_order(handle, _lib.host_ptr(order))
        inv = order.astype(np.intp)
        fwd = np.empty(n, dtype=np.intp)
        fwd[inv] = np.arange(n, dtype=np.intp)
        self.perm = Permutation(forward=fwd, inverse=inv)
        self.points = points[inv]
        self.dim = dim
        self._root = None

    def __len__(self):
        return self.points.shape[0]

    @property
    def handle(self):
        return self._h

    @property
    def root(self):
        if self._root is None:
            L = _lib.lib()
            nn = L.lh_tree_num_nodes(self._h)
            lohi = np.empty(2 * nn, dtype=np.int64)
            bbox = np.empty(2 * nn * self.dim, dtype=np.float64)
            kids = np.empty(2 * nn, dtype=np.int32)
            L.lh_tree_nodes(self._h, _lib.host_ptr(lohi), _lib.host_ptr(bbox), _lib.host_ptr(kids))
            bbox = bbox.reshape(nn, 2, self.dim)
            nodes = [None] * nn
            for i in range(nn - 1, -1, -1):  # children have larger ids than parents
                k0, k1 = int(kids[2 * i]), int(kids[2 * i + 1])
                ch = () if k0 < 0 else (nodes[k0], nodes[k1])
                nodes[i] = ClusterNode(int(lohi[2 * i]), int(lohi[2 * i + 1]), bbox[i, 0].copy(),
                                       bbox[i, 1].copy(), ch)
            self._root = nodes[0]
        return self._root

    def __del__(self):
        try:
            if self._h:
                _lib.lib().lh_tree_destroy(self._h)
                self._h = None
        except Exception:
            pass


def build_cluster_tree(pts, leaf_size=64, strategy="bisection"):
    """geometry.py:191-243: median bisection along the widest axis, or ``kmeans2``
    (geometry.py:157-188, deterministic 2-means) -- the same trees bit for bit."""
    if not isinstance(pts, PointSet):
        pts = PointSet(pts)
    if leaf_size < 1:
        raise ValueError("leaf_size must be >= 1")
    codes = {"bisection": 0, "kmeans2": 1}
    if strategy not in codes:
        raise ValueError(f"unknown strategy {strategy!r}")
    h = C.c_void_p()
    rc = _lib.lib().lh_tree_build_strategy(None, _lib.host_ptr(pts.points), pts.points.shape[0], pts.dim,
                                           int(leaf_size), codes[strategy], C.byref(h))
    _lib.check(rc)
    return ClusterTree(h, pts.points, pts.dim)


def bbox_distance(a, b):
    """geometry.py:246-250."""
    gap = np.maximum(a.bbox_lo - b.bbox_hi, b.bbox_lo - a.bbox_hi)
    gap = np.maximum(gap, 0.0)
    return float(np.linalg.norm(gap))


def admissible(a, b, eta):
    """geometry.py:253-263."""
    dist = bbox_distance(a, b)
    if dist <= 0.0:
        return False
    return min(a.diameter, b.diameter) <= eta * dist
