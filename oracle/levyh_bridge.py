"""Rebuild the REAL reference's block types (levyh.hmatrix Dense / LowRank / Hier /
FactoredDense, levyh.hops.HFactorization) from an H-matrix exported by the native library
(BASELINE INFRASTRUCTURE ONLY: bench.py's reference arm and tests).

The reference package is installed unmodified into baseline/_ref (DESIGN.md 6:
``pip install --no-index --no-build-isolation --no-deps --target baseline/_ref``).  It cannot
assemble or compress the BASELINE operators at N = 2^20 (dense N x N input, full SVDs:
SURVEY G7), so its own ``hops.matvec`` / ``hops.solve`` / ``hops.hlu`` are timed on factors
built on the GPU and exported in a separate process (bench.py --export-factors); the process
that times the reference never loads the native library.

The partition is replayed with the reference's own ``build_cluster_tree`` and ``admissible``
in the decision order of ``build_from_dense`` (hmatrix.py:319-337); leaves are zero-copy
views of the exported arena (dense leaves column-major = Fortran order, as scipy's
lu_factor leaves them).  A factored leaf gets the reference's ``pperm`` attribute
(hops.py:398: the net row permutation, which the export stores) and an identity ``piv``.
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

REF_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


def import_levyh():
    """The installed reference package (baseline/_ref), or None when it is not installed."""
    if os.path.isdir(os.path.join(REF_DIR, "levyh")) and REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import levyh  # noqa: F401
        import levyh.hmatrix
        import levyh.hops
        import levyh.geometry
    except Exception:
        return None
    return levyh


def _leaves(levyh, recs, arena, ranks, perm):
    H = levyh.hmatrix
    for rec in recs:
        r0, r1, c0, c1, kind, doff, uoff, voff, kcap, rslot, poff = (int(v) for v in rec)
        m, n = r1 - r0, c1 - c0
        if kind == 2:
            r = int(ranks[rslot])
            yield H.LowRank(arena[uoff:uoff + m * r].reshape(r, m).T, arena[voff:voff + n * r].reshape(r, n).T), r0, c0
        else:
            d = arena[doff:doff + m * n].reshape(n, m).T  # column-major leaf: F-contiguous view
            if kind == 3:
                b = H.FactoredDense(d, np.arange(m, dtype=np.int32))
                b.pperm = perm[poff:poff + m].astype(np.intp)
                yield b, r0, c0
            else:
                yield H.Dense(d), r0, c0


def hmatrix_from_export(levyh, points, leaf, recs, arena, ranks, perm, n_block=4, eta=1.0):
    """levyh.hmatrix.HMatrix over the exported leaves (same partition as build_from_dense)."""
    G, H = levyh.geometry, levyh.hmatrix
    ct = G.build_cluster_tree(np.asarray(points, dtype=float)[:, None], leaf_size=leaf)
    if not np.array_equal(ct.perm.inverse, np.arange(len(points))):
        raise ValueError("export bridge expects the identity tree permutation (1D sorted grid)")
    leaves = _leaves(levyh, recs, arena, ranks, perm)
    N = len(points)
    n_max = math.ceil(N / n_block)

    def build(rn, cn):
        m, n = rn.size, cn.size
        can_split = not rn.is_leaf and not cn.is_leaf
        if (m > n_max or n > n_max) and can_split:
            pass
        elif G.admissible(rn, cn, eta) and min(m, n) > leaf:
            return take(rn, cn)
        elif min(m, n) <= leaf or not can_split:
            return take(rn, cn)
        r0, r1 = rn.children
        c0, c1 = cn.children
        return H.Hier([[build(r0, c0), build(r0, c1)], [build(r1, c0), build(r1, c1)]],
                      row_split=r0.size, col_split=c0.size)

    def take(rn, cn):
        blk, r0, c0 = next(leaves)
        if (r0, c0) != (rn.start, cn.start):
            raise ValueError("export order does not follow the reference partition")
        return blk

    root = build(ct.root, ct.root)
    return H.HMatrix(root, ct, ct, N, N, eta)


def load_export(path):
    """(recs, arena, ranks, perm) written by bench.py --export-factors."""
    z = {k: np.load(os.path.join(path, k + ".npy")) for k in ("recs", "arena", "ranks", "perm")}
    return z["recs"], z["arena"], z["ranks"], z["perm"]
