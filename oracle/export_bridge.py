"""Rebuild oracle block trees (oracle/levyh_oracle.py types) from an H-matrix
exported by the native library (TEST / BASELINE INFRASTRUCTURE ONLY).

Used by tests and by bench.py's reference CPU arm to run the restated
reference algorithm (hops.matvec / hops.solve, SURVEY 8(c) "reference hops.*
on exported GPU factors") on GPU-built operators at sizes the reference
cannot assemble.  Leaf arrays are zero-copy views into the exported arena.
"""
from __future__ import annotations

import math

import numpy as np

from . import levyh_oracle as O


def leaf_blocks(recs, arena, ranks, perm):
    out = []
    for rec in recs:
        r0, r1, c0, c1, kind, doff, uoff, voff, kcap, rslot, poff = (int(v) for v in rec)
        m, n = r1 - r0, c1 - c0
        if kind == 2:  # low rank: first `rank` columns of U (m x kcap) and V (n x kcap)
            r = int(ranks[rslot])
            u = arena[uoff:uoff + m * r].reshape(r, m).T
            v = arena[voff:voff + n * r].reshape(r, n).T
            out.append((O.Blk("R", u=u, v=v), r0, c0))
        else:  # column-major dense leaf
            d = arena[doff:doff + m * n].reshape(n, m).T
            if kind == 3:
                b = O.Blk("F", d=d)
                b.perm = perm[poff:poff + m].astype(np.intp)
                out.append((b, r0, c0))
            else:
                out.append((O.Blk("D", d=d), r0, c0))
    return out


def tree_from_export(points, leaf, recs, arena, ranks, perm, n_block=4, eta=1.0):
    """Replay the partition recursion (hmatrix.py:319-337) and attach exported leaves."""
    root, _ = O.cluster_tree(points, leaf)
    leaves = iter(leaf_blocks(recs, arena, ranks, perm))
    N = root.size
    nmax = math.ceil(N / n_block)

    def rec(r, c):
        m, n = r.size, c.size
        splittable = (not r.leaf) and (not c.leaf)
        hier = False
        if splittable and (m > nmax or n > nmax):
            hier = True
        elif O.is_admissible(r, c, eta) and min(m, n) > leaf:
            hier = False
        elif min(m, n) <= leaf or not splittable:
            hier = False
        else:
            hier = True
        if not hier:
            blk, r0, c0 = next(leaves)
            assert (r0, c0) == (r.lo, c.lo), "export order does not follow the partition"
            return blk
        (ra, rb), (ca, cb) = r.kids, c.kids
        return O.Blk("H", k=[[rec(ra, ca), rec(ra, cb)], [rec(rb, ca), rec(rb, cb)]],
                     rs=ra.size, cs=ca.size)

    return rec(root, root)
