"""H-matrix / H-LU checkpoints (factor export and import, so an H-LU is
computed once and reused across runs; the reference recomputes it every time, cli.py:203-209).

``save_hmatrix(obj, path)`` writes an HMatrix or an HFactorization (csrc/checkpoint.cpp: one
self-contained file with both cluster trees and their points, the block tree, the storage
layout and the device arrays); ``load_hmatrix(path)`` returns the same type, bit-identical.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from .geometry import ClusterTree
from .hmatrix import HMatrix
from .hops import HFactorization

__all__ = ["save_hmatrix", "load_hmatrix"]


def save_hmatrix(obj, path):
    """Write an HMatrix or HFactorization to `path` (device arrays streamed to disk)."""
    if isinstance(obj, HFactorization):
        H, eps2 = obj.h, float(obj.eps2)
    elif isinstance(obj, HMatrix):
        H, eps2 = obj, -1.0
    else:
        raise TypeError("save_hmatrix takes an HMatrix or an HFactorization")
    _lib.check(_lib.lib().lh_hmat_save(H.ctx.h, H.handle, eps2, os.fsencode(path)), H.ctx.h)


def _tree(handle):
    """ClusterTree around a native tree handle (points come from the checkpoint)."""
    L = _lib.lib()
    nn = L.lh_tree_num_nodes(handle)
    lohi = np.empty(2 * nn, dtype=np.int64)
    L.lh_tree_nodes(handle, _lib.host_ptr(lohi), None, None)
    dim = L.lh_tree_points(handle, None)
    pts = np.empty((int(lohi[1] - lohi[0]), dim), dtype=np.float64)
    L.lh_tree_points(handle, _lib.host_ptr(pts))
    return ClusterTree(handle, pts, dim)


def load_hmatrix(path):
    """Read a checkpoint written by save_hmatrix: an HFactorization when a factor was saved,
    else an HMatrix (whose H-LU planning starts in the background, as after assembly)."""
    if not os.path.exists(path):
        raise FileNotFoundError(path)
    ctx = _lib.Context.get()
    rt, ct, h = C.c_void_p(), C.c_void_p(), C.c_void_p()
    fac, eps2 = C.c_int32(0), C.c_double(0.0)
    rc = _lib.lib().lh_hmat_load(ctx.h, os.fsencode(path), C.byref(rt), C.byref(ct), C.byref(h),
                                 C.byref(fac), C.byref(eps2))
    _lib.check(rc, ctx.h)
    H = HMatrix(h, _tree(rt), _tree(ct), None, ctx, None)
    if fac.value:
        H.factored = True
        return HFactorization(H, eps2.value)
    return H
