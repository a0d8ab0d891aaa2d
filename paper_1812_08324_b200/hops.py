"""H-matrix arithmetic on the GPU -- API of levyh.hops
(/root/reference/pkg/src/levyh/hops.py:30-432).

``matvec``/``mul_dense`` run the two-phase streaming kernel (csrc/matvec.cu);
``hlu`` runs the recursive H-LU as a static task DAG on a persistent
dataflow kernel (csrc/lu.cu); ``solve`` applies forward/backward substitution
(method "substitution"), the precomputed triangular-inverse factors
(method "inverse") or one H-matvec of the propagator Z = (LU)^{-1}
(method "propagator", the per-step fast path).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .hmatrix import HMatrix

__all__ = ["matvec", "mul_dense", "hlu", "HFactorization", "solve"]

SOLVE_METHODS = {"substitution": 0, "inverse": 1, "propagator": 2}


def _to_device(x, ctx):
    import torch

    if isinstance(x, torch.Tensor):
        return x.to(device=f"cuda:{ctx.device}", dtype=torch.float64), True
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).to(
        f"cuda:{ctx.device}"), False


def _colmajor(t):
    """(n,) or (n, k) tensor -> column-major storage tensor (k, n) view and k."""
    if t.ndim == 1:
        return t.contiguous().view(1, -1), 1
    return t.t().contiguous(), t.shape[1]


def matvec(H: HMatrix, x):
    """hops.py:65-70: y = H x, x in tree order (numpy in -> numpy out; torch stays on device)."""
    import torch

    ctx = H.ctx
    xt, was_torch = _to_device(x, ctx)
    if tuple(xt.shape) != (H.n_cols,):
        raise ValueError(f"vector length {tuple(xt.shape)} does not match n_cols={H.n_cols}")
    xt = xt.contiguous()
    y = torch.empty(H.n_rows, dtype=torch.float64, device=xt.device)
    _lib.check(_lib.lib().lh_hmat_matvec(ctx.h, H.handle, xt.data_ptr(), H.n_cols, y.data_ptr(),
                                         H.n_rows, 1), ctx.h)
    return y if was_torch else y.cpu().numpy()


def mul_dense(H: HMatrix, X):
    """hops.py:73-85: H @ X for a dense (n_cols, k) matrix."""
    import torch

    ctx = H.ctx
    xt, was_torch = _to_device(X, ctx)
    if xt.ndim == 1:
        return matvec(H, X)
    if xt.shape[0] != H.n_cols:
        raise ValueError("row count of X does not match n_cols")
    xc, k = _colmajor(xt)
    y = torch.empty((k, H.n_rows), dtype=torch.float64, device=xt.device)
    _lib.check(_lib.lib().lh_hmat_matvec(ctx.h, H.handle, xc.data_ptr(), H.n_cols, y.data_ptr(),
                                         H.n_rows, k), ctx.h)
    y = y.t()
    return y if was_torch else y.cpu().numpy()


@dataclass
class HFactorization:
    """In-place LU factors (hops.py:377-389); ``h`` is the consumed HMatrix."""

    h: HMatrix
    eps2: float
    inverse_ready: bool = False
    propagator_ready: bool = False

    def solve(self, b, method="substitution"):
        return solve(self, b, method)

    def prepare_inverse(self):
        if not self.inverse_ready:
            _lib.check(_lib.lib().lh_prepare_inverse(self.h.ctx.h, self.h.handle, float(self.eps2)),
                       self.h.ctx.h)
            self.inverse_ready = True

    def prepare_propagator(self):
        """Z = (LU)^{-1} as an H-matrix on the factor's block tree (method "propagator")."""
        if not self.propagator_ready:
            _lib.check(_lib.lib().lh_prepare_propagator(self.h.ctx.h, self.h.handle,
                                                        float(self.eps2)), self.h.ctx.h)
            self.propagator_ready = True

    def propagator_stats(self):
        """(task count, planning s, temp bytes, executor s) of the propagator build."""
        out = np.zeros(4)
        _lib.check(_lib.lib().lh_propagator_stats(self.h.handle, _lib.host_ptr(out)))
        return out


def hlu(H: HMatrix, eps2=1e-10):
    """hops.py:411-421: recursive H-LU in place (consumes H)."""
    if H.n_rows != H.n_cols:
        raise ValueError("LU requires a square matrix")
    _lib.check(_lib.lib().lh_hlu(H.ctx.h, H.handle, float(eps2)), H.ctx.h)
    H.factored = True
    return HFactorization(H, eps2)


def solve(F: HFactorization, b, method="substitution"):
    """hops.py:424-432: forward (unit L with leaf pivots) then backward (U)."""
    ctx = F.h.ctx
    bt, was_torch = _to_device(b, ctx)
    if bt.shape[0] != F.h.n_rows:
        raise ValueError("right-hand side length mismatch")
    m = SOLVE_METHODS[method]
    if m == 1:
        F.prepare_inverse()
    elif m == 2:
        F.prepare_propagator()
    shape = bt.shape
    bc, k = _colmajor(bt.reshape(shape[0], -1))
    bc = bc.clone()
    _lib.check(_lib.lib().lh_solve(ctx.h, F.h.handle, bc.data_ptr(), F.h.n_rows, k, m), ctx.h)
    out = bc.t().reshape(shape)
    return out if was_torch else out.cpu().numpy()
