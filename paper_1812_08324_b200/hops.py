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

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .hmatrix import HMatrix

__all__ = ["matvec", "mul_dense", "hlu", "HFactorization", "solve", "trisolve_lower",
           "trisolve_upper_right", "lowrank_add_recompress"]

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
    auto_prepare: bool = True   # default-method solves build the propagator after a few calls
    default_calls: int = 0

    def solve(self, b, method=None):
        return solve(self, b, method)

    @property
    def default_method(self):
        """The fastest method already prepared: propagator, then inverse factors, then
        substitution (which needs no preparation)."""
        if self.propagator_ready:
            return "propagator"
        if self.inverse_ready:
            return "inverse"
        return "substitution"

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
        """(task count, planning s, temp bytes, executor s, near-field leaves compressed,
        coarsening merges, single-RHS form (0 H, 1 shared leaf bases, 2 nested H2), its probe
        error against the H-form, mean leaf basis size, basis/transfer/coupling scalars, flops per
        right-hand side of the multi-RHS product and its form (2 H2 walk, 1 H-form)) of the
        propagator build."""
        out = np.zeros(12)
        _lib.check(_lib.lib().lh_propagator_stats(self.h.handle, _lib.host_ptr(out)))
        return out


def hlu(H: HMatrix, eps2=1e-10):
    """hops.py:411-421: recursive H-LU in place (consumes H)."""
    if H.n_rows != H.n_cols:
        raise ValueError("LU requires a square matrix")
    _lib.check(_lib.lib().lh_hlu(H.ctx.h, H.handle, float(eps2)), H.ctx.h)
    H.factored = True
    return HFactorization(H, eps2)


AUTO_PROPAGATOR_AFTER = 4


def solve(F: HFactorization, b, method=None):
    """hops.py:424-432: x = (LU)^-1 b.  ``method`` None uses the fastest method already
    prepared on F (F.default_method: one H-matvec of the propagator after
    prepare_propagator / CNSystem.prepare, else the triangular-inverse factors, else the
    reference's forward (unit L with leaf pivots) then backward (U) substitution; the fifth such
    default substitution solve on a 1D factor builds the propagator first, F.auto_prepare = False
    turns that off)."""
    ctx = F.h.ctx
    bt, was_torch = _to_device(b, ctx)
    if bt.shape[0] != F.h.n_rows:
        raise ValueError("right-hand side length mismatch")
    if method is None:
        method = F.default_method
        if method == "substitution" and F.auto_prepare and getattr(F.h.row_tree, "dim", 1) == 1:
            # repeated default solves on one factor (time stepping, preconditioning): after
            # AUTO_PROPAGATOR_AFTER substitution solves the propagator is built once (about ten
            # substitution solves' worth of time at N = 2^20) and every later solve is one
            # streaming H-matvec of Z; pass method="substitution" to keep the reference's solve
            F.default_calls += 1
            if F.default_calls > AUTO_PROPAGATOR_AFTER:
                try:
                    F.prepare_propagator()
                    method = "propagator"
                except (NotImplementedError, MemoryError, _lib.NativeError):
                    F.auto_prepare = False
    if method not in SOLVE_METHODS:
        raise ValueError(f"unknown solve method {method!r}; expected one of {sorted(SOLVE_METHODS)}")
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


# Truncation of the low-rank updates in block triangular solves.  The reference passes
# eps2 = 0 (hops.py:295, :310), which keeps every nonzero singular value -- rounding noise
# included -- so its ranks are decided by noise; a Frobenius tail of 1e-14 relative keeps the
# result within rounding of the exact solve with bounded ranks.
BLOCK_SOLVE_EPS2 = 1e-14


def _tri_solve_block(T, B, mode, unit):
    Th = T.h if isinstance(T, HFactorization) else T
    if not isinstance(Th, HMatrix):
        raise TypeError("triangular operand must be an HMatrix or HFactorization")
    if B.n_rows != Th.n_rows:
        raise ValueError("right-hand side shape mismatch")
    h = C.c_void_p()
    _lib.check(_lib.lib().lh_trisolve_block(Th.ctx.h, Th.handle, B.handle, int(mode), int(bool(unit)),
                                            float(BLOCK_SOLVE_EPS2), C.byref(h)), Th.ctx.h)
    return HMatrix(h, B.row_tree, B.col_tree, B.eta, B.ctx, B.cfg)


def _tri_solve(T, B, mode, unit):
    Th = T.h if isinstance(T, HFactorization) else T
    if not isinstance(Th, HMatrix):
        raise TypeError("triangular operand must be an HMatrix or HFactorization")
    if not (isinstance(B, np.ndarray) or _is_torch(B)):
        raise TypeError("right-hand side must be a dense array or an HMatrix")
    ctx = Th.ctx
    bt, was_torch = _to_device(B, ctx)
    return Th, ctx, bt, was_torch


def _is_torch(x):
    try:
        import torch
        return isinstance(x, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False


def trisolve_lower(L, B, unit_diagonal=False):
    """hops.py:282-295: solve L X = B with the lower triangle of L (dense B, (n,) or (n, k)).

    LU-factored diagonal leaves use their unit-L factor and pivots; plain dense leaves use
    their lower triangle (unit diagonal if requested) and raise LinAlgError("singular
    triangular diagonal block at L...") on a zero diagonal entry.  B is not modified.  An
    HMatrix B (same cluster trees) returns a new HMatrix: a deep copy of B solved block by
    block (_trisolve_block, hops.py:232-258)."""
    if isinstance(B, HMatrix):
        return _tri_solve_block(L, B, 0, unit_diagonal)
    Th, ctx, bt, was_torch = _tri_solve(L, B, 0, unit_diagonal)
    if bt.shape[0] != Th.n_rows:
        raise ValueError("right-hand side length mismatch")
    shape = bt.shape
    bc, k = _colmajor(bt.reshape(shape[0], -1))
    bc = bc.clone()
    _lib.check(_lib.lib().lh_trisolve_dense(ctx.h, Th.handle, 0, int(bool(unit_diagonal)),
                                            bc.data_ptr(), Th.n_rows, k), ctx.h)
    out = bc.t().reshape(shape)
    return out if was_torch else out.cpu().numpy()


def trisolve_upper_right(U, B, unit_diagonal=False):
    """hops.py:298-310: solve X U = B with the upper triangle of U, as U^T X^T = B^T
    (dense B of shape (m, n), or (n,) for one row)."""
    if isinstance(B, HMatrix):  # _trisolve_right_upper (hops.py:261-279) on a deep copy
        if unit_diagonal:
            raise ValueError("unit_diagonal right solves are not supported on blocks")
        return _tri_solve_block(U, B, 2, False)
    Th, ctx, bt, was_torch = _tri_solve(U, B, 2, unit_diagonal)
    n = Th.n_rows
    rows = bt.reshape(1, -1) if bt.ndim == 1 else bt.reshape(bt.shape[0], -1)
    if rows.shape[1] != n:
        raise ValueError("right-hand side width mismatch")
    bc = rows.contiguous().clone()  # (m, n) row-major == n x m column-major (B^T)
    k = rows.shape[0]
    _lib.check(_lib.lib().lh_trisolve_dense(ctx.h, Th.handle, 2, int(bool(unit_diagonal)),
                                            bc.data_ptr(), n, k), ctx.h)
    out = bc.reshape(bt.shape)
    return out if was_torch else out.cpu().numpy()


def lowrank_add_recompress(A, B, eps2):
    """hops.py:147-156: A + B recompressed (QR of [u1 u2], QR of [v1 v2], SVD of R_u R_v^T;
    smallest rank with Frobenius tail <= eps2 * ||A + B||_F), on the GPU.  A and B are
    LowRank (u: m x r, v: n x r); returns a LowRank of the same array type."""
    import torch

    from .hmatrix import LowRank

    if tuple(A.shape) != tuple(B.shape):
        raise ValueError("shape mismatch in low-rank addition")
    ctx = _lib.Context.get()
    m, n = A.shape
    was_torch = _is_torch(A.u)

    def dev(a):
        t, _ = _to_device(a, ctx)
        return t.reshape(t.shape[0], -1).t().contiguous()  # column-major storage

    u1, v1, u2, v2 = dev(A.u), dev(A.v), dev(B.u), dev(B.v)
    r1, r2 = u1.shape[0], u2.shape[0]
    cap = max(r1 + r2, 1)
    uo = torch.zeros((cap, m), dtype=torch.float64, device=u1.device)
    vo = torch.zeros((cap, n), dtype=torch.float64, device=u1.device)
    r = C.c_int32(0)
    _lib.check(_lib.lib().lh_lowrank_add_recompress(ctx.h, m, n, u1.data_ptr(), v1.data_ptr(), r1,
                                                    u2.data_ptr(), v2.data_ptr(), r2, float(eps2),
                                                    uo.data_ptr(), vo.data_ptr(), C.byref(r)), ctx.h)
    rr = r.value
    u, v = uo[:rr].t(), vo[:rr].t()
    if not was_torch:
        u, v = u.cpu().numpy(), v.cpu().numpy()
    return LowRank(u, v)
