"""Krylov solvers on the GPU -- API of levyh.solvers
(/root/reference/pkg/src/levyh/solvers.py:1-153).

``pcg`` and ``gmres_restarted`` keep the reference's signatures, stopping rules, residual
logging and exceptions.  The iteration runs in the native library (csrc/krylov.cu): the
vectors stay on the device, the operator and the inverse preconditioner are applied by the
GPU H-matvec / H-LU solve / dense matvec, and the host only sees the scalars the control
flow branches on.  Operators (solvers.py:39-43 ``_as_operator``) may be

* an ``HMatrix`` (y = H x, hops.matvec),
* an ``HFactorization`` (y = solve(F, x), method "substitution"; ``operator(F, method=...)``
  picks another solve method),
* a dense matrix (numpy or torch, uploaded once, row-major device GEMV),
* a callable.  It receives a torch CUDA float64 vector and returns an array-like of the
  same length (a torch CUDA tensor stays on the device; anything else is copied in).
"""
from __future__ import annotations

import csv
import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .hmatrix import HMatrix
from .hops import SOLVE_METHODS, HFactorization, _to_device

__all__ = ["IterationLog", "pcg", "gmres_restarted", "operator", "Operator"]

OP_IDENTITY, OP_HMATVEC, OP_HSOLVE, OP_DENSE, OP_CALLBACK = range(5)


@dataclass
class IterationLog:
    """Per-iteration relative residuals of a Krylov run (solvers.py:23-37)."""

    residuals: list = field(default_factory=list)
    iterations: int = 0
    converged: bool = False
    seconds: float = 0.0

    def write_csv(self, path):
        with open(path, "w", newline="") as fh:
            writer = csv.writer(fh, lineterminator="\n")
            writer.writerow(["iter", "relative_residual", "seconds"])
            last = len(self.residuals)
            for k, r in enumerate(self.residuals):
                writer.writerow([k + 1, f"{r:.17g}", f"{self.seconds:.6g}" if k + 1 == last else ""])


APPLY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)


class OperatorC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("hmat", C.c_void_p), ("method", C.c_int32),
                ("a_dev", C.c_void_p), ("lda", C.c_int64), ("fn", APPLY_FN), ("user", C.c_void_p)]


class _DevVec:
    """__cuda_array_interface__ view of a device vector (for torch.as_tensor)."""

    def __init__(self, ptr, n, readonly):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, readonly),
                                         "version": 3, "strides": None}


class Operator:
    """A Krylov operator bound to its native descriptor (keeps every referenced object alive)."""

    def __init__(self, op, n, ctx, method=None):
        import torch

        if method is None:  # the fastest method already prepared on a factor
            method = op.default_method if isinstance(op, HFactorization) else "substitution"

        self.keep = []
        self.error = None
        self.n = n
        c = OperatorC()
        if op is None:
            c.kind = OP_IDENTITY
        elif isinstance(op, Operator):
            if op.n != n:
                raise ValueError(f"operator size {op.n} does not match the right-hand side ({n},)")
            c = op.c
            self.keep.append(op)
        elif isinstance(op, HMatrix):
            if op.shape != (n, n):
                raise ValueError(f"operator shape {op.shape} does not match the right-hand side ({n},)")
            c.kind, c.hmat = OP_HMATVEC, op.handle.value
            self.keep.append(op)
        elif isinstance(op, HFactorization):
            if op.h.shape != (n, n):
                raise ValueError(f"preconditioner shape {op.h.shape} does not match ({n},)")
            if method not in SOLVE_METHODS:
                raise ValueError(f"unknown solve method {method!r}")
            if method == "inverse":
                op.prepare_inverse()
            elif method == "propagator":
                op.prepare_propagator()
            c.kind, c.hmat, c.method = OP_HSOLVE, op.h.handle.value, SOLVE_METHODS[method]
            self.keep.append(op)
        elif callable(op):
            dev = f"cuda:{ctx.device}"

            def trampoline(_user, x_ptr, y_ptr):
                try:
                    x = torch.as_tensor(_DevVec(x_ptr, n, False), device=dev)  # must not be modified
                    y = torch.as_tensor(_DevVec(y_ptr, n, False), device=dev)
                    r = op(x)
                    rt = r if isinstance(r, torch.Tensor) else torch.from_numpy(
                        np.ascontiguousarray(np.asarray(r, dtype=np.float64)))
                    if tuple(rt.shape) != (n,):
                        raise ValueError(f"operator returned shape {tuple(rt.shape)}, expected ({n},)")
                    y.copy_(rt.to(device=dev, dtype=torch.float64))
                    return _lib.LH_OK
                except BaseException as e:  # re-raised by the caller after the native loop unwinds
                    self.error = e
                    return _lib.LH_EINTERNAL

            fn = APPLY_FN(trampoline)
            self.keep.append(fn)
            c.kind, c.fn = OP_CALLBACK, fn
        else:
            a, _ = _to_device(op, ctx)
            if a.ndim != 2 or tuple(a.shape) != (n, n):
                raise ValueError(f"dense operator of shape {tuple(a.shape)} does not match ({n},)")
            a = a.contiguous()
            self.keep.append(a)
            c.kind, c.a_dev, c.lda = OP_DENSE, a.data_ptr(), n
        self.c = c


def operator(op, method=None, n=None):
    """Wrap an HFactorization with a chosen solve method (or any operator) for pcg / gmres;
    method None: the fastest method already prepared on the factor (substitution if none)."""
    ctx = _lib.Context.get()
    if method is None:
        method = op.default_method if isinstance(op, HFactorization) else "substitution"
    if n is None:
        n = op.h.n_rows if isinstance(op, HFactorization) else op.shape[0]
    return Operator(op, n, ctx, method)


def _prepare(apply_A, apply_M_inv, b):
    ctx = _lib.Context.get()
    bt, was_torch = _to_device(b, ctx)
    if bt.ndim != 1:
        raise ValueError("the Krylov solvers take one right-hand side (a 1-D vector)")
    bt = bt.contiguous()
    n = bt.shape[0]
    return ctx, bt, was_torch, n, Operator(apply_A, n, ctx), Operator(apply_M_inv, n, ctx)


def _finish(rc, ctx, ops, x, was_torch, res, iters, conv, t0):
    for op in ops:
        if op.error is not None:
            raise op.error
    _lib.check(rc, ctx.h)
    log = IterationLog(residuals=[float(r) for r in res[:iters.value]], iterations=int(iters.value),
                       converged=bool(conv.value), seconds=time.perf_counter() - t0)
    return (x if was_torch else x.cpu().numpy()), log


def pcg(apply_A, apply_M_inv, b, tol=1e-8, max_iter=500):
    """solvers.py:46-88: preconditioned conjugate gradient for SPD operators, from x = 0.

    Raises numpy.linalg.LinAlgError on breakdown (p'Ap <= 0).  Returns (x, IterationLog)."""
    import torch

    t0 = time.perf_counter()
    ctx, bt, was_torch, n, A, M = _prepare(apply_A, apply_M_inv, b)
    x = torch.empty_like(bt)
    res = np.zeros(max(int(max_iter), 1))
    iters, conv = C.c_int32(0), C.c_int32(0)
    rc = _lib.lib().lh_pcg(ctx.h, C.byref(A.c), C.byref(M.c), bt.data_ptr(), n, float(tol),
                           int(max_iter), x.data_ptr(), _lib.host_ptr(res), C.byref(iters),
                           C.byref(conv))
    return _finish(rc, ctx, (A, M), x, was_torch, res, iters, conv, t0)


def gmres_restarted(apply_A, apply_M_inv, b, tol=1e-8, restart=50, max_iter=500):
    """solvers.py:91-153: right-preconditioned restarted GMRES (MGS Arnoldi, Givens).

    The logged residual is the original system's; stagnation past max_iter returns with
    converged=False.  Returns (x, IterationLog)."""
    import torch

    t0 = time.perf_counter()
    ctx, bt, was_torch, n, A, M = _prepare(apply_A, apply_M_inv, b)
    x = torch.empty_like(bt)
    res = np.zeros(max(int(max_iter), 1))
    iters, conv = C.c_int32(0), C.c_int32(0)
    rc = _lib.lib().lh_gmres_restarted(ctx.h, C.byref(A.c), C.byref(M.c), bt.data_ptr(), n,
                                       float(tol), int(restart), int(max_iter), x.data_ptr(),
                                       _lib.host_ptr(res), C.byref(iters), C.byref(conv))
    return _finish(rc, ctx, (A, M), x, was_torch, res, iters, conv, t0)
