"""Crank-Nicolson stepping for the singular Levy generator on the GPU --
the composition SURVEY.md 8(c) describes on top of levyh.levy
(/root/reference/pkg/src/levyh/levy.py:131-330) and levyh.fractional.

Operator: u_t = a u_xx + b u_x + c u + int (u(x+y) - u(x) - u'(x) y 1_{|y|<1}) nu(dy)
on the interior nodes x_k = k h of [-L, L] with u = 0 outside.  A is the
negated singularity-subtraction stencil (fractional.py:362-405) plus the
local band of levy._entries_a_1d (levy.py:169-176) with b_eff = b + beta
(SURVEY G4), and A+- = I +- dt/2 A (levy.py:194-206).
"""
from __future__ import annotations

import numpy as np

from . import fractional as frac
from .geometry import build_cluster_tree
from .hmatrix import HConfig, build_toeplitz, derive_toeplitz
from .hops import SOLVE_METHODS, hlu, matvec, solve

__all__ = ["FracCNSystem", "step_cn", "run_cn"]


class FracCNSystem:
    """Assembled CN operators of the singular problem (cf. levy.CNSystem, levy.py:131-246).

    Parameters mirror the BASELINE.json configs: ``nu`` a LevyMeasure (power or CGMY
    evaluate on the GPU), grid h = L / n with N = 2n - 1 interior unknowns, window
    ``L_W`` (default 2L: every in-domain offset inside the near-field window),
    ``rho_r`` window radius, ``tail_mass`` (default: power formula or quadrature),
    ``drift_compensation`` adds beta to b.
    """

    def __init__(self, nu, a, b, c, n, dt, L=1.0, L_W=None, rho_r=0.2, tail_mass=None,
                 drift_compensation=True, s=None, distributed=False):
        if a < 0 or c > 0:
            raise ValueError("stability requires a >= 0 and c <= 0")
        self.nu, self.a, self.b, self.c, self.dt, self.L = nu, a, b, c, dt, L
        self.n = n
        self.h = L / n
        self.N = 2 * n - 1
        self.L_W = 2.0 * L if L_W is None else L_W
        self.rho_r = rho_r
        k = self.L_W / self.h
        if abs(k - round(k)) > 1e-9:
            raise ValueError("L_W must be an integer multiple of h")
        if not (0 < rho_r < self.L_W):
            raise ValueError("need 0 < rho_r < L_W")
        win = frac.quartic_window(rho_r)
        self.m2 = frac.windowed_second_moment(nu, win)
        if tail_mass is None:
            if nu.gpu is not None and nu.gpu[0] == "power":
                tail_mass = frac.tail_mass_power_1d(nu.gpu[2], self.L_W)
            else:
                tail_mass = frac.tail_mass_numeric(nu, self.L_W)
        self.tail = tail_mass
        self.beta = 0.0
        if drift_compensation and not nu.symmetric:
            self.beta = frac.drift_compensation_beta(nu, rho_r)
        self.b_eff = b + self.beta
        self.x = self.h * np.arange(-(n - 1), n)
        self.tA, self.tPlus, self.tMinus, self.sums = frac.frac_symbol_1d(
            nu, self.h, self.N, self.L_W, rho_r, self.tail, self.m2, a, self.b_eff, c, dt)
        self.tree = None
        self.factor = None
        self.h_minus = None
        self.h_plus = None
        # True / a process group: shard the ACA compression across the ranks
        self.distributed = distributed

    @property
    def size(self):
        return self.N

    def cluster_tree(self, leaf_size=64):
        if self.tree is None or self.tree_leaf != leaf_size:
            self.tree = build_cluster_tree(self.x[:, None], leaf_size=leaf_size)
            self.tree_leaf = leaf_size
        return self.tree

    def hmatrix(self, which="plus", cfg=None):
        """H-form of A+ / A- / A by matrix-free ACA on the GPU symbol (cf. levy.py:224-239)."""
        cfg = cfg or HConfig()
        ct = self.cluster_tree(cfg.n_min)
        t = {"A": self.tA, "plus": self.tPlus, "minus": self.tMinus}[which]
        return build_toeplitz(t, ct, ct, cfg, distributed=self.distributed)

    def build_pair(self, cfg=None):
        """H+ (capacity cfg.kcap, for H-LU) and H- derived from it: A-'s off-diagonal
        entries are exact negatives of A+'s, so its low-rank blocks are (-U, V) with
        identical ranks (hard part 4); dense leaves refilled from tMinus."""
        cfg = cfg or HConfig()
        Hp = self.hmatrix("plus", cfg)
        Hm = derive_toeplitz(Hp, self.tMinus, lr_scale=-1.0, kcap=0)
        return Hp, Hm

    def prepare(self, cfg=None, eps2=1e-10, method="inverse"):
        """Factorise A+ once and keep A- for stepping (levy.py:241-246)."""
        Hp, Hm = self.build_pair(cfg)
        self.h_minus = Hm
        self.factor = hlu(Hp, eps2)
        if method == "inverse":
            self.factor.prepare_inverse()
        elif method == "propagator":
            self.factor.prepare_propagator()
        self.method = method
        return self.factor


def step_cn(sys, u_n, F=None, method=None):
    """levy.py:295-306: solve A+ u = A- u_n."""
    F = F if F is not None else sys.factor
    if F is None or sys.h_minus is None:
        raise ValueError("call prepare() before stepping")
    perm = sys.tree.perm
    rhs = matvec(sys.h_minus, perm.to_tree(u_n))
    return perm.from_tree(solve(F, rhs, method or getattr(sys, "method", "substitution")))


def run_cn(sys, u0, n_steps, cfg=None, eps2=1e-10, method="inverse"):
    """levy.py:309-330: factor once, march n_steps on the device (CUDA-graph loop)."""
    import torch

    from . import _lib

    if sys.factor is None:
        sys.prepare(cfg, eps2, method)
    perm = sys.tree.perm
    ctx = sys.h_minus.ctx
    u = torch.as_tensor(perm.to_tree(np.asarray(u0, dtype=float))).to(f"cuda:{ctx.device}")
    uc = u.reshape(1, -1).contiguous() if u.ndim == 1 else u.t().contiguous()
    k = 1 if u.ndim == 1 else u.shape[1]
    m = SOLVE_METHODS[sys.method if method is None else method]
    if m == 2:
        sys.factor.prepare_propagator()
    elif m == 1:
        sys.factor.prepare_inverse()
    _lib.check(_lib.lib().lh_cn_steps(ctx.h, sys.h_minus.handle, sys.factor.h.handle, uc.data_ptr(),
                                      sys.N, k, int(n_steps), m), ctx.h)
    out = uc.reshape(-1) if k == 1 else uc.t()
    return perm.from_tree(out.cpu().numpy())
