"""Crank-Nicolson stepping for the singular Levy generator on the GPU --
the composition SURVEY.md 8(c) describes on top of levyh.levy
(/root/reference/pkg/src/levyh/levy.py:131-330) and levyh.fractional.

Operator: u_t = a u_xx + b u_x + c u + int (u(x+y) - u(x) - u'(x) y 1_{|y|<1}) nu(dy)
on the interior nodes x_k = k h of [-L, L] with u = 0 outside.  A is the
negated singularity-subtraction stencil (fractional.py:362-405) plus the
local band of levy._entries_a_1d (levy.py:169-176) with b_eff = b + beta
(SURVEY G4), and A+- = I +- dt/2 A (levy.py:194-206).

The smooth-measure system of the reference itself (levy.CNSystem with gaussian_measure,
assemble_cn_1d, the series H-builder; the reference's own `levyh bench` path, cli.py:163-224)
is CNSystem below: same Toeplitz machinery, low-rank blocks from the analytic expansion.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import fractional as frac
from .fractional import LevyMeasure
from .geometry import build_cluster_tree
from .hmatrix import (HConfig, ToeplitzEntries, build_from_expansion, build_toeplitz, derive_toeplitz,
                      gaussian_expansion_1d)
from .hops import SOLVE_METHODS, hlu, matvec, solve

__all__ = ["FracCNSystem", "CNSystem", "CNSystem2D", "LevyMeasure", "UniformGrid1D", "UniformGrid2D",
           "gaussian_measure", "assemble_cn_1d", "assemble_cn_2d", "step_cn", "run_cn"]


def gaussian_measure(eps_sq=5.0, scale=1.0):
    """levy.py:72-81: jump density scale * exp(-eps_sq y^2) (enables the series builder)."""
    return LevyMeasure(
        density=lambda y: scale * np.exp(-eps_sq * np.asarray(y, dtype=float) ** 2),
        kind="smooth_semi_heavy", symmetric=True,
        density2=lambda dx, dy: scale * np.exp(-eps_sq * (dx * dx + dy * dy)),
        gauss_eps_sq=eps_sq, scale=scale)


@dataclass(frozen=True)
class UniformGrid1D:
    """levy.py:84-102: n points x_i = lo + i h, h = (hi - lo) / n."""

    n: int
    lo: float = -1.0
    hi: float = 1.0

    @property
    def h(self):
        return (self.hi - self.lo) / self.n

    @property
    def points(self):
        return self.lo + self.h * np.arange(self.n)

    @property
    def size(self):
        return self.n


@dataclass(frozen=True)
class UniformGrid2D:
    """levy.py:106-128: tensor grid, row-major, point k = iy nx + ix at (lo + ix h, lo + iy h),
    h = (hi - lo) / nx, nx == ny."""

    nx: int
    ny: int
    lo: float = -1.0
    hi: float = 1.0

    @property
    def h(self):
        return (self.hi - self.lo) / self.nx

    @property
    def size(self):
        return self.nx * self.ny

    @property
    def points(self):
        ix = np.arange(self.nx)
        iy = np.arange(self.ny)
        X, Y = np.meshgrid(self.lo + self.h * ix, self.lo + self.h * iy)
        return np.column_stack([X.ravel(), Y.ravel()])


class CNSystem:
    """levy.py:131-246 for the smooth (Gaussian) jump density on a 1D uniform grid: the CN
    operators are Toeplitz, their symbols are generated on the GPU (lh_gauss_cn_symbol) and
    ``hmatrix`` runs the series builder (build_from_expansion with gaussian_expansion_1d and
    the exact entries as dense leaves, levy.py:224-239) on the device."""

    def __init__(self, grid, nu, a, b, c, dt, n_off, lam, dim, symbols):
        self.grid, self.nu, self.a, self.b, self.c, self.dt = grid, nu, a, b, c, dt
        self.n_off = n_off
        self.lam = lam
        self.dim = dim
        self.h = grid.h
        self.tA, self.tPlus, self.tMinus = symbols
        self.tree = None
        self.factor = None
        self.h_minus = None
        self.method = "propagator"
        self._host = {}

    @property
    def n(self):
        return self.grid.size

    @property
    def N(self):
        return self.grid.size

    size = n

    def weight(self, j):
        """levy.py:158-163."""
        j = np.asarray(j)
        w = np.full(j.shape, self.h, dtype=float)
        w[np.abs(j) >= self.n_off] = self.h / 2.0
        return w

    def _symbol(self, which):
        if which not in ("A", "plus", "minus"):
            raise ValueError(which)
        if which not in self._host:
            t = {"A": self.tA, "plus": self.tPlus, "minus": self.tMinus}[which]
            self._host[which] = t.cpu().numpy()
        return self._host[which]

    def entries(self, rows, cols, which="A"):
        """levy.py:194-206: exact entries for original-order index arrays (read from the
        device-generated symbol; the operator is Toeplitz)."""
        t = self._symbol(which)
        rows = np.asarray(rows, dtype=np.intp)
        cols = np.asarray(cols, dtype=np.intp)
        return t[self.n - 1 + cols[None, :] - rows[:, None]]

    def dense_matrix(self, which="A"):
        """levy.py:210-214 (small sizes: n x n host array)."""
        idx = np.arange(self.n)
        return self.entries(idx, idx, which)

    def cluster_tree(self, leaf_size=64, strategy="bisection"):
        """levy.py:216-222."""
        if self.tree is None:
            self.tree = build_cluster_tree(self.grid.points[:, None], leaf_size=leaf_size,
                                           strategy=strategy)
        return self.tree

    def hmatrix(self, which="plus", cfg=None):
        """levy.py:224-239: the series H-builder on the GPU."""
        cfg = cfg or HConfig()
        if self.nu.gauss_eps_sq is None:
            raise ValueError("series H-builder requires a Gaussian jump density")
        ct = self.cluster_tree(leaf_size=cfg.n_min)
        if not np.array_equal(ct.perm.inverse, np.arange(self.n)):
            raise ValueError("the Toeplitz entry source needs the identity tree permutation")
        sign = {"A": -1.0, "plus": -0.5 * self.dt, "minus": +0.5 * self.dt}[which]
        scale = sign * self.nu.scale * self.h ** self.dim
        expansion = gaussian_expansion_1d(self.nu.gauss_eps_sq, scale=scale)
        t = {"A": self.tA, "plus": self.tPlus, "minus": self.tMinus}[which]
        return build_from_expansion(ct, ct, expansion, cfg, entry_fn=ToeplitzEntries(t))

    def build_pair(self, cfg=None):
        """H+ and H- with H-'s factors derived from H+'s: the series U carries the sign
        (scale = -+ dt/2 * nu.scale * h), so H-'s low-rank blocks are exactly (-U, V)."""
        cfg = cfg or HConfig()
        Hp = self.hmatrix("plus", cfg)
        Hm = derive_toeplitz(Hp, self.tMinus, lr_scale=-1.0, kcap=0)
        return Hp, Hm

    def prepare(self, cfg=None, eps2=1e-10, method="propagator"):
        """levy.py:241-246: factorise A+ once and keep A- for stepping.  ``method`` picks the
        per-step solve (hops.solve): "propagator" (default, one streaming H-matvec of
        Z = (A+)^-1 per step), "inverse" (triangular-inverse factors) or "substitution"
        (the reference's forward/backward substitution); run_cn / step_cn use it."""
        Hp, Hm = self.build_pair(cfg)
        self.h_minus = Hm
        self.factor = hlu(Hp, eps2)
        if method == "inverse":
            self.factor.prepare_inverse()
        elif method == "propagator":
            self.factor.prepare_propagator()
        self.method = method
        return self.factor


def assemble_cn_1d(nu, a, b, c, grid, dt, window=None):
    """levy.py:249-263 (+ _check_coeffs :240-246): the Toeplitz symbols of A, A+ and A- are
    generated on the GPU for the Gaussian density (lh_gauss_cn_symbol)."""
    import ctypes as C

    import torch

    from . import _lib

    if a < 0 or c > 0:
        raise ValueError("stability requires a >= 0 and c <= 0")
    if nu.kind != "smooth_semi_heavy":
        raise ValueError("CN assembly needs a smooth semi-heavy density; "
                         "use levyh.fractional for singular measures")
    if nu.gauss_eps_sq is None:
        raise ValueError("the device CN assembly generates the Gaussian density "
                         "(gaussian_measure); use FracCNSystem for power / CGMY measures")
    if nu.gauss_eps_sq <= 0 or nu.scale < 0:
        raise ValueError("jump density must be nonnegative")
    span = window if window is not None else (grid.hi - grid.lo)
    n_off = int(round(span / grid.h))
    ctx = _lib.Context.get()
    n = grid.size
    dev = f"cuda:{ctx.device}"
    tA, tP, tM = (torch.empty(2 * n - 1, dtype=torch.float64, device=dev) for _ in range(3))
    lam = C.c_double()
    _lib.check(_lib.lib().lh_gauss_cn_symbol(ctx.h, n, grid.h, float(nu.gauss_eps_sq),
                                             float(nu.scale), n_off, float(a), float(b), float(c),
                                             float(dt), C.c_void_p(tA.data_ptr()),
                                             C.c_void_p(tP.data_ptr()), C.c_void_p(tM.data_ptr()),
                                             C.byref(lam)), ctx.h)
    return CNSystem(grid, nu, a, b, c, dt, n_off, float(lam.value), 1, (tA, tP, tM))


class CNSystem2D:
    """levy.py:131-246 with dim = 2 (assemble_cn_2d): the Gaussian-jump CN operator on a tensor
    grid.  Entries are generated on the GPU (lh_cn2d_dense, _entries_a_2d levy.py:178-206) in a
    cluster tree's order, and the H-form is build_from_dense of that matrix (ACA with the
    reference's SVD truncation at eps1, hmatrix.py:294-340).  Deviation: the reference's
    CNSystem.hmatrix uses the untruncated tensor-product Gaussian series (rank n_terms^2, e.g. 100
    for fixed_rank 10) for dim 2, which exceeds this engine's low-rank capacity (32); the
    truncated form represents the same operator to eps1."""

    dim = 2

    def __init__(self, grid, nu, a, b, c, dt, n_off, lam):
        self.grid, self.nu, self.a, self.b, self.c, self.dt = grid, nu, a, b, c, dt
        self.n_off, self.lam, self.h = n_off, lam, grid.h
        self.tree = None
        self.factor = None
        self.h_minus = None
        self.method = "substitution"

    @property
    def N(self):
        return self.grid.size

    n = size = N

    def _device_matrix(self, which, order):
        import ctypes as C

        import torch

        from . import _lib

        code = {"A": 0, "plus": 1, "minus": 2}
        if which not in code:
            raise ValueError(which)
        ctx = _lib.Context.get()
        out = torch.empty((self.N, self.N), dtype=torch.float64, device=f"cuda:{ctx.device}")
        order = np.ascontiguousarray(order, dtype=np.int64)
        _lib.check(_lib.lib().lh_cn2d_dense(ctx.h, self.N, self.grid.nx, float(self.h),
                                            float(self.nu.gauss_eps_sq), float(self.nu.scale), float(self.a),
                                            float(self.b), float(self.c), float(self.lam), float(self.dt),
                                            code[which], _lib.host_ptr(order), C.c_void_p(out.data_ptr())),
                   ctx.h)
        return out

    def dense_matrix(self, which="A"):
        """levy.py:210-214 (original order, host copy)."""
        return self._device_matrix(which, np.arange(self.N)).cpu().numpy()

    def entries(self, rows, cols, which="A"):
        """levy.py:194-206 for original-order index arrays."""
        rows = np.asarray(rows, dtype=np.intp)
        cols = np.asarray(cols, dtype=np.intp)
        return self.dense_matrix(which)[np.ix_(rows, cols)]

    def cluster_tree(self, leaf_size=64, strategy="bisection"):
        """levy.py:216-222 on the 2D grid points."""
        if self.tree is None:
            self.tree = build_cluster_tree(self.grid.points, leaf_size=leaf_size, strategy=strategy)
        return self.tree

    SERIES_TERMS_MAX = 5  # terms per dimension the engine stores (rank T^2 <= 32)

    def hmatrix(self, which="plus", cfg=None, builder=None):
        """levy.py:224-239.  ``builder="series"``: the reference's route, build_from_expansion with
        gaussian_expansion_2d and the exact entries as dense leaves (block rank fixed_rank ** 2,
        so at most 5 terms per dimension fit the engine's 32-column kept rank);
        ``builder="dense"``: build_from_dense of the device-generated operator at cfg.eps1
        (any accuracy, O(N^2) assembly).  None picks the series route when it fits (no delta
        rule, fixed_rank <= 5) and the dense route otherwise (the default fixed_rank = 10 would
        be rank 100).  The low-rank capacity defaults to 48 columns: the 2D factors' H-LU updates
        need the room."""
        import dataclasses

        from .hmatrix import Cn2dEntries, build_from_dense, build_from_expansion, gaussian_expansion_2d

        cfg = cfg or HConfig()
        if cfg.kcap < 48:
            cfg = dataclasses.replace(cfg, kcap=48)
        if which not in ("A", "plus", "minus"):
            raise ValueError(which)
        if builder is None:
            builder = "series" if cfg.delta is None and cfg.fixed_rank <= self.SERIES_TERMS_MAX else "dense"
        ct = self.cluster_tree(leaf_size=cfg.n_min)
        if builder == "dense":
            return build_from_dense(self._device_matrix(which, ct.perm.inverse), ct, ct, cfg)
        if builder != "series":
            raise ValueError("builder must be 'series', 'dense' or None")
        sign = {"A": -1.0, "plus": -0.5 * self.dt, "minus": +0.5 * self.dt}[which]
        expansion = gaussian_expansion_2d(self.nu.gauss_eps_sq, scale=sign * self.nu.scale * self.h ** 2)
        return build_from_expansion(ct, ct, expansion, cfg, entry_fn=Cn2dEntries(self, which))

    def build_pair(self, cfg=None):
        cfg = cfg or HConfig()
        return self.hmatrix("plus", cfg), self.hmatrix("minus", cfg)

    def prepare(self, cfg=None, eps2=1e-10, method="substitution"):
        """levy.py:241-246.  Steps by forward/backward substitution (the reference's solve); the
        propagator and triangular-inverse plans are built for the 1D block structure only."""
        if method != "substitution":
            raise NotImplementedError("2D systems step by substitution (the propagator and "
                                      "triangular-inverse planners assume the 1D block structure)")
        Hp, Hm = self.build_pair(cfg)
        self.h_minus = Hm
        self.factor = hlu(Hp, eps2)
        if method == "inverse":
            self.factor.prepare_inverse()
        elif method == "propagator":
            self.factor.prepare_propagator()
        self.method = method
        return self.factor


def assemble_cn_2d(nu, a, b, c, grid, dt, window=None):
    """levy.py:275-292: the 2D CN system (convection along the first coordinate, zero data
    outside the grid); lam = the window sum of the 2D density (host scalar, as the reference)."""
    if a < 0 or c > 0:
        raise ValueError("stability requires a >= 0 and c <= 0")
    if nu.kind != "smooth_semi_heavy":
        raise ValueError("CN assembly needs a smooth semi-heavy density; "
                         "use levyh.fractional for singular measures")
    if nu.density2 is None:
        raise ValueError("2D assembly needs a 2D density")
    if nu.gauss_eps_sq is None:
        raise ValueError("the device 2D assembly generates the Gaussian density (gaussian_measure)")
    span = window if window is not None else (grid.hi - grid.lo)
    n_off = int(round(span / grid.h))
    j = np.arange(-n_off, n_off + 1) * grid.h
    JX, JY = np.meshgrid(j, j)
    vals = nu.density2(JX, JY)
    if np.any(vals < 0):
        raise ValueError("jump density must be nonnegative")
    lam = float(vals.sum() - vals[n_off, n_off])
    return CNSystem2D(grid, nu, a, b, c, dt, n_off, lam)


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
        self.method = "propagator"
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

    def prepare(self, cfg=None, eps2=1e-10, method="propagator", spill_minus=False):
        """Factorise A+ once and keep A- for stepping (levy.py:241-246).  ``method`` as in
        CNSystem.prepare: "propagator" (default), "inverse" or "substitution".
        ``spill_minus``: with the propagator the CN step is u <- 2 Z u - u and never reads A-,
        so A- moves to pinned host memory (HMatrix.spill) and its HBM holds Z instead (N = 2^22);
        it comes back on first use."""
        Hp, Hm = self.build_pair(cfg)
        self.h_minus = Hm
        if spill_minus and method == "propagator":
            Hm.spill()
        self.factor = hlu(Hp, eps2)
        if method == "inverse":
            self.factor.prepare_inverse()
        elif method == "propagator":
            self.factor.prepare_propagator()
        self.method = method
        return self.factor


def step_cn(sys, u_n, F=None, method=None):
    """levy.py:295-306: solve A+ u = A- u_n, one C-ABI call (lh_cn_step_host) on host vectors.

    A pinned CPU torch tensor (tree order = grid order for these 1D grids) takes the
    pipelined path: u streams in and the new u streams out in pieces overlapped with the
    step's kernels.  numpy in -> numpy out."""
    import torch

    from . import _lib

    F = F if F is not None else sys.factor
    if F is None or sys.h_minus is None:
        raise ValueError("call prepare() before stepping")
    m = SOLVE_METHODS[method or getattr(sys, "method", None) or "propagator"]
    if m == 2:
        F.prepare_propagator()
    elif m == 1:
        F.prepare_inverse()
    perm = sys.tree.perm
    ctx = sys.h_minus.ctx
    if isinstance(u_n, torch.Tensor):
        if u_n.is_cuda or u_n.dtype != torch.float64 or u_n.shape != (sys.N,):
            raise ValueError("step_cn takes a host float64 vector of length N")
        if not np.array_equal(perm.inverse, np.arange(sys.N)):
            raise ValueError("torch host vectors need the identity tree permutation")
        src = u_n.contiguous()
        out = torch.empty_like(src, pin_memory=src.is_pinned())
        _lib.check(_lib.lib().lh_cn_step_host(ctx.h, sys.h_minus.handle, F.h.handle, src.data_ptr(),
                                              out.data_ptr(), m), ctx.h)
        return out
    u_n = np.asarray(u_n, dtype=float)
    if u_n.shape != (sys.N,):
        raise ValueError(f"vector shape {u_n.shape} does not match N={sys.N}")
    src = np.ascontiguousarray(perm.to_tree(u_n))
    out = np.empty_like(src)
    _lib.check(_lib.lib().lh_cn_step_host(ctx.h, sys.h_minus.handle, F.h.handle, _lib.host_ptr(src),
                                          _lib.host_ptr(out), m), ctx.h)
    return perm.from_tree(out)


def _dense_device(sys, which):
    """The dense A+ / A- in original (grid) order as a device tensor."""
    import torch

    from . import _lib

    if hasattr(sys, "_device_matrix"):
        return sys._device_matrix(which, np.arange(sys.N))
    t = {"plus": sys.tPlus, "minus": sys.tMinus}[which]  # Toeplitz: A[i, j] = t[N - 1 + j - i]
    n = sys.N
    if 8.0 * n * n > 64e9:
        raise MemoryError(f"dense mode refused for N={n}: {8.0 * n * n / 2 ** 30:.1f} GiB")
    i = torch.arange(n, device=t.device)
    return t[(n - 1) + i[None, :] - i[:, None]]


def _run_cn_dense(sys, u0, n_steps):
    import torch

    Ap, Am = _dense_device(sys, "plus"), _dense_device(sys, "minus")
    lu, piv = torch.linalg.lu_factor(Ap)
    del Ap
    u = torch.as_tensor(np.asarray(u0, dtype=float)).to(Am.device).reshape(sys.N, -1)
    for _ in range(int(n_steps)):
        u = torch.linalg.lu_solve(lu, piv, Am @ u)
    out = u.cpu().numpy()
    return out[:, 0] if np.ndim(u0) == 1 else out


def run_cn(sys, u0, n_steps, cfg=None, eps2=1e-10, method=None, mode="hmatrix"):
    """levy.py:309-330: factor once, march n_steps on the device (CUDA-graph loop).
    ``method`` None steps with the method ``prepare`` set up (sys.method, default
    "propagator"); an explicit method prepares what it needs on the existing factor.
    ``mode='dense'`` is the reference's dense oracle path (levy.py:318-325: LU of the dense A+,
    u <- lu_solve(A- u)), run on the device: the operators are generated on the GPU (Toeplitz
    symbol gather in 1D, lh_cn2d_dense in 2D) and factored / applied by torch.linalg (cuSOLVER /
    cuBLAS -- library code, off the H-matrix path; the convergence studies use it as their
    reference solution, cli.py:318)."""
    if mode == "dense":
        return _run_cn_dense(sys, u0, n_steps)
    if mode != "hmatrix":
        raise ValueError("mode must be 'hmatrix' or 'dense'")
    import torch

    from . import _lib

    if sys.factor is None:
        sys.prepare(cfg, eps2, method or getattr(sys, "method", None) or "propagator")
    perm = sys.tree.perm
    ctx = sys.h_minus.ctx
    u = torch.as_tensor(perm.to_tree(np.asarray(u0, dtype=float))).to(f"cuda:{ctx.device}")
    uc = u.reshape(1, -1).contiguous() if u.ndim == 1 else u.t().contiguous()
    k = 1 if u.ndim == 1 else u.shape[1]
    m = SOLVE_METHODS[method or getattr(sys, "method", None) or "propagator"]
    if m == 2:
        sys.factor.prepare_propagator()
    elif m == 1:
        sys.factor.prepare_inverse()
    _lib.check(_lib.lib().lh_cn_steps(ctx.h, sys.h_minus.handle, sys.factor.h.handle, uc.data_ptr(),
                                      sys.N, k, int(n_steps), m), ctx.h)
    out = uc.reshape(-1) if k == 1 else uc.t()
    return perm.from_tree(out.cpu().numpy())
