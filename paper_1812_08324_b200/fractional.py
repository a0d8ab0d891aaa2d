"""Singular-measure entry generation -- API of levyh.fractional (1D part,
/root/reference/pkg/src/levyh/fractional.py:65-405).

Scalar set-up (c_{d,s}, the graded second moment m2, tail masses, the drift
compensator beta of SURVEY G4) is host arithmetic; the O(M) window sums
S0, Sg, Sd and the Toeplitz symbol of the operator are generated on the GPU
(csrc/build.cu: window_sums_kernel, symbol_fill_kernel).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
from scipy.special import gammaln

from . import _lib

__all__ = ["LevyMeasure", "WindowFn", "quartic_window", "frac_kernel_constant", "power_measure",
           "cgmy_measure", "FracConfig", "FracStencil", "windowed_second_moment",
           "tail_mass_power_1d", "tail_mass_numeric", "drift_compensation_beta", "frac_symbol_1d",
           "frac_stencil_1d", "assemble_fractional_poisson_1d"]


@dataclass
class LevyMeasure:
    """levy.py:51-69, plus ``gpu``: the device evaluation spec
    (("power", c, s) or ("cgmy", C, G, M, Y)); None -> host-tabulated."""

    density: object
    kind: str = "smooth_semi_heavy"
    symmetric: bool | None = None
    density2: object = None
    gauss_eps_sq: float | None = None
    scale: float = 1.0
    gpu: tuple | None = None

    def __call__(self, y):
        return self.density(np.asarray(y, dtype=float))


@dataclass(frozen=True)
class WindowFn:
    """fractional.py:65-75."""

    radius: float
    profile: object

    def __call__(self, y):
        t = np.abs(np.asarray(y, dtype=float)) / self.radius
        return np.where(t < 1.0, self.profile(np.minimum(t, 1.0)), 0.0)


def quartic_window(radius):
    """fractional.py:78-86: (1 - (|y|/r)^4)^2."""
    if radius <= 0:
        raise ValueError("window radius must be positive")
    return WindowFn(radius, lambda t: (1.0 - t ** 4) ** 2)


def frac_kernel_constant(d, s):
    """fractional.py:89-105: 4^s Gamma(d/2+s) / (pi^{d/2} |Gamma(-s)|)."""
    if d not in (1, 2):
        raise ValueError("d must be 1 or 2")
    if not (1e-12 < s < 1.0 - 1e-12):
        raise ValueError("order s must lie strictly inside (0, 1)")
    log_c = (2 * s * math.log(2.0) + gammaln(d / 2.0 + s) - (d / 2.0) * math.log(math.pi)
             - (gammaln(1.0 - s) - math.log(s)))
    return float(np.exp(log_c))


def power_measure(d, s):
    """fractional.py:108-127 (1D GPU-evaluated)."""
    c = frac_kernel_constant(d, s)

    def density(y):
        y = np.asarray(y, dtype=float)
        with np.errstate(divide="ignore"):
            return c * np.abs(y) ** (-d - 2 * s)

    def density2(dx, dy):
        r2 = np.asarray(dx, dtype=float) ** 2 + np.asarray(dy, dtype=float) ** 2
        with np.errstate(divide="ignore"):
            return c * r2 ** (-(d + 2 * s) / 2.0)

    return LevyMeasure(density=density, kind="singular_heavy_tail", symmetric=True,
                       density2=density2 if d == 2 else None, gpu=("power", c, s) if d == 1 else None)


def cgmy_measure(C_, G, M, Y):
    """Tempered-stable density C e^{-G|y|}|y|^{-1-Y} (y<0), C e^{-M y} y^{-1-Y} (y>0)."""
    if not (0 < Y < 2):
        raise ValueError("CGMY requires 0 < Y < 2")

    def density(y):
        y = np.asarray(y, dtype=float)
        ay = np.abs(y)
        with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
            rate = np.where(y < 0, G, M)
            return C_ * np.exp(-rate * ay) * ay ** (-1.0 - Y)

    return LevyMeasure(density=density, kind="singular_heavy_tail", symmetric=(G == M),
                       gpu=("cgmy", C_, G, M, Y))


@dataclass
class FracConfig:
    """fractional.py:130-176 (1D)."""

    s: float
    h: float
    L: float
    L_W: float
    rho_r: float = 0.2
    far_field: object = None
    tail_mass: float | None = None
    nu: LevyMeasure | None = None
    dim: int = 1

    def __post_init__(self):
        if not (0 < self.rho_r < self.L_W):
            raise ValueError("need 0 < rho_r < L_W")
        if not (1e-12 < self.s < 1 - 1e-12):
            raise ValueError("order s must lie strictly inside (0, 1)")
        if self.nu is None:
            self.nu = power_measure(self.dim, self.s)
        for name, val in (("L", self.L), ("L_W", self.L_W)):
            k = val / self.h
            if abs(k - round(k)) > 1e-9:
                raise ValueError(f"{name} must be an integer multiple of h")

    @property
    def n_window(self):
        return int(round(self.L_W / self.h))

    @property
    def n_main(self):
        return int(round(self.L / self.h))

    @property
    def window(self):
        return quartic_window(self.rho_r)


@dataclass
class FracStencil:
    weights: np.ndarray
    offset: np.ndarray
    x: np.ndarray


_GL_X, _GL_W = np.polynomial.legendre.leggauss(16)


def _graded(f, radius, rel_tol=1e-12, max_levels=60):
    """Dyadic Gauss-Legendre panels toward 0 with geometric completion (fractional.py:200-232)."""
    total, hi = 0.0, radius
    prev_part = prev_val = None
    for _ in range(max_levels):
        lo = hi / 2.0
        mid, rad = 0.5 * (lo + hi), 0.5 * (hi - lo)
        part = rad * float(f(mid + rad * _GL_X) @ _GL_W)
        total += part
        val = total
        if prev_part is not None and 0 < abs(part) < abs(prev_part):
            q = part / prev_part
            if 0 < q < 1:
                val = total + part * q / (1.0 - q)
        if abs(part) < rel_tol * max(abs(val), 1e-300):
            return val
        if prev_val is not None and abs(val - prev_val) <= rel_tol * max(abs(val), 1e-300):
            return val
        prev_part, prev_val = part, val
        hi = lo
    raise RuntimeError("graded quadrature did not converge within 60 levels")


def windowed_second_moment(nu, window, rel_tol=1e-12):
    """fractional.py:235-246: int rho nu y^2 (both sides)."""
    up = _graded(lambda y: window(y) * nu.density(y) * y * y, window.radius, rel_tol)
    dn = _graded(lambda y: window(-y) * nu.density(-y) * y * y, window.radius, rel_tol)
    return up + dn


def tail_mass_power_1d(s, L_W):
    """fractional.py:261-263."""
    return frac_kernel_constant(1, s) * L_W ** (-2 * s) / s


def tail_mass_numeric(nu, L_W):
    """int_{|y|>L_W} nu (adaptive quadrature; for measures without a closed form)."""
    from scipy.integrate import quad

    f = lambda y: float(nu.density(np.array(y)))  # noqa: E731
    g = lambda y: float(nu.density(np.array(-y)))  # noqa: E731
    return (quad(f, L_W, np.inf, epsabs=0, epsrel=1e-12)[0]
            + quad(g, L_W, np.inf, epsabs=0, epsrel=1e-12)[0])


def drift_compensation_beta(nu, rho_r):
    """beta = int (rho(y) - 1_{|y|<1}) y nu(y) dy, so that the generator with the
    1_{|y|<1} compensator equals the rho-compensated one plus beta u'."""
    from scipy.integrate import quad

    win = quartic_window(rho_r)

    def g(y):
        return float((win(y) - 1.0) * y * nu.density(np.array(y)))

    return (quad(g, 0.0, 1.0, limit=400, epsabs=0.0, epsrel=1e-13, points=[rho_r])[0]
            + quad(g, -1.0, 0.0, limit=400, epsabs=0.0, epsrel=1e-13, points=[-rho_r])[0])


def _measure_native(nu, h, M, ctx):
    import torch

    spec = nu.gpu
    keep = None
    if spec is not None and spec[0] == "power":
        m = _lib.MeasureC(0, spec[1], spec[2], 0, 0, 0, 0, None)
    elif spec is not None and spec[0] == "cgmy":
        m = _lib.MeasureC(1, 0, 0, spec[1], spec[2], spec[3], spec[4], None)
    else:
        y = np.arange(-M, M + 1) * h
        with np.errstate(all="ignore"):
            tab = np.asarray(nu.density(y), dtype=np.float64)
        tab[M] = 0.0
        keep = torch.from_numpy(tab).to(f"cuda:{ctx.device}")
        m = _lib.MeasureC(2, 0, 0, 0, 0, 0, 0, C.c_void_p(keep.data_ptr()))
    return m, keep


def frac_symbol_1d(nu, h, N, L_W, rho_r, tail, m2, a=0.0, b=0.0, c=0.0, dt=0.0):
    """GPU Toeplitz symbols of A (composed CN operator) and A+- = I +- dt/2 A.

    Returns (tA, tPlus, tMinus, sums) with torch device tensors of length 2N-1,
    entry k + N - 1 = A[i, i + k], and sums = (S0, Sg, Sd) from the GPU reduction.
    """
    import torch

    ctx = _lib.Context.get()
    M = int(round(L_W / h))
    meas, keep = _measure_native(nu, h, M, ctx)
    dev = f"cuda:{ctx.device}"
    tA = torch.empty(2 * N - 1, dtype=torch.float64, device=dev)
    tP = torch.empty_like(tA)
    tM = torch.empty_like(tA)
    sums = np.zeros(3)
    p = _lib.CNParamsC(float(h), int(N), int(M), float(rho_r), float(tail), float(m2), float(a),
                       float(b), float(c), float(dt))
    _lib.check(_lib.lib().lh_cn_symbol(ctx.h, C.byref(meas), C.byref(p), tA.data_ptr(), tP.data_ptr(),
                                       tM.data_ptr(), _lib.host_ptr(sums)), ctx.h)
    del keep
    return tA, tP, tM, tuple(float(v) for v in sums)


def frac_stencil_1d(cfg: FracConfig):
    """fractional.py:362-390 (dense W on the main grid; small n only)."""
    M, K = cfg.n_window, cfg.n_main
    n = 2 * K + 1
    m2 = windowed_second_moment(cfg.nu, cfg.window)
    tail = cfg.tail_mass if cfg.tail_mass is not None else tail_mass_power_1d(cfg.s, cfg.L_W)
    tA, _, _, _ = frac_symbol_1d(cfg.nu, cfg.h, n, cfg.L_W, cfg.rho_r, tail, m2)
    t = -tA.cpu().numpy()
    i = np.arange(n)
    W = t[(i[None, :] - i[:, None]) + n - 1]
    x = cfg.h * np.arange(-K, K + 1)
    f = cfg.far_field(x) if cfg.far_field is not None else np.zeros(n)
    return FracStencil(weights=W, offset=np.asarray(f, dtype=float), x=x)


def assemble_fractional_poisson_1d(s, n, L=1.0, L_W=2.0, rho_r=0.2):
    """fractional.py:393-405 (dense; small n only)."""
    h = L / n
    cfg = FracConfig(s=s, h=h, L=L, L_W=L_W, rho_r=rho_r)
    st = frac_stencil_1d(cfg)
    return -st.weights[1:-1, 1:-1], st.x[1:-1]
