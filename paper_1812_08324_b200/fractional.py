"""Singular-measure entry generation -- API of levyh.fractional
(/root/reference/pkg/src/levyh/fractional.py:65-635).

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
           "frac_stencil_1d", "assemble_fractional_poisson_1d", "eval_i1", "eval_i2", "eval_i3",
           "frac_apply_1d", "frac_apply_2d", "windowed_second_moment_radial_2d", "tail_mass_square_2d",
           "lshape_grid", "lshape_boundary_distance", "variable_order_field", "three_bump_source",
           "assemble_variable_order", "write_field_csv"]


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

    spec = getattr(nu, "gpu", None)  # a levyh LevyMeasure (no device spec) is tabulated
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


# ---------------------------------------------------------------------------
# matrix-free evaluators (fractional.py:304-361, :413-477) -- csrc/apply.cu
# ---------------------------------------------------------------------------
def _dev_f64(a, ctx):
    import torch

    if isinstance(a, torch.Tensor):
        return a.to(device=f"cuda:{ctx.device}", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.array(a, dtype=np.float64, order="C")).to(f"cuda:{ctx.device}")


def _like_input(out, src):
    import torch

    return out if isinstance(src, torch.Tensor) else out.cpu().numpy()


def _tail_1d(cfg):
    return cfg.tail_mass if cfg.tail_mass is not None else tail_mass_power_1d(cfg.s, cfg.L_W)


def _apply_1d(u, cfg, M, K, far, part, tail, m2):
    import torch

    ctx = _lib.Context.get()
    ud = _dev_f64(u, ctx)
    meas, keep = _measure_native(cfg.nu, cfg.h, M, ctx)
    out = torch.empty(2 * K + 1, dtype=torch.float64, device=ud.device)
    fd = None if far is None else _dev_f64(np.broadcast_to(np.asarray(far, dtype=float), (2 * K + 1,)), ctx)
    sums = np.zeros(3)
    _lib.check(_lib.lib().lh_frac_apply_1d(ctx.h, C.byref(meas), float(cfg.h), M, K, float(cfg.rho_r),
                                           float(tail), float(m2), ud.data_ptr(),
                                           None if fd is None else fd.data_ptr(), part, out.data_ptr(),
                                           _lib.host_ptr(sums)), ctx.h)
    del keep
    return out, sums


def eval_i1(u, p, cfg, sums=None):
    """fractional.py:304-319: near-field compensated trapezoid sum at padded index p (the device
    evaluates the window sums itself; ``sums`` is accepted for signature compatibility)."""
    if cfg.rho_r >= cfg.L_W:
        raise ValueError("window radius must be smaller than L_W")
    M = cfg.n_window
    if p - M < 0 or p + M + 1 > len(u):
        raise ValueError("p must leave a full window inside u")
    out, _ = _apply_1d(u[p - M: p + M + 1], cfg, M, 0, None, 1, 0.0, 0.0)
    return float(out[0])


def eval_i2(u_x, x, cfg):
    """fractional.py:322-326: far-field term f_x - u(x) tail_mass (host scalars)."""
    f = cfg.far_field(x) if cfg.far_field is not None else 0.0
    return float(f - u_x * _tail_1d(cfg))


def eval_i3(u, p, cfg, moment=None):
    """fractional.py:329-335: windowed diffusion term via the central second difference."""
    if moment is None:
        moment = windowed_second_moment(cfg.nu, cfg.window)
    d2 = (u[p + 1] + u[p - 1] - 2 * u[p]) / (2 * cfg.h ** 2)
    return float(d2 * moment)


def frac_apply_1d(u, cfg):
    """fractional.py:338-361: the generator on the main grid [-L, L] from 2(n_main + n_window) + 1
    samples on the padded grid, evaluated on the GPU (lh_frac_apply_1d).  numpy in -> numpy out,
    torch CUDA tensor in -> tensor out."""
    M, K = cfg.n_window, cfg.n_main
    if u.shape[0] != 2 * (M + K) + 1:
        raise ValueError("u must be sampled on the padded grid")
    far = None
    if cfg.far_field is not None:
        far = cfg.far_field(cfg.h * np.arange(-K, K + 1))
    m2 = windowed_second_moment(cfg.nu, cfg.window)
    out, _ = _apply_1d(u, cfg, M, K, far, 0, _tail_1d(cfg), m2)
    return _like_input(out, u)


_GL64_X, _GL64_W = np.polynomial.legendre.leggauss(64)


def windowed_second_moment_radial_2d(nu_radial, window, rel_tol=1e-12):
    """fractional.py:249-258: int rho(|y|) nu(|y|) y_1^2 dy = pi int_0^r rho nu r^3 dr."""
    return _graded(lambda r: math.pi * window(r) * nu_radial(r) * r ** 3, window.radius, rel_tol)


def tail_mass_square_2d(s, L_W, n_quad=64):
    """fractional.py:266-278: mass of the 2D power density outside [-L_W, L_W]^2."""
    c = frac_kernel_constant(2, s)
    x, w = (_GL64_X, _GL64_W) if n_quad == 64 else np.polynomial.legendre.leggauss(n_quad)
    r0 = L_W / np.cos((x + 1.0) * (math.pi / 8.0))
    return float(8.0 * (math.pi / 8.0) * ((c * r0 ** (-2 * s) / (2 * s)) @ w))


def frac_apply_2d(u, cfg):
    """fractional.py:435-477: the generator on the main grid [-L, L]^2 from u[kx, ky] on the padded
    grid (square near-field window), evaluated on the GPU (lh_frac_apply_2d)."""
    import torch

    M, K = cfg.n_window, cfg.n_main
    side = 2 * (M + K) + 1
    if tuple(u.shape) != (side, side):
        raise ValueError("u must be sampled on the padded 2D grid")
    if cfg.nu.density2 is None:
        raise ValueError("the measure has no 2D density")
    ctx = _lib.Context.get()
    ud = _dev_f64(u, ctx)
    tail = cfg.tail_mass if cfg.tail_mass is not None else tail_mass_square_2d(cfg.s, cfg.L_W)
    m2 = windowed_second_moment_radial_2d(lambda r: cfg.nu.density2(r, 0.0), cfg.window)
    j = np.arange(-M, M + 1) * cfg.h
    with np.errstate(all="ignore"):
        tab = np.array(cfg.nu.density2(j[:, None], j[None, :]), dtype=np.float64)
    tab[M, M] = 0.0
    td = _dev_f64(tab, ctx)
    fd = None
    if cfg.far_field is not None:
        xs = cfg.h * np.arange(-K, K + 1)
        fd = _dev_f64(np.broadcast_to(np.asarray(cfg.far_field(xs[:, None], xs[None, :]), dtype=float),
                                      (2 * K + 1, 2 * K + 1)), ctx)
    out = torch.empty((2 * K + 1, 2 * K + 1), dtype=torch.float64, device=ud.device)
    _lib.check(_lib.lib().lh_frac_apply_2d(ctx.h, 0.0, float(cfg.s), td.data_ptr(), float(cfg.h), M, K,
                                           float(cfg.rho_r), float(tail), float(m2), ud.data_ptr(),
                                           None if fd is None else fd.data_ptr(), out.data_ptr(), None),
               ctx.h)
    return _like_input(out, u)


# ---------------------------------------------------------------------------
# variable-order L-shape assembly (fractional.py:480-622)
# ---------------------------------------------------------------------------
_LSHAPE_CORNERS = np.array([(-1.0, -1.0), (1.0, -1.0), (1.0, 0.0), (0.0, 0.0), (0.0, 1.0), (-1.0, 1.0)])


def lshape_grid(n):
    """fractional.py:504-520: cell centres of [-1,1]^2 without [0,1]^2, n cells per side (even);
    returns (points, integer cell coordinates), 3 n^2 / 4 of each, x-major."""
    if n % 2:
        raise ValueError("n must be even for the L-shape grid")
    h = 2.0 / n
    gx, gy = (a.ravel() for a in np.meshgrid(np.arange(n), np.arange(n), indexing="ij"))
    x, y = -1.0 + (gx + 0.5) * h, -1.0 + (gy + 0.5) * h
    keep = ~((x > 0) & (y > 0))
    return np.column_stack([x[keep], y[keep]]), np.column_stack([gx[keep], gy[keep]])


def lshape_boundary_distance(pts):
    """fractional.py:523-533: distance to the boundary polygon of the L-shape."""
    pts = np.atleast_2d(np.asarray(pts, dtype=float))
    best = np.full(pts.shape[0], np.inf)
    for k in range(6):
        p, q = _LSHAPE_CORNERS[k], _LSHAPE_CORNERS[(k + 1) % 6]
        d = q - p
        t = np.clip(((pts - p) @ d) / (d @ d), 0.0, 1.0)
        best = np.minimum(best, np.linalg.norm(pts - (p + t[:, None] * d), axis=1))
    return best


def variable_order_field(pts):
    """fractional.py:536-538: s(x) = 0.9 - 0.8 d(x)."""
    return 0.9 - 0.8 * lshape_boundary_distance(pts)


def three_bump_source(pts):
    """fractional.py:541-547: Gaussian bumps at (-.5,.5), (.5,-.5), (-.5,-.5)."""
    pts = np.atleast_2d(np.asarray(pts, dtype=float))
    out = np.zeros(pts.shape[0])
    for cx, cy in ((-0.5, 0.5), (0.5, -0.5), (-0.5, -0.5)):
        out += np.exp(-10.0 * ((pts[:, 0] - cx) ** 2 + (pts[:, 1] - cy) ** 2))
    return out


def assemble_variable_order(n, s_field=None, f_field=None, L_W=2.0, rho_r=0.2, threads=None, device=False):
    """fractional.py:550-622: variable-order stiffness matrix and source on the L-shape, rows
    assembled on the GPU (lh_assemble_variable_order: one CTA per row; ``threads`` is accepted and
    ignored).  Returns (A, b, pts); ``device=True`` keeps A as a torch CUDA tensor (row-major), the
    form build_from_dense takes without a host round trip."""
    import torch

    pts, cells = lshape_grid(n)
    m = pts.shape[0]
    s = np.ascontiguousarray((s_field or variable_order_field)(pts), dtype=np.float64)
    if np.any((s <= 0) | (s >= 1)):
        raise ValueError("order field must map into (0, 1)")
    b = (f_field or three_bump_source)(pts)
    if rho_r <= 0:
        raise ValueError("window radius must be positive")
    ctx = _lib.Context.get()
    A = torch.empty((m, m), dtype=torch.float64, device=f"cuda:{ctx.device}")
    c32 = np.ascontiguousarray(cells, dtype=np.int32)
    gl16 = np.concatenate([_GL_X, _GL_W])
    gl64 = np.concatenate([_GL64_X, _GL64_W])
    _lib.check(_lib.lib().lh_assemble_variable_order(ctx.h, int(n), int(m), _lib.host_ptr(c32), _lib.host_ptr(s),
                                                     float(L_W), float(rho_r), _lib.host_ptr(gl16),
                                                     _lib.host_ptr(gl64), A.data_ptr(), None), ctx.h)
    return (A if device else A.cpu().numpy()), b, pts


def write_field_csv(path, points, values, meta=()):
    """fractional.py:625-635: scalar field as CSV rows (x, y, value) under '# ' metadata lines."""
    points = np.atleast_2d(np.asarray(points, dtype=float))
    values = np.asarray(values, dtype=float).ravel()
    with open(path, "w", newline="") as fh:
        fh.writelines(f"# {line}\n" for line in meta)
        fh.write("x,y,value\n")
        for p, v in zip(points, values):
            fh.write(",".join([*(f"{c:.17g}" for c in p), f"{v:.17g}"]) + "\n")
