"""CPU oracle for the matrix-free evaluators and the variable-order assembly (TEST INFRASTRUCTURE
ONLY; same rules as levyh_oracle.py: imported by tests/ and nothing else).

numpy restatement of /root/reference/pkg/src/levyh/fractional.py:285-361 (1D window sums,
eval_i1..i3, frac_apply_1d), :413-477 (2D window sums, frac_apply_2d) and :504-622 (L-shape grid,
order field, assemble_variable_order).  Pinned to fixtures the real reference produced
(tests/golden/make_golden_apply.py -> tests/golden/apply.npz; tests/test_oracle_apply.py).
"""
from __future__ import annotations

import math

import numpy as np

from .levyh_oracle import frac_const, graded_integral, window, window_sums


def power2(s):
    """2D power density c r^(-2-2s) on offsets (dx, dy) (fractional.py:117-120)."""
    c = frac_const(2, s)

    def f(dx, dy):
        r2 = np.asarray(dx, dtype=float) ** 2 + np.asarray(dy, dtype=float) ** 2
        with np.errstate(divide="ignore"):
            return c * r2 ** (-(2 + 2 * s) / 2.0)
    return f


def apply_1d(u, nu, h, M, K, rho_r, tail, m2, far=0.0):
    """frac_apply_1d (fractional.py:338-361); returns (values, i1)."""
    u = np.asarray(u, dtype=float)
    kern, S0, Sg, Sd = window_sums(nu, h, M, rho_r)
    conv = np.correlate(u, kern, mode="valid")
    uc, ue, uw = u[M: M + 2 * K + 1], u[M + 1: M + 2 * K + 2], u[M - 1: M + 2 * K]
    d1 = (ue - uw) / (2 * h)
    d2 = (ue + uw - 2 * uc) / (2 * h * h)
    i1 = conv - uc * S0 - d1 * Sg - d2 * Sd
    return i1 + far - uc * tail + d2 * m2, i1


def window_sums_2d(nu2, h, M, rho_r):
    """_window_sums_2d (fractional.py:413-432): kern and S0, Sgx, Sgy, Sdxx, Sdyy, Sdxy."""
    j = np.arange(-M, M + 1)
    JX, JY = np.meshgrid(j * h, j * h, indexing="ij")
    with np.errstate(all="ignore"):
        nu_l = np.array(nu2(JX, JY), dtype=float)
    nu_l[M, M] = 0.0
    w1 = np.full(j.shape, h)
    w1[0] = w1[-1] = h / 2.0
    kern = nu_l * np.outer(w1, w1)
    rho = window(np.hypot(JX, JY), rho_r)
    return kern, np.array([kern.sum(), (rho * JX * kern).sum(), (rho * JY * kern).sum(),
                           (rho * JX * JX * kern).sum(), (rho * JY * JY * kern).sum(),
                           (rho * JX * JY * kern).sum()])


def moment_radial_2d(nu_radial, rho_r, rel_tol=1e-12):
    """windowed_second_moment_radial_2d (fractional.py:249-258)."""
    return graded_integral(lambda r: math.pi * window(r, rho_r) * nu_radial(r) * r ** 3, rho_r, rel_tol)


def tail_square_2d(s, L_W, n_quad=64):
    """tail_mass_square_2d (fractional.py:266-278)."""
    c = frac_const(2, s)
    x, w = np.polynomial.legendre.leggauss(n_quad)
    r0 = L_W / np.cos((x + 1.0) * (math.pi / 8.0))
    return float(8.0 * (math.pi / 8.0) * ((c * r0 ** (-2 * s) / (2 * s)) @ w))


def apply_2d(u, nu2, h, M, K, rho_r, tail, m2, far=0.0):
    """frac_apply_2d (fractional.py:435-477) with a direct (not FFT) window correlation."""
    u = np.asarray(u, dtype=float)
    kern, S = window_sums_2d(nu2, h, M, rho_r)
    n = 2 * K + 1
    conv = np.zeros((n, n))
    for jx in range(2 * M + 1):
        for jy in range(2 * M + 1):
            conv += u[jx: jx + n, jy: jy + n] * kern[jx, jy]
    c, e, w = slice(M, M + n), slice(M + 1, M + n + 1), slice(M - 1, M + n - 1)
    uc = u[c, c]
    ux = (u[e, c] - u[w, c]) / (2 * h)
    uy = (u[c, e] - u[c, w]) / (2 * h)
    uxx = (u[e, c] + u[w, c] - 2 * uc) / h ** 2
    uyy = (u[c, e] + u[c, w] - 2 * uc) / h ** 2
    uxy = (u[e, e] + u[w, w] - u[e, w] - u[w, e]) / (4 * h ** 2)
    i1 = (conv - uc * S[0] - ux * S[1] - uy * S[2] - 0.5 * uxx * S[3] - 0.5 * uyy * S[4] - uxy * S[5])
    return i1 + far - uc * tail + 0.5 * (uxx + uyy) * m2


def lshape_cells(n):
    """lshape_grid (fractional.py:504-520)."""
    h = 2.0 / n
    gx, gy = (a.ravel() for a in np.meshgrid(np.arange(n), np.arange(n), indexing="ij"))
    x, y = -1.0 + (gx + 0.5) * h, -1.0 + (gy + 0.5) * h
    keep = ~((x > 0) & (y > 0))
    return np.column_stack([x[keep], y[keep]]), np.column_stack([gx[keep], gy[keep]])


def assemble_vo(n, s, L_W=2.0, rho_r=0.2, rows=None):
    """assemble_variable_order (fractional.py:550-622) for a given per-row order array s
    (rows: assemble only these rows, the others stay zero)."""
    pts, cells = lshape_cells(n)
    m, h = pts.shape[0], 2.0 / n
    Mw = int(round(L_W / h))
    off = np.arange(-Mw, Mw + 1)
    DX, DY = np.meshgrid(off * h, off * h, indexing="ij")
    R2 = DX * DX + DY * DY
    R2[Mw, Mw] = 1.0
    logR2 = np.log(R2)
    w1 = np.full(off.shape, h)
    w1[0] = w1[-1] = h / 2.0
    w2 = np.outer(w1, w1)
    rho = window(np.sqrt(R2), rho_r)
    table = -np.ones((n, n), dtype=np.intp)
    table[cells[:, 0], cells[:, 1]] = np.arange(m)
    A = np.zeros((m, m))
    info = np.zeros((m, 8))
    for i in (range(m) if rows is None else rows):
        si = s[i]
        ci = frac_const(2, si)
        k = ci * np.exp(-(1.0 + si) * logR2)
        k[Mw, Mw] = 0.0
        kw = k * w2
        S0 = kw.sum()
        sgx, sgy = (rho * DX * kw).sum(), (rho * DY * kw).sum()
        sdxx, sdyy, sdxy = (rho * DX * DX * kw).sum(), (rho * DY * DY * kw).sum(), (rho * DX * DY * kw).sum()
        m2 = moment_radial_2d(lambda r: ci * r ** (-2.0 - 2.0 * si), rho_r)
        tail = tail_square_2d(si, L_W)
        info[i] = S0, sgx, sgy, sdxx, sdyy, sdxy, m2, tail
        gx, gy = cells[i]
        x0, x1 = max(0, gx - Mw), min(n, gx + Mw + 1)
        y0, y1 = max(0, gy - Mw), min(n, gy + Mw + 1)
        cols = table[x0:x1, y0:y1].ravel()
        vals = (k[x0 - gx + Mw: x1 - gx + Mw, y0 - gy + Mw: y1 - gy + Mw] * h * h).ravel()
        A[i, cols[cols >= 0]] = vals[cols >= 0]
        cxx, cyy, cxy = 0.5 * (m2 - sdxx) / h ** 2, 0.5 * (m2 - sdyy) / h ** 2, -sdxy / (4 * h ** 2)
        for dx, dy, val in ((0, 0, -S0 - tail - 2 * cxx - 2 * cyy), (1, 0, cxx - sgx / (2 * h)),
                            (-1, 0, cxx + sgx / (2 * h)), (0, 1, cyy - sgy / (2 * h)),
                            (0, -1, cyy + sgy / (2 * h)), (1, 1, cxy), (-1, -1, cxy), (1, -1, -cxy),
                            (-1, 1, -cxy)):
            cx, cy = gx + dx, gy + dy
            if 0 <= cx < n and 0 <= cy < n and table[cx, cy] >= 0:
                A[i, table[cx, cy]] += val
    return A, info
