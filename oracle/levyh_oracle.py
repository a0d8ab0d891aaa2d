"""CPU oracle for the Crank-Nicolson H-matrix hot path (TEST INFRASTRUCTURE ONLY).

This module is a numpy restatement of the reference package `levyh`
(/root/reference/pkg/src/levyh, arxiv 1812.08324) for the one path the
B200 build accelerates: singular-measure entry generation, dense-to-H
compression by truncated SVD, recursive H-LU and forward/backward solve,
the H-matvec, and the CN stepping loop.  Every function cites the
reference file:line it restates.

Only `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` /
`--impl reference` legs of `bench.py` may import this file, and only as the
checker or as the timed CPU baseline.  The product package never imports
it; the product path fails loudly without its CUDA library.

Pinning: `tests/golden/make_golden.py` runs the real reference (importable
in the build container) and writes `tests/golden/*.npz`; `tests/test_oracle.py`
checks this restatement against those fixtures bit-for-bit where the
arithmetic is identical (partition, symbol, ranks) and to 1e-13 where LAPACK
call shapes differ.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.linalg as sla
from scipy.linalg.blas import dtrsm
from scipy.special import gammaln

# ---------------------------------------------------------------------------
# cluster tree + admissibility   (geometry.py:142-263)
# ---------------------------------------------------------------------------


class Cluster:
    """Contiguous tree-order range [lo, hi) with its bounding box."""

    __slots__ = ("lo", "hi", "blo", "bhi", "kids")

    def __init__(self, lo, hi, blo, bhi, kids=()):
        self.lo, self.hi, self.blo, self.bhi, self.kids = lo, hi, blo, bhi, kids

    @property
    def size(self):
        return self.hi - self.lo

    @property
    def leaf(self):
        return not self.kids

    def diam(self):  # geometry.py:89-91 (norm of bbox diagonal)
        d = self.bhi - self.blo
        return float(math.sqrt(float(np.dot(d, d))))


def cluster_tree(points, leaf_size):
    """Median bisection along the widest axis (geometry.py:146-154, 191-243).

    Returns (root, order) with order[i_tree] = i_orig.
    """
    pts = np.asarray(points, dtype=float)
    if pts.ndim == 1:
        pts = pts[:, None]
    n = pts.shape[0]
    order = np.empty(n, dtype=np.intp)

    def rec(idx, start):
        sub = pts[idx]
        blo, bhi = sub.min(axis=0), sub.max(axis=0)
        if idx.shape[0] <= leaf_size:
            order[start:start + idx.shape[0]] = idx
            return Cluster(start, start + idx.shape[0], blo, bhi)
        ax = int(np.argmax(bhi - blo))
        srt = np.argsort(sub[:, ax], kind="stable")
        left = np.zeros(idx.shape[0], dtype=bool)
        left[srt[: idx.shape[0] // 2]] = True
        a = rec(idx[left], start)
        b = rec(idx[~left], a.hi)
        return Cluster(start, b.hi, blo, bhi, (a, b))

    root = rec(np.arange(n, dtype=np.intp), 0)
    return root, order


def is_admissible(a, b, eta):
    """bbox test min(diam) <= eta * dist, dist <= 0 never (geometry.py:246-263)."""
    gap = np.maximum(np.maximum(a.blo - b.bhi, b.blo - a.bhi), 0.0)
    dist = float(math.sqrt(float(np.dot(gap, gap))))
    if dist <= 0.0:
        return False
    return min(a.diam(), b.diam()) <= eta * dist


# ---------------------------------------------------------------------------
# H-matrix blocks   (hmatrix.py:51-118)
# ---------------------------------------------------------------------------


class Blk:
    """kind in {'D' dense, 'R' low-rank u@v.T, 'H' 2x2, 'F' factored dense}."""

    __slots__ = ("kind", "d", "u", "v", "k", "rs", "cs", "piv", "perm")

    def __init__(self, kind, **kw):
        self.kind = kind
        self.d = kw.get("d")
        self.u = kw.get("u")
        self.v = kw.get("v")
        self.k = kw.get("k")
        self.rs = kw.get("rs")
        self.cs = kw.get("cs")
        self.piv = None
        self.perm = None

    @property
    def shape(self):
        if self.kind in "DF":
            return self.d.shape
        if self.kind == "R":
            return (self.u.shape[0], self.v.shape[0])
        return (self.k[0][0].shape[0] + self.k[1][0].shape[0],
                self.k[0][0].shape[1] + self.k[0][1].shape[1])


def svd_truncate(blk, eps1):
    """Full SVD, keep s > eps1*s[0]; None when rank > min//2 (hmatrix.py:294-303)."""
    u, s, vt = np.linalg.svd(blk, full_matrices=False)
    r = 0 if (s.size == 0 or s[0] == 0.0) else int(np.count_nonzero(s > eps1 * s[0]))
    if r > min(blk.shape) // 2:
        return None
    return Blk("R", u=u[:, :r] * s[:r], v=vt[:r].T.copy())


def compress_dense(A, root, eps1, n_min=64, n_block=4, eta=1.0):
    """Partition + compression decision order of build_from_dense (hmatrix.py:306-340)."""
    A = np.asarray(A, dtype=float)
    if not np.all(np.isfinite(A)):
        raise ValueError("matrix has non-finite entries")
    nmax = math.ceil(max(A.shape) / n_block)

    def rec(r, c):
        m, n = r.size, c.size
        sub = A[r.lo:r.hi, c.lo:c.hi]
        splittable = (not r.leaf) and (not c.leaf)
        if splittable and (m > nmax or n > nmax):
            pass
        elif is_admissible(r, c, eta) and min(m, n) > n_min:
            lr = svd_truncate(sub, eps1)
            return lr if lr is not None else Blk("D", d=sub.copy())
        elif min(m, n) <= n_min or not splittable:
            return Blk("D", d=sub.copy())
        (r0, r1), (c0, c1) = r.kids, c.kids
        return Blk("H", k=[[rec(r0, c0), rec(r0, c1)], [rec(r1, c0), rec(r1, c1)]],
                   rs=r0.size, cs=c0.size)

    return rec(root, root)


def leaves(b, r0=0, c0=0, out=None):
    """Depth-first (11,12,21,22) leaf walk (hmatrix.py:343-351)."""
    if out is None:
        out = []
    if b.kind == "H":
        leaves(b.k[0][0], r0, c0, out)
        leaves(b.k[0][1], r0, c0 + b.cs, out)
        leaves(b.k[1][0], r0 + b.rs, c0, out)
        leaves(b.k[1][1], r0 + b.rs, c0 + b.cs, out)
    else:
        out.append((b, r0, c0))
    return out


def structure(b):
    """Records as in structure_summary (hmatrix.py:376-389): (r0,r1,c0,c1,kind,rank)."""
    recs = []
    for blk, r0, c0 in leaves(b):
        m, n = blk.shape
        kind = {"D": 0, "R": 1, "F": 2}[blk.kind]
        rank = blk.u.shape[1] if blk.kind == "R" else -1
        recs.append((r0, r0 + m, c0, c0 + n, kind, rank))
    return np.array(recs, dtype=np.int64).reshape(-1, 6)


def stored_scalars(b):
    """memory_report stored_scalars (hmatrix.py:354-373)."""
    tot = 0
    for blk, _, _ in leaves(b):
        m, n = blk.shape
        tot += blk.u.shape[1] * (m + n) if blk.kind == "R" else m * n
    return tot


def densify(b):
    """to_dense (hmatrix.py:402-413)."""
    if b.kind == "D":
        return b.d.copy()
    if b.kind == "R":
        return b.u @ b.v.T
    if b.kind == "F":
        raise ValueError("cannot densify an LU-factored leaf")
    return np.vstack([np.hstack([densify(b.k[0][0]), densify(b.k[0][1])]),
                      np.hstack([densify(b.k[1][0]), densify(b.k[1][1])])])


# ---------------------------------------------------------------------------
# products   (hops.py:50-100)
# ---------------------------------------------------------------------------


def bmul(b, X):
    """b @ X for dense X, vector or matrix (hops.py:50-62, 73-85)."""
    if b.kind == "D":
        return b.d @ X
    if b.kind == "R":
        return b.u @ (b.v.T @ X)
    if b.kind == "H":
        X1, X2 = X[:b.cs], X[b.cs:]
        top = bmul(b.k[0][0], X1) + bmul(b.k[0][1], X2)
        bot = bmul(b.k[1][0], X1) + bmul(b.k[1][1], X2)
        return np.concatenate([top, bot]) if X.ndim == 1 else np.vstack([top, bot])
    raise TypeError(f"cannot multiply block of kind {b.kind}")


def bmul_t(b, X):
    """b.T @ X (hops.py:88-100)."""
    if b.kind == "D":
        return b.d.T @ X
    if b.kind == "R":
        return b.v @ (b.u.T @ X)
    if b.kind == "H":
        X1, X2 = X[:b.rs], X[b.rs:]
        top = bmul_t(b.k[0][0], X1) + bmul_t(b.k[1][0], X2)
        bot = bmul_t(b.k[0][1], X1) + bmul_t(b.k[1][1], X2)
        return np.vstack([top, bot])
    raise TypeError(f"cannot multiply block of kind {b.kind}")


def hmatvec(b, x):
    """matvec (hops.py:65-70)."""
    x = np.asarray(x, dtype=float)
    if x.ndim != 1 or x.shape[0] != b.shape[1]:
        raise ValueError("vector length does not match n_cols")
    return bmul(b, x)


# ---------------------------------------------------------------------------
# recompression   (hops.py:124-163)
# ---------------------------------------------------------------------------


def frob_tail_rank(s, eps2):
    """Smallest r with ||s[r:]|| <= eps2 ||s|| (hops.py:124-131)."""
    sq = s * s
    tot = float(np.sqrt(sq.sum()))
    if tot == 0.0:
        return 0
    tails = np.sqrt(np.concatenate([np.cumsum(sq[::-1])[::-1], [0.0]]))
    return int(np.argmax(tails <= eps2 * tot))


def lr_add(u1, v1, u2, v2, eps2):
    """QR-QR-SVD recompression of u1 v1' + u2 v2' (hops.py:134-144)."""
    U = np.hstack([u1, u2])
    V = np.hstack([v1, v2])
    if U.shape[1] == 0:
        return U, V
    qu, ru = np.linalg.qr(U)
    qv, rv = np.linalg.qr(V)
    w, s, zt = np.linalg.svd(ru @ rv.T)
    r = frob_tail_rank(s, eps2)
    return qu @ (w[:, :r] * s[:r]), qv @ zt[:r].T


def dense_to_lr(D, eps2):
    """hops.py:159-163."""
    u, s, vt = np.linalg.svd(D, full_matrices=False)
    r = frob_tail_rank(s, eps2)
    return u[:, :r] * s[:r], vt[:r].T.copy()


# ---------------------------------------------------------------------------
# triangular solves   (hops.py:171-279)
# ---------------------------------------------------------------------------


def _pivot_perm(piv):
    """Net permutation of LAPACK ipiv (hops.py:171-177)."""
    p = np.arange(piv.shape[0])
    for i, j in enumerate(piv):
        if j != i:
            p[i], p[j] = p[j], p[i]
    return p


def _blas_trsm(a, B, lower, trans, unit):
    return dtrsm(1.0, a, np.asfortranarray(B, dtype=float), side=0, lower=lower,
                 trans_a=trans, diag=unit, overwrite_b=1)


def _leaf_trsm(T, B, mode, unit, path):
    """hops.py:191-208."""
    lo, tr = {"L": (1, 0), "U": (0, 0), "Ut": (0, 1)}[mode]
    if T.kind == "F":
        if mode == "L":
            return _blas_trsm(T.d, B[T.perm], 1, 0, 1)
        return _blas_trsm(T.d, B, lo, tr, 0)
    if np.any(np.diag(T.d) == 0.0):
        raise np.linalg.LinAlgError(f"singular triangular diagonal block at {path}")
    return _blas_trsm(T.d, B, lo, tr, int(unit))


def solve_dense(T, B, mode, unit, path):
    """Recursive dense-RHS triangular solve (hops.py:211-229)."""
    if T.kind != "H":
        return _leaf_trsm(T, B, mode, unit, path)
    c, s = T.k, T.rs
    B1, B2 = B[:s], B[s:]
    if mode == "L":
        y1 = solve_dense(c[0][0], B1, mode, unit, path + ".11")
        y2 = solve_dense(c[1][1], B2 - bmul(c[1][0], y1), mode, unit, path + ".22")
    elif mode == "U":
        y2 = solve_dense(c[1][1], B2, mode, unit, path + ".22")
        y1 = solve_dense(c[0][0], B1 - bmul(c[0][1], y2), mode, unit, path + ".11")
    elif mode == "Ut":
        y1 = solve_dense(c[0][0], B1, mode, unit, path + ".11")
        y2 = solve_dense(c[1][1], B2 - bmul_t(c[0][1], y1), mode, unit, path + ".22")
    else:
        raise ValueError(mode)
    return np.vstack([y1, y2])


def solve_block_left(T, B, mode, unit, eps2, path):
    """T X = B in place on block B (hops.py:232-258)."""
    if B.kind == "R":
        B.u = solve_dense(T, B.u, mode, unit, path)
        return B
    if B.kind == "D":
        B.d = solve_dense(T, B.d, mode, unit, path)
        return B
    if T.kind != "H":
        return Blk("D", d=solve_dense(T, densify(B), mode, unit, path))
    c, b = T.k, B.k
    if mode == "L":
        b[0][0] = solve_block_left(c[0][0], b[0][0], mode, unit, eps2, path + ".11")
        b[0][1] = solve_block_left(c[0][0], b[0][1], mode, unit, eps2, path + ".11")
        schur(b[1][0], c[1][0], b[0][0], eps2)
        schur(b[1][1], c[1][0], b[0][1], eps2)
        b[1][0] = solve_block_left(c[1][1], b[1][0], mode, unit, eps2, path + ".22")
        b[1][1] = solve_block_left(c[1][1], b[1][1], mode, unit, eps2, path + ".22")
    else:
        b[1][0] = solve_block_left(c[1][1], b[1][0], mode, unit, eps2, path + ".22")
        b[1][1] = solve_block_left(c[1][1], b[1][1], mode, unit, eps2, path + ".22")
        schur(b[0][0], c[0][1], b[1][0], eps2)
        schur(b[0][1], c[0][1], b[1][1], eps2)
        b[0][0] = solve_block_left(c[0][0], b[0][0], mode, unit, eps2, path + ".11")
        b[0][1] = solve_block_left(c[0][0], b[0][1], mode, unit, eps2, path + ".11")
    return B


def solve_block_right_upper(T, B, eps2, path):
    """X U = B in place on B (hops.py:261-279)."""
    if B.kind == "R":
        B.v = solve_dense(T, B.v, "Ut", True, path)
        return B
    if B.kind == "D":
        B.d = solve_dense(T, B.d.T, "Ut", True, path).T
        return B
    if T.kind != "H":
        return Blk("D", d=solve_dense(T, densify(B).T, "Ut", True, path).T)
    c, b = T.k, B.k
    b[0][0] = solve_block_right_upper(c[0][0], b[0][0], eps2, path + ".11")
    b[1][0] = solve_block_right_upper(c[0][0], b[1][0], eps2, path + ".11")
    schur(b[0][1], b[0][0], c[0][1], eps2)
    schur(b[1][1], b[1][0], c[0][1], eps2)
    b[0][1] = solve_block_right_upper(c[1][1], b[0][1], eps2, path + ".22")
    b[1][1] = solve_block_right_upper(c[1][1], b[1][1], eps2, path + ".22")
    return B


# ---------------------------------------------------------------------------
# Schur updates   (hops.py:318-369)
# ---------------------------------------------------------------------------


def sub_lowrank(C, U, V, eps2):
    """C -= U V' (hops.py:318-331)."""
    if U.shape[1] == 0:
        return
    if C.kind == "D":
        C.d -= U @ V.T
    elif C.kind == "R":
        C.u, C.v = lr_add(C.u, C.v, -U, V, eps2)
    else:
        rs, cs = C.rs, C.cs
        sub_lowrank(C.k[0][0], U[:rs], V[:cs], eps2)
        sub_lowrank(C.k[0][1], U[:rs], V[cs:], eps2)
        sub_lowrank(C.k[1][0], U[rs:], V[:cs], eps2)
        sub_lowrank(C.k[1][1], U[rs:], V[cs:], eps2)


def sub_dense(C, D, eps2):
    """C -= D (hops.py:334-345)."""
    if C.kind == "D":
        C.d -= D
    elif C.kind == "R":
        C.u, C.v = dense_to_lr(C.u @ C.v.T - D, eps2)
    else:
        rs, cs = C.rs, C.cs
        sub_dense(C.k[0][0], D[:rs, :cs], eps2)
        sub_dense(C.k[0][1], D[:rs, cs:], eps2)
        sub_dense(C.k[1][0], D[rs:, :cs], eps2)
        sub_dense(C.k[1][1], D[rs:, cs:], eps2)


def schur(C, A, B, eps2):
    """C -= A @ B in block arithmetic (hops.py:348-369)."""
    if A.kind == "R":
        sub_lowrank(C, A.u, bmul_t(B, A.v), eps2)
    elif B.kind == "R":
        sub_lowrank(C, bmul(A, B.u), B.v, eps2)
    elif A.kind == "D" and B.kind == "D":
        sub_dense(C, A.d @ B.d, eps2)
    elif A.kind == "D":
        sub_dense(C, bmul_t(B, A.d.T).T, eps2)
    elif B.kind == "D":
        sub_dense(C, bmul(A, B.d), eps2)
    elif C.kind == "H" and A.kind == "H" and B.kind == "H":
        if A.cs != B.rs or C.rs != A.rs or C.cs != B.cs:
            sub_dense(C, bmul(A, densify(B)), eps2)
            return
        for i in (0, 1):
            for j in (0, 1):
                for k in (0, 1):
                    schur(C.k[i][j], A.k[i][k], B.k[k][j], eps2)
    else:
        sub_dense(C, bmul(A, densify(B)), eps2)


# ---------------------------------------------------------------------------
# H-LU and solve   (hops.py:392-432)
# ---------------------------------------------------------------------------


def lu_inplace(b, eps2, path="root"):
    """Recursive in-place block LU (hops.py:392-408)."""
    if b.kind == "D":
        lu, piv = sla.lu_factor(b.d, check_finite=False)
        if np.any(np.diag(lu) == 0.0):
            raise np.linalg.LinAlgError(f"zero pivot in dense diagonal leaf at {path}")
        f = Blk("F", d=lu)
        f.piv = piv
        f.perm = _pivot_perm(piv)
        return f
    if b.kind != "H":
        raise TypeError(f"cannot LU-factorize diagonal block of kind {b.kind} at {path}")
    c = b.k
    c[0][0] = lu_inplace(c[0][0], eps2, path + ".11")
    c[0][1] = solve_block_left(c[0][0], c[0][1], "L", True, eps2, path + ".12")
    c[1][0] = solve_block_right_upper(c[0][0], c[1][0], eps2, path + ".21")
    schur(c[1][1], c[1][0], c[0][1], eps2)
    c[1][1] = lu_inplace(c[1][1], eps2, path + ".22")
    return b


def hlu(root, eps2=1e-10):
    """hops.py:411-421 (consumes `root`)."""
    if root.shape[0] != root.shape[1]:
        raise ValueError("LU requires a square matrix")
    return lu_inplace(root, eps2, "root")


def lu_solve(F, b):
    """Forward (unit L, leaf pivots) then backward (U) (hops.py:424-432)."""
    b = np.asarray(b, dtype=float)
    if b.shape[0] != F.shape[0]:
        raise ValueError("right-hand side length mismatch")
    rhs = b.reshape(b.shape[0], -1)
    y = solve_dense(F, rhs, "L", True, "root")
    x = solve_dense(F, y, "U", False, "root")
    return x.reshape(b.shape)


# ---------------------------------------------------------------------------
# singular-measure entries   (fractional.py:65-405, levy.py:169-206)
# ---------------------------------------------------------------------------

_GLX, _GLW = np.polynomial.legendre.leggauss(16)


def frac_const(d, s):
    """c_{d,s} via log-Gamma (fractional.py:89-105)."""
    if not (1e-12 < s < 1.0 - 1e-12):
        raise ValueError("order s must lie strictly inside (0, 1)")
    lc = (2 * s * math.log(2.0) + gammaln(d / 2.0 + s) - (d / 2.0) * math.log(math.pi)
          - (gammaln(1.0 - s) - math.log(s)))
    return float(np.exp(lc))


def nu_power(s):
    """1D power density c|y|^{-1-2s} (fractional.py:108-127)."""
    c = frac_const(1, s)

    def f(y):
        y = np.asarray(y, dtype=float)
        with np.errstate(divide="ignore"):
            return c * np.abs(y) ** (-1 - 2 * s)
    return f


def nu_cgmy(C, G, M, Y):
    """CGMY density: C e^{-G|y|}|y|^{-1-Y} (y<0), C e^{-M y} y^{-1-Y} (y>0)."""
    def f(y):
        y = np.asarray(y, dtype=float)
        ay = np.abs(y)
        with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
            rate = np.where(y < 0, G, M)
            return C * np.exp(-rate * ay) * ay ** (-1.0 - Y)
    return f


def window(y, radius):
    """Quartic window (1-(|y|/r)^4)^2 (fractional.py:65-86)."""
    t = np.abs(np.asarray(y, dtype=float)) / radius
    return np.where(t < 1.0, (1.0 - np.minimum(t, 1.0) ** 4) ** 2, 0.0)


def window_sums(nu, h, M, rho_r):
    """Trapezoid kern, S0, Sg, Sd over offsets |j| <= M, j != 0 (fractional.py:285-301)."""
    j = np.arange(-M, M + 1)
    y = j * h
    nj = nu(y)
    nj[M] = 0.0
    w = np.full(j.shape, h)
    w[0] = w[-1] = h / 2.0
    rho = window(y, rho_r)
    kern = nj * w
    return kern, float(kern.sum()), float((rho * y * kern).sum()), float((rho * y * y * kern).sum())


def graded_integral(f, radius, rel_tol=1e-12, max_levels=60):
    """Dyadic GL-16 panels with geometric tail completion (fractional.py:200-232)."""
    acc, hi = 0.0, radius
    last_part = last_val = None
    for _ in range(max_levels):
        lo = hi / 2.0
        mid, rad = 0.5 * (lo + hi), 0.5 * (hi - lo)
        part = rad * float(f(mid + rad * _GLX) @ _GLW)
        acc += part
        val = acc
        if last_part is not None and 0 < abs(part) < abs(last_part):
            q = part / last_part
            if 0 < q < 1:
                val = acc + part * q / (1.0 - q)
        if abs(part) < rel_tol * max(abs(val), 1e-300):
            return val
        if last_val is not None and abs(val - last_val) <= rel_tol * max(abs(val), 1e-300):
            return val
        last_part, last_val = part, val
        hi = lo
    raise RuntimeError("graded quadrature did not converge within 60 levels")


def second_moment(nu, rho_r, rel_tol=1e-12):
    """m2 = int rho nu y^2 (fractional.py:235-246)."""
    up = graded_integral(lambda y: window(y, rho_r) * nu(y) * y * y, rho_r, rel_tol)
    dn = graded_integral(lambda y: window(-y, rho_r) * nu(-y) * y * y, rho_r, rel_tol)
    return up + dn


def tail_power(s, L_W):
    """fractional.py:261-263."""
    return frac_const(1, s) * L_W ** (-2 * s) / s


def symbol_A(nu, h, N, L_W, rho_r, tail, a=0.0, b=0.0, c=0.0):
    """Toeplitz symbol tA[k + N - 1] = A[i, i+k] of the composed CN operator A.

    A = -W[1:-1,1:-1] (fractional.py:362-405) with the local band of
    levy._entries_a_1d (levy.py:169-176) added afterwards.
    Floating-point order follows the reference statements exactly.
    Returns (tA, scalars dict).
    """
    M = int(round(L_W / h))
    kern, S0, Sg, Sd = window_sums(nu, h, M, rho_r)
    m2 = second_moment(nu, rho_r)
    t = np.zeros(2 * N - 1)
    kmax = min(N - 1, M)
    ks = np.arange(-kmax, kmax + 1)
    Wv = np.zeros(2 * N - 1)
    Wv[ks + N - 1] = kern[ks + M]
    Wv[N - 1] = 0.0 + ((-S0 - tail) - (m2 - Sd) / h ** 2)
    cside = (m2 - Sd) / (2 * h ** 2)
    if N > 1:
        Wv[N] += cside - Sg / (2 * h)
        Wv[N - 2] += cside + Sg / (2 * h)
    t[:] = -Wv
    t[N - 1] += 2 * a / h ** 2 - c
    if N > 1:
        t[N] += -a / h ** 2 - b / (2 * h)
        t[N - 2] += -a / h ** 2 + b / (2 * h)
    return t, dict(S0=S0, Sg=Sg, Sd=Sd, m2=m2, tail=tail, M=M)


def symbol_pm(tA, dt, which):
    """A+- = I +- dt/2 A on the symbol (levy.py:201-205)."""
    N = (tA.shape[0] + 1) // 2
    hd = 0.5 * dt
    if which == "plus":
        t = 0.0 + hd * tA
        t[N - 1] = 1.0 + hd * tA[N - 1]
    else:
        t = 0.0 - hd * tA
        t[N - 1] = 1.0 - hd * tA[N - 1]
    return t


def toeplitz_dense(t):
    """Dense N x N matrix with entry (i, j) = t[j - i + N - 1]."""
    N = (t.shape[0] + 1) // 2
    i = np.arange(N)
    return t[(i[None, :] - i[:, None]) + N - 1]


def drift_beta(nu, rho_r):
    """beta = int (rho(y) - 1_{|y|<1}) y nu(y) dy, by scipy quad."""
    from scipy.integrate import quad

    def g(y):
        return float((window(y, rho_r) - 1.0) * y * nu(np.array(y)))
    pos = quad(g, 0.0, 1.0, limit=400, epsabs=0.0, epsrel=1e-13, points=[rho_r])[0]
    neg = quad(g, -1.0, 0.0, limit=400, epsabs=0.0, epsrel=1e-13, points=[-rho_r])[0]
    return pos + neg


# ---------------------------------------------------------------------------
# CN stepping   (levy.py:295-330)
# ---------------------------------------------------------------------------


def run_cn(Hm, F, u0, n_steps):
    """Factor-once loop u <- solve(F, H- u) (levy.py:309-330), identity perm."""
    u = np.asarray(u0, dtype=float).copy()
    for _ in range(n_steps):
        u = lu_solve(F, hmatvec(Hm, u))
    return u


def build_cn(tA, dt, x, leaf, eps1, n_block=4, eta=1.0):
    """Cluster tree + H+ / H- of the composed CN operator."""
    root, order = cluster_tree(x, leaf)
    Ap = toeplitz_dense(symbol_pm(tA, dt, "plus"))
    Am = toeplitz_dense(symbol_pm(tA, dt, "minus"))
    Hp = compress_dense(Ap[np.ix_(order, order)], root, eps1, leaf, n_block, eta)
    Hm = compress_dense(Am[np.ix_(order, order)], root, eps1, leaf, n_block, eta)
    return root, order, Hp, Hm


# ---------------------------------------------------------------------------
# smooth-measure (Gaussian) system + series H-builder
# (levy.py:72-81, :169-206, :249-263; hmatrix.py:156-186, :243-291)
# ---------------------------------------------------------------------------


def gauss_density(eps_sq, scale=1.0):
    """levy.py:72-81: nu(y) = scale * exp(-eps_sq y^2)."""
    return lambda y: scale * np.exp(-eps_sq * np.asarray(y, dtype=float) ** 2)


def gauss_cn_symbol(n, h, eps_sq, scale, a, b, c, n_off):
    """Toeplitz symbol t[k + n - 1] = A[i, i + k] of levy.CNSystem's A (levy.py:169-176) with
    lam = sum over the window offsets (assemble_cn_1d, levy.py:257-262)."""
    nu = gauss_density(eps_sq, scale)
    j = np.arange(1, n_off + 1)
    lam = float(np.concatenate([nu(-j * h), nu(j * h)]).sum())
    k = np.arange(-(n - 1), n)
    t = -nu(k * h) * h
    if n > 1:
        t[n] += -a / h ** 2 - b / (2 * h)
        t[n - 2] += -a / h ** 2 + b / (2 * h)
    t[n - 1] = 2 * a / h ** 2 - c + lam * h
    return t, lam


def series_cols(t, eps_sq, n_terms, alpha, scale=1.0):
    """hmatrix.py:156-169: column k = scale (2 eps_sq t)^k e^{-eps_sq t^2} / k! (alpha) or
    t^k e^{-eps_sq t^2}, by the recurrence col_k = col_{k-1} * base / k."""
    cols = [scale * np.exp(-eps_sq * t * t)]
    base = 2.0 * eps_sq * t if alpha else t
    for k in range(1, n_terms):
        cols.append(cols[-1] * base / (k if alpha else 1))
    return np.stack(cols, axis=1)


def series_terms(eps_sq, D, fixed_rank, delta):
    """_expansion_terms + rank_bound_gaussian (hmatrix.py:270-290)."""
    if delta is None:
        return fixed_rank
    if D <= 0:
        return 1
    eps = math.sqrt(eps_sq)
    e2 = 2.0 * eps * eps * D * D
    bound = max(e2 / math.log(2.0) - math.log2(delta) - 1.0, 6.0 * e2 - 1.0)
    return max(0, math.floor(bound) + 1) + 1


def build_series(x, leaf, eps_sq, scale, t, fixed_rank=10, delta=None, n_block=4, eta=1.0):
    """build_from_expansion (hmatrix.py:243-291) with gaussian_expansion_1d around the row
    cluster centre, dense leaves from the Toeplitz symbol t (the CNSystem entry_fn,
    levy.py:235-237).  Returns (root, order, blk)."""
    x = np.asarray(x, dtype=float)
    root, order = cluster_tree(x, leaf)
    pts = x[order]
    n = x.shape[0]
    nmax = math.ceil(n / n_block)

    def dense(r, c):
        rows = order[r.lo:r.hi]
        cols = order[c.lo:c.hi]
        return Blk("D", d=t[n - 1 + cols[None, :] - rows[:, None]].copy())

    def rec(r, c):
        m, k = r.size, c.size
        splittable = (not r.leaf) and (not c.leaf)
        if splittable and (m > nmax or k > nmax):
            pass
        elif is_admissible(r, c, eta) and min(m, k) > leaf:
            ctr = 0.5 * (r.blo + r.bhi)
            K = series_terms(eps_sq, r.diam(), fixed_rank, delta)
            u = series_cols(pts[r.lo:r.hi] - ctr[0], eps_sq, K, True, scale)
            v = series_cols(pts[c.lo:c.hi] - ctr[0], eps_sq, K, False)
            return Blk("R", u=u, v=v)
        elif min(m, k) <= leaf or not splittable:
            return dense(r, c)
        (r0, r1), (c0, c1) = r.kids, c.kids
        return Blk("H", k=[[rec(r0, c0), rec(r0, c1)], [rec(r1, c0), rec(r1, c1)]],
                   rs=r0.size, cs=c0.size)

    return root, order, rec(root, root)


def build_gauss_cn(n, eps_sq, scale, a, b, c, dt, leaf, fixed_rank=10, delta=None, lo=-1.0, hi=1.0):
    """levy.assemble_cn_1d + CNSystem.hmatrix('plus'/'minus') (levy.py:224-263) on
    UniformGrid1D(n, lo, hi) (levy.py:84-102).  Returns (x, tA, lam, root, Hp, Hm)."""
    h = (hi - lo) / n
    x = lo + h * np.arange(n)
    n_off = int(round((hi - lo) / h))
    tA, lam = gauss_cn_symbol(n, h, eps_sq, scale, a, b, c, n_off)
    tP = symbol_pm(tA, dt, "plus")
    tM = symbol_pm(tA, dt, "minus")
    root, _, Hp = build_series(x, leaf, eps_sq, -0.5 * dt * scale * h, tP, fixed_rank, delta)
    _, _, Hm = build_series(x, leaf, eps_sq, +0.5 * dt * scale * h, tM, fixed_rank, delta)
    return x, tA, lam, root, Hp, Hm


# ---------------------------------------------------------------------------
# Krylov consumers   (solvers.py:46-153)
# ---------------------------------------------------------------------------


def _op(f):
    """solvers.py:39-43: callables pass through, arrays become a matvec."""
    if f is None:
        return lambda v: v
    if callable(f):
        return f
    mat = np.asarray(f)
    return lambda v: mat @ v


def pcg(A, Minv, b, tol=1e-8, max_iter=500):
    """Preconditioned CG from x = 0 (solvers.py:46-88).  Returns (x, residuals, converged);
    raises LinAlgError when p'Ap <= 0 (solvers.py:71-72)."""
    A, M = _op(A), _op(Minv)
    b = np.asarray(b, dtype=float)
    x = np.zeros_like(b)
    nb = np.linalg.norm(b)
    if nb == 0:
        return x, [], True
    r = b.copy()
    z = M(r)
    p = np.array(z, copy=True)
    rz = float(np.dot(r, z))
    hist = []
    for _ in range(max_iter):
        q = A(p)
        curv = float(np.dot(p, q))
        if curv <= 0:
            raise np.linalg.LinAlgError("PCG breakdown: operator is not positive definite")
        step = rz / curv
        x += step * p
        r -= step * q
        hist.append(float(np.linalg.norm(r) / nb))
        if hist[-1] <= tol:
            return x, hist, True
        z = M(r)
        rz_next = float(np.dot(r, z))
        p = z + (rz_next / rz) * p
        rz = rz_next
    return x, hist, False


def gmres_restarted(A, Minv, b, tol=1e-8, restart=50, max_iter=500):
    """Right-preconditioned restarted GMRES (solvers.py:91-153): modified Gram-Schmidt
    Arnoldi, Givens rotations, residual of the original system.  Returns
    (x, residuals, converged)."""
    A, M = _op(A), _op(Minv)
    b = np.asarray(b, dtype=float)
    n = b.size
    x = np.zeros_like(b)
    nb = np.linalg.norm(b)
    if nb == 0:
        return x, [], True
    hist, done, count = [], False, 0
    while count < max_iter and not done:
        r = b - A(x)
        beta = float(np.linalg.norm(r))
        if beta / nb <= tol:
            done = True
            break
        m = min(restart, max_iter - count)
        Q = np.zeros((n, m + 1))
        Hs = np.zeros((m + 1, m))
        rot = np.zeros((m, 2))  # (cos, sin)
        g = np.zeros(m + 1)
        g[0] = beta
        Q[:, 0] = r / beta
        k = 0
        for j in range(m):
            w = A(M(Q[:, j]))
            for i in range(j + 1):  # MGS
                Hs[i, j] = float(np.dot(w, Q[:, i]))
                w = w - Hs[i, j] * Q[:, i]
            Hs[j + 1, j] = float(np.linalg.norm(w))
            if Hs[j + 1, j] > 0:
                Q[:, j + 1] = w / Hs[j + 1, j]
            for i in range(j):  # earlier rotations on the new column
                c, s = rot[i]
                hi, hn = Hs[i, j], Hs[i + 1, j]
                Hs[i, j], Hs[i + 1, j] = c * hi + s * hn, -s * hi + c * hn
            rho = np.hypot(Hs[j, j], Hs[j + 1, j])
            rot[j] = Hs[j, j] / rho, Hs[j + 1, j] / rho
            Hs[j, j], Hs[j + 1, j] = rho, 0.0
            g[j], g[j + 1] = rot[j, 0] * g[j], -rot[j, 1] * g[j]
            k = j + 1
            count += 1
            hist.append(float(abs(g[j + 1]) / nb))
            if hist[-1] <= tol:
                break
        y = np.linalg.solve(Hs[:k, :k], g[:k]) if k else np.zeros(0)
        x = x + M(Q[:, :k] @ y)
        if hist and hist[-1] <= tol:
            done = True
    return x, hist, done
