"""Golden fixtures of the reference's Krylov consumers (levyh.solvers.pcg / gmres_restarted,
solvers.py:46-153), made by running the REAL reference package in the build container:

    python tests/golden/make_golden_krylov.py

Cases follow the reference's own call sites:
* cli.frac_poisson1d_study (cli.py:410-426): CG on the dense fractional Dirichlet operator
  with a unit source, tol 1e-12, max_iter 10 N;
* cli.frac_lshape_study (cli.py:442-477): restarted GMRES (restart 50) on the exact operator,
  right-preconditioned by solve(F, .) with F = hlu of a coarse (eps1 = 1e-1; the reference study uses 1e-4) H-matrix, and
  unpreconditioned;
plus CG preconditioned by the H-LU and a short-restart GMRES.  Operators are 1D (the
hot path's): the cfg1 fractional Laplacian and the cfg2-style convection-diffusion operator.
Writes tests/golden/krylov.npz.  Nothing here runs on the GPU box.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from levyh import fractional as F  # noqa: E402
from levyh import geometry as G  # noqa: E402
from levyh import hmatrix as HM  # noqa: E402
from levyh import hops as HO  # noqa: E402
from levyh import solvers as S  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def struct_array(H):
    kinds = {"dense": 0, "lowrank": 1, "dense_lu": 2}
    return np.array([(d["row0"], d["row1"], d["col0"], d["col1"], kinds[d["kind"]], d.get("rank", -1))
                     for d in HM.structure_summary(H)], dtype=np.int64).reshape(-1, 6)


def conv_diff_A(s, n, a, b_eff, c):
    """SURVEY 8(c) composition (as tests/golden/make_golden.py: composed_A)."""
    h = 1.0 / n
    cfg = F.FracConfig(s=s, h=h, L=1.0, L_W=2.0, rho_r=0.2)
    A = -F.frac_stencil_1d(cfg).weights[1:-1, 1:-1]
    N = A.shape[0]
    i = np.arange(N)
    A[i, i] += 2 * a / h ** 2 - c
    A[i[:-1], i[:-1] + 1] += -a / h ** 2 - b_eff / (2 * h)
    A[i[1:], i[1:] - 1] += -a / h ** 2 + b_eff / (2 * h)
    x = h * np.arange(-n + 1, n)
    return A, x


def coarse_factor(A, x, leaf, eps1):
    ct = G.build_cluster_tree(x[:, None], leaf_size=leaf)
    assert np.array_equal(ct.perm.inverse, np.arange(len(x)))
    H = HM.build_from_dense(A, ct, ct, HM.HConfig(n_min=leaf, n_block=4, eta=1.0, eps1=eps1))
    st = struct_array(H)
    return HO.hlu(H, 1e-10), st


def main():
    out = {}

    def put(tag, x, log, **extra):
        out[f"{tag}_x"] = x
        out[f"{tag}_res"] = np.array(log.residuals, dtype=np.float64)
        out[f"{tag}_iters"] = np.int64(log.iterations)
        out[f"{tag}_conv"] = np.int64(log.converged)
        for k, v in extra.items():
            out[f"{tag}_{k}"] = v

    # cli.frac_poisson1d_study: pcg(A, None, ones, tol=1e-12, max_iter=10 N)
    for n in (64, 128):
        A, x = F.assemble_fractional_poisson_1d(0.5, n, L_W=2.0, rho_r=0.2)
        u, log = S.pcg(A, None, np.ones_like(x), tol=1e-12, max_iter=10 * A.shape[0])
        put(f"poisson{n}", u, log)

    # CG on the cfg1 operator (N = 1023), preconditioned by a coarse H-LU
    A, x = F.assemble_fractional_poisson_1d(0.5, 512, L_W=2.0, rho_r=0.2)
    Fc, st = coarse_factor(A, x, 32, 1e-1)
    b = np.exp(-50 * x ** 2)
    u, log = S.pcg(A, lambda v: HO.solve(Fc, v), b, tol=1e-10, max_iter=200)
    put("pcg_hlu", u, log, struct=st)

    # cli.frac_lshape_study pattern on the cfg2-style operator (s = 0.25, a = .5, b = 1, c = -1)
    A, x = conv_diff_A(0.25, 512, 0.5, 1.0, -1.0)
    Fc, st = coarse_factor(A, x, 32, 1e-1)
    b = np.exp(-50 * x ** 2)
    u, log = S.gmres_restarted(lambda v: A @ v, lambda v: HO.solve(Fc, v), b, tol=1e-10,
                               restart=50, max_iter=400)
    put("gmres_hlu", u, log, struct=st)
    u, log = S.gmres_restarted(lambda v: A @ v, None, b, tol=1e-10, restart=20, max_iter=60)
    put("gmres_raw", u, log)

    # short restarts on the CN matrix A+ = I + dt/2 A (dt = h)
    h = 1.0 / 512
    Ap = np.eye(A.shape[0]) + 0.5 * h * A
    u, log = S.gmres_restarted(Ap, None, b, tol=1e-12, restart=5, max_iter=60)
    put("gmres_r5", u, log)

    np.savez_compressed(os.path.join(OUT, "krylov.npz"), **out)
    for k in sorted(out):
        if k.endswith("_iters") or k.endswith("_conv"):
            print(k, int(out[k]))


if __name__ == "__main__":
    main()
