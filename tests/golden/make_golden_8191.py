"""Reference-generated fixtures at N = 8191 for the cfg2 (s = 0.25) and cfg3 (CGMY) operators
(pin the ACA ranks and the CN solution on blocks of thousands of rows).

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_8191.py

Same composition as make_golden.py (cn_case: the reference's frac_stencil_1d, build_from_dense,
hlu, solve, matvec); only the grid is 8x finer.  About a minute per case (two full-SVD
compressions of 8191 x 8191 matrices)."""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import make_golden as MG  # noqa: E402
from make_golden import F, LV  # noqa: E402


def main():
    n = 4096
    cfg = F.FracConfig(s=0.25, h=1.0 / n, L=1.0, L_W=2.0, rho_r=0.2)
    MG.cn_case("cfg2_s025_n8191", cfg, 0.5, 1.0, -1.0, 1.0 / n, 64, 1e-10, lambda x: np.exp(-50 * x ** 2), 20)

    nu = MG.cgmy_density(1.0, 5.0, 10.0, 0.5)
    from scipy.integrate import quad
    tail = (quad(lambda y: nu(np.array(y)), 8, np.inf, epsabs=0, epsrel=1e-12)[0]
            + quad(lambda y: nu(np.array(-y)), 8, np.inf, epsabs=0, epsrel=1e-12)[0])
    beta = MG.drift_beta(nu, 0.2)
    h = 4.0 / n
    meas = LV.LevyMeasure(density=nu, kind="singular_heavy_tail", symmetric=False)
    cfg = F.FracConfig(s=0.25, h=h, L=4.0, L_W=8.0, rho_r=0.2, nu=meas, tail_mass=tail)
    MG.cn_case("cfg3_cgmy_n8191", cfg, 0.05, 0.1 + beta, -0.05, 16 * h, 64, 1e-9,
               lambda x: np.maximum(np.exp(x) - 1.0, 0.0), 10)


if __name__ == "__main__":
    main()
