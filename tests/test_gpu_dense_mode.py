"""GPU: run_cn(mode='dense') -- the reference's dense oracle path (levy.py:318-325), which its
convergence studies use as the reference solution (cli.py:288-343) -- against the reference's own
dense CN results in the fixtures, and the 2D temporal-study pattern (cli.levy2d_temporal_study)."""
import os

import numpy as np
import pytest

from tests import cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1812_08324_b200 as P
    return P


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_dense_mode_fractional_1d(P):
    g = cases.load("cfg1")
    s = cases.make_system("cfg1", g)
    u = P.run_cn(s, g["u0"], int(g["n_steps"]), mode="dense")
    assert _rel(u, g["uT_dense"]) <= 1e-10
    with pytest.raises(ValueError):
        P.run_cn(s, g["u0"], 1, mode="sparse")


def test_dense_mode_2d_and_temporal_order(P):
    g = dict(np.load(os.path.join(cases.GOLDEN, "golden_2d.npz")))
    s = P.assemble_cn_2d(P.gaussian_measure(5.0), 0.1, 0.5, -0.2, P.UniformGrid2D(24, 24), 0.05)
    u = P.run_cn(s, g["cn2_u0"], 10, mode="dense")
    assert _rel(u, g["cn2_uT_dense"]) <= 1e-11
    # cli.levy2d_temporal_study: H path at nt steps against the dense path at ref_nt steps, T = 1
    grid = P.UniformGrid2D(24, 24)
    nu = P.gaussian_measure(5.0)
    u0 = g["cn2_u0"]
    ref = P.run_cn(P.assemble_cn_2d(nu, 0, 0, 0, grid, 1.0 / 160), u0, 160, mode="dense")
    errs = []
    for nt in (5, 10, 20):
        cfg = P.HConfig(n_min=32, eps1=1e-6)  # the 2D engine limit (tests/test_gpu_2d.py)
        uh = P.run_cn(P.assemble_cn_2d(nu, 0, 0, 0, grid, 1.0 / nt), u0, nt, cfg, 1e-10)
        errs.append(float(np.abs(uh - ref).max()))
    order = P.fit_order([5, 10, 20], errs)
    assert 1.7 <= order <= 2.3, (errs, order)


def test_dense_mode_gaussian_1d_multi_rhs(P):
    s = P.assemble_cn_1d(P.gaussian_measure(5.0), 0.05, 0.2, -0.1, P.UniformGrid1D(400), 0.02)
    U0 = np.random.default_rng(2).standard_normal((400, 3))
    Ud = P.run_cn(s, U0, 5, mode="dense")
    Ap, Am = s.dense_matrix("plus"), s.dense_matrix("minus")
    want = U0.copy()
    for _ in range(5):
        want = np.linalg.solve(Ap, Am @ want)
    assert Ud.shape == (400, 3) and _rel(Ud, want) <= 1e-12
    uh = P.run_cn(s, U0[:, 0], 5, P.HConfig(n_min=32, fixed_rank=12), 1e-12)
    assert _rel(uh, want[:, 0]) <= 1e-6   # the series rank's accuracy
