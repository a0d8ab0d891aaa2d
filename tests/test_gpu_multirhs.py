"""Multi-RHS path (BASELINE configs[3] / SURVEY 8(d) cfg4): the DMMA matmat behind
mul_dense / solve / run_cn with K >= 8 right-hand sides must match the single-RHS path
column by column (and the oracle) on the golden operators."""
import numpy as np
import pytest

from oracle import levyh_oracle as O
from tests import cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1812_08324_b200 as P
    return P


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _bumps(x, K, seed=0):
    """cfg4-style initial conditions: sums of 8 Gaussian bumps per column (seeded)."""
    rng = np.random.default_rng(seed)
    U = np.zeros((x.shape[0], K))
    for k in range(K):
        c = rng.uniform(-0.8, 0.8, 8)
        w = rng.uniform(0.02, 0.2, 8)
        a = rng.normal(0.0, 1.0, 8)
        U[:, k] = (a[None, :] * np.exp(-((x[:, None] - c[None, :]) / w[None, :]) ** 2)).sum(1)
    return U


@pytest.mark.parametrize("name", ["cfg1", "cfg3_cgmy", "cfg5_leaf128"])
@pytest.mark.parametrize("K", [8, 67])
def test_mul_dense_matches_columns(P, name, K):
    g = cases.load(name)
    s = cases.make_system(name, g)
    cfg = P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"]))
    Hp, Hm = s.build_pair(cfg)
    X = np.random.default_rng(K).standard_normal((s.N, K))
    Y = P.mul_dense(Hm, X)
    cols = np.stack([P.matvec(Hm, X[:, k]) for k in range(K)], axis=1)
    assert Y.shape == (s.N, K)
    assert _rel(Y, cols) <= 1e-13
    root, order, Op, Om = O.build_cn(g["tA"], float(g["dt"]), g["x"], int(g["leaf"]), float(g["eps1"]))
    assert _rel(Y[:, :3], np.stack([O.hmatvec(Om, X[:, k]) for k in range(3)], 1)) <= 1e-12


def test_propagator_solve_multi(P):
    g = cases.load("cfg3_cgmy")
    s = cases.make_system("cfg3_cgmy", g)
    cfg = P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"]))
    Hp, Hm = s.build_pair(cfg)
    F = P.hlu(Hp, 1e-10)
    B = np.random.default_rng(3).standard_normal((s.N, 20))
    Xm = P.solve(F, B, method="propagator")
    Xs = P.solve(F, B, method="substitution")
    assert _rel(Xm, Xs) <= 1e-9


@pytest.mark.parametrize("name", ["cfg1", "cfg2_s075"])
def test_run_cn_multi_rhs(P, name):
    g = cases.load(name)
    s = cases.make_system(name, g)
    cfg = P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"]))
    s.prepare(cfg, float(g["eps2"]), method="propagator")
    K, steps = 16, 10
    U0 = _bumps(s.x, K)
    UK = P.run_cn(s, U0, steps)  # (N, K): one DMMA matmat per step
    ref = np.stack([P.run_cn(s, U0[:, k], steps) for k in range(4)], axis=1)
    assert UK.shape == (s.N, K)
    assert _rel(UK[:, :4], ref) <= 1e-11
    root, order, Op, Om = O.build_cn(g["tA"], float(g["dt"]), g["x"], int(g["leaf"]), float(g["eps1"]))
    Fo = O.hlu(Op, 1e-10)
    uo = O.run_cn(Om, Fo, U0[:, 5], steps)
    assert _rel(UK[:, 5], uo) <= 1e-8


def test_run_cn_multi_rhs_coarsened_propagator(P):
    """cfg4's operator at N = 32767: the coarsened propagator has fewer low-rank blocks than A-,
    so the two matmat plans size the shared multi-RHS scratch differently (regression: the
    first plan's scratch pointers must survive the second plan's request)."""
    n = 2 ** 14
    s = P.FracCNSystem(P.power_measure(1, 0.5), 0.0, 0.0, 0.0, n, 1.0 / n)
    s.prepare(P.HConfig(n_min=64, eps1=1e-10), 1e-10, method="propagator")
    U0 = np.random.default_rng(3).standard_normal((s.N, 64))
    UK = P.run_cn(s, U0, 3)
    for k in (0, 37, 63):
        uk = P.run_cn(s, U0[:, k], 3)
        assert np.linalg.norm(UK[:, k] - uk) <= 1e-10 * np.linalg.norm(uk)
