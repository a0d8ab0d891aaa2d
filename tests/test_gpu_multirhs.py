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


def _path(P, F):
    out = np.zeros(4, dtype=np.int32)
    P._lib.check(P._lib.lib().lh_cn_last_path(F.h.handle, P._lib.host_ptr(out)))
    return out


def _oracle_multi(g, U0, steps):
    """The reference's multi-RHS CN loop: U <- solve(F, mul_dense(H-.root, U))
    (levy.py:309-330 with hops.py:73-85 and :424-432 on (N, K) right-hand sides)."""
    root, order, Op, Om = O.build_cn(g["tA"], float(g["dt"]), g["x"], int(g["leaf"]), float(g["eps1"]))
    Fo = O.hlu(Op, 1e-10)
    U = np.array(U0, dtype=float)
    for _ in range(steps):
        U = O.lu_solve(Fo, O.bmul(Om, U))
    return U


@pytest.mark.parametrize("name", ["cfg1", "cfg2_s075", "cfg3_cgmy"])
@pytest.mark.parametrize("K", [16, 67])
def test_run_cn_multi_rhs(P, name, K):
    """K >= 8 columns through run_cn(method="propagator"): every step is ONE DMMA matmat of the
    propagator, U <- 2 Z U - U (lh_cn_steps' multi-RHS branch), compared column by column with
    the reference's own multi-RHS loop (oracle) and with single-RHS H2-path runs."""
    g = cases.load(name)
    s = cases.make_system(name, g)
    cfg = P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"]))
    s.prepare(cfg, float(g["eps2"]), method="propagator")
    steps = 10
    U0 = _bumps(s.x, K)
    UK = P.run_cn(s, U0, steps, method="propagator")
    assert list(_path(P, s.factor)[:3]) == [2, 2, 0]  # CN pair, DMMA walk of the H2 form
    assert UK.shape == (s.N, K)
    ref = _oracle_multi(g, U0, steps)
    for k in range(K):
        assert _rel(UK[:, k], ref[:, k]) <= 1e-8, k
    assert _rel(UK, ref) <= 1e-9
    single = np.stack([P.run_cn(s, U0[:, k], steps) for k in (0, K // 2, K - 1)], axis=1)
    assert list(_path(P, s.factor)[:3]) == [2, 0, 0]
    assert _rel(UK[:, [0, K // 2, K - 1]], single) <= 1e-10


@pytest.mark.parametrize("K", [16, 67])
def test_run_cn_multi_rhs_general_hminus(P, K):
    """The multi-RHS branch with an A- that is NOT 2I - A+ (shape 3: U <- Z (A- U), two DMMA
    matmats per step) against the oracle loop on the same operator."""
    g = cases.load("cfg1")
    s = cases.make_system("cfg1", g)
    cfg = P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"]))
    s.prepare(cfg, float(g["eps2"]), method="propagator")
    t = s.tMinus.clone().zero_()
    t[s.N - 1] = 0.5
    Hq = P.derive_toeplitz(s.h_minus, t, lr_scale=0.5, kcap=0)  # 0.5 I + 0.5 (admissible part of A-)
    s.h_minus = Hq
    U0 = _bumps(s.x, K, seed=5)
    steps = 4
    UK = P.run_cn(s, U0, steps, method="propagator")
    assert list(_path(P, s.factor)[:3]) == [3, 2, 0]
    want = U0.copy()
    for _ in range(steps):
        want = P.solve(s.factor, P.mul_dense(Hq, want), method="substitution")
    assert _rel(UK, want) <= 1e-9
    u1 = P.run_cn(s, U0[:, 3], steps, method="propagator")
    assert list(_path(P, s.factor)[:3]) == [3, 0, 0]
    assert _rel(UK[:, 3], u1) <= 1e-10


def test_run_cn_multi_rhs_coarsened_propagator(P):
    """cfg4's operator at N = 32767: the coarsened propagator has fewer low-rank blocks than A-,
    so the two matmat plans size the shared multi-RHS scratch differently (regression: the
    first plan's scratch pointers must survive the second plan's request).  K = 64 columns on
    the DMMA branch against single-RHS runs of the H2 path and against the reference algorithm
    (A- matvec + substitution solve)."""
    n = 2 ** 14
    s = P.FracCNSystem(P.power_measure(1, 0.5), 0.0, 0.0, 0.0, n, 1.0 / n)
    s.prepare(P.HConfig(n_min=64, eps1=1e-10), 1e-10, method="propagator")
    U0 = np.random.default_rng(3).standard_normal((s.N, 64))
    UK = P.run_cn(s, U0, 3, method="propagator")
    form = int(s.factor.propagator_stats()[6])  # this operator's nested bases exceed 32 columns
    assert list(_path(P, s.factor)[:3]) == [2, 2 if form == 2 else 1, 0]
    for k in (0, 37, 63):
        uk = P.run_cn(s, U0[:, k], 3, method="propagator")
        assert np.linalg.norm(UK[:, k] - uk) <= 1e-10 * np.linalg.norm(uk)
        us = P.run_cn(s, U0[:, k], 3, method="substitution")
        assert list(_path(P, s.factor)[:3]) == [0, 0, 0]
        assert np.linalg.norm(UK[:, k] - us) <= 1e-9 * np.linalg.norm(us)


@pytest.mark.parametrize("name", ["cfg1", "cfg3_cgmy_n8191", "cfg5_leaf128"])
def test_multi_rhs_h2_walk_matches_h_form_matmat(P, name, monkeypatch):
    """The two multi-RHS forms of Z: the nested-basis walk as batched DMMA products (h2mm.cu:
    leaves, up levels, couplings, down levels, then the segment matmat of the dense leaves and
    row bases) and the DMMA matmat of Z's H-form (LEVYH_NO_H2MM), against each other, against
    single-RHS steps and against the reference multi-RHS loop (oracle, N <= 1023).  Leaf-128
    operators have no H2 form: both runs take the H-form."""
    g = cases.load(name)
    s = cases.make_system(name, g)
    s.prepare(P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"])), float(g["eps2"]))
    K, steps = 72, 5
    U0 = _bumps(s.x, K, seed=11)
    UH2 = P.run_cn(s, U0, steps)
    form = int(s.factor.propagator_stats()[6])
    assert _path(P, s.factor)[1] == (2 if form == 2 else 1)
    monkeypatch.setenv("LEVYH_NO_H2MM", "1")
    UH = P.run_cn(s, U0, steps)
    assert _path(P, s.factor)[1] == 1
    monkeypatch.delenv("LEVYH_NO_H2MM")
    assert _rel(UH2, UH) <= 1e-10
    for k in (0, 35, 71):
        assert _rel(UH2[:, k], P.run_cn(s, U0[:, k], steps)) <= 1e-10
    if s.N <= 1023:
        ref = _oracle_multi(g, U0[:, :8], steps)
        assert _rel(UH2[:, :8], ref) <= 1e-8
