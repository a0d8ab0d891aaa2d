"""Parity at BASELINE.json's full sizes through size-independent properties (the CPU oracle
cannot run these sizes; the golden-fixture tests pin the algorithms at small N):

* cfg3 (N = 2^20 - 1, CGMY): the three solve paths agree; the substitution solve (the
  reference algorithm, hops.py:424-432) has an eps-level residual against a separately
  assembled A+; one propagator CN step equals A- matvec + substitution solve; the CN step is
  linear.
* cfg2 (N = 2^16 - 1, s in {0.25, 0.75}, a=0.5, b=1, c=-1): 200 propagator steps equal 200
  steps of the reference algorithm.
* cfg4 (N = 2^18 - 1): a multi-RHS CN run equals single-RHS runs column by column.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1812_08324_b200 as P
    return P


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def cfg3(P):
    s = P.FracCNSystem(P.cgmy_measure(1.0, 5.0, 10.0, 0.5), 0.05, 0.1, -0.05, 2 ** 19, 8.0 / 2 ** 20 * 16,
                       L=4.0, L_W=8.0, drift_compensation=True)
    cfg = P.HConfig(n_min=64, eps1=1e-9)
    s.prepare(cfg, 1e-10, method="propagator")
    return s, cfg


def test_cfg3_solves_agree_and_residual(P, cfg3):
    s, cfg = cfg3
    F = s.factor
    b = np.random.default_rng(0).standard_normal(s.N)
    x_sub = P.solve(F, b, method="substitution")
    x_prop = P.solve(F, b, method="propagator")
    assert _rel(x_prop, x_sub) <= 1e-9
    Ap = s.hmatrix("plus", cfg)  # a second, unfactored A+
    assert _rel(P.matvec(Ap, x_sub), b) <= 1e-8


def test_cfg3_step_and_linearity(P, cfg3):
    s, _ = cfg3
    perm = s.tree.perm
    u0 = np.maximum(np.exp(s.x) - 1.0, 0.0)
    u_prop = P.run_cn(s, u0, 1, method="propagator")
    rhs = P.matvec(s.h_minus, perm.to_tree(u0))
    u_ref = perm.from_tree(P.solve(s.factor, rhs, method="substitution"))
    assert _rel(u_prop, u_ref) <= 1e-9
    rng = np.random.default_rng(1)
    v, w = rng.standard_normal(s.N), rng.standard_normal(s.N)
    lhs = P.run_cn(s, 2.0 * v - 3.0 * w, 3, method="propagator")
    rhs3 = 2.0 * P.run_cn(s, v, 3, method="propagator") - 3.0 * P.run_cn(s, w, 3, method="propagator")
    assert _rel(lhs, rhs3) <= 1e-11


@pytest.mark.parametrize("sfrac", [0.25, 0.75])
def test_cfg2_full_200_steps(P, sfrac):
    n = 2 ** 15
    s = P.FracCNSystem(P.power_measure(1, sfrac), 0.5, 1.0, -1.0, n, 1.0 / n)
    s.prepare(P.HConfig(n_min=64, eps1=1e-10), 1e-10, method="propagator")
    u0 = np.exp(-50.0 * s.x ** 2)
    u_prop = P.run_cn(s, u0, 200, method="propagator")
    u_ref = P.run_cn(s, u0, 200, method="substitution")
    assert _rel(u_prop, u_ref) <= 1e-8
    assert np.all(np.isfinite(u_prop)) and np.linalg.norm(u_prop) < np.linalg.norm(u0)


def test_cfg4_multi_rhs_columns(P):
    n = 2 ** 17
    s = P.FracCNSystem(P.power_measure(1, 0.5), 0.0, 0.0, 0.0, n, 1.0 / n)
    s.prepare(P.HConfig(n_min=64, eps1=1e-10), 1e-10, method="propagator")
    rng = np.random.default_rng(0)
    K = 32
    U0 = np.zeros((s.N, K))
    for k in range(K):
        c, w, a = rng.uniform(-0.8, 0.8, 8), rng.uniform(0.02, 0.2, 8), rng.normal(0, 1, 8)
        U0[:, k] = (a[None, :] * np.exp(-((s.x[:, None] - c[None, :]) / w[None, :]) ** 2)).sum(1)
    UK = P.run_cn(s, U0, 10)
    for k in (0, 13, 31):
        assert _rel(UK[:, k], P.run_cn(s, U0[:, k], 10)) <= 1e-11


def test_cfg3_propagator_nested_bases(P, cfg3):
    """At N = 2^20 the CN step streams Z in nested (H2) form, checked at build time against the
    H-form of Z on a probe vector."""
    s, _ = cfg3
    st = s.factor.propagator_stats()
    assert st[6] == 2.0  # nested H2 bases in use
    assert st[7] <= 1e-10  # probe relative error of the H2 form against the H-form
    assert 4.0 <= st[8] <= 32.0  # mean leaf basis size


def test_cfg3_100_steps_propagator_vs_substitution(P, cfg3):
    """The headline run (cfg3, N = 2^20 - 1, 100 CN steps) on the default path (one H2 matvec of
    Z per step) against the reference algorithm on the same factors (A- matvec + forward /
    backward substitution, hops.py:65-70 + :424-432), 100 steps each."""
    s, _ = cfg3
    u0 = np.maximum(np.exp(s.x) - 1.0, 0.0)
    u_prop = P.run_cn(s, u0, 100)
    u_sub = P.run_cn(s, u0, 100, method="substitution")
    assert _rel(u_prop, u_sub) <= 1e-8
