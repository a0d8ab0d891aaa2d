"""Convergence order of the CN scheme on the GPU path (temporal order 2.0 on the
cfg1 operator, as measured with the reference; joint dt = h refinement is ~0.6-0.75)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _solve(P, n, n_steps, T=1.0):
    h = 1.0 / n
    s = P.FracCNSystem(P.power_measure(1, 0.5), 0.0, 0.0, 0.0, n, T / n_steps)
    s.prepare(P.HConfig(n_min=32, eps1=1e-10), 1e-10, method="inverse")
    u0 = (1 - s.x ** 2) ** 2
    return s.x, P.run_cn(s, u0, n_steps)


def test_temporal_order_two():
    import paper_1812_08324_b200 as P

    n = 512  # N = 1023 interior unknowns (cfg1 grid)
    _, ref = _solve(P, n, 1024)
    nts = (16, 32, 64, 128)
    errs = [np.abs(_solve(P, n, nt)[1] - ref).max() for nt in nts]
    slope = np.polyfit(np.log(nts), np.log(errs), 1)[0]
    assert 1.8 <= -slope <= 2.2, (errs, slope)


def _restrict(ref, n_ref, n):
    """Values of the n_ref grid (x = k / n_ref, |k| < n_ref) at the points of the n grid."""
    stride = n_ref // n
    k = np.arange(-(n - 1), n) * stride
    return ref[k + n_ref - 1]


def test_joint_order_dt_eq_h():
    """Joint refinement dt = h (cli.py:288-309 pattern, fit_order cli.py:116-118) on the cfg1
    operator with the default stepping path (propagator): the zero-exterior, boundary-singular
    regime gives max-norm orders 0.57-0.74 with the reference (PAPER.md:57-60
    "reduced to O(dt^2 + h)").  The coarse solutions are also pinned to the oracle's dense CN
    (oracle/levyh_oracle.py: symbol_A / symbol_pm, fractional.py:362-405, levy.py:201-205)."""
    import paper_1812_08324_b200 as P
    from oracle import levyh_oracle as O

    def run(n):
        s = P.FracCNSystem(P.power_measure(1, 0.5), 0.0, 0.0, 0.0, n, 1.0 / n)
        s.prepare(P.HConfig(n_min=32, eps1=1e-10), 1e-10)
        u0 = (1 - s.x ** 2) ** 2
        return s, P.run_cn(s, u0, n)

    n_ref = 2048  # N = 4095 interior nodes, 2048 steps (the reference study's N)
    _, ref = run(n_ref)
    ns = (128, 256, 512)  # N = 255 .. 1023
    errs = []
    for n in ns:
        s, u = run(n)
        errs.append(float(np.abs(u - _restrict(ref, n_ref, n)).max()))
        if n <= 256:  # the same solution from the oracle's dense CN
            tA, _ = O.symbol_A(O.nu_power(0.5), s.h, s.N, 2.0, 0.2, O.tail_power(0.5, 2.0))
            Ap = O.toeplitz_dense(O.symbol_pm(tA, 1.0 / n, "plus"))
            Am = O.toeplitz_dense(O.symbol_pm(tA, 1.0 / n, "minus"))
            uo = (1 - s.x ** 2) ** 2
            for _ in range(n):
                uo = np.linalg.solve(Ap, Am @ uo)
            assert np.linalg.norm(u - uo) <= 1e-8 * np.linalg.norm(uo), n
    orders = [np.log(errs[i] / errs[i + 1]) / np.log(2.0) for i in range(len(ns) - 1)]
    import paper_1812_08324_b200 as P
    fitted = P.fit_order(np.asarray(ns, float), errs)  # cli.py:116-118 on the parameter N
    print("joint dt = h: max errors", errs, "orders", orders, "fitted", fitted)
    assert all(0.5 <= o <= 0.8 for o in orders), (errs, orders)
    assert 0.55 <= fitted <= 0.8, (errs, fitted)
