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
