"""Parity at BASELINE.json's full sizes against exact, independent references:

* the device Toeplitz symbol of the CN operator against the oracle's restatement of the
  reference stencil (fractional.py:285-405 + levy.py:169-206, bit-identical to the reference
  at small N: tests/test_oracle.py) at N = 2^20 - 1 (cfg3, CGMY) and N = 2^22 - 1 (cfg5);
* the H-matvec of A+ / A- against the EXACT Toeplitz product computed by FFT, at the same
  sizes: the compressed operator differs from the exact one only by the ACA truncation at eps1
  (hmatrix.py:294-303), so the relative error must stay within 10 eps1.
"""
import numpy as np
import pytest

from oracle import levyh_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1812_08324_b200 as P
    return P


def toeplitz_fft(t, x):
    """y_i = sum_j t[N - 1 + j - i] x_j as one full convolution (numpy FFT)."""
    N = x.shape[0]
    L = 1 << int(np.ceil(np.log2(3 * N)))
    y = np.fft.irfft(np.fft.rfft(t[::-1], L) * np.fft.rfft(x, L), L)
    return y[N - 1:2 * N - 1]


def _cfg3(P):
    return P.FracCNSystem(P.cgmy_measure(1.0, 5.0, 10.0, 0.5), 0.05, 0.1, -0.05, 2 ** 19, 8.0 / 2 ** 20 * 16,
                          L=4.0, L_W=8.0, drift_compensation=True)


def _cfg5(P):
    n = 2 ** 21
    return P.FracCNSystem(P.power_measure(1, 0.8), 0.1, 0.0, 0.0, n, 1.0 / n)


def _check_symbol(s, nu):
    tA = s.tA.cpu().numpy()
    ref, sc = O.symbol_A(nu, s.h, s.N, s.L_W, s.rho_r, s.tail, s.a, s.b_eff, s.c)
    assert sc["m2"] == s.m2
    N = s.N
    scale = np.abs(ref).max()
    off = np.ones(2 * N - 1, dtype=bool)
    off[N - 2:N + 1] = False  # the diagonal and +-1 carry the window sums S0, Sg, Sd
    # off-band entries are pointwise nu(kh) w_k: GPU pow / exp within a few ulp (measured <= 3 ulp,
    # 6.4e-16 relative at cfg3, 4.2e-16 at cfg5)
    e_off = np.abs(tA[off] - ref[off])
    assert (e_off <= 1e-15 * np.abs(ref[off]) + 1e-300).all(), (e_off / np.maximum(np.abs(ref[off]), 1e-300)).max()
    # band: sums over 2M + 1 offsets in a different order (device tree reduction vs numpy)
    e_band = np.abs(tA[~off] - ref[~off])
    assert (e_band <= 1e-14 * scale).all(), e_band.max() / scale
    # A+- = I +- dt/2 A on the device symbol: off-diagonals exact negatives
    tp, tm = s.tPlus.cpu().numpy(), s.tMinus.cpu().numpy()
    o = np.arange(2 * N - 1) != N - 1
    assert np.array_equal(tp[o], -tm[o])
    return tA


def test_symbol_cfg3_full_size(P):
    s = _cfg3(P)
    _check_symbol(s, O.nu_cgmy(1.0, 5.0, 10.0, 0.5))


def test_symbol_cfg5_full_size(P):
    s = _cfg5(P)
    _check_symbol(s, O.nu_power(0.8))


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_matvec_vs_fft_toeplitz_cfg3(P):
    s = _cfg3(P)
    eps1 = 1e-9
    Hp, Hm = s.build_pair(P.HConfig(n_min=64, eps1=eps1))
    x = np.random.default_rng(7).standard_normal(s.N)
    for H, t in ((Hp, s.tPlus), (Hm, s.tMinus)):
        y = P.matvec(H, x)
        assert _rel(y, toeplitz_fft(t.cpu().numpy(), x)) <= 10 * eps1
    # smooth input (the CN state): same bound
    u = np.maximum(np.exp(s.x) - 1.0, 0.0)
    assert _rel(P.matvec(Hm, u), toeplitz_fft(s.tMinus.cpu().numpy(), u)) <= 10 * eps1


def test_matvec_vs_fft_toeplitz_cfg5(P):
    s = _cfg5(P)
    eps1 = 1e-10
    Hm = s.hmatrix("minus", P.HConfig(n_min=128, eps1=eps1, kcap=12))
    x = np.random.default_rng(8).standard_normal(s.N)
    y = P.matvec(Hm, x)
    assert _rel(y, toeplitz_fft(s.tMinus.cpu().numpy(), x)) <= 10 * eps1
    Hm.release()
