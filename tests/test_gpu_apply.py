"""GPU: the matrix-free evaluators (fractional.py:304-361 frac_apply_1d / eval_i1..i3, :435-477
frac_apply_2d) and the variable-order L-shape assembly (fractional.py:550-622) through the C ABI
(lh_frac_apply_1d / lh_frac_apply_2d / lh_assemble_variable_order) against fixtures the real
reference produced (tests/golden/make_golden_apply.py), against the oracle on larger seeded
inputs, and through size-independent properties at sizes the CPU cannot reach in seconds."""
import os

import numpy as np
import pytest

from oracle import frac_oracle as FO
from oracle import levyh_oracle as O
from tests import cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1812_08324_b200 as P
    return P


@pytest.fixture(scope="module")
def g():
    return cases.load("apply")


def _cfg_1d(P, c, far):
    nu = None
    if c["measure"][0] == "cgmy":
        nu = P.cgmy_measure(*c["measure"][1:])
    return P.FracConfig(s=c["s"], h=c["h"], L=c["L"], L_W=c["L_W"], rho_r=c["rho_r"], far_field=far,
                        tail_mass=c.get("tail"), nu=nu)


# The correlation sums 2M+1 products in a different order than numpy: the error bound is a few
# ulps of sum |u_j kern_j| (which exceeds the result: the compensator cancels most of it).
def _conv_scale(kern, u):
    return np.abs(kern).sum() * np.abs(u).max()


@pytest.mark.parametrize("name", list(cases.APPLY_1D))
def test_frac_apply_1d_vs_reference(P, g, name):
    c = cases.APPLY_1D[name]
    u, far = cases.apply_inputs_1d(c)
    cfg = _cfg_1d(P, c, far)
    out = P.frac_apply_1d(u, cfg)
    ref = g[f"{name}_out"]
    M, K = cfg.n_window, cfg.n_main
    kern = O.window_sums(cfg.nu.density, c["h"], M, c["rho_r"])[0]
    assert out.shape == ref.shape
    assert np.abs(out - ref).max() <= 1e-13 * _conv_scale(kern, u)
    ps = [M, M + K, M + 2 * K]
    i1 = np.array([P.eval_i1(u, p, cfg) for p in ps])
    assert np.abs(i1 - g[f"{name}_i1"]).max() <= 1e-13 * _conv_scale(kern, u)
    i2 = np.array([P.eval_i2(u[p], c["h"] * (p - M - K), cfg) for p in ps])
    i3 = np.array([P.eval_i3(u, p, cfg) for p in ps])
    assert np.allclose(i2, g[f"{name}_i2"], rtol=1e-14, atol=0)
    assert np.allclose(i3, g[f"{name}_i3"], rtol=1e-13, atol=0)
    # eval_i1 + eval_i2 + eval_i3 is the full evaluator at that point (fractional.py:304-361)
    assert np.allclose(i1 + i2 + i3, out[[0, K, 2 * K]], rtol=0, atol=1e-12 * _conv_scale(kern, u))


def test_frac_apply_1d_tabulated_measure(P, g):
    """A measure without a device evaluation spec (e.g. a levyh LevyMeasure: density only) is
    tabulated on the window offsets by the host layer; same result."""
    c = cases.APPLY_1D["ap1_power"]
    u, far = cases.apply_inputs_1d(c)
    nu = P.LevyMeasure(density=P.power_measure(1, c["s"]).density, kind="singular_heavy_tail")
    assert nu.gpu is None
    cfg = P.FracConfig(s=c["s"], h=c["h"], L=c["L"], L_W=c["L_W"], rho_r=c["rho_r"], far_field=far, nu=nu)
    kern = O.window_sums(nu.density, c["h"], cfg.n_window, c["rho_r"])[0]
    assert np.abs(P.frac_apply_1d(u, cfg) - g["ap1_power_out"]).max() <= 1e-13 * _conv_scale(kern, u)


def test_frac_apply_1d_errors(P):
    cfg = P.FracConfig(s=0.5, h=1.0 / 16, L=1.0, L_W=2.0)
    with pytest.raises(ValueError):
        P.frac_apply_1d(np.zeros(10), cfg)
    with pytest.raises(ValueError):
        P.eval_i1(np.zeros(40), 3, cfg)


def test_frac_apply_1d_vs_oracle_mid_size(P):
    """K = 4096, M = 8192 (several tiles and window parts) against the oracle; torch in/out."""
    import torch

    s, h, K = 0.7, 1.0 / 4096, 4096
    cfg = P.FracConfig(s=s, h=h, L=1.0, L_W=2.0, rho_r=0.2)
    M = cfg.n_window
    rng = np.random.default_rng(7)
    x = h * np.arange(-(M + K), M + K + 1)
    u = np.exp(-2 * x * x) + 0.01 * rng.standard_normal(x.shape)
    nu = O.nu_power(s)
    ref, _ = FO.apply_1d(u, nu, h, M, K, 0.2, O.tail_power(s, 2.0), O.second_moment(nu, 0.2))
    out = P.frac_apply_1d(torch.from_numpy(u).cuda(), cfg)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    kern = O.window_sums(nu, h, M, 0.2)[0]
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-13 * _conv_scale(kern, u)


def test_frac_apply_1d_full_size_properties(P):
    """N = 2^18 + 1 main points, 2^19 window offsets per side (1.4e11 multiply-adds): constants are
    annihilated up to the tail mass (out = -c tail), the evaluator is linear, and on functions
    supported in the main grid it equals the negated Toeplitz operator of frac_symbol_1d (the
    stencil form, fractional.py:362-390) applied by FFT."""
    import torch

    s, K = 0.5, 2 ** 17
    h = 1.0 / K
    cfg = P.FracConfig(s=s, h=h, L=1.0, L_W=2.0, rho_r=0.2)
    M, n = cfg.n_window, 2 * K + 1
    tail = P.tail_mass_power_1d(s, 2.0)
    const = torch.full((2 * (M + K) + 1,), 1.5, dtype=torch.float64, device="cuda")
    out = P.frac_apply_1d(const, cfg)
    S0 = float(O.window_sums(O.nu_power(s), h, M, 0.2)[1])
    assert float((out + 1.5 * tail).abs().max()) <= 1e-12 * 1.5 * S0
    gen = torch.Generator(device="cuda").manual_seed(11)
    a = torch.zeros_like(const)
    b = torch.zeros_like(const)
    a[M:M + n] = torch.randn(n, generator=gen, dtype=torch.float64, device="cuda")
    b[M:M + n] = torch.randn(n, generator=gen, dtype=torch.float64, device="cuda")
    oa, ob, oab = P.frac_apply_1d(a, cfg), P.frac_apply_1d(b, cfg), P.frac_apply_1d(2.0 * a - 3.0 * b, cfg)
    scale = float(oa.abs().max())
    assert float((oab - (2.0 * oa - 3.0 * ob)).abs().max()) <= 1e-11 * scale
    m2 = P.windowed_second_moment(cfg.nu, cfg.window)
    tA, _, _, _ = P.frac_symbol_1d(cfg.nu, h, n, 2.0, 0.2, tail, m2)
    # y_i = sum_j t[j - i + n - 1] x_j by a circular convolution of length >= 3n - 2
    L = 1 << int(np.ceil(np.log2(3 * n)))
    y = torch.fft.irfft(torch.fft.rfft(torch.flip(tA, [0]), L) * torch.fft.rfft(a[M:M + n], L), L)[n - 1:2 * n - 1]
    assert float((oa + y).abs().max()) <= 1e-9 * scale


@pytest.mark.parametrize("name", list(cases.APPLY_2D))
def test_frac_apply_2d_vs_reference(P, g, name):
    c = cases.APPLY_2D[name]
    u, far = cases.apply_inputs_2d(c)
    cfg = P.FracConfig(s=c["s"], h=c["h"], L=c["L"], L_W=c["L_W"], rho_r=c["rho_r"], far_field=far, dim=2)
    out = P.frac_apply_2d(u, cfg)
    kern, _ = FO.window_sums_2d(FO.power2(c["s"]), c["h"], cfg.n_window, c["rho_r"])
    assert out.shape == g[f"{name}_out"].shape
    # the reference convolves by FFT (error ~1e-16 * sum|kern| * max|u| * log), the device directly
    assert np.abs(out - g[f"{name}_out"]).max() <= 1e-12 * _conv_scale(kern, u)
    M, K = cfg.n_window, cfg.n_main
    xs = c["h"] * np.arange(-K, K + 1)
    fv = far(xs[:, None], xs[None, :]) if far else 0.0
    m2, tail = g[f"{name}_m2_tail"]
    ref = FO.apply_2d(u, FO.power2(c["s"]), c["h"], M, K, c["rho_r"], tail, m2, fv)
    assert np.abs(out - ref).max() <= 1e-13 * _conv_scale(kern, u)
    with pytest.raises(ValueError):
        P.frac_apply_2d(u[:-1], cfg)


def test_frac_apply_2d_properties(P):
    """65 x 65 main grid under a 129 x 129 window: constants give -c tail; linearity."""
    import torch

    cfg = P.FracConfig(s=0.6, h=1.0 / 32, L=1.0, L_W=2.0, rho_r=0.25, dim=2)
    M, K = cfg.n_window, cfg.n_main
    side = 2 * (M + K) + 1
    tail = P.tail_mass_square_2d(0.6, 2.0)
    out = P.frac_apply_2d(torch.full((side, side), 2.0, dtype=torch.float64, device="cuda"), cfg)
    kern, S = FO.window_sums_2d(FO.power2(0.6), cfg.h, M, 0.25)
    assert float((out + 2.0 * tail).abs().max()) <= 1e-12 * 2.0 * S[0]
    gen = torch.Generator(device="cuda").manual_seed(3)
    a = torch.randn((side, side), generator=gen, dtype=torch.float64, device="cuda")
    b = torch.randn((side, side), generator=gen, dtype=torch.float64, device="cuda")
    oa, ob, oab = P.frac_apply_2d(a, cfg), P.frac_apply_2d(b, cfg), P.frac_apply_2d(a + 0.5 * b, cfg)
    assert float((oab - (oa + 0.5 * ob)).abs().max()) <= 1e-11 * float(oa.abs().max())


@pytest.mark.parametrize("name", list(cases.VARIABLE_ORDER))
def test_assemble_variable_order_vs_reference(P, g, name):
    c = cases.VARIABLE_ORDER[name]
    A, b, pts = P.assemble_variable_order(c["n"], s_field=cases.order_field(c), L_W=c["L_W"], rho_r=c["rho_r"])
    ref = g[f"{name}_A"]
    assert np.array_equal(pts, g[f"{name}_pts"]) and np.array_equal(b, g[f"{name}_b"])
    assert np.array_equal(A == 0.0, ref == 0.0)                       # the same sparsity (short windows)
    off = ~np.eye(len(ref), dtype=bool) & (ref != 0.0)
    assert np.abs(A[off] / ref[off] - 1.0).max() <= 1e-12             # entrywise, off the diagonal
    # the diagonal is -S0 - tail - stencil: a sum over the window, compared at its scale
    assert np.abs(np.diag(A) / np.diag(ref) - 1.0).max() <= 1e-12
    with pytest.raises(ValueError):
        P.assemble_variable_order(c["n"], s_field=lambda p: np.full(len(p), 1.0))
    with pytest.raises(ValueError):
        P.assemble_variable_order(7)


def test_variable_order_device_pipeline(P):
    """cli.frac_lshape_study (cli.py:442-477) end to end on the device: assembly (n = 24, the
    reference's matrix in golden_2d.npz), kmeans2 tree, build_from_dense from the device matrix,
    hlu, solve."""
    import torch

    g2 = dict(np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_2d.npz")))
    A, b, pts = P.assemble_variable_order(24, device=True)
    assert isinstance(A, torch.Tensor) and A.is_cuda
    assert np.array_equal(pts, g2["ls_pts"]) and np.array_equal(b, g2["ls_b"])
    ref = g2["ls_A"]
    assert np.abs(A.cpu().numpy() / ref - 1.0).max() <= 1e-12
    ct = P.build_cluster_tree(pts, leaf_size=32, strategy="kmeans2")
    perm = ct.perm
    idx = torch.from_numpy(np.asarray(perm.inverse)).cuda()
    H = P.build_from_dense(A[idx][:, idx], ct, ct, P.HConfig(n_min=32, eps1=1e-6))
    st, rs = H.structure_array(), g2["ls_struct"]
    assert np.array_equal(st[:, :5], rs[:, :5])
    lr = rs[:, 4] == 1
    diff = st[lr, 5] - rs[lr, 5]
    cases.report_rank_mismatch("lshape24_device_assembly", "build_from_dense", int(lr.sum()), diff)
    assert np.count_nonzero(diff) == 0, diff
    F = P.hlu(H, 1e-10)
    uh = perm.from_tree(P.solve(F, perm.to_tree(b)))
    assert np.linalg.norm(uh - g2["ls_uh"]) <= 1e-9 * np.linalg.norm(g2["ls_uh"])


def test_variable_order_large(P):
    """n = 96 (m = 6912, 193 x 193 window offsets per row, 382 MB matrix): finite, and rows are
    independent, so single rows equal the oracle's recomputation of those rows alone."""
    import torch

    A, b, pts = P.assemble_variable_order(96, device=True)
    assert A.shape == (6912, 6912) and bool(torch.isfinite(A).all())
    small, _, _ = P.assemble_variable_order(8, device=True)
    assert small.shape == (48, 48)
    s = P.variable_order_field(pts)
    rows = [0, 3456, 6911]
    Ao, _ = FO.assemble_vo(96, s, rows=rows)
    for r in rows:
        got, row = A[r].cpu().numpy(), Ao[r]
        nz = row != 0
        assert np.array_equal(got != 0, nz)
        assert np.abs(got[nz] / row[nz] - 1.0).max() <= 1e-12
