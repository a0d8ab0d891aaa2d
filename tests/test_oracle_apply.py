"""The evaluator / variable-order oracle (oracle/frac_oracle.py) against fixtures the real
reference produced (tests/golden/make_golden_apply.py), and the host-side pieces of the product's
fractional API that need no GPU (L-shape grid, order field, tails, moments, CSV writer)."""
import numpy as np
import pytest

from oracle import frac_oracle as FO
from oracle import levyh_oracle as O
from tests import cases


@pytest.fixture(scope="module")
def g():
    return cases.load("apply")


def _nu_1d(c):
    return cases.cgmy_density(*c["measure"][1:]) if c["measure"][0] == "cgmy" else O.nu_power(c["s"])


@pytest.mark.parametrize("name", list(cases.APPLY_1D))
def test_oracle_apply_1d(g, name):
    c = cases.APPLY_1D[name]
    u, far = cases.apply_inputs_1d(c)
    M, K = int(round(c["L_W"] / c["h"])), int(round(c["L"] / c["h"]))
    nu = _nu_1d(c)
    tail = c.get("tail", None)
    tail = O.tail_power(c["s"], c["L_W"]) if tail is None else tail
    m2 = O.second_moment(nu, c["rho_r"])
    fv = far(c["h"] * np.arange(-K, K + 1)) if far else 0.0
    out, i1 = FO.apply_1d(u, nu, c["h"], M, K, c["rho_r"], tail, m2, fv)
    assert np.array_equal(out, g[f"{name}_out"])          # the same numpy operations: bit-exact
    assert np.allclose(i1[[0, K, 2 * K]], g[f"{name}_i1"], rtol=0, atol=1e-12 * np.abs(i1).max())
    _, S0, Sg, Sd = O.window_sums(nu, c["h"], M, c["rho_r"])
    assert np.array_equal([S0, Sg, Sd], g[f"{name}_sums"])


@pytest.mark.parametrize("name", list(cases.APPLY_2D))
def test_oracle_apply_2d(g, name):
    c = cases.APPLY_2D[name]
    u, far = cases.apply_inputs_2d(c)
    M, K = int(round(c["L_W"] / c["h"])), int(round(c["L"] / c["h"]))
    nu2 = FO.power2(c["s"])
    kern, S = FO.window_sums_2d(nu2, c["h"], M, c["rho_r"])
    assert np.array_equal(S, g[f"{name}_sums"])
    m2 = FO.moment_radial_2d(lambda r: nu2(r, 0.0), c["rho_r"])
    tail = FO.tail_square_2d(c["s"], c["L_W"])
    assert np.array_equal([m2, tail], g[f"{name}_m2_tail"])
    xs = c["h"] * np.arange(-K, K + 1)
    fv = far(xs[:, None], xs[None, :]) if far else 0.0
    out = FO.apply_2d(u, nu2, c["h"], M, K, c["rho_r"], tail, m2, fv)
    ref = g[f"{name}_out"]                                  # the reference convolves by FFT
    assert np.abs(out - ref).max() <= 1e-11 * np.abs(kern).sum() * np.abs(u).max()


@pytest.mark.parametrize("name", list(cases.VARIABLE_ORDER))
def test_oracle_variable_order(g, name):
    c = cases.VARIABLE_ORDER[name]
    pts, _ = FO.lshape_cells(c["n"])
    assert np.array_equal(pts, g[f"{name}_pts"])
    field = cases.order_field(c)
    import paper_1812_08324_b200.fractional as PF
    s = field(pts) if field else PF.variable_order_field(pts)
    A, _ = FO.assemble_vo(c["n"], s, c["L_W"], c["rho_r"])
    assert np.array_equal(A, g[f"{name}_A"])


def test_lshape_host_api(g, tmp_path):
    import paper_1812_08324_b200.fractional as PF

    pts, cells = PF.lshape_grid(12)
    assert pts.shape == (108, 2) and cells.shape == (108, 2)
    assert np.array_equal(PF.lshape_boundary_distance(pts), g["lshape12_dist"])
    assert np.array_equal(PF.variable_order_field(pts), g["lshape12_s"])
    assert np.array_equal(PF.three_bump_source(g["vo8_pts"]), g["vo8_b"])
    with pytest.raises(ValueError):
        PF.lshape_grid(7)
    for name, c in cases.APPLY_2D.items():
        nu = PF.power_measure(2, c["s"])
        m2 = PF.windowed_second_moment_radial_2d(lambda r: nu.density2(r, 0.0), PF.quartic_window(c["rho_r"]))
        assert np.array_equal([m2, PF.tail_mass_square_2d(c["s"], c["L_W"])], g[f"{name}_m2_tail"])
    p = tmp_path / "f.csv"
    PF.write_field_csv(p, pts[:3], [1.0, 2.5, -1e-3], meta=("n=12", "field=test"))
    lines = p.read_text().splitlines()
    assert lines[:3] == ["# n=12", "# field=test", "x,y,value"] and len(lines) == 6
    assert lines[3] == ",".join(f"{v:.17g}" for v in (*pts[0], 1.0))
