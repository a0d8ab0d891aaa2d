"""Reference-generated fixtures for the matrix-free evaluators (fractional.py:304-361,
:435-477) and the variable-order L-shape assembly (fractional.py:550-622).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_apply.py

Inputs are seeded and rebuilt by the tests (tests/cases.py: apply_inputs), so only the
reference's outputs are stored (tests/golden/apply.npz).
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from levyh import fractional as F  # noqa: E402
from levyh import levy as LV  # noqa: E402
from tests import cases  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    res = {}
    # --- 1D ---------------------------------------------------------------------------
    for name, c in cases.APPLY_1D.items():
        u, far = cases.apply_inputs_1d(c)
        nu = None
        if c["measure"][0] == "cgmy":
            nu = LV.LevyMeasure(density=cases.cgmy_density(*c["measure"][1:]), kind="singular_heavy_tail",
                                symmetric=False)
        cfg = F.FracConfig(s=c["s"], h=c["h"], L=c["L"], L_W=c["L_W"], rho_r=c["rho_r"], far_field=far,
                           tail_mass=c.get("tail"), nu=nu)
        res[f"{name}_out"] = F.frac_apply_1d(u, cfg)
        M = cfg.n_window
        ps = [M, M + cfg.n_main, M + 2 * cfg.n_main]
        res[f"{name}_i1"] = np.array([F.eval_i1(u, p, cfg) for p in ps])
        res[f"{name}_i2"] = np.array([F.eval_i2(u[p], cfg.h * (p - M - cfg.n_main), cfg) for p in ps])
        res[f"{name}_i3"] = np.array([F.eval_i3(u, p, cfg) for p in ps])
        sums = F._window_sums_1d(cfg)
        res[f"{name}_sums"] = np.array([sums["S0"], sums["Sg"], sums["Sd"]])
    # --- 2D ---------------------------------------------------------------------------
    for name, c in cases.APPLY_2D.items():
        u, far = cases.apply_inputs_2d(c)
        cfg = F.FracConfig(s=c["s"], h=c["h"], L=c["L"], L_W=c["L_W"], rho_r=c["rho_r"], far_field=far, dim=2)
        res[f"{name}_out"] = F.frac_apply_2d(u, cfg)
        sums = F._window_sums_2d(cfg)
        res[f"{name}_sums"] = np.array([sums[k] for k in ("S0", "Sgx", "Sgy", "Sdxx", "Sdyy", "Sdxy")])
        res[f"{name}_m2_tail"] = np.array([
            F.windowed_second_moment_radial_2d(lambda r: cfg.nu.density2(r, 0.0), cfg.window),
            F.tail_mass_square_2d(cfg.s, cfg.L_W)])
    # --- variable order ---------------------------------------------------------------
    for name, c in cases.VARIABLE_ORDER.items():
        A, b, pts = F.assemble_variable_order(c["n"], s_field=cases.order_field(c), L_W=c["L_W"], rho_r=c["rho_r"])
        res[f"{name}_A"] = A
        res[f"{name}_b"] = b
        res[f"{name}_pts"] = pts
    pts = F.lshape_grid(12)[0]
    res["lshape12_dist"] = F.lshape_boundary_distance(pts)
    res["lshape12_s"] = F.variable_order_field(pts)
    np.savez_compressed(os.path.join(OUT, "apply.npz"), **res)
    print({k: v.shape for k, v in res.items()})


if __name__ == "__main__":
    main()
