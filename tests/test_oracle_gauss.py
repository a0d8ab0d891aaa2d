"""Pin the oracle's restatement of the reference's smooth-measure path (gaussian_measure ->
assemble_cn_1d -> CNSystem.hmatrix via build_from_expansion -> hlu -> CN steps) against
fixtures made by the real reference (tests/golden/make_golden_gauss.py).  CPU only."""
import os

import numpy as np
import pytest

from oracle import levyh_oracle as O

CASES = ["bench", "delta"]


def _load(golden_dir, name):
    return dict(np.load(os.path.join(golden_dir, f"gauss_{name}.npz")))


def _build(g):
    delta = float(g["delta"])
    return O.build_gauss_cn(int(g["n"]), float(g["eps_sq"]), float(g["scale"]), float(g["a"]),
                            float(g["b"]), float(g["c"]), float(g["dt"]), int(g["leaf"]),
                            int(g["fixed_rank"]), None if delta < 0 else delta)


def _lowrank(blk):
    recs, us, vs = [], [], []
    for (b, r0, c0) in O.leaves(blk):
        if b.kind == "R":
            recs.append((r0, c0, b.u.shape[0], b.v.shape[0], b.u.shape[1]))
            us.append(b.u.ravel(order="F"))
            vs.append(b.v.ravel(order="F"))
    return np.array(recs), np.concatenate(us), np.concatenate(vs)


@pytest.mark.parametrize("name", CASES)
def test_symbol_and_series_factors(name, golden_dir):
    g = _load(golden_dir, name)
    x, tA, lam, root, Hp, Hm = _build(g)
    assert lam == float(g["lam"])
    assert np.array_equal(tA, g["symbol"])
    assert np.array_equal(O.structure(Hp), g["struct_plus"])
    recs, u, v = _lowrank(Hp)
    assert np.array_equal(recs, g["lr_recs"])
    # same recurrence, same arithmetic order: bit-exact
    assert np.array_equal(u, g["lr_u"]) and np.array_equal(v, g["lr_v"])


@pytest.mark.parametrize("name", CASES)
def test_matvec_lu_and_steps(name, golden_dir):
    g = _load(golden_dir, name)
    x, tA, lam, root, Hp, Hm = _build(g)
    for H, key in ((Hp, "y_plus"), (Hm, "y_minus")):
        y = O.hmatvec(H, g["x"])
        assert np.linalg.norm(y - g[key]) <= 1e-14 * np.linalg.norm(g[key])
    F = O.hlu(Hp, 1e-10)
    assert np.array_equal(O.structure(F), g["struct_lu"])
    xs = O.lu_solve(F, g["b_solve"])
    assert np.linalg.norm(xs - g["x_solve"]) <= 1e-12 * np.linalg.norm(g["x_solve"])
    uT = O.run_cn(Hm, F, g["u0"], int(g["steps"]))
    assert np.linalg.norm(uT - g["uT"]) <= 1e-12 * np.linalg.norm(g["uT"])


def test_rank_bound_pins():
    # hmatrix.py:270-281 on hand-checked values: e2 = 2 eps^2 D^2
    assert O.series_terms(5.0, 0.5, 10, None) == 10
    assert O.series_terms(5.0, 0.0, 10, 1e-6) == 1
    e2 = 2.0 * 3.0 * 0.25
    expect = int(np.floor(max(e2 / np.log(2.0) - np.log2(1e-6) - 1.0, 6 * e2 - 1.0))) + 1 + 1
    assert O.series_terms(3.0, 0.5, 10, 1e-6) == expect
