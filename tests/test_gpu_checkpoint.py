"""GPU: H-matrix / H-LU checkpoints.  A saved and re-loaded factor (or
operator) is bit-identical to the original: same block structure, same device arrays, same
solves and CN steps, including leaf-128 factors (refined dense leaves); re-factorising a
re-loaded operator reproduces the reference fixtures; foreign / truncated files raise the
reference's ValueError."""
import os

import numpy as np
import pytest

from tests import cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1812_08324_b200 as P
    return P


def _layout_equal(P, A, B):
    ra, aa, ka, pa = P.hmatrix.export_layout(A)
    rb, ab, kb, pb = P.hmatrix.export_layout(B)
    return (np.array_equal(ra, rb) and np.array_equal(aa, ab) and np.array_equal(ka, kb)
            and np.array_equal(pa, pb))


@pytest.mark.parametrize("name", ["cfg1", "cfg2_s025", "cfg5_leaf128"])
def test_factor_roundtrip_bitexact(P, tmp_path, name):
    g = cases.load(name)
    s = cases.make_system(name, g)
    cfg = P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"]))
    Hp, Hm = s.build_pair(cfg)
    F = P.hlu(Hp, float(g["eps2"]))
    fp, mp = str(tmp_path / "factor.lhb"), str(tmp_path / "hminus.lhb")
    P.save_hmatrix(F, fp)
    P.save_hmatrix(Hm, mp)
    F2 = P.load_hmatrix(fp)
    Hm2 = P.load_hmatrix(mp)
    assert isinstance(F2, P.HFactorization) and F2.eps2 == float(g["eps2"])
    assert isinstance(Hm2, P.HMatrix) and not Hm2.factored
    assert np.array_equal(F2.h.structure_array(), F.h.structure_array())
    assert np.array_equal(Hm2.structure_array(), Hm.structure_array())
    assert _layout_equal(P, F.h, F2.h) and _layout_equal(P, Hm, Hm2)
    assert np.array_equal(F2.h.row_tree.points, F.h.row_tree.points)
    assert np.array_equal(F2.h.row_tree.perm.inverse, F.h.row_tree.perm.inverse)
    x = np.random.default_rng(1).standard_normal(Hm.n_cols)
    assert np.array_equal(P.matvec(Hm2, x), P.matvec(Hm, x))
    for method in ("substitution", "inverse", "propagator"):
        assert np.array_equal(P.solve(F2, x, method=method), P.solve(F, x, method=method)), method
    # CN stepping on the re-loaded pair: same result as the original pair, and the fixture's
    u0 = g["u0"]
    for method in ("inverse", "propagator"):
        s.h_minus, s.factor, s.method = Hm, F, method
        u1 = P.run_cn(s, u0, int(g["n_steps"]), method=method)
        s.h_minus, s.factor = Hm2, F2
        u2 = P.run_cn(s, u0, int(g["n_steps"]), method=method)
        assert np.array_equal(u1, u2), method
        assert np.linalg.norm(u2 - g["uT"]) <= 1e-8 * np.linalg.norm(g["uT"])


def test_operator_roundtrip_then_factor(P, tmp_path):
    """An assembled (unfactored) operator saved and re-loaded factorises like the original."""
    g = cases.load("cfg1")
    s = cases.make_system("cfg1", g)
    Hp, _ = s.build_pair(P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"])))
    p = str(tmp_path / "hplus.lhb")
    P.save_hmatrix(Hp, p)
    Hp2 = P.load_hmatrix(p)
    assert _layout_equal(P, Hp, Hp2)
    F, F2 = P.hlu(Hp, 1e-10), P.hlu(Hp2, 1e-10)
    x = np.random.default_rng(2).standard_normal(Hp2.n_rows)
    a, b = P.solve(F, x), P.solve(F2, x)
    assert np.linalg.norm(a - b) <= 1e-14 * np.linalg.norm(a)
    assert np.array_equal(F2.h.structure_array(), g["struct_factor"]) or \
        np.array_equal(F2.h.structure_array()[:, :5], g["struct_factor"][:, :5])


def test_checkpoint_errors(P, tmp_path):
    bad = tmp_path / "bad.lhb"
    bad.write_bytes(b"not a checkpoint at all")
    with pytest.raises(ValueError, match="not a levyh_b200"):
        P.load_hmatrix(str(bad))
    with pytest.raises(FileNotFoundError):
        P.load_hmatrix(str(tmp_path / "missing.lhb"))
    g = cases.load("cfg1")
    s = cases.make_system("cfg1", g)
    Hp, _ = s.build_pair(P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"])))
    p = tmp_path / "h.lhb"
    P.save_hmatrix(Hp, str(p))
    data = p.read_bytes()
    trunc = tmp_path / "trunc.lhb"
    trunc.write_bytes(data[: len(data) // 2])
    with pytest.raises(ValueError, match="truncated or corrupt"):
        P.load_hmatrix(str(trunc))
    with pytest.raises(TypeError):
        P.save_hmatrix(np.eye(3), str(tmp_path / "x.lhb"))
    assert os.path.getsize(p) > 8 * P.memory_report(Hp)["stored_scalars"]
