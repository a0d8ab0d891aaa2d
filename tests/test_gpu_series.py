"""GPU parity of the reference's smooth-measure path: gaussian_measure ->
assemble_cn_1d -> CNSystem.hmatrix (build_from_expansion with gaussian_expansion_1d) -> hlu ->
CN steps, against fixtures made by the real reference (tests/golden/make_golden_gauss.py),
plus size-independent properties at the reference bench's N = 2^20."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ["bench", "delta"]


@pytest.fixture(scope="module")
def P():
    import paper_1812_08324_b200 as P
    return P


def _load(name):
    return dict(np.load(os.path.join(GOLDEN, f"gauss_{name}.npz")))


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _system(P, g):
    nu = P.gaussian_measure(float(g["eps_sq"]), float(g["scale"]))
    s = P.assemble_cn_1d(nu, float(g["a"]), float(g["b"]), float(g["c"]), P.UniformGrid1D(int(g["n"])),
                         float(g["dt"]))
    delta = float(g["delta"])
    cfg = P.HConfig(n_min=int(g["leaf"]), fixed_rank=int(g["fixed_rank"]),
                    delta=None if delta < 0 else delta)
    return s, cfg


@pytest.mark.parametrize("name", CASES)
def test_symbol(P, name):
    g = _load(name)
    s, _ = _system(P, g)
    assert s.n_off == int(g["n_off"])
    assert abs(s.lam - float(g["lam"])) <= 1e-14 * abs(float(g["lam"]))
    t = s.tA.cpu().numpy()
    assert np.abs(t - g["symbol"]).max() <= 1e-14 * np.abs(g["symbol"]).max()


@pytest.mark.parametrize("name", CASES)
def test_series_build(P, name):
    g = _load(name)
    s, cfg = _system(P, g)
    Hp = s.hmatrix("plus", cfg)
    assert np.array_equal(Hp.structure_array(), g["struct_plus"])  # partition + series ranks
    lr = [(r0, c0, b) for (r0, c0, b) in P.export_blocks(Hp) if isinstance(b, P.hmatrix.LowRank)]
    recs = np.array([(r0, c0, b.u.shape[0], b.v.shape[0], b.u.shape[1]) for r0, c0, b in lr])
    assert np.array_equal(recs, g["lr_recs"])
    u = np.concatenate([b.u.ravel(order="F") for _, _, b in lr])
    v = np.concatenate([b.v.ravel(order="F") for _, _, b in lr])
    # the reference's recurrence on device: exp() may differ from numpy's by an ulp
    assert np.abs(u - g["lr_u"]).max() <= 1e-14 * np.abs(g["lr_u"]).max()
    assert np.abs(v - g["lr_v"]).max() <= 1e-13 * np.abs(g["lr_v"]).max()
    assert _rel(P.matvec(Hp, g["x"]), g["y_plus"]) <= 1e-14
    Hp2, Hm = s.build_pair(cfg)
    assert np.array_equal(Hm.structure_array(), g["struct_plus"])
    assert _rel(P.matvec(Hm, g["x"]), g["y_minus"]) <= 1e-14


@pytest.mark.parametrize("name", CASES)
def test_hlu_solve_and_steps(P, name):
    g = _load(name)
    s, cfg = _system(P, g)
    F = s.prepare(cfg, 1e-10, method="propagator")
    st = F.h.structure_array()
    ref = g["struct_lu"]
    assert np.array_equal(st[:, :5], ref[:, :5])
    lrm = ref[:, 4] == 1
    assert np.abs(st[lrm, 5] - ref[lrm, 5]).max() <= 1
    for method in ("substitution", "inverse", "propagator"):
        assert _rel(P.solve(F, g["b_solve"], method=method), g["x_solve"]) <= 1e-9, method
        uT = P.run_cn(s, g["u0"], int(g["steps"]), method=method)
        assert _rel(uT, g["uT"]) <= 1e-9, method


def test_kernel_dense_leaves_without_entry_fn(P):
    """build_from_expansion without entry_fn fills dense leaves from the expansion kernel."""
    n = 512
    x = np.linspace(-1.0, 1.0, n, endpoint=False)
    ct = P.build_cluster_tree(x[:, None], leaf_size=32)
    ex = P.gaussian_expansion_1d(4.0, scale=0.7)
    H = P.build_from_expansion(ct, ct, ex, P.HConfig(n_min=32))
    for r0, c0, b in P.export_blocks(H):
        if isinstance(b, P.hmatrix.Dense):
            m, k = b.data.shape
            ref = ex.kernel(x[r0:r0 + m, None], x[c0:c0 + k, None])
            assert np.abs(b.data - ref).max() <= 1e-15
        else:
            ctr = 0.5 * (x[r0] + x[r0 + b.u.shape[0] - 1])
            ru = ex.row_factors(x[r0:r0 + b.u.shape[0], None], [ctr], b.u.shape[1])
            rv = ex.col_factors(x[c0:c0 + b.v.shape[0], None], [ctr], b.v.shape[1])
            assert np.abs(b.u - ru).max() <= 1e-14 * np.abs(ru).max()
            assert np.abs(b.v - rv).max() <= 1e-13 * np.abs(rv).max()


def test_errors(P):
    g = _load("bench")
    s, cfg = _system(P, g)
    with pytest.raises(ValueError):
        P.assemble_cn_1d(P.gaussian_measure(5.0), -1.0, 0.0, 0.0, P.UniformGrid1D(64), 0.01)
    ct = s.cluster_tree(cfg.n_min)
    with pytest.raises(TypeError):
        P.build_from_expansion(ct, ct, P.KernelExpansion(None, None, None), cfg)
    with pytest.raises(TypeError):
        P.build_from_expansion(ct, ct, P.gaussian_expansion_1d(5.0), cfg, entry_fn=lambda r, c: 0)
    with pytest.raises(P._lib.NativeError):
        # rank bound above the low-rank capacity (kcap = 32)
        P.build_from_expansion(ct, ct, P.gaussian_expansion_1d(50.0), P.HConfig(n_min=64, delta=1e-12))


def test_bench_system_full_size(P):
    """The reference bench system at N = 2^20 (cli.py:173-177, rank 10, leaf 64): factor
    solves a separately built A+ to the eps2 level; the three solve paths agree; the
    CN step is linear."""
    n = 2 ** 20
    s = P.assemble_cn_1d(P.gaussian_measure(5.0), 0.0, 0.0, 0.0, P.UniformGrid1D(n), 0.01)
    cfg = P.HConfig(n_min=64, fixed_rank=10)
    F = s.prepare(cfg, 1e-10, method="propagator")
    rng = np.random.default_rng(0)
    b = rng.standard_normal(n)
    x_sub = P.solve(F, b, method="substitution")
    assert _rel(P.solve(F, b, method="propagator"), x_sub) <= 1e-9
    Ap = s.hmatrix("plus", cfg)
    assert _rel(P.matvec(Ap, x_sub), b) <= 1e-8
    v, w = rng.standard_normal(n), rng.standard_normal(n)
    lhs = P.run_cn(s, 2.0 * v - 3.0 * w, 2, method="propagator")
    rhs = 2.0 * P.run_cn(s, v, 2, method="propagator") - 3.0 * P.run_cn(s, w, 2, method="propagator")
    assert _rel(lhs, rhs) <= 1e-11
