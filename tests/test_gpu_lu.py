"""GPU parity: H-LU factorisation, substitution / inverse-factor / propagator solves, and
the CN stepping loop against the reference golden fixtures (rel. L2 1e-8,
the BASELINE.json contract) and the oracle."""
import numpy as np
import pytest

from oracle import levyh_oracle as O
from tests import cases

pytestmark = pytest.mark.gpu

NAMES = list(cases.CASES)


@pytest.fixture(scope="module")
def P():
    import paper_1812_08324_b200 as P
    return P


def _factor(P, name, g):
    s = cases.make_system(name, g)
    cfg = P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"]))
    Hp, Hm = s.build_pair(cfg)
    F = P.hlu(Hp, float(g["eps2"]))
    return s, F, Hm


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("name", NAMES)
def test_hlu_solve_substitution(P, name):
    g = cases.load(name)
    s, F, Hm = _factor(P, name, g)
    st = F.h.structure_array()
    ref = g["struct_factor"]
    assert np.array_equal(st[:, :5], ref[:, :5])  # same blocks, leaves LU-factored
    # factor ranks follow the same eps2 recompression (hops.py:124-131): count and report
    # every block whose rank differs from the reference's
    lr = ref[:, 4] == 1
    diff = st[lr, 5] - ref[lr, 5]
    cases.report_rank_mismatch(name, "factor", int(lr.sum()), diff)
    assert np.count_nonzero(diff) == 0, diff
    sol = P.solve(F, g["probe"], method="substitution")
    assert _rel(sol, g["solve_probe"]) <= 1e-9


@pytest.mark.parametrize("name", NAMES)
def test_inverse_solve_matches_substitution(P, name):
    g = cases.load(name)
    s, F, Hm = _factor(P, name, g)
    a = P.solve(F, g["probe"], method="substitution")
    b = P.solve(F, g["probe"], method="inverse")
    assert _rel(b, a) <= 1e-9
    assert _rel(b, g["solve_probe"]) <= 1e-9


def test_hlu_streamed_chunks(P, monkeypatch):
    """H-LU executed in plan chunks while the background planner is still running
    (N = 2^17 - 1, where planning outlasts assembly) gives the same factor as the
    one-DAG run, and solves A+ x = b to the eps2-level residual."""
    n = 1 << 16
    h = 1.0 / n
    x = np.random.default_rng(3).standard_normal(2 * n - 1)

    def factor(stream):
        if stream:
            monkeypatch.setenv("LEVYH_STREAM_MIN_CHUNK", "2000")
            monkeypatch.delenv("LEVYH_NO_STREAM_LU", raising=False)
        else:
            monkeypatch.setenv("LEVYH_NO_STREAM_LU", "1")
        s = P.FracCNSystem(P.power_measure(1, 0.5), 0.0, 0.0, 0.0, n, h)
        cfg = P.HConfig(n_min=64, eps1=1e-10)
        Hp, _ = s.build_pair(cfg)
        F = P.hlu(Hp, 1e-10)
        st = np.zeros(8)
        P._lib.check(P._lib.lib().lh_hlu_stats(F.h.handle, P._lib.host_ptr(st)))
        return s, cfg, F, st

    s, cfg, F1, st1 = factor(True)
    assert st1[4] >= 2, st1  # ran as more than one chunk
    _, _, F0, st0 = factor(False)
    assert st0[4] == 1
    # algorithmic flops / bytes of the factorisation: the same task list both ways; at least the
    # diagonal leaves' LU (2/3 64^3 flops each), at most a dense LU of the whole matrix
    nleaf = s.N // 64
    assert st0[5] > nleaf * (2.0 / 3.0) * 64 ** 3 and st0[5] < (2.0 / 3.0) * float(s.N) ** 3
    assert st0[6] > 8.0 * 2 * nleaf * 64 * 64
    assert abs(st1[5] / st0[5] - 1.0) < 1e-2 and abs(st1[6] / st0[6] - 1.0) < 1e-2
    x1 = P.solve(F1, x, method="substitution")
    x0 = P.solve(F0, x, method="substitution")
    assert _rel(x1, x0) <= 1e-12
    Ap = s.hmatrix("plus", cfg)
    assert _rel(P.matvec(Ap, x1), x) <= 1e-8


@pytest.mark.parametrize("name", NAMES)
def test_propagator_solve(P, name):
    g = cases.load(name)
    s, F, Hm = _factor(P, name, g)
    a = P.solve(F, g["probe"], method="substitution")
    b = P.solve(F, g["probe"], method="propagator")
    assert _rel(b, a) <= 1e-9
    assert _rel(b, g["solve_probe"]) <= 1e-9
    st = F.propagator_stats()
    assert st[0] > 0 and st[3] > 0  # tasks, executor seconds
    assert st[6] in (0.0, 1.0, 2.0) and st[7] <= 1e-10  # single-RHS form of Z and its probe error


def test_propagator_general_hminus(P):
    """cn_steps method 2 with an hminus that is NOT 2I - A+ must run Z (Hm u), not 2Zu - u."""
    g = cases.load("cfg1")
    s, F, Hm = _factor(P, "cfg1", g)
    t = s.tMinus.clone().zero_()
    t[s.N - 1] = 0.5
    Hq = P.derive_toeplitz(Hm, t, lr_scale=0.5, kcap=0)  # 0.5 I + 0.5 (admissible blocks of A-)
    u0 = np.asarray(g["u0"], dtype=float)
    perm = s.tree.perm
    s.h_minus, s.factor, s.method = Hq, F, "propagator"
    u = P.run_cn(s, u0, 3)  # method None: the prepared method (propagator)
    path = np.zeros(4, dtype=np.int32)
    P._lib.check(P._lib.lib().lh_cn_last_path(F.h.handle, P._lib.host_ptr(path)))
    assert list(path[:3]) == [3, 0, 0]  # shape 3: u <- Z (A- u), single RHS
    want = u0
    for _ in range(3):
        want = perm.from_tree(P.solve(F, P.matvec(Hq, perm.to_tree(want)), method="substitution"))
    assert _rel(u, want) <= 1e-9


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("method", ["propagator", "inverse", "substitution"])
def test_cn_end_to_end(P, name, method):
    g = cases.load(name)
    s = cases.make_system(name, g)
    cfg = P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"]))
    s.prepare(cfg, float(g["eps2"]), method=method)
    n_steps = int(g["n_steps"]) if method != "substitution" or name != "cfg1" else 64
    u = P.run_cn(s, g["u0"], n_steps, method=method)
    if n_steps == int(g["n_steps"]):
        assert _rel(u, g["uT"]) <= 1e-8, "solution differs from the reference beyond 1e-8"
    else:
        # shorter run: compare with the oracle composition at the same step count
        tA = g["tA"]
        root, order, Hp, Hm = O.build_cn(tA, float(g["dt"]), g["x"], int(g["leaf"]), float(g["eps1"]))
        Fo = O.hlu(Hp, 1e-10)
        uo = O.run_cn(Hm, Fo, g["u0"], n_steps)
        assert _rel(u, uo) <= 1e-8


@pytest.mark.parametrize("method", ["propagator", "inverse"])
def test_cfg1_golden_pins(P, method):
    g = cases.load("cfg1")
    s = cases.make_system("cfg1", g)
    s.prepare(P.HConfig(n_min=32, eps1=1e-10), 1e-10, method=method)
    u = P.run_cn(s, g["u0"], 512)
    assert abs(np.linalg.norm(u) - 6.179677103303214) <= 1e-8 * 6.18
    assert abs(u[511] - 0.25498164269386925) <= 1e-8


def test_singular_leaf_raises_with_path(P):
    N = 255
    x = (2.0 / (N + 1)) * np.arange(-(N // 2), N // 2 + 1)
    A = np.eye(N) * 4.0
    A[40:48, 40:48] = 0.0  # inside the second leaf of size 32: rows 32..63
    ct = P.build_cluster_tree(x[:, None], leaf_size=32)
    H = P.build_from_dense(A, ct, ct, P.HConfig(n_min=32, eps1=1e-10))
    root, _ = O.cluster_tree(x, 32)
    Ho = O.compress_dense(A, root, 1e-10, 32)
    with pytest.raises(np.linalg.LinAlgError) as ref_exc:
        O.hlu(Ho)
    with pytest.raises(np.linalg.LinAlgError) as exc:
        P.hlu(H)
    assert str(exc.value) == str(ref_exc.value)
    assert "zero pivot in dense diagonal leaf at root." in str(exc.value)


def test_solve_shape_errors(P):
    g = cases.load("cfg1")
    s, F, Hm = _factor(P, "cfg1", g)
    with pytest.raises(ValueError):
        P.solve(F, np.ones(7))
    with pytest.raises(ValueError):
        P.hlu(F.h)  # already factored / consumed


@pytest.mark.parametrize("n,leaf", [(256, 64), (200, 32)])
def test_hlu_leaf_pivoting_dense(P, n, leaf):
    """Leaves that need row exchanges (a random matrix with weak diagonal): the GETRF task's
    pivoted path (the speculative no-exchange pass fails its |a_jj| >= |a_ij| check) gives
    the same solution as LAPACK (rel. 1e-9), for 64- and 32-row leaves.  (Refined 128-row
    leaves pivot within their 64-row halves only; a cross-half pivot raises ValueError with
    the leaf's path.)"""
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n)) + 0.5 * np.eye(n)
    x = np.linspace(-1, 1, n)
    ct = P.build_cluster_tree(x[:, None], leaf_size=leaf)
    H = P.build_from_dense(A, ct, ct, P.HConfig(n_min=leaf, eps1=1e-14))
    F = P.hlu(H, 1e-14)
    b = rng.standard_normal(n)
    want = np.linalg.solve(A, b)
    for method in ("substitution", "inverse", "propagator"):
        got = P.solve(F, b, method=method)
        assert _rel(got, want) <= 1e-9, method
    # the leaf permutations are not all the identity (row exchanges happened)
    recs, arena, ranks, perm = P.hmatrix.export_layout(F.h)
    assert (perm[: n] != np.arange(n) % leaf).any() or (perm != np.sort(perm)).any()


def test_hlu_leaf128_cross_half_pivot_raises(P):
    n = 512
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n)) + 0.5 * np.eye(n)
    ct = P.build_cluster_tree(np.linspace(-1, 1, n)[:, None], leaf_size=128)
    H = P.build_from_dense(A, ct, ct, P.HConfig(n_min=128, eps1=1e-14))
    with pytest.raises(ValueError, match="root"):
        P.hlu(H, 1e-14)


def test_reference_levyh_on_exported_factors(P):
    """The unmodified reference (levyh installed in baseline/_ref) runs hops.matvec / hops.solve
    on GPU-built factors rebuilt as its own block types (oracle/levyh_bridge.py, the bench's
    reference arm) and agrees with the GPU path: checks the bridge and pins the GPU solve to the
    real reference code on identical factors."""
    from oracle import levyh_bridge as LB

    levyh = LB.import_levyh()
    if levyh is None:
        pytest.skip("reference not installed in baseline/_ref")
    g = cases.load("cfg3_cgmy")
    s, F, Hm = _factor(P, "cfg3_cgmy", g)
    leaf = int(g["leaf"])
    Fr = levyh.hops.HFactorization(LB.hmatrix_from_export(levyh, s.x, leaf, *P.hmatrix.export_layout(F.h)), 1e-10)
    Hr = LB.hmatrix_from_export(levyh, s.x, leaf, *P.hmatrix.export_layout(Hm))
    b = np.asarray(g["probe"])[:, 0].copy()
    assert _rel(levyh.hops.matvec(Hr, b), P.matvec(Hm, b)) <= 1e-13
    assert _rel(levyh.hops.solve(Fr, b), P.solve(F, b, method="substitution")) <= 1e-12
    u = np.asarray(g["u0"], dtype=float)
    s.h_minus, s.factor = Hm, F
    F.prepare_propagator()
    s.method = "propagator"
    want = u.copy()
    for _ in range(10):
        want = levyh.hops.solve(Fr, levyh.hops.matvec(Hr, want))
    assert _rel(P.run_cn(s, u, 10), want) <= 1e-9


@pytest.mark.parametrize("name", ["cfg3_cgmy_n8191", "cfg5_leaf128"])
def test_propagator_column_parts_path(P, name, monkeypatch):
    """The large-N propagator path (N = 2^22: the DAG's column parts run one after another into a
    scratch buffer, each part packed at capacity max(rank, 1); the factor is compacted first and
    the plans still to run re-pointed), forced at fixture size: same Z action, same CN solution
    (reference fixture, rel. L2 1e-8), and substitution solves on the compacted factor still
    match the reference."""
    monkeypatch.setenv("LEVYH_PROP_PARTS_GB", "0")
    g = cases.load(name)
    s, F, Hm = _factor(P, name, g)
    b = P.solve(F, g["probe"], method="propagator")
    assert _rel(b, g["solve_probe"]) <= 1e-9
    a = P.solve(F, g["probe"], method="substitution")  # plans re-cut on the compacted factor
    assert _rel(a, g["solve_probe"]) <= 1e-9
    monkeypatch.delenv("LEVYH_PROP_PARTS_GB")
    s2, F2, Hm2 = _factor(P, name, g)
    b2 = P.solve(F2, g["probe"], method="propagator")
    assert _rel(b, b2) <= 1e-12, "part-by-part propagator differs from the merged DAG"
    s.h_minus, s.factor, s.method = Hm, F, "propagator"
    u = P.run_cn(s, g["u0"], int(g["n_steps"]))
    assert _rel(u, g["uT"]) <= 1e-8


def test_levyh_style_run_cn_takes_the_two_kernel_step(P):
    """prepare() -> run_cn(sys, u0, n) with defaults (levy.py:241-330 call pattern) steps with the
    propagator in nested-basis form: the captured step graph is the two persistent kernels
    (h2step.cu K1 + K2, the state kept in the staging copy between steps), and the result is
    the reference's."""
    g = cases.load("cfg3_cgmy_n8191")
    s = cases.make_system("cfg3_cgmy_n8191", g)
    s.prepare(P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"])), float(g["eps2"]))
    u = P.run_cn(s, g["u0"], int(g["n_steps"]))
    assert _rel(u, g["uT"]) <= 1e-8
    st = s.factor.propagator_stats()
    assert st[6] == 2.0, "nested-basis (H2) form not installed"
    path = np.zeros(4, dtype=np.int32)
    P._lib.check(P._lib.lib().lh_cn_last_path(s.factor.h.handle, P._lib.host_ptr(path)))
    assert list(path[:3]) == [2, 0, 0]  # u <- 2 Z u - u, single RHS, device-resident
    assert int(P._lib.lib().lh_step_graph_kernels(s.factor.h.handle)) == 2


def test_row_walk_one_cta_per_subtree_equals_one_per_sm(P, monkeypatch):
    """K2 of the two-kernel step cuts its chunk lists per row subtree (two CTAs per SM, 32 KB
    slots) when there are between one and two subtrees per SM, and per SM otherwise: the same
    arithmetic in the same order, so both cuttings give the same step (and the reference's)."""
    n = 2 ** 15
    h = 1.0 / n
    outs = []
    for one_per_sm in (False, True):
        if one_per_sm:
            monkeypatch.setenv("LEVYH_H2S_ONE_PER_SM", "1")
        else:
            monkeypatch.delenv("LEVYH_H2S_ONE_PER_SM", raising=False)
        s = P.FracCNSystem(P.power_measure(1, 0.25), 0.5, 1.0, -1.0, n, h)   # cfg2 at N = 2^16 - 1
        s.prepare(P.HConfig(n_min=64, eps1=1e-10), 1e-10)
        assert s.factor.propagator_stats()[6] == 2.0                           # 256 row subtrees
        u0 = np.maximum(1.0 - s.x ** 2, 0.0) ** 3
        outs.append(P.run_cn(s, u0, 25))
        assert int(P._lib.lib().lh_step_graph_kernels(s.factor.h.handle)) == 2
        if not one_per_sm:
            ref = u0
            perm = s.tree.perm
            for _ in range(3):
                ref = perm.from_tree(P.solve(s.factor, P.matvec(s.h_minus, perm.to_tree(ref)), method="substitution"))
            assert _rel(P.run_cn(s, u0, 3), ref) <= 1e-9
    assert _rel(outs[0], outs[1]) <= 1e-13


def test_default_solve_builds_the_propagator_after_a_few_calls(P):
    """hops.solve(F, b) with default arguments: the reference's substitution for the first calls,
    then (fifth call on the same factor) the propagator is built once and used from there on;
    every answer stays within 1e-9 of the substitution solve; auto_prepare = False keeps
    substitution."""
    g = cases.load("cfg1")
    s, F, Hm = _factor(P, "cfg1", g)
    ref = P.solve(F, g["probe"], method="substitution")
    for k in range(6):
        x = P.solve(F, g["probe"])
        assert _rel(x, ref) <= 1e-9
        assert F.propagator_ready == (k >= P.hops.AUTO_PROPAGATOR_AFTER)
    x, log = P.gmres_restarted(s.hmatrix("plus", P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"]))), F,
                               g["probe"][:, 0], tol=1e-10, restart=20, max_iter=40)
    assert log.converged and log.iterations <= 3      # preconditioned by the prepared propagator
    s2, F2, _ = _factor(P, "cfg1", g)
    F2.auto_prepare = False
    for k in range(6):
        assert _rel(P.solve(F2, g["probe"]), ref) <= 1e-12
    assert not F2.propagator_ready
