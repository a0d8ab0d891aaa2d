"""GPU parity of the Krylov consumers: pcg / gmres_restarted
(solvers.py:46-153) run in csrc/krylov.cu with the GPU dense matvec, H-matvec and H-LU solve
as operators, against fixtures made by the real reference (tests/golden/krylov.npz,
tests/golden/make_golden_krylov.py) and the numpy oracle; plus properties at N = 2^16 and the
reference's exception behaviour.

Tolerances: dense-operator runs follow the reference's arithmetic up to summation order, so
iteration counts are equal and residual histories agree to 1e-6 relative.  Runs
preconditioned by the coarse (eps1 = 0.1) H-LU use the GPU's ACA-compressed factors, whose
rank-1 blocks differ from the reference's SVD truncation at the ACA tolerance (1e-4
relative): iteration counts equal, solutions within 1e-7, histories within 5e-2."""
import numpy as np
import pytest

from tests.cases import krylov_operators

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1812_08324_b200 as P
    return P


@pytest.fixture(scope="module")
def G(golden_dir):
    return dict(np.load(f"{golden_dir}/krylov.npz"))


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _check(G, tag, x, log, res_rtol, x_rtol):
    assert log.iterations == int(G[f"{tag}_iters"])
    assert log.converged == bool(G[f"{tag}_conv"])
    assert len(log.residuals) == log.iterations
    np.testing.assert_allclose(log.residuals, G[f"{tag}_res"], rtol=res_rtol, atol=1e-14)
    assert _rel(x, G[f"{tag}_x"]) <= x_rtol


@pytest.mark.parametrize("n", [64, 128])
def test_pcg_poisson_dense(P, G, n):
    """cli.frac_poisson1d_study's solve: pcg(A, None, ones, tol=1e-12, max_iter=10 N)."""
    A, x = krylov_operators(f"poisson{n}")
    u, log = P.pcg(A, None, np.ones_like(x), tol=1e-12, max_iter=10 * A.shape[0])
    assert isinstance(u, np.ndarray)
    _check(G, f"poisson{n}", u, log, 1e-6, 1e-10)


def test_pcg_poisson_hmatrix_operator(P, G):
    """Same solve with the operator as a GPU H-matrix (eps1 = 1e-12): same iterations."""
    A, x = krylov_operators("poisson128")
    ct = P.build_cluster_tree(x[:, None], leaf_size=32)
    H = P.build_from_dense(A, ct, ct, P.HConfig(n_min=32, eps1=1e-12))
    u, log = P.pcg(H, None, np.ones_like(x), tol=1e-12, max_iter=10 * A.shape[0])
    assert abs(log.iterations - int(G["poisson128_iters"])) <= 1 and log.converged
    assert _rel(u, G["poisson128_x"]) <= 1e-9


def _coarse_factor(P, G, tag, A, x):
    ct = P.build_cluster_tree(x[:, None], leaf_size=32)
    H = P.build_from_dense(A, ct, ct, P.HConfig(n_min=32, eps1=1e-1))
    assert np.array_equal(H.structure_array(), G[f"{tag}_struct"])  # partition + ranks
    return P.hlu(H, 1e-10)


def test_pcg_hlu_preconditioned(P, G):
    A, x = krylov_operators("pcg_hlu")
    F = _coarse_factor(P, G, "pcg_hlu", A, x)
    b = np.exp(-50 * x ** 2)
    u, log = P.pcg(A, F, b, tol=1e-10, max_iter=200)
    _check(G, "pcg_hlu", u, log, 5e-2, 1e-7)
    assert _rel(A @ u, b) <= 1e-10


def test_gmres_hlu_preconditioned(P, G):
    """cli.frac_lshape_study's pattern: exact operator, right preconditioner solve(F, .)."""
    A, x = krylov_operators("gmres_hlu")
    F = _coarse_factor(P, G, "gmres_hlu", A, x)
    b = np.exp(-50 * x ** 2)
    for method in ("substitution", "inverse", "propagator"):
        u, log = P.gmres_restarted(A, P.operator(F, method), b, tol=1e-10, restart=50, max_iter=400)
        _check(G, "gmres_hlu", u, log, 5e-2, 1e-7)
        assert _rel(A @ u, b) <= 1e-10


@pytest.mark.parametrize("tag,restart,tol", [("gmres_raw", 20, 1e-10), ("gmres_r5", 5, 1e-12)])
def test_gmres_restarts_dense(P, G, tag, restart, tol):
    """Unconverged runs across several restart cycles: same history, converged=False."""
    A, x = krylov_operators(tag)
    b = np.exp(-50 * x ** 2)
    u, log = P.gmres_restarted(A, None, b, tol=tol, restart=restart, max_iter=60)
    _check(G, tag, u, log, 1e-6, 1e-8)


def test_callable_operators_on_device(P, G):
    """Callables get torch CUDA vectors (solvers.py:39-41); results equal the dense path."""
    import torch

    A, x = krylov_operators("gmres_raw")
    At = torch.from_numpy(A).cuda()
    b = np.exp(-50 * x ** 2)
    calls = []

    def apply(v):
        calls.append(v.device.type)
        return At @ v

    u, log = P.gmres_restarted(apply, None, torch.from_numpy(b).cuda(), tol=1e-10, restart=20,
                               max_iter=60)
    assert isinstance(u, torch.Tensor) and u.is_cuda
    assert set(calls) == {"cuda"}
    _check(G, "gmres_raw", u.cpu().numpy(), log, 1e-6, 1e-8)


def test_errors_and_edge_cases(P):
    import torch

    with pytest.raises(np.linalg.LinAlgError, match="not positive definite"):
        P.pcg(-np.eye(8), None, np.ones(8))
    for solver in (P.pcg, P.gmres_restarted):
        u, log = solver(np.eye(5), None, np.zeros(5))
        assert log.converged and log.residuals == [] and log.iterations == 0 and not u.any()
        with pytest.raises(ValueError):
            solver(np.eye(5), None, np.ones(6))
        with pytest.raises(ValueError):
            solver(np.eye(5), None, np.ones((5, 2)))

        def bad(v):
            raise KeyError("user operator failed")

        with pytest.raises(KeyError, match="user operator failed"):
            solver(bad, None, np.ones(5))
    # max_iter = 0: nothing runs, not converged (solvers.py:108 loop guard)
    u, log = P.gmres_restarted(np.eye(5), None, np.ones(5), max_iter=0)
    assert not log.converged and log.iterations == 0
    u, log = P.pcg(torch.eye(3, dtype=torch.float64).cuda() * 2, None, np.ones(3))
    assert np.allclose(u, 0.5) and log.converged


def test_oracle_agreement_fullsize_cn(P):
    """N = 2^16 - 1 (cfg2 size, s = 0.25, a = .5, b = 1, c = -1): GMRES on the H-matrix A+
    preconditioned by its H-LU, and CG on the SPD CN matrix of the s = 0.5 operator; the
    solutions satisfy the system to the requested tolerance (checked with an independent
    H-matvec) and agree with the direct H-LU solve."""
    n = 2 ** 15
    cfg = P.HConfig(n_min=64, eps1=1e-10)
    sys_ = P.FracCNSystem(P.power_measure(1, 0.25), 0.5, 1.0, -1.0, n, 1.0 / n)
    Hp, _ = sys_.build_pair(cfg)
    Hp2 = Hp.clone()
    F = P.hlu(Hp, 1e-10)
    b = np.exp(-50 * sys_.x ** 2)
    u, log = P.gmres_restarted(Hp2, F, b, tol=1e-12, restart=50, max_iter=50)
    assert log.converged and log.iterations <= 3
    assert _rel(P.matvec(Hp2, u), b) <= 1e-11
    assert _rel(u, P.solve(F, b)) <= 1e-10

    sym = P.FracCNSystem(P.power_measure(1, 0.5), 0.0, 0.0, 0.0, n, 1.0 / n)
    Sp, _ = sym.build_pair(cfg)
    u, log = P.pcg(Sp, None, b, tol=1e-12, max_iter=500)
    assert log.converged
    assert _rel(P.matvec(Sp, u), b) <= 1e-11
    assert all(np.diff(log.residuals[:3]) < 0)
