"""Oracle pin for the Krylov consumers (CPU): the numpy restatement of levyh.solvers
(oracle.levyh_oracle.pcg / gmres_restarted, solvers.py:46-153) reproduces the residual
histories and solutions the REAL reference produced (tests/golden/krylov.npz, made by
tests/golden/make_golden_krylov.py) on the same operators."""
import numpy as np
import pytest

from oracle import levyh_oracle as O
from tests.cases import krylov_operators

G = None


def golden(golden_dir):
    global G
    if G is None:
        G = dict(np.load(f"{golden_dir}/krylov.npz"))
    return G


def _check(g, tag, x, hist, conv, rtol_res=1e-9):
    assert len(hist) == int(g[f"{tag}_iters"])
    assert int(conv) == int(g[f"{tag}_conv"])
    np.testing.assert_allclose(hist, g[f"{tag}_res"], rtol=rtol_res, atol=1e-15)
    ref = g[f"{tag}_x"]
    assert np.linalg.norm(x - ref) <= 1e-10 * np.linalg.norm(ref)


def test_oracle_pcg_poisson(golden_dir):
    g = golden(golden_dir)
    for n in (64, 128):
        A, x = krylov_operators(f"poisson{n}")
        u, hist, conv = O.pcg(A, None, np.ones_like(x), tol=1e-12, max_iter=10 * A.shape[0])
        _check(g, f"poisson{n}", u, hist, conv)


def test_oracle_pcg_and_gmres_hlu(golden_dir):
    g = golden(golden_dir)
    for tag in ("pcg_hlu", "gmres_hlu"):
        A, x = krylov_operators(tag)
        root, _ = O.cluster_tree(x[:, None], 32)
        H = O.compress_dense(A, root, 1e-1, n_min=32)
        assert np.array_equal(O.structure(H), g[f"{tag}_struct"])
        Fc = O.hlu(H, 1e-10)
        b = np.exp(-50 * x ** 2)
        if tag == "pcg_hlu":
            u, hist, conv = O.pcg(A, lambda v: O.lu_solve(Fc, v), b, tol=1e-10, max_iter=200)
        else:
            u, hist, conv = O.gmres_restarted(lambda v: A @ v, lambda v: O.lu_solve(Fc, v), b,
                                              tol=1e-10, restart=50, max_iter=400)
        _check(g, tag, u, hist, conv, rtol_res=1e-7)


def test_oracle_gmres_restarts(golden_dir):
    g = golden(golden_dir)
    A, x = krylov_operators("gmres_raw")
    b = np.exp(-50 * x ** 2)
    u, hist, conv = O.gmres_restarted(lambda v: A @ v, None, b, tol=1e-10, restart=20, max_iter=60)
    _check(g, "gmres_raw", u, hist, conv, rtol_res=1e-8)
    Ap, _ = krylov_operators("gmres_r5")
    u, hist, conv = O.gmres_restarted(Ap, None, b, tol=1e-12, restart=5, max_iter=60)
    _check(g, "gmres_r5", u, hist, conv, rtol_res=1e-8)


def test_oracle_breakdown_and_zero_rhs():
    A = -np.eye(4)
    with pytest.raises(np.linalg.LinAlgError, match="not positive definite"):
        O.pcg(A, None, np.ones(4))
    x, hist, conv = O.pcg(np.eye(3), None, np.zeros(3))
    assert conv and hist == [] and not x.any()
    x, hist, conv = O.gmres_restarted(np.eye(3), None, np.zeros(3))
    assert conv and hist == [] and not x.any()


def test_iteration_log_csv(tmp_path):
    """IterationLog.write_csv keeps the reference's format (solvers.py:30-37)."""
    from paper_1812_08324_b200.solvers import IterationLog

    log = IterationLog(residuals=[0.5, 0.25, 1e-9], iterations=3, converged=True, seconds=1.25)
    p = tmp_path / "log.csv"
    log.write_csv(p)
    assert p.read_text() == ("iter,relative_residual,seconds\n1,0.5,\n2,0.25,\n"
                             "3,1.0000000000000001e-09,1.25\n")
