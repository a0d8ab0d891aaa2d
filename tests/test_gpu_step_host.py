"""GPU: the reference-facing CN step on HOST vectors (levy.step_cn, levy.py:295-306) through
lh_cn_step_host.  Pinned buffers take the pipelined graph (u streams in / out in pieces
overlapped with the kernels); it must give exactly the device-resident step's result; numpy
vectors take the copy-in / step / copy-out path; both match the reference fixtures over the
full step counts (rel. L2 1e-8)."""
import numpy as np
import pytest

from tests import cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1812_08324_b200 as P
    return P


@pytest.mark.parametrize("name", ["cfg1", "cfg2_s075", "cfg3_cgmy"])
@pytest.mark.parametrize("method", ["propagator", "inverse"])
def test_step_host_matches_device_steps(P, name, method):
    import torch

    g = cases.load(name)
    s = cases.make_system(name, g)
    s.prepare(P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"])), float(g["eps2"]), method=method)
    n_steps = int(g["n_steps"])
    u_dev = P.run_cn(s, g["u0"], n_steps, method=method)
    # pinned torch host vector: pipelined path (method propagator)
    u = torch.from_numpy(g["u0"].copy()).pin_memory()
    for _ in range(n_steps):
        u = P.step_cn(s, u, method=method)
    assert u.is_pinned()
    assert np.array_equal(u.numpy(), u_dev), "host-buffer step differs from the device step"
    # numpy vector: copy-in / step / copy-out
    v = g["u0"].copy()
    for _ in range(min(n_steps, 20)):
        v = P.step_cn(s, v, method=method)
    w = P.run_cn(s, g["u0"], min(n_steps, 20), method=method)
    assert np.array_equal(v, w)
    assert np.linalg.norm(u.numpy() - g["uT"]) <= 1e-8 * np.linalg.norm(g["uT"])


def test_step_host_in_place_and_errors(P):
    import torch

    g = cases.load("cfg1")
    s = cases.make_system("cfg1", g)
    s.prepare(P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"])), 1e-10, method="propagator")
    L = P._lib.lib()
    u = torch.from_numpy(g["u0"].copy()).pin_memory()
    ref = P.run_cn(s, g["u0"], 3, method="propagator")
    for _ in range(3):  # u_out == u_in
        P._lib.check(L.lh_cn_step_host(s.h_minus.ctx.h, s.h_minus.handle, s.factor.h.handle,
                                       u.data_ptr(), u.data_ptr(), 2), s.h_minus.ctx.h)
    assert np.array_equal(u.numpy(), ref)
    with pytest.raises(ValueError):
        P.step_cn(s, np.ones(s.N + 1))
    with pytest.raises(ValueError):
        P.step_cn(s, torch.ones(s.N, dtype=torch.float64).cuda())


def test_spilled_minus_steps_and_restores(P):
    """prepare(spill_minus=True): A- of the CN pair lives in pinned host memory while the
    propagator step u <- 2 Z u - u runs (it never reads A-); the fixture's CN solution is
    unchanged, and the first call that reads A- (matvec) brings it back bit-identically."""
    g = cases.load("cfg2_s075")
    s = cases.make_system("cfg2_s075", g)
    s.prepare(P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"])), float(g["eps2"]), spill_minus=True)
    assert not s.h_minus.resident
    n_steps = int(g["n_steps"])
    u = P.run_cn(s, g["u0"], n_steps)
    assert not s.h_minus.resident, "the CN-pair propagator step read the spilled A-"
    assert np.linalg.norm(u - g["uT"]) <= 1e-8 * np.linalg.norm(g["uT"])
    x = np.random.default_rng(3).standard_normal(s.N)
    y = P.matvec(s.h_minus, x)
    assert s.h_minus.resident
    t = cases.make_system("cfg2_s075", g)
    Hp, Hm = t.build_pair(P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"])))
    assert np.array_equal(y, P.matvec(Hm, x))
    with pytest.raises(ValueError):
        s.factor.h.spill()  # factored: refused
