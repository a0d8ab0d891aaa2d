"""Generate golden fixtures by running the REAL reference package.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/*.npz.  Every number comes from the reference's own
public functions (levyh.fractional / geometry / hmatrix / hops); the
composition of the singular CN operator follows SURVEY.md 8(c) (G2-G5).
The tests pin oracle/levyh_oracle.py against these files, and the GPU
parity tests use them as known answers.  Nothing here runs on the GPU box.
"""

from __future__ import annotations

import hashlib
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from levyh import fractional as F  # noqa: E402
from levyh import geometry as G  # noqa: E402
from levyh import hmatrix as HM  # noqa: E402
from levyh import hops as HO  # noqa: E402
from levyh import levy as LV  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def struct_array(H):
    kinds = {"dense": 0, "lowrank": 1, "dense_lu": 2}
    return np.array([(d["row0"], d["row1"], d["col0"], d["col1"], kinds[d["kind"]], d.get("rank", -1))
                     for d in HM.structure_summary(H)], dtype=np.int64).reshape(-1, 6)


def composed_A(stencil_weights, h, a, b_eff, c):
    """A = -W_int, then the local band with levy._entries_a_1d's rules."""
    A = -stencil_weights[1:-1, 1:-1]
    n = A.shape[0]
    i = np.arange(n)
    A[i, i] += 2 * a / h ** 2 - c
    A[i[:-1], i[:-1] + 1] += -a / h ** 2 - b_eff / (2 * h)
    A[i[1:], i[1:] - 1] += -a / h ** 2 + b_eff / (2 * h)
    return A


def cgmy_density(C, Gc, Mc, Y):
    def f(y):
        y = np.asarray(y, dtype=float)
        ay = np.abs(y)
        with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
            rate = np.where(y < 0, Gc, Mc)
            return C * np.exp(-rate * ay) * ay ** (-1.0 - Y)
    return f


def drift_beta(nu, rho_r):
    from scipy.integrate import quad
    win = F.quartic_window(rho_r)

    def g(y):
        return float((win(y) - 1.0) * y * nu(np.array(y)))
    return (quad(g, 0.0, 1.0, limit=400, epsabs=0.0, epsrel=1e-13, points=[rho_r])[0]
            + quad(g, -1.0, 0.0, limit=400, epsabs=0.0, epsrel=1e-13, points=[-rho_r])[0])


def cn_case(name, cfg, a, b_eff, c, dt, leaf, eps1, u0_fn, n_steps, eps2=1e-10, nrhs_probe=3):
    st = F.frac_stencil_1d(cfg)
    h = cfg.h
    A = composed_A(st.weights, h, a, b_eff, c)
    x = st.x[1:-1]
    N = A.shape[0]
    eye = np.eye(N)
    Ap = eye + 0.5 * dt * A
    Am = eye - 0.5 * dt * A
    ct = G.build_cluster_tree(x[:, None], leaf_size=leaf)
    assert np.array_equal(ct.perm.inverse, np.arange(N))
    hc = HM.HConfig(n_min=leaf, n_block=4, eta=1.0, eps1=eps1)
    Hp = HM.build_from_dense(Ap, ct, ct, hc)
    Hm = HM.build_from_dense(Am, ct, ct, hc)
    sp, sm = struct_array(Hp), struct_array(Hm)
    mem = HM.memory_report(Hp)
    rng = np.random.default_rng(1234)
    probe = rng.standard_normal((N, nrhs_probe))
    mv = np.stack([HO.matvec(Hp, probe[:, k]) for k in range(nrhs_probe)], axis=1)
    mvm = np.stack([HO.matvec(Hm, probe[:, k]) for k in range(nrhs_probe)], axis=1)
    F_ = HO.hlu(Hp, eps2)
    sf = struct_array(F_.h)
    sol = HO.solve(F_, probe)
    u0 = u0_fn(x)
    u = u0.copy()
    for _ in range(n_steps):
        u = HO.solve(F_, HO.matvec(Hm, u))
    # dense CN for the record
    import scipy.linalg as sla
    lu = sla.lu_factor(Ap)
    ud = u0.copy()
    for _ in range(n_steps):
        ud = sla.lu_solve(lu, Am @ ud)
    # the symbol, read back from the dense matrix (first row / first column)
    tA = np.concatenate([A[::-1, 0][:-1], A[0, :]])
    out = dict(N=N, h=h, dt=dt, a=a, b_eff=b_eff, c=c, leaf=leaf, eps1=eps1, eps2=eps2,
               n_steps=n_steps, x=x, tA=tA, struct_plus=sp, struct_minus=sm,
               struct_factor=sf, stored_scalars=mem["stored_scalars"], probe=probe,
               matvec_plus=mv, matvec_minus=mvm, solve_probe=sol, u0=u0, uT=u,
               uT_dense=ud, rel_h_vs_dense=np.linalg.norm(u - ud) / np.linalg.norm(ud))
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(name, N, sp.shape[0], "blocks", mem, "rel H vs dense", out["rel_h_vs_dense"])
    return out


def main():
    # --- config 1 (BASELINE.json configs[0]) -----------------------------------
    s = 0.5
    n = 512
    h = 1.0 / n
    cfg = F.FracConfig(s=s, h=h, L=1.0, L_W=2.0, rho_r=0.2)
    sums = F._window_sums_1d(cfg)
    m2 = F.windowed_second_moment(cfg.nu, cfg.window)
    out = cn_case("cfg1", cfg, 0.0, 0.0, 0.0, h, 32, 1e-10,
                  lambda x: (1 - x ** 2) ** 2, 512)
    np.savez_compressed(os.path.join(OUT, "cfg1_scalars.npz"), S0=sums["S0"], Sg=sums["Sg"],
                        Sd=sums["Sd"], m2=m2, tail=F.tail_mass_power_1d(s, 2.0),
                        M=cfg.n_window, c_half=F.frac_kernel_constant(1, 0.5),
                        c2_half=F.frac_kernel_constant(2, 0.5))

    # --- config 2 style (s in {0.25, 0.75}, a,b,c local terms), reduced N -------
    for s2, tag in ((0.25, "cfg2_s025"), (0.75, "cfg2_s075")):
        n = 1024
        h = 1.0 / n
        cfg = F.FracConfig(s=s2, h=h, L=1.0, L_W=2.0, rho_r=0.2)
        cn_case(tag, cfg, 0.5, 1.0, -1.0, h, 64, 1e-10, lambda x: np.exp(-50 * x ** 2), 20)

    # --- config 3 style (CGMY on [-4,4], drift compensation), reduced N ---------
    nu = cgmy_density(1.0, 5.0, 10.0, 0.5)
    from scipy.integrate import quad
    tail = (quad(lambda y: nu(np.array(y)), 8, np.inf, epsabs=0, epsrel=1e-12)[0]
            + quad(lambda y: nu(np.array(-y)), 8, np.inf, epsabs=0, epsrel=1e-12)[0])
    beta = drift_beta(nu, 0.2)
    n = 512
    h = 4.0 / n
    meas = LV.LevyMeasure(density=nu, kind="singular_heavy_tail", symmetric=False)
    cfg = F.FracConfig(s=0.25, h=h, L=4.0, L_W=8.0, rho_r=0.2, nu=meas, tail_mass=tail)
    o3 = cn_case("cfg3_cgmy", cfg, 0.05, 0.1 + beta, -0.05, 16 * h, 64, 1e-9,
                 lambda x: np.maximum(np.exp(x) - 1.0, 0.0), 10)
    np.savez_compressed(os.path.join(OUT, "cfg3_scalars.npz"), beta=beta, tail=tail)

    # --- config 5 style (s=0.8, a=0.1) -------------------------------------------
    n = 512
    h = 1.0 / n
    cfg = F.FracConfig(s=0.8, h=h, L=1.0, L_W=2.0, rho_r=0.2)
    cn_case("cfg5_s08", cfg, 0.1, 0.0, 0.0, h, 32, 1e-10,
            lambda x: np.maximum(1 - x ** 2, 0.0) ** 3, 10)

    # --- SPEC pins ---------------------------------------------
    rng = np.random.default_rng(7)
    m_, n_ = 40, 30
    A = HM.LowRank(rng.standard_normal((m_, 5)), rng.standard_normal((n_, 5)))
    negA = HO.lowrank_add_recompress(A, HM.LowRank(-A.u, A.v), 1e-10)
    dbl = HO.lowrank_add_recompress(A, A, 1e-10)
    B1 = HM.LowRank(rng.standard_normal((m_, 2)), rng.standard_normal((n_, 2)))
    B2 = HM.LowRank(rng.standard_normal((m_, 2)), rng.standard_normal((n_, 2)))
    disj = HO.lowrank_add_recompress(B1, B2, 1e-12)
    np.savez_compressed(os.path.join(OUT, "spec_lowrank.npz"), Au=A.u, Av=A.v,
                        B1u=B1.u, B1v=B1.v, B2u=B2.u, B2v=B2.v,
                        rank_neg=negA.rank, rank_dbl=dbl.rank, rank_disj=disj.rank,
                        dense_neg=negA.u @ negA.v.T, dense_dbl=dbl.u @ dbl.v.T)
    print("spec ranks A-A", negA.rank, "A+A", dbl.rank, "disjoint", disj.rank)

    # --- partition pins at the full config sizes (cheap expansion builder) ------
    parts = {}
    for tag, N, leaf, lo, hi in (("cfg1", 1023, 32, -1.0, 1.0), ("cfg2", 65535, 64, -1.0, 1.0),
                                 ("cfg3", 1048575, 64, -4.0, 4.0), ("cfg4", 262143, 64, -1.0, 1.0),
                                 ("cfg5", 4194303, 128, -1.0, 1.0)):
        hh = (hi - lo) / (N + 1)
        x = hh * np.arange(-(N // 2), N // 2 + 1)
        ct = G.build_cluster_tree(x[:, None], leaf_size=leaf)
        ident = bool(np.array_equal(ct.perm.inverse, np.arange(N)))
        Hx = HM.build_from_expansion(ct, ct, HM.gaussian_expansion_1d(1.0), HM.HConfig(
            n_min=leaf, n_block=4, eta=1.0, fixed_rank=1),
            entry_fn=lambda r, c: np.zeros((r.shape[0], c.shape[0])))
        sa = struct_array(Hx)[:, :5]
        nh = 0

        def count_h(b):
            nonlocal nh
            if isinstance(b, HM.Hier):
                nh += 1
                for row in b.children:
                    for ch in row:
                        count_h(ch)
        count_h(Hx.root)
        lr = sa[sa[:, 4] == 1]
        parts[tag] = dict(N=N, leaf=leaf, identity_perm=ident, dense=int((sa[:, 4] == 0).sum()),
                          lowrank=int(lr.shape[0]), hier=nh,
                          sum_mn_lowrank=int(((lr[:, 1] - lr[:, 0]) + (lr[:, 3] - lr[:, 2])).sum()),
                          sha256=hashlib.sha256(np.ascontiguousarray(sa).tobytes()).hexdigest())
        print(tag, parts[tag])
        del Hx, ct
    import json
    with open(os.path.join(OUT, "partitions.json"), "w") as f:
        json.dump(parts, f, indent=1)


if __name__ == "__main__":
    main()
