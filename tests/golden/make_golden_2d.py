"""Reference-generated fixtures for the 2D rows of SURVEY 8(f) (row 4): kmeans2 / bisection
cluster trees on 2D point sets (geometry.py:146-243), the variable-order L-shape system through
build_from_dense / hlu / solve / gmres_restarted (cli.frac_lshape_study, cli.py:442-477), and the
2D Gaussian CN system (levy.assemble_cn_2d, levy.py:275-292, _entries_a_2d :178-192) with the
reference's dense CN solution and its build_from_dense partition and ranks.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_2d.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from levyh import fractional as F  # noqa: E402
from levyh import geometry as G  # noqa: E402
from levyh import hmatrix as HM  # noqa: E402
from levyh import hops as HO  # noqa: E402
from levyh import levy as LV  # noqa: E402
from levyh import solvers as SV  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def struct_array(H):
    kinds = {"dense": 0, "lowrank": 1, "dense_lu": 2}
    return np.array([(d["row0"], d["row1"], d["col0"], d["col1"], kinds[d["kind"]], d.get("rank", -1))
                     for d in HM.structure_summary(H)], dtype=np.int64).reshape(-1, 6)


def tree_ranges(ct):
    out = []

    def walk(nd):
        out.append((nd.start, nd.end))
        if not nd.is_leaf:
            for c in nd.children:
                walk(c)
    walk(ct.root)
    return np.array(out, dtype=np.int64)


def main():
    res = {}
    # --- trees on 2D point sets ------------------------------------------------------
    sets = {
        "lshape24": F.lshape_grid(24)[0],
        "grid20": LV.UniformGrid2D(20, 20).points,
        "rand500": np.random.default_rng(0).uniform(-1, 1, (500, 2)) * np.array([1.0, 0.3]),
    }
    for name, pts in sets.items():
        res[f"pts_{name}"] = pts
        for strat in ("kmeans2", "bisection"):
            for leaf in (16, 32):
                ct = G.build_cluster_tree(pts, leaf_size=leaf, strategy=strat)
                res[f"order_{name}_{strat}_{leaf}"] = ct.perm.inverse.astype(np.int64)
                res[f"ranges_{name}_{strat}_{leaf}"] = tree_ranges(ct)
    # --- variable-order L-shape (cli.frac_lshape_study pattern) ------------------------
    n = 24
    A, b, pts = F.assemble_variable_order(n)
    ct = G.build_cluster_tree(pts, leaf_size=32, strategy="kmeans2")
    perm = ct.perm
    At = A[np.ix_(perm.inverse, perm.inverse)]
    cfg = HM.HConfig(n_min=32, n_block=4, eta=1.0, eps1=1e-6)
    H = HM.build_from_dense(At, ct, ct, cfg)
    sH = struct_array(H)
    Fh = HO.hlu(H, 1e-10)
    uh = perm.from_tree(HO.solve(Fh, perm.to_tree(b)))
    bt = perm.to_tree(b)
    _, log_pre = SV.gmres_restarted(lambda v: At @ v, lambda v: HO.solve(Fh, v), bt, tol=1e-8, restart=50,
                                    max_iter=400)
    res.update(ls_A=A, ls_b=b, ls_pts=pts, ls_struct=sH, ls_struct_factor=struct_array(Fh.h), ls_uh=uh,
               ls_udense=np.linalg.solve(A, b), ls_gmres_iters=log_pre.iterations,
               ls_gmres_res=np.array(log_pre.residuals))
    print("lshape", A.shape, sH.shape, "gmres", log_pre.iterations)
    # --- 2D Gaussian CN system ---------------------------------------------------------
    grid = LV.UniformGrid2D(24, 24)
    nu = LV.gaussian_measure(5.0)
    sysm = LV.assemble_cn_2d(nu, 0.1, 0.5, -0.2, grid, 0.05)
    Ap, Am = sysm.dense_matrix("plus"), sysm.dense_matrix("minus")
    ctg = sysm.cluster_tree(leaf_size=32)
    pg = ctg.perm
    hc = HM.HConfig(n_min=32, eps1=1e-6)
    Hp = HM.build_from_dense(Ap[np.ix_(pg.inverse, pg.inverse)], ctg, ctg, hc)
    sp = struct_array(Hp)
    Hm = HM.build_from_dense(Am[np.ix_(pg.inverse, pg.inverse)], ctg, ctg, hc)
    Fp = HO.hlu(Hp, 1e-10)
    x = grid.points
    u0 = np.exp(-20.0 * (x[:, 0] ** 2 + x[:, 1] ** 2))
    ut = pg.to_tree(u0)
    for _ in range(10):  # levy.run_cn's H loop on the build_from_dense operators
        ut = HO.solve(Fp, HO.matvec(Hm, ut))
    uh = pg.from_tree(ut)
    ud = LV.run_cn(sysm, u0, 10, mode="dense")
    res.update(cn2_Aplus=Ap, cn2_Aminus=Am, cn2_lam=sysm.lam, cn2_h=grid.h, cn2_struct_plus=sp,
               cn2_u0=u0, cn2_uT_dense=ud, cn2_uT_h=uh, cn2_order=pg.inverse.astype(np.int64))
    print("cn2d H vs dense", np.linalg.norm(uh - ud) / np.linalg.norm(ud), "ranks", sp[sp[:, 4] == 1, 5])
    print("cn2d", Ap.shape, "lam", sysm.lam)
    np.savez_compressed(os.path.join(OUT, "golden_2d.npz"), **res)


if __name__ == "__main__":
    main()
