"""Golden fixtures of the reference's smooth-measure path (the series H-builder), made by
running the REAL reference package in the build container:

    python tests/golden/make_golden_gauss.py

Path (the reference's own `levyh bench` system, cli.py:163-224):
levy.gaussian_measure -> levy.assemble_cn_1d -> CNSystem.hmatrix (hmatrix.build_from_expansion
with gaussian_expansion_1d, levy.py:224-239) -> hops.hlu -> CN stepping (levy.run_cn).
Writes tests/golden/gauss_*.npz.  Nothing here runs on the GPU box.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from levyh import hmatrix as HM  # noqa: E402
from levyh import hops as HO  # noqa: E402
from levyh import levy as LV  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def struct_array(H):
    kinds = {"dense": 0, "lowrank": 1, "dense_lu": 2}
    return np.array([(d["row0"], d["row1"], d["col0"], d["col1"], kinds[d["kind"]], d.get("rank", -1))
                     for d in HM.structure_summary(H)], dtype=np.int64).reshape(-1, 6)


def lowrank_blocks(H):
    """(row0, col0, m, n, rank) and the concatenated u / v of every low-rank leaf, walk order."""
    recs, us, vs = [], [], []

    def walk(b, r0, c0):
        if isinstance(b, HM.Hier):
            rs, cs = b.row_split, b.col_split
            walk(b.children[0][0], r0, c0)
            walk(b.children[0][1], r0, c0 + cs)
            walk(b.children[1][0], r0 + rs, c0)
            walk(b.children[1][1], r0 + rs, c0 + cs)
        elif isinstance(b, HM.LowRank):
            recs.append((r0, c0, b.u.shape[0], b.v.shape[0], b.u.shape[1]))
            us.append(b.u.ravel(order="F"))
            vs.append(b.v.ravel(order="F"))

    walk(H.root, 0, 0)
    return np.array(recs, dtype=np.int64), np.concatenate(us), np.concatenate(vs)


def case(name, n, eps_sq, scale, a, b, c, dt, leaf, fixed_rank, delta, steps, seed):
    nu = LV.gaussian_measure(eps_sq, scale)
    grid = LV.UniformGrid1D(n)
    sysm = LV.assemble_cn_1d(nu, a, b, c, grid, dt)
    cfg = HM.HConfig(n_min=leaf, n_block=4, eta=1.0, fixed_rank=fixed_rank, delta=delta)
    Hp = sysm.hmatrix("plus", cfg)
    Hm = sysm.hmatrix("minus", cfg)
    lr_recs, lr_u, lr_v = lowrank_blocks(Hp)
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n)
    y_plus = HO.matvec(Hp, x)
    y_minus = HO.matvec(Hm, x)
    idx = np.arange(n)
    # Toeplitz symbol t[k + n - 1] = A[i, i + k] read off the first and last rows
    row0 = sysm.entries(np.zeros(1, dtype=np.intp), idx, "A")[0]
    rowl = sysm.entries(np.full(1, n - 1), idx, "A")[0]
    symbol = np.concatenate([rowl[:-1], row0])
    struct_plus = struct_array(Hp)
    F = HO.hlu(Hp, 1e-10)
    struct_lu = struct_array(F.h)
    b_solve = rng.standard_normal(n)
    x_solve = HO.solve(F, b_solve)
    u0 = np.exp(-20.0 * grid.points ** 2)
    sysm.factor, sysm.h_minus = F, Hm
    sysm.tree = sysm.cluster_tree(leaf)
    uT = LV.run_cn(sysm, u0, steps)
    np.savez_compressed(os.path.join(OUT, f"gauss_{name}.npz"),
                        n=n, eps_sq=eps_sq, scale=scale, a=a, b=b, c=c, dt=dt, leaf=leaf,
                        fixed_rank=fixed_rank, delta=(-1.0 if delta is None else delta), steps=steps,
                        lam=sysm.lam, n_off=sysm.n_off, symbol=symbol, struct_plus=struct_plus,
                        lr_recs=lr_recs, lr_u=lr_u, lr_v=lr_v, x=x, y_plus=y_plus, y_minus=y_minus,
                        struct_lu=struct_lu, b_solve=b_solve, x_solve=x_solve, u0=u0, uT=uT)
    print(name, "n", n, "lowrank", len(lr_recs), "ranks", np.unique(lr_recs[:, 4]),
          "LU ranks", np.unique(struct_lu[struct_lu[:, 4] == 1, 5]), "|uT|", np.linalg.norm(uT))


if __name__ == "__main__":
    # the reference bench system (cli.py:173-177): eps_sq 5, a = b = c = 0, dt = 0.01, rank 10
    case("bench", 1024, 5.0, 1.0, 0.0, 0.0, 0.0, 0.01, 64, 10, None, 20, 0)
    # convection-diffusion with a scaled density and per-block ranks from the Gaussian bound
    case("delta", 1024, 3.0, 2.0, 0.05, 0.3, -0.1, 0.005, 64, 10, 1e-6, 20, 1)
