"""Reference-generated fixtures for the 2D series H-builder (levy.CNSystem.hmatrix with
gaussian_expansion_2d, hmatrix.py:189-216, :243-291, levy.py:224-246) at 4 and 5 terms per
dimension (block ranks 16 and 25): structure, factors of one block, matvecs, H-LU solve, CN steps.

    python tests/golden/make_golden_2d_series.py
"""
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


def first_lowrank(b):
    if isinstance(b, HM.LowRank):
        return b
    if isinstance(b, HM.Hier):
        for row in b.children:
            for k in row:
                r = first_lowrank(k)
                if r is not None:
                    return r
    return None


def main():
    res = {}
    rng = np.random.default_rng(3)
    for T in (4, 5):
        s = LV.assemble_cn_2d(LV.gaussian_measure(5.0), 0.1, 0.5, -0.2, LV.UniformGrid2D(24, 24), 0.05)
        cfg = HM.HConfig(n_min=32, fixed_rank=T)
        Hp, Hm = s.hmatrix("plus", cfg), s.hmatrix("minus", cfg)
        perm = s.tree.perm
        X = rng.standard_normal((s.n, 2))
        res[f"t{T}_order"] = perm.inverse.astype(np.int64)
        res[f"t{T}_struct"] = struct_array(Hp)
        res[f"t{T}_X"] = X
        res[f"t{T}_mv_plus"] = np.column_stack([HO.matvec(Hp, X[:, k]) for k in range(2)])
        res[f"t{T}_mv_minus"] = np.column_stack([HO.matvec(Hm, X[:, k]) for k in range(2)])
        dense_plus = HM.to_dense(Hp)
        lr = first_lowrank(Hp.root)
        res[f"t{T}_lr_u"], res[f"t{T}_lr_v"] = lr.u, lr.v
        F = HO.hlu(s.hmatrix("plus", cfg), 1e-10)
        res[f"t{T}_struct_factor"] = struct_array(F.h)
        res[f"t{T}_solve"] = HO.solve(F, X[:, 0])
        u0 = np.exp(-4.0 * (s.grid.points ** 2).sum(axis=1))
        res[f"t{T}_u0"] = u0
        res[f"t{T}_uT"] = LV.run_cn(LV.assemble_cn_2d(LV.gaussian_measure(5.0), 0.1, 0.5, -0.2,
                                                      LV.UniformGrid2D(24, 24), 0.05), u0, 10, cfg, 1e-10)
        print(T, "blocks", len(res[f"t{T}_struct"]), "rank", lr.u.shape,
              "series vs exact", np.linalg.norm(dense_plus - s.dense_matrix("plus")[np.ix_(perm.inverse, perm.inverse)]))
    np.savez_compressed(os.path.join(OUT, "golden_2d_series.npz"), **res)


if __name__ == "__main__":
    main()
