"""CPU check of the H-arithmetic planner: the task DAGs exported by the native
library (H-LU, substitution solve, lower/upper triangular inverses, propagator
Z = (LU)^{-1}) are executed
by a numpy emulator of the device task semantics (tests/plan_emulator.py) on the
oracle's compressed operator, and compared with the oracle's hlu / solve."""
import numpy as np
import pytest

from oracle import levyh_oracle as O
from tests import cases
from tests import plan_emulator as E


@pytest.mark.parametrize("name", ["cfg1", "cfg3_cgmy", "cfg5_leaf128"])
def test_planned_dags_match_oracle(name, tmp_path):
    import paper_1812_08324_b200 as P
    from paper_1812_08324_b200 import _lib

    g = cases.load(name)
    leaf, N = int(g["leaf"]), int(g["N"])
    root, order, Hp, Hm = O.build_cn(g["tA"], float(g["dt"]), g["x"], leaf, float(g["eps1"]))
    ct = P.build_cluster_tree(g["x"][:, None], leaf)
    path = str(tmp_path / "plans.bin")
    assert _lib.testing().lh_debug_dump_plans(ct.handle, ct.handle, leaf, 4, 1.0, 32, 48, path.encode()) == 0
    D = E.load(path)
    # --- H-LU
    arenaF, ranks = E.fill_from_oracle(D["F0"], Hp, O.leaves)
    lu = D["lu"]
    rk = np.zeros(lu["nslots_total"] + 1, dtype=np.int64)
    rk[:ranks.shape[0]] = ranks
    perm = np.zeros(max(D["F"]["perm_len"], 1), dtype=np.int64)
    M = E.Machine({E.B_F: arenaF, E.B_TMP: np.zeros(max(lu["temp_len"], 1))}, rk, perm)
    M.run(lu, np.random.default_rng(0))
    Fo = O.hlu(Hp, 1e-10)
    b = g["probe"][:, :2].copy()
    ref = O.lu_solve(Fo, b)
    # --- substitution solve DAG on a 2-column right-hand side
    sp = D["solve"]
    nsF = D["F"]["nslots"]
    rk2 = np.zeros(sp["nslots_total"] + 1, dtype=np.int64)
    rk2[:nsF] = rk[:nsF]
    rk2[sp["rhs_slot"]] = 2
    rhs = np.zeros(N * 4)
    rhs[:2 * N] = b.T.ravel()
    M2 = E.Machine({E.B_F: arenaF, E.B_TMP: np.zeros(max(sp["temp_len"], 1)), E.B_RHS: rhs}, rk2, perm)
    M2.run(sp, np.random.default_rng(0))
    x = rhs[:2 * N].reshape(2, N).T
    assert np.linalg.norm(x - ref) <= 1e-12 * np.linalg.norm(ref)
    # --- triangular inverses: X b == forward / backward substitution; propagator Z b == solve
    for key, pk, mode in (("XL", "invL", "L"), ("XU", "invU", "U"), ("Z", "prop", "LU")):
        lay, ip = D[key], D[pk]
        ar = np.zeros(max(lay["arena"], 1))
        rk3 = np.zeros(ip["nslots_total"] + 1, dtype=np.int64)
        rk3[:nsF] = rk[:nsF]
        M3 = E.Machine({E.B_F: arenaF, E.B_TMP: np.zeros(max(ip["temp_len"], 1)), E.B_X: ar}, rk3, perm)
        M3.run(ip, np.random.default_rng(1))
        y = np.zeros_like(b)
        for rec in lay["recs"]:
            R0, R1, C0, C1, kind, doff, uoff, voff, kcap, rslot, poff = (int(q) for q in rec)
            m, n = R1 - R0, C1 - C0
            if kind == 4:
                continue
            if kind == 2:
                r = int(rk3[ip["slot_off_x"] + rslot])
                U = ar[uoff + np.arange(m)[:, None] + np.arange(r)[None, :] * m]
                V = ar[voff + np.arange(n)[:, None] + np.arange(r)[None, :] * n]
                y[R0:R1] += U @ (V.T @ b[C0:C1])
            else:
                y[R0:R1] += ar[doff + np.arange(m)[:, None] + np.arange(n)[None, :] * m] @ b[C0:C1]
        if mode == "LU":
            want = ref
        else:
            want = O.solve_dense(Fo, b.copy(), mode, mode == "L", "root")
        assert np.linalg.norm(y - want) <= 1e-11 * np.linalg.norm(want), key
