"""Pin the CPU oracle (oracle/levyh_oracle.py) against fixtures produced by the
real reference (tests/golden/make_golden.py).  CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import levyh_oracle as O

CASES = ["cfg1", "cfg2_s025", "cfg2_s075", "cfg3_cgmy", "cfg5_s08", "cfg5_leaf128"]
BIG = ["cfg2_s025_n8191", "cfg3_cgmy_n8191"]  # symbol only (compression: GPU tests)


def _load(golden_dir, name):
    return dict(np.load(os.path.join(golden_dir, name + ".npz")))


def _case_symbol(name, g, golden_dir):
    h = float(g["h"])
    N = int(g["N"])
    if name.startswith("cfg3_cgmy"):
        sc = _load(golden_dir, "cfg3_scalars")
        nu = O.nu_cgmy(1.0, 5.0, 10.0, 0.5)
        tail = float(sc["tail"])
        L_W = 8.0
    else:
        s = {"cfg1": 0.5, "cfg2_s025": 0.25, "cfg2_s075": 0.75, "cfg5_s08": 0.8,
             "cfg5_leaf128": 0.8, "cfg2_s025_n8191": 0.25}[name]
        nu = O.nu_power(s)
        L_W = 2.0
        tail = O.tail_power(s, L_W)
    tA, sc = O.symbol_A(nu, h, N, L_W, 0.2, tail, float(g["a"]), float(g["b_eff"]), float(g["c"]))
    return tA, sc


@pytest.mark.parametrize("name", CASES + BIG)
def test_symbol_bitexact(name, golden_dir):
    g = _load(golden_dir, name)
    tA, _ = _case_symbol(name, g, golden_dir)
    assert np.array_equal(tA, g["tA"])


def test_cfg1_scalars(golden_dir):
    g = _load(golden_dir, "cfg1")
    sc = _load(golden_dir, "cfg1_scalars")
    _, mine = _case_symbol("cfg1", g, golden_dir)
    for k in ("S0", "Sg", "Sd", "m2", "tail"):
        assert mine[k] == float(sc[k]), k
    assert mine["M"] == int(sc["M"]) == 1024
    assert abs(O.frac_const(1, 0.5) - 1 / np.pi) < 1e-15
    assert float(sc["c_half"]) == O.frac_const(1, 0.5)


def test_cgmy_beta_and_tail(golden_dir):
    sc = _load(golden_dir, "cfg3_scalars")
    nu = O.nu_cgmy(1.0, 5.0, 10.0, 0.5)
    assert abs(O.drift_beta(nu, 0.2) - float(sc["beta"])) < 1e-14
    assert abs(float(sc["beta"]) - 0.133343) < 1e-6


@pytest.mark.parametrize("name", CASES)
def test_partition_ranks_and_solution(name, golden_dir):
    g = _load(golden_dir, name)
    tA, _ = _case_symbol(name, g, golden_dir)
    leaf, eps1 = int(g["leaf"]), float(g["eps1"])
    root, order, Hp, Hm = O.build_cn(tA, float(g["dt"]), g["x"], leaf, eps1)
    assert np.array_equal(order, np.arange(int(g["N"])))
    assert np.array_equal(O.structure(Hp), g["struct_plus"])
    assert np.array_equal(O.structure(Hm), g["struct_minus"])
    assert O.stored_scalars(Hp) == int(g["stored_scalars"])
    probe = g["probe"]
    mv = np.stack([O.hmatvec(Hp, probe[:, k]) for k in range(probe.shape[1])], axis=1)
    assert np.abs(mv - g["matvec_plus"]).max() <= 1e-13 * np.abs(g["matvec_plus"]).max()
    F = O.hlu(Hp, float(g["eps2"]))
    assert np.array_equal(O.structure(F), g["struct_factor"])
    sol = O.lu_solve(F, probe)
    assert np.abs(sol - g["solve_probe"]).max() <= 1e-12 * np.abs(g["solve_probe"]).max()
    if name != "cfg1":  # cfg1's 512 steps are covered by test_cfg1_end_to_end
        u = O.run_cn(Hm, F, g["u0"], int(g["n_steps"]))
        assert np.linalg.norm(u - g["uT"]) <= 1e-12 * np.linalg.norm(g["uT"])


def test_cfg1_end_to_end(golden_dir):
    g = _load(golden_dir, "cfg1")
    tA, _ = _case_symbol("cfg1", g, golden_dir)
    root, order, Hp, Hm = O.build_cn(tA, float(g["dt"]), g["x"], 32, 1e-10)
    ranks = O.structure(Hp)[:, 5]
    assert sorted(np.unique(ranks[ranks >= 0], return_counts=True)[1].tolist()) == [22, 44]
    F = O.hlu(Hp, 1e-10)
    u = O.run_cn(Hm, F, g["u0"], 512)
    assert np.linalg.norm(u - g["uT"]) <= 1e-12 * np.linalg.norm(g["uT"])
    # SURVEY 8(c) golden pins
    assert abs(np.linalg.norm(u) - 6.179677103303214) < 1e-11
    assert abs(u.sum() - 185.84434969900343) < 1e-9
    assert abs(u[511] - 0.25498164269386925) < 1e-13


def test_spec_lowrank_pins(golden_dir):
    g = _load(golden_dir, "spec_lowrank")
    u, v = O.lr_add(g["Au"], g["Av"], -g["Au"], g["Av"], 1e-10)
    assert u.shape[1] == int(g["rank_neg"]) == 10  # the reference keeps rank 10
    u, v = O.lr_add(g["Au"], g["Av"], g["Au"], g["Av"], 1e-10)
    assert u.shape[1] == int(g["rank_dbl"]) == 5
    assert np.abs(u @ v.T - g["dense_dbl"]).max() < 1e-12 * np.abs(g["dense_dbl"]).max()
    u, v = O.lr_add(g["B1u"], g["B1v"], g["B2u"], g["B2v"], 1e-12)
    assert u.shape[1] == int(g["rank_disj"]) == 4


def test_partition_counts_small(golden_dir):
    parts = json.load(open(os.path.join(golden_dir, "partitions.json")))
    p = parts["cfg1"]
    N = p["N"]
    x = (2.0 / (N + 1)) * np.arange(-(N // 2), N // 2 + 1)
    root, order = O.cluster_tree(x, p["leaf"])
    A = np.eye(N)
    H = O.compress_dense(A, root, 1e-10, p["leaf"])
    st = O.structure(H)
    assert int((st[:, 4] == 0).sum()) == p["dense"]
    assert int((st[:, 4] == 1).sum()) == p["lowrank"]
    # identity: all low-rank blocks rank 0 and matvec exact
    assert (st[st[:, 4] == 1, 5] == 0).all()
    xv = np.random.default_rng(0).standard_normal(N)
    assert np.array_equal(O.hmatvec(H, xv), xv)
