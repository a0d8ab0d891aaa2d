"""Shared parity-case definitions (parameters of tests/golden/*.npz)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

CASES = {
    # name: (measure spec, L, n, L_W, tail or None)
    "cfg1": (("power", 0.5), 1.0, 512, 2.0),
    "cfg2_s025": (("power", 0.25), 1.0, 1024, 2.0),
    "cfg2_s075": (("power", 0.75), 1.0, 1024, 2.0),
    "cfg3_cgmy": (("cgmy", 1.0, 5.0, 10.0, 0.5), 4.0, 512, 8.0),
    "cfg5_s08": (("power", 0.8), 1.0, 512, 2.0),
    "cfg5_leaf128": (("power", 0.8), 1.0, 1024, 2.0),  # cfg5's leaf size (128)
    # N = 8191 (tests/golden/make_golden_8191.py): blocks of up to 2048 rows
    "cfg2_s025_n8191": (("power", 0.25), 1.0, 4096, 2.0),
    "cfg3_cgmy_n8191": (("cgmy", 1.0, 5.0, 10.0, 0.5), 4.0, 4096, 8.0),
}


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def make_system(name, g=None):
    """FracCNSystem with exactly the golden case's parameters."""
    import paper_1812_08324_b200 as P

    g = g if g is not None else load(name)
    spec, L, n, L_W = CASES[name]
    if spec[0] == "power":
        nu = P.power_measure(1, spec[1])
        tail = None
        b = float(g["b_eff"])
        drift = False
    else:
        nu = P.cgmy_measure(*spec[1:])
        sc = load("cfg3_scalars")
        tail = float(sc["tail"])
        b = float(g["b_eff"]) - float(sc["beta"])
        drift = True
    sys_ = P.FracCNSystem(nu, float(g["a"]), b, float(g["c"]), n, float(g["dt"]), L=L, L_W=L_W,
                          tail_mass=tail, drift_compensation=drift)
    return sys_


def struct_from_golden(arr):
    return arr.copy()


def krylov_operators(tag):
    """Dense operator and grid of a tests/golden/krylov.npz case (oracle restatement of
    make_golden_krylov.py's operators: the cfg1 fractional Laplacian, and the cfg2-style
    convection-diffusion operator and its CN matrix)."""
    from oracle import levyh_oracle as O

    if tag.startswith("poisson") or tag == "pcg_hlu":
        n = int(tag[7:]) if tag.startswith("poisson") else 512
        s, a, b, c = 0.5, 0.0, 0.0, 0.0
    else:
        n, s, a, b, c = 512, 0.25, 0.5, 1.0, -1.0
    h = 1.0 / n
    N = 2 * n - 1
    tA, _ = O.symbol_A(O.nu_power(s), h, N, 2.0, 0.2, O.tail_power(s, 2.0), a, b, c)
    A = O.toeplitz_dense(tA)
    x = h * np.arange(-n + 1, n)
    if tag == "gmres_r5":
        A = np.eye(N) + 0.5 * h * A
    return A, x


def report_rank_mismatch(name, what, nblocks, diff):
    """Record per-block rank differences against the reference (G1: report, do not hide):
    printed (visible with -s / in the captured log) and appended to
    gpurun_out/rank_mismatch.jsonl when that directory exists."""
    import json

    diff = np.asarray(diff)
    rec = {"case": name, "what": what, "lowrank_blocks": int(nblocks),
           "mismatches": int(np.count_nonzero(diff)),
           "max_abs": int(np.abs(diff).max(initial=0)),
           "higher": int((diff > 0).sum()), "lower": int((diff < 0).sum())}
    print("rank-mismatch", json.dumps(rec))
    out = os.path.join(os.path.dirname(GOLDEN), "..", "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "rank_mismatch.jsonl"), "a") as f:
            f.write(json.dumps(rec) + "\n")
    return rec


# ---------------------------------------------------------------------------
# matrix-free evaluators / variable-order assembly: seeded inputs shared by the fixture
# generator (tests/golden/make_golden_apply.py) and the tests
# ---------------------------------------------------------------------------
APPLY_1D = {
    "ap1_power": dict(measure=("power",), s=0.5, h=1.0 / 32, L=1.0, L_W=2.0, rho_r=0.2, far=True, seed=1),
    "ap1_s08_ragged": dict(measure=("power",), s=0.8, h=1.0 / 50, L=0.74, L_W=1.5, rho_r=0.3, far=False, seed=2),
    "ap1_cgmy": dict(measure=("cgmy", 1.0, 5.0, 10.0, 0.5), s=0.25, h=1.0 / 40, L=1.0, L_W=2.0, rho_r=0.2,
                     far=False, tail=0.0123, seed=3),
    "ap1_point": dict(measure=("power",), s=0.3, h=1.0 / 16, L=0.0, L_W=1.0, rho_r=0.25, far=False, seed=4),
}
APPLY_2D = {
    "ap2_s04": dict(s=0.4, h=1.0 / 8, L=0.5, L_W=1.0, rho_r=0.3, far=True, seed=5),
    "ap2_s075": dict(s=0.75, h=1.0 / 10, L=0.7, L_W=1.2, rho_r=0.25, far=False, seed=6),
}
VARIABLE_ORDER = {
    "vo8": dict(n=8, L_W=2.0, rho_r=0.2, field="default"),
    "vo12_short_window": dict(n=12, L_W=0.5, rho_r=0.2, field="wave"),
    "vo16": dict(n=16, L_W=2.0, rho_r=0.3, field="default"),
}


def cgmy_density(C, G, M, Y):
    def f(y):
        y = np.asarray(y, dtype=float)
        ay = np.abs(y)
        with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
            return C * np.exp(-np.where(y < 0, G, M) * ay) * ay ** (-1.0 - Y)
    return f


def apply_inputs_1d(c):
    M, K = int(round(c["L_W"] / c["h"])), int(round(c["L"] / c["h"]))
    x = c["h"] * np.arange(-(M + K), M + K + 1)
    rng = np.random.default_rng(c["seed"])
    u = np.exp(-x * x) * np.cos(3 * x) + 0.05 * rng.standard_normal(x.shape)
    far = (lambda t: 0.3 * np.sin(2 * np.asarray(t)) + 0.1) if c["far"] else None
    return u, far


def apply_inputs_2d(c):
    M, K = int(round(c["L_W"] / c["h"])), int(round(c["L"] / c["h"]))
    x = c["h"] * np.arange(-(M + K), M + K + 1)
    rng = np.random.default_rng(c["seed"])
    u = np.exp(-(x[:, None] ** 2 + 0.5 * x[None, :] ** 2)) * np.cos(2 * x[:, None] + x[None, :])
    u = u + 0.05 * rng.standard_normal(u.shape)
    far = (lambda a, b: 0.2 * np.cos(np.asarray(a)) * np.asarray(b) + 0.05) if c["far"] else None
    return u, far


def order_field(c):
    if c["field"] == "default":
        return None
    return lambda pts: 0.5 + 0.35 * np.sin(2.0 * pts[:, 0]) * np.cos(3.0 * pts[:, 1])
