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
