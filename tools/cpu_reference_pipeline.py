"""The reference's own CPU pipeline for the cfg3 operator (CGMY, leaf 64, ACA tol 1e-9), timed
phase by phase with levyh.cli.median_time (cli.py:96-106): the unmodified levyh from
baseline/_ref (frac_stencil_1d, build_from_dense of A+ and A-, hlu, and the CN loop
solve(F, matvec(H-, u)) of levy.run_cn, levy.py:309-330), composed as tests/golden/make_golden.py
does.  Baseline infrastructure: not part of the product.

    python tools/cpu_reference_pipeline.py [n=8192 -> N = 2n - 1] [steps=100] [repeat=1] [warmup=0]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(1, os.path.join(ROOT, "tests", "golden"))
import make_golden as MG  # noqa: E402  (its levyh imports resolve to baseline/_ref)
from levyh import cli as CLI  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
repeat = int(sys.argv[3]) if len(sys.argv) > 3 else 1
warmup = int(sys.argv[4]) if len(sys.argv) > 4 else 0
F, G, HM, HO, LV = MG.F, MG.G, MG.HM, MG.HO, MG.LV

nu = MG.cgmy_density(1.0, 5.0, 10.0, 0.5)
from scipy.integrate import quad  # noqa: E402

tail = (quad(lambda y: nu(np.array(y)), 8, np.inf, epsabs=0, epsrel=1e-12)[0]
        + quad(lambda y: nu(np.array(-y)), 8, np.inf, epsabs=0, epsrel=1e-12)[0])
beta = MG.drift_beta(nu, 0.2)
h = 4.0 / n
dt = 16 * h
meas = LV.LevyMeasure(density=nu, kind="singular_heavy_tail", symmetric=False)
cfg = F.FracConfig(s=0.25, h=h, L=4.0, L_W=8.0, rho_r=0.2, nu=meas, tail_mass=tail)
out = {"what": "levyh (unmodified, baseline/_ref) CPU pipeline, cfg3 operator", "n": n, "N": 2 * n - 1,
       "steps": steps, "repeat": repeat, "warmup": warmup, "cores": os.cpu_count(),
       "blas_threads": os.environ.get("OMP_NUM_THREADS", "default")}


def timed(key, fn):
    t, r = CLI.median_time(fn, repeat, warmup)
    out[key] = round(t, 3)
    print(key, out[key], flush=True)
    return r


st = timed("stencil_s", lambda: F.frac_stencil_1d(cfg))
A = MG.composed_A(st.weights, h, 0.05, 0.1 + beta, -0.05)
x = st.x[1:-1]
N = A.shape[0]
eye = np.eye(N)
Ap, Am = eye + 0.5 * dt * A, eye - 0.5 * dt * A
ct = G.build_cluster_tree(x[:, None], leaf_size=64)
hc = HM.HConfig(n_min=64, n_block=4, eta=1.0, eps1=1e-9)
Hp = timed("build_plus_s", lambda: HM.build_from_dense(Ap, ct, ct, hc))
Hm = timed("build_minus_s", lambda: HM.build_from_dense(Am, ct, ct, hc))
out["stored_scalars_plus"] = HM.memory_report(Hp)["stored_scalars"]
builds = [Hp] + [HM.build_from_dense(Ap, ct, ct, hc) for _ in range(repeat + warmup - 1)]
ts = []
for Hb in builds:  # hlu consumes its input (cli.bench_point's convention)
    t0 = time.perf_counter()
    Fh = HO.hlu(Hb, 1e-10)
    ts.append(time.perf_counter() - t0)
out["hlu_s"] = round(float(np.median(ts[warmup:])), 3)
print("hlu_s", out["hlu_s"], flush=True)
u0 = np.maximum(np.exp(x) - 1.0, 0.0)


def run():
    u = u0.copy()
    for _ in range(steps):
        u = HO.solve(Fh, HO.matvec(Hm, u))
    return u


timed("steps_s", run)
out["steps_per_s"] = round(steps / out["steps_s"], 4)
out["setup_s"] = round(out["stencil_s"] + out["build_plus_s"] + out["build_minus_s"] + out["hlu_s"], 3)
print(json.dumps(out), flush=True)
