"""compute-sanitizer target: the persistent dataflow executor (lu.cu: exec_kernel) on the cfg1
operator at N = 1023 (assembly, H-LU, substitution / inverse / propagator solves, 4 CN steps),
checked against the oracle so a silent corruption also fails.

    compute-sanitizer --tool racecheck python tools/sanitize_exec.py
    compute-sanitizer --tool memcheck python tools/sanitize_exec.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_08324_b200 as P  # noqa: E402
from oracle import levyh_oracle as O  # noqa: E402

n, s = 512, 0.5
h = 1.0 / n
sy = P.FracCNSystem(P.power_measure(1, s), 0.0, 0.0, 0.0, n, h)
cfg = P.HConfig(n_min=32, eps1=1e-10)
Hp, Hm = sy.build_pair(cfg)
F = P.hlu(Hp, 1e-10)
tA, _ = O.symbol_A(O.nu_power(s), h, sy.N, 2.0, 0.2, O.tail_power(s, 2.0))
root, order, Op, Om = O.build_cn(tA, h, sy.x, 32, 1e-10)
Fo = O.hlu(Op, 1e-10)
x = np.random.default_rng(0).standard_normal(sy.N)
ref = O.lu_solve(Fo, x)
for method in ("substitution", "inverse", "propagator"):
    z = P.solve(F, x, method=method)
    err = np.linalg.norm(z - ref) / np.linalg.norm(ref)
    print(method, "rel err", err)
    assert err <= 1e-9
sy.h_minus, sy.factor, sy.method = Hm, F, "propagator"
u0 = (1 - sy.x ** 2) ** 2
u = P.run_cn(sy, u0, 4)
uo = O.run_cn(Om, Fo, u0, 4)
assert np.linalg.norm(u - uo) <= 1e-8 * np.linalg.norm(uo)
print("sanitize target ok: N =", sy.N)
