"""H2 probe errors for several subtree splits / tolerances on a cfg3-like operator (stderr log)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_08324_b200 as P

os.environ["LEVYH_PLAN_VERBOSE"] = "1"
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 13
for split, eps in [("5", None), ("20", None), ("0", None), ("2", None), ("5", "1e-14")]:
    os.environ["LEVYH_H2_SPLIT"] = split
    if eps:
        os.environ["LEVYH_SB_EPS"] = eps
    print(f"=== split {split} eps {eps}", file=sys.stderr, flush=True)
    s = P.FracCNSystem(P.cgmy_measure(1.0, 5.0, 10.0, 0.5), 0.05, 0.1, -0.05, n, 8.0 / 2 ** 20 * 16,
                       L=4.0, L_W=8.0, drift_compensation=True)
    s.prepare(P.HConfig(n_min=64, eps1=1e-9), 1e-10, method="propagator")
    del s
