import sys, numpy as np
sys.path.insert(0, '.')
import paper_1812_08324_b200 as P
n = int(sys.argv[1])
s = P.FracCNSystem(P.power_measure(1, 0.5), 0.0, 0.0, 0.0, n, 1.0 / n)
s.prepare(P.HConfig(n_min=64, eps1=1e-10), 1e-10, method="propagator")
print("N", s.N, "stats", s.factor.propagator_stats())
