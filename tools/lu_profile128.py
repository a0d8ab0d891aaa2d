"""Task-level profile of the H-LU DAG on a cfg5-style operator (s=0.8, a=0.1, leaf 128).

    LEVYH_TASK_PROFILE=gpurun_out/tasks128.txt python tools/lu_profile128.py [n]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1812_08324_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 19
leaf = int(sys.argv[2]) if len(sys.argv) > 2 else 128
t = time.time()
s = P.FracCNSystem(P.power_measure(1, 0.8), 0.1, 0.0, 0.0, n, 1.0 / n)
Hp, Hm = s.build_pair(P.HConfig(n_min=leaf, eps1=1e-10, kcap=24))
t1 = time.time()
F = P.hlu(Hp, 1e-10)
import numpy as np  # noqa: E402
st = np.zeros(8)
P._lib.lib().lh_hlu_stats(F.h.handle, P._lib.host_ptr(st))
print(f"N={s.N} leaf={leaf}: build {t1 - t:.2f} s, hlu {time.time() - t1:.2f} s, tasks {int(st[0])}, "
      f"plan {st[1]:.2f} s, exec {st[3]:.2f} s, chunks {int(st[4])}", flush=True)
