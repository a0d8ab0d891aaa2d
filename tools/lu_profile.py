"""Task-level profile of H-LU and inverse-factor DAGs on the cfg3 operator.

    LEVYH_TASK_PROFILE=gpurun_out/tasks.txt python tools/lu_profile.py [n]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1812_08324_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 15
t = time.time()
s, F, Hm, times = bench.build_system(P, n=n)
print({k: v for k, v in times.items()}, "wall", time.time() - t, flush=True)
