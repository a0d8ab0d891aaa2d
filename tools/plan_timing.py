"""Host planner timing and device footprints (no GPU): H-LU and propagator plans on the 1D
partition of size N = 2n - 1.   python tools/plan_timing.py [n] [which=3] [leaf=64] [kcap_f=32] [kcap_z=32]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_08324_b200 as P  # noqa: E402
from paper_1812_08324_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
which = int(sys.argv[2]) if len(sys.argv) > 2 else 3
leaf = int(sys.argv[3]) if len(sys.argv) > 3 else 64
kf = int(sys.argv[4]) if len(sys.argv) > 4 else 32
kz = int(sys.argv[5]) if len(sys.argv) > 5 else 32
x = np.linspace(-1, 1, 2 * n + 1)[1:-1]
ct = P.build_cluster_tree(x[:, None], leaf)
out = np.zeros(16)
t = time.time()
rc = _lib.testing().lh_debug_plan_timing(ct.handle, ct.handle, leaf, 4, 1.0, kf, kz, which, _lib.host_ptr(out))
print(f"rc={rc} N={2 * n - 1} leaf {leaf}: H-LU plan {out[0]:.3f} s ({int(out[1])} tasks, temp {out[4] / 1e9:.2f} GB, "
      f"device {out[7] / 1e9:.2f} GB), propagator plan {out[2]:.3f} s ({int(out[3])} tasks, temp {out[5] / 1e9:.2f} GB, "
      f"device {out[8] / 1e9:.2f} GB); arenas F {out[9] / 1e9:.2f} GB (kcap {kf}), Z {out[6] / 1e9:.2f} GB (kcap {kz}); "
      f"wall {time.time() - t:.2f} s")
