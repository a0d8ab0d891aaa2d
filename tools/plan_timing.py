"""Host planner timing (no GPU): H-LU and propagator plans on the 1D partition of size
N = 2n - 1, leaf 64.   python tools/plan_timing.py [n] [which=3]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_08324_b200 as P  # noqa: E402
from paper_1812_08324_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
which = int(sys.argv[2]) if len(sys.argv) > 2 else 3
x = np.linspace(-1, 1, 2 * n + 1)[1:-1]
ct = P.build_cluster_tree(x[:, None], 64)
out = np.zeros(4)
t = time.time()
rc = _lib.lib().lh_debug_plan_timing(ct.handle, ct.handle, 64, 4, 1.0, 32, 48, which, _lib.host_ptr(out))
print(f"rc={rc} N={2 * n - 1}: H-LU plan {out[0]:.3f} s ({int(out[1])} tasks, {out[0] / max(out[1], 1) * 1e6:.2f} us/task), "
      f"propagator plan {out[2]:.3f} s ({int(out[3])} tasks); wall {time.time() - t:.2f} s")
