import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_1812_08324_b200 as P
ctx = P._lib.Context.get(); L = P._lib.testing(); out = np.zeros(2)
for kind, name in ((0, "GETRF+inv"), (3, "GETRF")):
    P._lib.check(L.lh_debug_task_bench(ctx.h, kind, 2000, 64, 1, P._lib.host_ptr(out)), ctx.h)
    print(f"{name:10s} chain: wall {out[0]:8.2f} us/task, body {out[1]:8.2f} us", flush=True)
