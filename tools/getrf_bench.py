"""GETRF task micro-benchmark: chained 64x64 leaf LU with (kind 0) / without (kind 3) the
packed leaf inverse, independent (throughput).  python tools/getrf_bench.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1812_08324_b200 as P  # noqa: E402

ctx = P._lib.Context.get()
L = P._lib.testing()
out = np.zeros(2)
for kind, name in ((0, "GETRF+inverse"), (3, "GETRF only")):
    for chain in (1, 0):
        R = 2000 if chain else 20000
        P._lib.check(L.lh_debug_task_bench(ctx.h, kind, R, 64, chain, P._lib.host_ptr(out)), ctx.h)
        print(f"{name:14s} {'chain' if chain else 'indep'}: wall {out[0]:8.2f} us/task, body {out[1]:8.2f} us",
              flush=True)
