"""Executor micro-benchmark (chains of synthetic tasks): python tools/task_bench.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1812_08324_b200 as P  # noqa: E402

ctx = P._lib.Context.get()
L = P._lib.testing()
out = np.zeros(2)
for kind, name in ((0, "GETRF"), (1, "TRSM"), (2, "SEGMUL")):
    for k in ((64,) if kind == 0 else (7, 64)):
        for chain in (1, 0):
            R = 2000 if chain else 20000
            P._lib.check(L.lh_debug_task_bench(ctx.h, kind, R, k, chain, P._lib.host_ptr(out)), ctx.h)
            print(f"{name:7s} k={k:3d} {'chain' if chain else 'indep'}: wall {out[0]:8.2f} us/task, body {out[1]:8.2f} us",
                  flush=True)
