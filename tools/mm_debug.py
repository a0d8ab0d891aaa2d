"""Multi-RHS propagator steps on the cfg4 operator at a given n and K; checks against K single-RHS
runs (debugging aid).  python tools/mm_debug.py n K"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_08324_b200 as P

n, K = int(sys.argv[1]), int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "both"
s = P.FracCNSystem(P.power_measure(1, 0.5), 0.0, 0.0, 0.0, n, 1.0 / n)
s.prepare(P.HConfig(n_min=64, eps1=1e-10), 1e-10, method="propagator")
F, Hm, L = s.factor, s.h_minus, P._lib.lib()
U = np.random.default_rng(0).standard_normal((s.N, K))
u = torch.from_numpy(np.asfortranarray(U).T.copy()).cuda()
if mode != "single":
    P._lib.check(L.lh_cn_steps(Hm.ctx.h, Hm.handle, F.h.handle, u.data_ptr(), s.N, K, 2, 2), Hm.ctx.h)
    torch.cuda.synchronize()
    print("multi ok", flush=True)
Y = u.cpu().numpy().T
v = torch.from_numpy(U[:, 0].copy()).cuda()
P._lib.check(L.lh_cn_steps(Hm.ctx.h, Hm.handle, F.h.handle, v.data_ptr(), s.N, 1, 2, 2), Hm.ctx.h)
print("n", n, "K", K, "col0 rel", np.linalg.norm(Y[:, 0] - v.cpu().numpy()) / np.linalg.norm(v.cpu().numpy()))
