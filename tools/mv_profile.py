"""Build the cfg3 operator pair at full size (no factorisation) and run H-matvecs;
used under ncu to profile the streaming kernels.   python tools/mv_profile.py [n] [iters]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1812_08324_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 19
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = bench.CFG3
nu = P.cgmy_measure(1.0, 5.0, 10.0, 0.5)
s = P.FracCNSystem(nu, cfg["a"], cfg["b"], cfg["c"], n, cfg["dt"], L=cfg["L"], L_W=cfg["L_W"])
Hp, Hm = s.build_pair(P.HConfig(n_min=cfg["leaf"], eps1=cfg["eps1"]))
x = torch.rand(s.N, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
L = P._lib.lib()
torch.cuda.synchronize()
t = time.time()
for _ in range(iters):
    L.lh_hmat_matvec(Hm.ctx.h, Hm.handle, x.data_ptr(), s.N, y.data_ptr(), s.N, 1)
Hm.ctx.sync()
dt = (time.time() - t) / iters
st = P.memory_report(Hm)["stored_scalars"]
print(f"matvec {dt*1e3:.3f} ms, {8*st/dt/1e9:.0f} GB/s algorithmic (stored {st})")
