import sys, os; sys.path.insert(0,'.')
import numpy as np, paper_1812_08324_b200 as P
g=dict(np.load('tests/golden/golden_2d.npz'))
cfg=P.HConfig(n_min=32, eps1=1e-6)
for method in ("substitution", "inverse", "propagator"):
    t=P.assemble_cn_2d(P.gaussian_measure(5.0),0.1,0.5,-0.2,P.UniformGrid2D(24,24),0.05)
    try:
        t.prepare(cfg, 1e-10, method=method)
        u=P.run_cn(t, g['cn2_u0'], 10)
        st=t.factor.h.structure_array(); print(method, 'ok', np.linalg.norm(u-g['cn2_uT_h'])/np.linalg.norm(g['cn2_uT_h']), 'max factor rank', st[st[:,4]==1,5].max())
    except Exception as e: print(method, 'ERR', e)
