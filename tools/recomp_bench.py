"""Phase timing of the device recompression (QR, QR, Ru Rv^T, Jacobi SVD, apply) on inputs
shaped like the H-LU / propagator LRADD updates: [U1 U2][V1 V2]^T with both terms eps-truncated
approximations of smooth far-field blocks.  Usage: python tools/recomp_bench.py"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_1812_08324_b200 as P


def lowrank(G, eps, rmax):
    u, s, vt = np.linalg.svd(G, full_matrices=False)
    r = min(rmax, int(np.sum(s > eps * s[0])))
    return u[:, :r] * s[:r], vt[:r].T


def case(m, n, r_each):
    x = np.linspace(0, 1, m)
    y = np.linspace(2, 3, n)
    G1 = 1.0 / np.abs(x[:, None] - y[None, :]) ** 1.5
    G2 = 0.3 / np.abs(x[:, None] - y[None, :] - 0.1) ** 1.7
    U1, V1 = lowrank(G1, 1e-12, r_each)
    U2, V2 = lowrank(G2, 1e-12, r_each)
    return np.asfortranarray(np.hstack([U1, U2])), np.asfortranarray(np.hstack([V1, V2]))


ctx = P._lib.Context.get()
L = P._lib.testing()
names = ["stage", "qr_u", "qr_v", "C", "jacobi", "apply"]
for m, r_each in ((64, 7), (128, 9), (128, 11), (256, 11), (256, 16), (192, 11)):
    U, V = case(m, m, r_each)
    K = U.shape[1]
    out = np.zeros(8)
    P._lib.check(L.lh_debug_recomp_bench(ctx.h, m, m, K, 50, P._lib.host_ptr(U), P._lib.host_ptr(V),
                                         P._lib.host_ptr(out)), ctx.h)
    tot = out[:6].sum() / 1e3
    print(f"m=n={m:4d} K={K:2d} r={out[6]:.0f} sweeps={out[7]:.0f}: total {tot:7.1f} us  " +
          " ".join(f"{nm} {v / 1e3:6.1f}" for nm, v in zip(names, out[:6])), flush=True)
