"""Sharded assembly (SURVEY 8(e), cfg5 phase 1): W ranks each compress a share of the
admissible blocks and exchange packed factors.  Emulated here in one process (W shards
built on one GPU, buffers handed over directly, as the all-gather would); every finalized
shard must equal the unsharded build bit for bit, and solve the same CN problem."""
import ctypes as C

import numpy as np
import pytest
import torch

from tests import cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1812_08324_b200 as P
    return P


def _content(H, P):
    """(structure, per-block stored values) with only the meaningful U/V columns."""
    recs, arena, ranks, _ = P.hmatrix.export_layout(H)
    out = []
    for rec in recs:
        r0, r1, c0, c1, kind, doff, uoff, voff, kcap, slot, _ = (int(v) for v in rec)
        m, n = r1 - r0, c1 - c0
        if kind == 2:
            r = int(ranks[slot])
            out.append((kind, r, arena[uoff:uoff + m * r].copy(), arena[voff:voff + n * r].copy()))
        else:
            out.append((kind, -1, arena[doff:doff + m * n].copy(), None))
    return recs[:, :5].copy(), out


def _sharded(P, t, ct, cfg, world):
    L = P._lib.lib()
    ctx = P._lib.Context.get()
    shards, bufs = [], []
    for q in range(world):
        h = C.c_void_p()
        P._lib.check(L.lh_hmat_build_toeplitz_shard(ctx.h, ct.handle, ct.handle, C.c_void_p(t.data_ptr()),
                                                    C.byref(cfg.native()), q, world, C.byref(h)), ctx.h)
        H = P.HMatrix(h, ct, ct, cfg.eta, ctx, cfg)
        n = C.c_int64(0)
        P._lib.check(L.lh_hmat_shard_pack(ctx.h, H.handle, None, 0, C.byref(n)), ctx.h)
        buf = torch.empty(max(n.value, 1), dtype=torch.float64, device="cuda")
        P._lib.check(L.lh_hmat_shard_pack(ctx.h, H.handle, C.c_void_p(buf.data_ptr()), buf.numel(),
                                          C.byref(n)), ctx.h)
        shards.append(H)
        bufs.append(buf[:n.value])
    for q, H in enumerate(shards):
        for src, b in enumerate(bufs):
            P._lib.check(L.lh_hmat_shard_unpack(ctx.h, H.handle, src, C.c_void_p(b.data_ptr()), b.numel()),
                         ctx.h)
        P._lib.check(L.lh_hmat_shard_finalize(ctx.h, H.handle), ctx.h)
    return shards


@pytest.mark.parametrize("name,world", [("cfg3_cgmy", 2), ("cfg2_s075", 3), ("cfg5_leaf128", 4)])
def test_sharded_build_bit_exact(P, name, world):
    g = cases.load(name)
    s = cases.make_system(name, g)
    cfg = P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"]))
    ct = s.cluster_tree(cfg.n_min)
    full = P.build_toeplitz(s.tPlus, ct, ct, cfg)
    st_f, val_f = _content(full, P)
    for H in _sharded(P, s.tPlus, ct, cfg, world):
        st, val = _content(H, P)
        assert np.array_equal(st, st_f)
        for a, b in zip(val, val_f):
            assert a[0] == b[0] and a[1] == b[1]
            assert np.array_equal(a[2], b[2])
            if a[3] is not None:
                assert np.array_equal(a[3], b[3])


def test_sharded_build_solves_cn(P):
    g = cases.load("cfg3_cgmy")
    s = cases.make_system("cfg3_cgmy", g)
    cfg = P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"]))
    ct = s.cluster_tree(cfg.n_min)
    Hp = _sharded(P, s.tPlus, ct, cfg, 2)[1]
    Hm = P.derive_toeplitz(Hp, s.tMinus, lr_scale=-1.0, kcap=0)
    s.h_minus, s.factor, s.method = Hm, P.hlu(Hp, float(g["eps2"])), "propagator"
    s.factor.prepare_propagator()
    u = P.run_cn(s, g["u0"], int(g["n_steps"]))
    assert np.linalg.norm(u - g["uT"]) <= 1e-8 * np.linalg.norm(g["uT"])


@pytest.mark.parametrize("name,stages", [("cfg3_cgmy", 1), ("cfg3_cgmy_n8191", 4), ("cfg5_leaf128", 3)])
def test_nccl_staged_build_bit_exact(P, name, stages):
    """The library's own NCCL communicator (lh_nccl_unique_id / lh_nccl_init, one rank on this
    GPU) and the staged, exchange-overlapped sharded build (lh_hmat_build_toeplitz_nccl): the
    same partition, ranks and factor bits as the single-GPU build; lh_bcast_factors from rank 0
    leaves it unchanged."""
    ctx = P._lib.Context.get()
    if not ctx.nccl_ready():
        uid = (C.c_char * 128)()
        P._lib.check(P._lib.lib().lh_nccl_unique_id(C.cast(uid, C.c_void_p)))
        P._lib.check(P._lib.lib().lh_nccl_init(ctx.h, 0, 1, C.cast(uid, C.c_void_p)), ctx.h)
    g = cases.load(name)
    s = cases.make_system(name, g)
    cfg = P.HConfig(n_min=int(g["leaf"]), eps1=float(g["eps1"]))
    ct = s.cluster_tree(cfg.n_min)
    full = P.build_toeplitz(s.tPlus, ct, ct, cfg)
    st_f, val_f = _content(full, P)
    H = P.build_toeplitz_nccl(s.tPlus, ct, ct, cfg, stages=stages)
    assert H.shard_stats["bytes_sent"] > 0
    for Hx in (H, P.bcast_factors(H, 0)):
        st, val = _content(Hx, P)
        assert np.array_equal(st, st_f)
        for a, b in zip(val, val_f):
            assert a[0] == b[0] and a[1] == b[1]
            assert np.array_equal(a[2], b[2])
            if a[3] is not None:
                assert np.array_equal(a[3], b[3])
