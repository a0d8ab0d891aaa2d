"""CPU emulator of the B200 H-arithmetic task DAG (TEST INFRASTRUCTURE ONLY).

Reads the plans exported by ``lh_debug_dump_plans`` and executes every task in
plan order with numpy, with the semantics of the device tasks in
paper_1812_08324_b200/csrc/lu.cu.  Used to check the planner (the replay of the
reference recursion, dependency order, views, temporaries) against the oracle
without a GPU.  The product never uses this file.
"""
from __future__ import annotations

import struct

import numpy as np
import scipy.linalg as sla

(T_GETRF, T_TRSM, T_SEGMUL, T_VTX, T_LRADD, T_DGEMM, T_DADD, T_DENSIFY, T_IDENT, T_NOP, T_RAND,
 T_ORTH, T_CHECK) = range(1, 14)
B_F, B_TMP, B_RHS, B_X = range(4)
KC = 32
KC_MAX = 32


class Reader:
    def __init__(self, path):
        self.b = open(path, "rb").read()
        self.p = 0

    def i64(self, n=None):
        if n is None:
            v = struct.unpack_from("<q", self.b, self.p)[0]
            self.p += 8
            return v
        a = np.frombuffer(self.b, dtype="<i8", count=n, offset=self.p).copy()
        self.p += 8 * n
        return a

    def f64(self, n):
        a = np.frombuffer(self.b, dtype="<f8", count=n, offset=self.p).copy()
        self.p += 8 * n
        return a

    def nodes(self):
        nb = self.i64()
        arena, nslots, perm_len = self.i64(), self.i64(), self.i64()
        recs = self.i64(11 * nb).reshape(nb, 11)
        return dict(recs=recs, arena=arena, nslots=nslots, perm_len=perm_len)

    def plan(self):
        nt, nd, npc = self.i64(), self.i64(), self.i64()
        temp_len, nslots_total, slot_off_x, rhs_slot = self.i64(), self.i64(), self.i64(), self.i64()
        ints = np.empty((nt, 36), dtype=np.int64)
        dbl = np.empty((nt, 2))
        for t in range(nt):
            ints[t] = self.i64(36)
            dbl[t] = self.f64(2)
        deps = self.i64(nd)
        pcs = self.i64(15 * npc).reshape(npc, 15)
        return dict(ints=ints, dbl=dbl, deps=deps, pieces=pcs, temp_len=temp_len,
                    nslots_total=nslots_total, slot_off_x=slot_off_x, rhs_slot=rhs_slot)


def load(path):
    r = Reader(path)
    assert r.i64() == 0x4c48504c414e31
    out = {"F0": r.nodes(), "F": r.nodes(), "lu": r.plan(), "solve": r.plan()}
    out["XL"] = r.nodes()
    out["invL"] = r.plan()
    out["XU"] = r.nodes()
    out["invU"] = r.plan()
    out["Z"] = r.nodes()
    out["prop"] = r.plan()
    return out


class View:
    __slots__ = ("off", "rows", "cols", "ld", "wslot", "base", "trans")

    def __init__(self, a):
        self.off, self.rows, self.cols, self.ld, self.wslot, self.base, self.trans = (int(x) for x in a)


class Machine:
    def __init__(self, bases, ranks, perm):
        self.bases = bases
        self.ranks = ranks
        self.perm = perm

    def ncols(self, v):
        return int(self.ranks[v.wslot]) if v.wslot >= 0 else v.cols

    def idx(self, v, rows, cols):
        i = np.arange(rows)[:, None]
        j = np.arange(cols)[None, :]
        return v.off + (j + i * v.ld if v.trans else i + j * v.ld)

    def get(self, v, rows=None, cols=None):
        rows = v.rows if rows is None else rows
        cols = self.ncols(v) if cols is None else cols
        return self.bases[v.base][self.idx(v, rows, cols)]

    def put(self, v, val):
        rows, cols = val.shape
        self.bases[v.base][self.idx(v, rows, cols)] = val

    def run(self, plan, rng):
        ints, dbl, pcs = plan["ints"], plan["dbl"], plan["pieces"]
        for t in range(ints.shape[0]):
            row = ints[t]
            typ, flags, path, aux = (int(x) for x in row[:4])
            pc_beg, pc_end = int(row[6]), int(row[7])
            v = [View(row[8 + 7 * k: 15 + 7 * k]) for k in range(4)]
            alpha, alpha2 = dbl[t]
            if typ == T_GETRF:
                A = self.get(v[0])
                lu, piv = sla.lu_factor(A, check_finite=False)
                self.put(v[0], lu)
                m = A.shape[0]
                p = np.arange(m)
                for i, q in enumerate(piv):
                    if q != i:
                        p[i], p[q] = p[q], p[i]
                self.perm[aux:aux + m] = p
                if np.any(np.diag(lu) == 0):
                    raise np.linalg.LinAlgError(f"path {path}")
            elif typ == T_TRSM:
                m = v[0].rows
                T = self.get(v[0], m, m)
                B = self.get(v[1])
                if B.shape[1] == 0:
                    continue
                mode, unit = flags & 15, bool(flags & 16)
                if flags & 128 and np.any(np.diag(T) == 0):
                    raise np.linalg.LinAlgError(f"path {path}")
                if mode == 0:
                    if flags & 32:
                        B = B[self.perm[aux:aux + m]]
                    X = sla.solve_triangular(T, B, lower=True, unit_diagonal=unit)
                elif mode == 1:
                    X = sla.solve_triangular(T, B, lower=False, unit_diagonal=unit)
                else:
                    X = sla.solve_triangular(T, B, lower=False, trans="T", unit_diagonal=unit)
                self.put(v[1], X)
            elif typ == T_SEGMUL:
                Y = self.get(v[0])
                acc = np.zeros_like(Y)
                k = Y.shape[1]
                for p in range(pc_beg, pc_end):
                    kind = int(pcs[p, 0])
                    mv, xv = View(pcs[p, 1:8]), View(pcs[p, 8:15])
                    if kind == 0:
                        M = self.get(mv, mv.rows, mv.cols)
                        X = self.get(xv, mv.cols, k)
                    else:
                        r = self.ncols(mv)
                        M = self.get(mv, mv.rows, r)
                        X = self.get(xv, r, k)
                    acc += M @ X
                self.put(v[0], (0.0 if flags & 1 else Y) + alpha * acc)
            elif typ == T_VTX:
                F = self.get(v[0])
                X = self.get(v[1])
                r, k = F.shape[1], X.shape[1]
                if r and k:
                    self.put(v[2], F.T @ X)
            elif typ == T_LRADD:
                cu, cv, u2, v2 = v
                r2 = self.ncols(u2)
                if r2 == 0:
                    continue
                r1 = int(self.ranks[cu.wslot])
                K = r1 + r2
                assert K <= cu.cols and K <= 48, "rank capacity"
                U = np.hstack([self.get(cu, cu.rows, r1), alpha * self.get(u2)])
                V = np.hstack([self.get(cv, cv.rows, r1), self.get(v2)])
                qu, ru = np.linalg.qr(U)
                qv, rv = np.linalg.qr(V)
                w, s, zt = np.linalg.svd(ru @ rv.T)
                sq = s * s
                tot = np.sqrt(sq.sum())
                if tot == 0:
                    r = 0
                else:
                    tails = np.sqrt(np.concatenate([np.cumsum(sq[::-1])[::-1], [0.0]]))
                    r = int(np.argmax(tails <= alpha2 * tot))
                assert r <= min(cu.cols, KC_MAX)
                if r:
                    self.put(cu, qu @ (w[:, :r] * s[:r]))
                    self.put(cv, qv @ zt[:r].T)
                self.ranks[cu.wslot] = r
            elif typ == T_DGEMM:
                C = self.get(v[0])
                A = self.get(v[1])
                inner = A.shape[1]
                if flags & 1:
                    B = self.get(v[2], v[0].cols, inner).T
                else:
                    B = self.get(v[2], inner, v[0].cols)
                self.put(v[0], (0.0 if flags & 2 else C) + alpha * (A @ B))
            elif typ == T_DADD:
                C = self.get(v[0])
                self.put(v[0], C + alpha * self.get(v[1], v[0].rows, v[0].cols))
            elif typ == T_DENSIFY:
                if flags & 1:
                    U = self.get(v[1])
                    V = self.get(v[2], v[0].cols, U.shape[1])
                    self.put(v[0], U @ V.T)
                else:
                    self.put(v[0], self.get(v[1], v[0].rows, v[0].cols))
            elif typ == T_IDENT:
                k = self.ncols(v[0])
                self.put(v[0], np.zeros((v[0].rows, k)) if flags & 1 else np.eye(v[0].rows, k))
            elif typ == T_RAND:
                self.put(v[0], rng.standard_normal((v[0].rows, v[0].cols)))
            elif typ == T_ORTH:
                Y = self.get(v[0])
                q, _ = np.linalg.qr(Y)
                self.put(v[0], q)
            elif typ == T_NOP:
                pass
            elif typ == T_CHECK:
                assert np.abs(self.get(v[0])).max() <= alpha, f"cross-half pivot (path {path})"
            else:
                raise ValueError(f"unknown task type {typ}")


def fill_from_oracle(layout, oracle_root, leaves_fn):
    """Arena + ranks from an oracle block tree with the same partition."""
    recs = layout["recs"]
    arena = np.zeros(max(layout["arena"], 1))
    ranks = np.zeros(max(layout["nslots"], 1), dtype=np.int64)
    blocks = leaves_fn(oracle_root)
    assert len(blocks) == recs.shape[0]
    for (blk, r0, c0), rec in zip(blocks, recs):
        R0, R1, C0, C1, kind, doff, uoff, voff, kcap, rslot, poff = (int(x) for x in rec)
        assert (r0, c0) == (R0, C0)
        m, n = R1 - R0, C1 - C0
        if blk.kind == "R":
            r = blk.u.shape[1]
            arena[uoff + np.arange(m)[:, None] + np.arange(r)[None, :] * m] = blk.u
            arena[voff + np.arange(n)[:, None] + np.arange(r)[None, :] * n] = blk.v
            ranks[rslot] = r
        else:
            arena[doff + np.arange(m)[:, None] + np.arange(n)[None, :] * m] = blk.d
    return arena, ranks
