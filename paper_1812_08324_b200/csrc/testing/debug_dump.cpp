// Host-only export of the H-arithmetic task DAGs for a given partition, so the
// planner's semantics can be verified on the CPU (tests/plan_emulator.py) against
// the oracle.  No device memory is touched.
#include <cstdio>

#include "../abi_types.h"
#include "../plan_impl.h"
#include "../../../include/levyh_b200_testing.h"

namespace lh {
void triangle_layout(HMat &X, const HMat &F, bool lower, int kcap);
void block_layout(HMat &X, const HMat &F, int part, int kcap);
void task_bench(Ctx &ctx, int kind, int R, int k, bool chain, double *out);
void recomp_bench(Ctx &ctx, int m, int n, int K, int reps, const double *u, const double *v, double *out);
}

using namespace lh;

namespace {

void put_i64(FILE *f, int64_t v) { fwrite(&v, 8, 1, f); }

void dump_nodes(FILE *f, const HMat &H) {
    put_i64(f, (int64_t)H.leafblocks.size());
    put_i64(f, H.arena_len);
    put_i64(f, H.nslots);
    put_i64(f, H.perm_len);
    for (int32_t b : H.leafblocks) {
        const Node &n = H.nodes[b];
        int64_t rec[11] = {n.r0, n.r0 + n.m, n.c0, n.c0 + n.n, n.kind, n.doff, n.uoff, n.voff,
                           n.kcap, n.rslot, n.poff};
        fwrite(rec, 8, 11, f);
    }
}

void view_ints(const DView &v, int64_t *o) {
    o[0] = v.off;
    o[1] = v.rows;
    o[2] = v.cols;
    o[3] = v.ld;
    o[4] = v.wslot;
    o[5] = v.base;
    o[6] = v.trans;
}

void dump_plan(FILE *f, const Plan &P) {
    put_i64(f, (int64_t)P.tasks.size());
    put_i64(f, (int64_t)P.deps.size());
    put_i64(f, (int64_t)P.pieces.size());
    put_i64(f, P.temp_len);
    put_i64(f, P.nslots_total);
    put_i64(f, P.slot_off_x);
    put_i64(f, P.rhs_slot);
    for (const DTask &t : P.tasks) {
        int64_t o[8 + 28];
        o[0] = t.type;
        o[1] = t.flags;
        o[2] = t.path;
        o[3] = t.aux;
        o[4] = t.dep_beg;
        o[5] = t.dep_cnt;
        o[6] = t.pc_beg;
        o[7] = t.pc_end;
        for (int k = 0; k < 4; ++k) view_ints(t.v[k], o + 8 + 7 * k);
        fwrite(o, 8, 36, f);
        double d[2] = {t.alpha, t.alpha2};
        fwrite(d, 8, 2, f);
    }
    for (int32_t d : P.deps) put_i64(f, d);
    for (const DPiece &p : P.pieces) {
        int64_t o[15];
        o[0] = p.kind;
        view_ints(p.mat, o + 1);
        view_ints(p.x, o + 8);
        fwrite(o, 8, 15, f);
    }
}

}  // namespace

extern "C" int lh_debug_dump_plans(const lh_tree *rt, const lh_tree *ct, int n_min, int n_block,
                                   double eta, int kcap_f, int kcap_x, const char *path) {
    try {
        HMat F;
        partition(F, *rt->t, *ct->t, n_min, n_block, eta);
        i64 off = 0;
        int32_t slots = 0;
        for (int32_t b : F.leafblocks) {
            Node &nd = F.nodes[b];
            if (nd.kind == K_DENSE) {
                nd.doff = off;
                off += nd.m * nd.n;
            }
        }
        for (int32_t b : F.leafblocks) {
            Node &nd = F.nodes[b];
            if (nd.kind == K_LR) {
                nd.kcap = kcap_f;
                nd.rslot = slots++;
                nd.uoff = off;
                off += nd.m * kcap_f;
                nd.voff = off;
                off += nd.n * kcap_f;
            }
        }
        F.arena_len = off;
        F.nslots = slots;
        FILE *f = fopen(path, "wb");
        if (!f) return LH_EINVAL;
        put_i64(f, 0x4c48504c414e31LL);  // "LHPLAN1"
        dump_nodes(f, F);                   // F before factorisation (dense kinds)
        i64 perm_len = 0;
        auto Plu = plan_hlu(F, 1e-10, perm_len);
        F.perm_len = perm_len;
        dump_nodes(f, F);                   // F after planning (FDENSE + perm offsets)
        dump_plan(f, *Plu);
        F.factored = true;
        auto Ps = plan_solve(F, F.nrows, 4);
        dump_plan(f, *Ps);
        for (int mode = 0; mode < 2; ++mode) {
            HMat X;
            triangle_layout(X, F, mode == 0, kcap_x);
            dump_nodes(f, X);
            auto Pi = plan_inverse(F, X, mode, 1e-10);
            dump_plan(f, *Pi);
        }
        {
            HMat Z;
            block_layout(Z, F, 2, kcap_x);
            dump_nodes(f, Z);
            auto Pz = plan_propagator(F, Z, 1e-10);
            dump_plan(f, *Pz);
        }
        fclose(f);
        return LH_OK;
    } catch (const std::exception &e) {
        fprintf(stderr, "lh_debug_dump_plans: %s\n", e.what());
        return LH_EINTERNAL;
    }
}

// Host-only planner timing on a partition: out[0] H-LU plan seconds, out[1] its tasks,
// out[2] propagator plan seconds (column-split, from mark_lu_leaves), out[3] its tasks.
extern "C" int lh_debug_plan_timing(const lh_tree *rt, const lh_tree *ct, int n_min, int n_block,
                                    double eta, int kcap_f, int kcap_x, int which, double *out) {
    try {
        HMat F;
        partition(F, *rt->t, *ct->t, n_min, n_block, eta);
        i64 off = 0;
        int32_t slots = 0;
        for (int32_t b : F.leafblocks) {
            Node &nd = F.nodes[b];
            if (nd.kind == K_DENSE) {
                nd.doff = off;
                off += nd.m * nd.n;
            }
        }
        for (int32_t b : F.leafblocks) {
            Node &nd = F.nodes[b];
            if (nd.kind == K_LR) {
                nd.kcap = kcap_f;
                nd.rslot = slots++;
                nd.uoff = off;
                off += nd.m * kcap_f;
                nd.voff = off;
                off += nd.n * kcap_f;
            }
        }
        F.arena_len = off;
        F.nslots = slots;
        refine_dense_leaves(F);
        for (int k = 0; k < 10; ++k) out[k] = 0.0;
        HMat G = F;  // structure copies for the two planners
        G.d_arena = nullptr;
        G.d_ranks = nullptr;
        if (which & 1) {
            i64 pl = 0;
            auto P = plan_hlu(F, 1e-10, pl);
            out[0] = P->build_seconds;
            out[1] = (double)P->tasks.size();
            out[4] = 8.0 * (double)P->temp_len;
            out[7] = plan_device_bytes(*P);
        }
        if (which & 2) {
            i64 pl = 0, il = 0;
            mark_lu_leaves(G, pl, il);
            G.factored = true;
            HMat Z;
            block_layout(Z, G, 2, kcap_x);
            auto Pz = plan_propagator(G, Z, 1e-10);
            out[2] = Pz->build_seconds;
            out[3] = (double)Pz->tasks.size();
            out[5] = 8.0 * (double)Pz->temp_len;
            out[6] = 8.0 * (double)Z.arena_len;
            out[8] = plan_device_bytes(*Pz);
            out[9] = 8.0 * (double)F.arena_len;
        }
        F.d_arena = nullptr;
        return LH_OK;
    } catch (const std::exception &e) {
        fprintf(stderr, "lh_debug_plan_timing: %s\n", e.what());
        return LH_EINTERNAL;
    }
}

// executor / recompression micro-benchmarks (lu.cu: task_bench, recomp_bench)
template <class F>
static int tguard(lh_ctx *ctx, F &&f) {
    try {
        f();
        return LH_OK;
    } catch (const lh::Error &e) {
        if (ctx) ctx->c.last_error = e.what();
        return e.code;
    } catch (const std::exception &e) {
        if (ctx) ctx->c.last_error = e.what();
        return LH_EINTERNAL;
    }
}

extern "C" int lh_debug_task_bench(lh_ctx *ctx, int kind, int R, int k, int chain, double *out) {
    return tguard(ctx, [&] { task_bench(ctx->c, kind, R, k, chain != 0, out); });
}

extern "C" int lh_debug_recomp_bench(lh_ctx *ctx, int m, int n, int K, int reps, const double *u,
                                     const double *v, double *out) {
    return tguard(ctx, [&] { recomp_bench(ctx->c, m, n, K, reps, u, v, out); });
}
