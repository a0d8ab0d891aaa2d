// C-ABI of the B200 H-matrix engine (include/levyh_b200.h).
#include <atomic>
#include <cstdlib>
#include <cstring>

#include <sys/mman.h>

#include "abi_types.h"
#include "core.h"
#include "matvec.h"
#include "plan_impl.h"

namespace lh {
void cn_symbol(Ctx &ctx, const lh_measure &m, const lh_cn_params &p, double *tA, double *tP,
               double *tM, double *sums_host);
void build_toeplitz(Ctx &ctx, HMat &H, const double *t, const lh_hconfig &cfg);
void frac_apply_1d(Ctx &ctx, const lh_measure &m, double h, i64 M, i64 K, double rho_r, double tail, double m2,
                   const double *u, const double *far, int part, double *out, double *sums_host);
void frac_apply_2d(Ctx &ctx, double c, double s, const double *table, double h, i64 M, i64 K, double rho_r,
                   double tail, double m2, const double *u, const double *far, double *out, double *sums_host);
void assemble_variable_order(Ctx &ctx, int n, i64 m, const int32_t *cells_host, const double *s_host, double L_W,
                             double rho_r, const double *gl16, const double *gl64, double *A, double *rowinfo_host);
void cn2d_dense(Ctx &ctx, i64 N, int nx, double h, double eps_sq, double scale, double a, double b, double c,
                double lam, double dt, int which, const int64_t *order_host, double *out_dev);
void build_toeplitz_nccl(Ctx &ctx, HMat &H, const double *t, const lh_hconfig &cfg, int stages, double *stats);
void build_gauss_series(Ctx &ctx, HMat &H, const double *t, const double *xr, const double *yc,
                        double eps_sq, double scale, int fixed_rank, double delta,
                        const lh_hconfig &cfg);
int gauss_series_terms(double eps_sq, double D, int fixed_rank, double delta);
void build_gauss_series_2d(Ctx &ctx, HMat &H, const double *xr, const double *yc, double eps_sq, double scale,
                           int fixed_rank, double delta, const lh_hconfig &cfg, const lh_cn2d_entries *ent);
void gauss_cn_symbol(Ctx &ctx, i64 N, double h, double eps_sq, double scale, i64 n_off, double a,
                     double b, double c, double dt, double *tA, double *tP, double *tM,
                     double *lam_host);
void build_dense(Ctx &ctx, HMat &H, const double *A, i64 lda, int row_major, const lh_hconfig &cfg);
void derive(Ctx &ctx, const HMat &S, HMat &D, const double *t, double scale, int kcap);
void hlu(Ctx &ctx, HMat &H, double eps2);
void solve(Ctx &ctx, HMat &F, double *b, i64 ldb, int nrhs, int method);
void prepare_inverse(Ctx &ctx, HMat &F, double eps2);
void cn_steps(Ctx &ctx, HMat &Hm, HMat &F, double *u, i64 ldu, int nrhs, int nsteps, int method);
void cn_step_host(Ctx &ctx, HMat &Hm, HMat &F, const double *u_in, double *u_out, int method);
void step_profile(Ctx &ctx, HMat &Hm, HMat &F, double *u, int iters, int method, double *out);
void prepare_propagator(Ctx &ctx, HMat &F, double eps2);
void propagator_stats(HMat &F, double *out);
int step_graph_kernels(HMat &F);
void cn_last_path(HMat &F, int32_t *out);
void trisolve_dense(Ctx &ctx, HMat &T, int mode, bool unit, double *b, i64 ldb, int nrhs);
void trisolve_block(Ctx &ctx, HMat &T, HMat &X, int mode, bool unit, double eps2);
void build_toeplitz_shard(Ctx &ctx, HMat &H, const double *t, const lh_hconfig &cfg, int rank,
                          int world);
i64 shard_pack(Ctx &ctx, HMat &H, double *buf, i64 cap);
void shard_unpack(Ctx &ctx, HMat &H, int src_rank, const double *buf, i64 len);
void shard_finalize(Ctx &ctx, HMat &H);
int lowrank_add_recompress(Ctx &ctx, i64 m, i64 n, const double *u1, const double *v1, int r1,
                           const double *u2, const double *v2, int r2, double eps2, double *uo,
                           double *vo);
void start_background_plans(HMat &H);
struct KOp {
    int kind = LH_OP_IDENTITY;
    HMat *h = nullptr;
    int method = 0;
    const double *a = nullptr;
    i64 lda = 0;
    lh_apply_fn fn = nullptr;
    void *user = nullptr;
};
void pcg(Ctx &ctx, const KOp &A, const KOp &M, const double *b, i64 n, double tol, int max_iter,
         double *x, double *res, int *iters, int *conv);
void gmres(Ctx &ctx, const KOp &A, const KOp &M, const double *b, i64 n, double tol, int restart,
           int max_iter, double *x, double *res, int *iters, int *conv);
void dense_gemv(Ctx &ctx, const double *A, i64 lda, i64 m, i64 n, const double *x, double *y);
void save_hmat(Ctx &ctx, HMat &H, double eps2, const char *path);
void load_hmat(Ctx &ctx, const char *path, HMat &H, std::shared_ptr<Tree> &rt,
               std::shared_ptr<Tree> &ct, double &eps2);

double *DevBuf::ensure(i64 n) {
    if (n > cap) {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        p = dalloc<double>(n);
        cap = n;
    }
    return p;
}
DevBuf::~DevBuf() {
    if (p) cudaFree(p);
}

void *Ctx::ensure_scratch(size_t bytes) {
    if (bytes > scratch_bytes) {
        if (scratch) {
            cudaStreamSynchronize(stream);
            cudaFree(scratch);
        }
        scratch = nullptr;
        LH_CUDA(cudaMalloc(&scratch, bytes));
        scratch_bytes = bytes;
    }
    return scratch;
}
Ctx::~Ctx() {
    if (scratch) cudaFree(scratch);
    if (owns_stream) cudaStreamDestroy(stream);
}
uint64_t next_hmat_id() {
    static std::atomic<uint64_t> ctr{1};
    return ctr.fetch_add(1);
}

HMat::~HMat() {
    mv_plan.reset();
    solve_plan.reset();
    inv_plan.reset();
    if (d_arena) cudaFree(d_arena);
    if (d_ranks) cudaFree(d_ranks);
    if (d_perm) cudaFree(d_perm);
    if (d_inv) cudaFree(d_inv);
    if (h_spill) std::free(h_spill);
}
void spill_arena(HMat &H, cudaStream_t s) {
    if (H.h_spill || !H.d_arena) return;
    LH_REQUIRE(!H.shard, LH_EINVAL, "cannot spill an H-matrix with a pending sharded assembly");
    {  // refuse rather than push the host into swap / the OOM killer: keep half of it free
        long long avail_kb = -1;
        if (FILE *f = fopen("/proc/meminfo", "r")) {
            char key[64];
            long long v = 0;
            while (fscanf(f, "%63s %lld kB\n", key, &v) == 2)
                if (!strcmp(key, "MemAvailable:")) {
                    avail_kb = v;
                    break;
                }
            fclose(f);
        }
        const double need = 8.0 * (double)H.arena_len;
        LH_REQUIRE(avail_kb < 0 || need <= 0.5 * 1024.0 * (double)avail_kb, LH_ENOMEM,
                   "spill: not enough available host memory for the arena");
    }
    // pageable host memory on transparent huge pages (pinning tens of GB page by page costs
    // more than the driver's staged copies)
    const size_t bytes = sizeof(double) * (size_t)std::max<i64>(H.arena_len, 1);
    const size_t HP = (size_t)2 << 20;
    double *hp = static_cast<double *>(std::aligned_alloc(HP, (bytes + HP - 1) / HP * HP));
    LH_REQUIRE(hp != nullptr, LH_ENOMEM, "spill: host allocation failed");
    madvise(hp, (bytes + HP - 1) / HP * HP, MADV_HUGEPAGE);
    cudaError_t e = cudaMemcpyAsync(hp, H.d_arena, sizeof(double) * (size_t)H.arena_len, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        std::free(hp);
        LH_CUDA(e);
    }
    H.mv_plan.reset();
    cudaFree(H.d_arena);
    H.d_arena = nullptr;
    H.h_spill = hp;
    ++H.gen;
}
void ensure_resident(HMat &H, cudaStream_t s) {
    if (!H.h_spill) return;
    double *d = dalloc<double>(std::max<i64>(H.arena_len, 1));
    cudaError_t e = cudaMemcpyAsync(d, H.h_spill, sizeof(double) * (size_t)H.arena_len, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        cudaFree(d);
        LH_CUDA(e);
    }
    std::free(H.h_spill);
    H.h_spill = nullptr;
    H.d_arena = d;
    ++H.gen;
}
void HMat::sync_ranks(cudaStream_t s) {
    h_ranks.assign(std::max(nslots, 0), 0);
    if (nslots > 0) {
        LH_CUDA(cudaMemcpyAsync(h_ranks.data(), d_ranks, sizeof(int32_t) * nslots,
                                cudaMemcpyDeviceToHost, s));
        LH_CUDA(cudaStreamSynchronize(s));
    }
}
}  // namespace lh

using namespace lh;

template <class F>
static int guard(lh_ctx *ctx, F &&f) {
    try {
        f();
        return LH_OK;
    } catch (const lh::Error &e) {
        if (ctx) ctx->c.last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc &) {
        if (ctx) ctx->c.last_error = "host allocation failed";
        return LH_ENOMEM;
    } catch (const std::exception &e) {
        if (ctx) ctx->c.last_error = e.what();
        return LH_EINTERNAL;
    }
}

// the H-matrix with its arena on the device (brings a spilled arena back first)
static HMat &resident(lh_ctx *ctx, const lh_hmat *h) {
    HMat &H = const_cast<HMat &>(h->h);
    ensure_resident(H, ctx->c.stream);
    return H;
}

static void check_cfg(const lh_hconfig *cfg) {
    LH_REQUIRE(cfg != nullptr, LH_EINVAL, "null HConfig");
    LH_REQUIRE(cfg->n_block >= 2, LH_EINVAL, "n_block must be >= 2");
    LH_REQUIRE(cfg->n_min >= 1, LH_EINVAL, "n_min must be >= 1");
    LH_REQUIRE(cfg->eta > 0, LH_EINVAL, "eta must be positive");
}

extern "C" {

int lh_version(void) { return 1; }

int lh_ctx_create(int device, void *stream, lh_ctx **out) {
    lh_ctx *c = new lh_ctx();
    int rc = guard(c, [&] {
        LH_CUDA(cudaSetDevice(device));
        c->c.device = device;
        c->c.stream = (cudaStream_t)stream;
        if (c->c.stream == nullptr) {
            // the legacy default stream cannot be graph-captured; a blocking stream still
            // orders implicitly with work that callers put on the legacy default stream
            LH_CUDA(cudaStreamCreate(&c->c.stream));
            c->c.owns_stream = true;
        }
        int sms = 0;
        LH_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        c->c.num_sms = sms;
    });
    if (rc != LH_OK) {
        // keep the context so the caller can read the message
    }
    *out = c;
    return rc;
}

void lh_ctx_destroy(lh_ctx *ctx) { delete ctx; }

const char *lh_ctx_last_error(const lh_ctx *ctx) { return ctx ? ctx->c.last_error.c_str() : ""; }

void *lh_ctx_stream(const lh_ctx *ctx) { return ctx ? (void *)ctx->c.stream : nullptr; }

int lh_ctx_synchronize(lh_ctx *ctx) {
    return guard(ctx, [&] { LH_CUDA(cudaStreamSynchronize(ctx->c.stream)); });
}

int lh_tree_build(lh_ctx *ctx, const double *pts, int64_t n, int dim, int leaf_size, lh_tree **out) {
    return guard(ctx, [&] {
        std::shared_ptr<Tree> t(build_tree(pts, n, dim, leaf_size));
        lh_tree *o = new lh_tree();
        o->t = t;
        *out = o;
    });
}

int lh_tree_build_strategy(lh_ctx *ctx, const double *pts, int64_t n, int dim, int leaf_size, int strategy,
                           lh_tree **out) {
    return guard(ctx, [&] {
        std::shared_ptr<Tree> t(build_tree(pts, n, dim, leaf_size, strategy));
        lh_tree *o = new lh_tree();
        o->t = t;
        *out = o;
    });
}

void lh_tree_destroy(lh_tree *t) { delete t; }

int64_t lh_tree_num_nodes(const lh_tree *t) { return (int64_t)t->t->nodes.size(); }

int lh_tree_nodes(const lh_tree *t, int64_t *lohi, double *bbox, int32_t *kids) {
    const Tree &T = *t->t;
    for (size_t i = 0; i < T.nodes.size(); ++i) {
        const Cluster &c = T.nodes[i];
        if (lohi) {
            lohi[2 * i] = c.lo;
            lohi[2 * i + 1] = c.hi;
        }
        if (bbox)
            for (int d = 0; d < T.dim; ++d) {
                bbox[(2 * i) * T.dim + d] = c.blo[d];
                bbox[(2 * i + 1) * T.dim + d] = c.bhi[d];
            }
        if (kids) {
            kids[2 * i] = c.kid[0];
            kids[2 * i + 1] = c.kid[1];
        }
    }
    return LH_OK;
}

int lh_tree_order(const lh_tree *t, int64_t *order) {
    std::memcpy(order, t->t->order.data(), sizeof(int64_t) * t->t->order.size());
    return LH_OK;
}

int lh_partition(const lh_tree *rt, const lh_tree *ct, int n_min, int n_block, double eta,
                 int64_t *recs, int64_t *nblocks, int64_t *nhier) {
    return guard(nullptr, [&] {
        HMat H;
        partition(H, *rt->t, *ct->t, n_min, n_block, eta);
        int64_t nh = 0;
        for (const Node &nd : H.nodes) nh += nd.kind == K_HIER;
        if (nblocks) *nblocks = (int64_t)H.leafblocks.size();
        if (nhier) *nhier = nh;
        if (recs)
            for (size_t k = 0; k < H.leafblocks.size(); ++k) {
                const Node &nd = H.nodes[H.leafblocks[k]];
                int64_t *r = recs + 5 * k;
                r[0] = nd.r0;
                r[1] = nd.r0 + nd.m;
                r[2] = nd.c0;
                r[3] = nd.c0 + nd.n;
                r[4] = nd.kind == K_LR ? 1 : 0;
            }
    });
}

int lh_plan_stats(const lh_tree *rt, const lh_tree *ct, int n_min, int n_block, double eta,
                  int kcap, double *stats) {
    return guard(nullptr, [&] {
        HMat H;
        partition(H, *rt->t, *ct->t, n_min, n_block, eta);
        i64 off = 0;
        int32_t slots = 0;
        for (int32_t b : H.leafblocks) {
            Node &nd = H.nodes[b];
            if (nd.kind == K_DENSE) {
                nd.doff = off;
                off += nd.m * nd.n;
            } else if (nd.kind == K_LR) {
                nd.kcap = kcap;
                nd.rslot = slots++;
                nd.uoff = off;
                off += nd.m * kcap;
                nd.voff = off;
                off += nd.n * kcap;
            }
        }
        H.nslots = slots;
        i64 pl = 0;
        auto P = plan_hlu(H, 1e-10, pl);
        stats[0] = (double)P->tasks.size();
        stats[1] = (double)P->deps.size();
        stats[2] = (double)P->temp_len;
        stats[3] = P->build_seconds;
        stats[7] = (double)critical_path(*P);
        H.factored = true;
        auto S = plan_solve(H, H.nrows, 1);
        stats[4] = (double)S->tasks.size();
        stats[5] = (double)S->deps.size();
        stats[6] = (double)critical_path(*S);
    });
}

static lh_hmat *new_hmat(const lh_tree *rt, const lh_tree *ct) {
    lh_hmat *o = new lh_hmat();
    o->h.rt_hold = rt->t;
    o->h.ct_hold = ct->t;
    return o;
}

int lh_hmat_build_toeplitz_shard(lh_ctx *ctx, const lh_tree *rt, const lh_tree *ct,
                                 const double *t_dev, const lh_hconfig *cfg, int32_t rank,
                                 int32_t world, lh_hmat **out) {
    lh_hmat *o = nullptr;
    int rc = guard(ctx, [&] {
        check_cfg(cfg);
        o = new_hmat(rt, ct);
        partition(o->h, *rt->t, *ct->t, cfg->n_min, cfg->n_block, cfg->eta);
        build_toeplitz_shard(ctx->c, o->h, t_dev, *cfg, rank, world);
        start_background_plans(o->h);  // plans depend on the partition only
    });
    if (rc != LH_OK) {
        delete o;
        o = nullptr;
    }
    *out = o;
    return rc;
}

int lh_hmat_shard_pack(lh_ctx *ctx, lh_hmat *h, double *buf_dev, int64_t cap, int64_t *len) {
    return guard(ctx, [&] { *len = shard_pack(ctx->c, resident(ctx, h), buf_dev, cap); });
}

int lh_hmat_shard_unpack(lh_ctx *ctx, lh_hmat *h, int32_t src_rank, const double *buf_dev,
                         int64_t len) {
    return guard(ctx, [&] { shard_unpack(ctx->c, h->h, src_rank, buf_dev, len); });
}

int lh_hmat_shard_finalize(lh_ctx *ctx, lh_hmat *h) {
    return guard(ctx, [&] { shard_finalize(ctx->c, h->h); });
}

int lh_hmat_build_gauss_series(lh_ctx *ctx, const lh_tree *rt, const lh_tree *ct, const double *t_dev,
                               const double *row_pts_dev, const double *col_pts_dev, double eps_sq,
                               double scale, int fixed_rank, double delta, const lh_hconfig *cfg,
                               lh_hmat **out) {
    lh_hmat *o = nullptr;
    int rc = guard(ctx, [&] {
        check_cfg(cfg);
        LH_REQUIRE(row_pts_dev && col_pts_dev, LH_EINVAL, "series builder needs the tree-order points");
        o = new_hmat(rt, ct);
        partition(o->h, *rt->t, *ct->t, cfg->n_min, cfg->n_block, cfg->eta);
        build_gauss_series(ctx->c, o->h, t_dev, row_pts_dev, col_pts_dev, eps_sq, scale, fixed_rank,
                           delta, *cfg);
        start_background_plans(o->h);
    });
    if (rc != LH_OK) {
        delete o;
        o = nullptr;
    }
    *out = o;
    return rc;
}

int lh_hmat_build_gauss_series_2d(lh_ctx *ctx, const lh_tree *rt, const lh_tree *ct,
                                  const double *row_pts_dev, const double *col_pts_dev, double eps_sq,
                                  double scale, int fixed_rank, double delta, const lh_hconfig *cfg,
                                  const lh_cn2d_entries *entries, lh_hmat **out) {
    lh_hmat *o = nullptr;
    int rc = guard(ctx, [&] {
        check_cfg(cfg);
        LH_REQUIRE(row_pts_dev && col_pts_dev, LH_EINVAL, "series builder needs the tree-order points");
        o = new_hmat(rt, ct);
        partition(o->h, *rt->t, *ct->t, cfg->n_min, cfg->n_block, cfg->eta);
        build_gauss_series_2d(ctx->c, o->h, row_pts_dev, col_pts_dev, eps_sq, scale, fixed_rank, delta, *cfg,
                              entries);
        start_background_plans(o->h);
    });
    if (rc != LH_OK) {
        delete o;
        o = nullptr;
    }
    *out = o;
    return rc;
}

int lh_gauss_series_terms(double eps_sq, double diameter, int fixed_rank, double delta) {
    return gauss_series_terms(eps_sq, diameter, fixed_rank, delta);
}

int lh_gauss_cn_symbol(lh_ctx *ctx, int64_t N, double h, double eps_sq, double scale, int64_t n_off,
                       double a, double b, double c, double dt, double *tA_dev, double *tPlus_dev,
                       double *tMinus_dev, double *lam_host) {
    return guard(ctx, [&] {
        gauss_cn_symbol(ctx->c, N, h, eps_sq, scale, n_off, a, b, c, dt, tA_dev, tPlus_dev,
                        tMinus_dev, lam_host);
    });
}

int lh_cn2d_dense(lh_ctx *ctx, int64_t N, int32_t nx, double h, double eps_sq, double scale, double a,
                  double b, double c, double lam, double dt, int32_t which, const int64_t *order_host,
                  double *out_dev) {
    return guard(ctx, [&] { cn2d_dense(ctx->c, N, nx, h, eps_sq, scale, a, b, c, lam, dt, which, order_host, out_dev); });
}

int lh_hmat_build_toeplitz(lh_ctx *ctx, const lh_tree *rt, const lh_tree *ct, const double *t_dev,
                           const lh_hconfig *cfg, lh_hmat **out) {
    lh_hmat *o = nullptr;
    int rc = guard(ctx, [&] {
        check_cfg(cfg);
        o = new_hmat(rt, ct);
        partition(o->h, *rt->t, *ct->t, cfg->n_min, cfg->n_block, cfg->eta);
        build_toeplitz(ctx->c, o->h, t_dev, *cfg);
        start_background_plans(o->h);
    });
    if (rc != LH_OK) {
        delete o;
        o = nullptr;
    }
    *out = o;
    return rc;
}

int lh_nccl_unique_id(void *uid128_host) {
    return guard(nullptr, [&] { nccl_unique_id(uid128_host); });
}

int lh_nccl_init(lh_ctx *ctx, int32_t rank, int32_t world, const void *uid128_host) {
    return guard(ctx, [&] { nccl_init(ctx->c, rank, world, uid128_host); });
}

int lh_nccl_ready(lh_ctx *ctx) { return nccl_ready(ctx->c) ? 1 : 0; }

int lh_hmat_build_toeplitz_nccl(lh_ctx *ctx, const lh_tree *rt, const lh_tree *ct, const double *t_dev,
                                const lh_hconfig *cfg, int32_t stages, double *stats_host, lh_hmat **out) {
    lh_hmat *o = nullptr;
    int rc = guard(ctx, [&] {
        check_cfg(cfg);
        o = new_hmat(rt, ct);
        partition(o->h, *rt->t, *ct->t, cfg->n_min, cfg->n_block, cfg->eta);
        build_toeplitz_nccl(ctx->c, o->h, t_dev, *cfg, stages, stats_host);
        start_background_plans(o->h);
    });
    if (rc != LH_OK) {
        delete o;
        o = nullptr;
    }
    *out = o;
    return rc;
}

int lh_bcast_factors(lh_ctx *ctx, lh_hmat *h, int32_t root) {
    return guard(ctx, [&] { bcast_hmat(ctx->c, h->h, root); });
}

int lh_hmat_build_dense(lh_ctx *ctx, const lh_tree *rt, const lh_tree *ct, const double *A_dev,
                        int64_t lda, int row_major, const lh_hconfig *cfg, lh_hmat **out) {
    lh_hmat *o = nullptr;
    int rc = guard(ctx, [&] {
        check_cfg(cfg);
        o = new_hmat(rt, ct);
        partition(o->h, *rt->t, *ct->t, cfg->n_min, cfg->n_block, cfg->eta);
        build_dense(ctx->c, o->h, A_dev, lda, row_major, *cfg);
        start_background_plans(o->h);
    });
    if (rc != LH_OK) {
        delete o;
        o = nullptr;
    }
    *out = o;
    return rc;
}

int lh_hmat_derive_toeplitz(lh_ctx *ctx, const lh_hmat *src, const double *t_dev, double lr_scale,
                            int32_t kcap, lh_hmat **out) {
    lh_hmat *o = nullptr;
    int rc = guard(ctx, [&] {
        o = new lh_hmat();
        derive(ctx->c, resident(ctx, src), o->h, t_dev, lr_scale, kcap);
    });
    if (rc != LH_OK) {
        delete o;
        o = nullptr;
    }
    *out = o;
    return rc;
}

int lh_hmat_clone(lh_ctx *ctx, const lh_hmat *src, int32_t kcap, lh_hmat **out) {
    lh_hmat *o = nullptr;
    int rc = guard(ctx, [&] {
        o = new lh_hmat();
        derive(ctx->c, resident(ctx, src), o->h, nullptr, 1.0, kcap);
    });
    if (rc != LH_OK) {
        delete o;
        o = nullptr;
    }
    *out = o;
    return rc;
}

void lh_hmat_destroy(lh_hmat *h) { delete h; }

int64_t lh_hmat_num_blocks(const lh_hmat *h) { return (int64_t)h->h.leafblocks.size(); }

int lh_hmat_spill(lh_ctx *ctx, lh_hmat *h) {
    return guard(ctx, [&] {
        HMat &H = h->h;
        LH_REQUIRE(!H.factored && !H.solve_plan && !H.inv_plan, LH_EINVAL,
                   "only an unfactored H-matrix without solve plans can be spilled");
        spill_arena(H, ctx->c.stream);
    });
}

int lh_hmat_resident(const lh_hmat *h) { return h->h.h_spill ? 0 : 1; }

int lh_hmat_structure(lh_ctx *ctx, const lh_hmat *h, int64_t *recs) {
    return guard(ctx, [&] {
        const HMat &H = h->h;
        const_cast<HMat &>(H).sync_ranks(ctx->c.stream);
        for (size_t k = 0; k < H.leafblocks.size(); ++k) {
            const Node &nd = H.nodes[H.leafblocks[k]];
            int64_t *r = recs + 6 * k;
            r[0] = nd.r0;
            r[1] = nd.r0 + nd.m;
            r[2] = nd.c0;
            r[3] = nd.c0 + nd.n;
            r[4] = nd.kind == K_LR ? 1 : (nd.kind == K_FDENSE ? 2 : 0);
            r[5] = nd.kind == K_LR ? H.h_ranks[nd.rslot] : -1;
        }
    });
}

int lh_hmat_memory(lh_ctx *ctx, const lh_hmat *h, int64_t *stats) {
    return guard(ctx, [&] {
        const HMat &H = h->h;
        const_cast<HMat &>(H).sync_ranks(ctx->c.stream);
        int64_t nd_ = 0, nl = 0, sc = 0, nh = 0;
        for (const Node &nd : H.nodes) {
            if (nd.vpar >= 0) continue;  // virtual children of refined leaves
            if (nd.kind == K_HIER) {
                ++nh;
            } else if (nd.kind == K_LR) {
                ++nl;
                sc += (int64_t)H.h_ranks[nd.rslot] * (nd.m + nd.n);
            } else {
                ++nd_;
                sc += nd.m * nd.n;
            }
        }
        stats[0] = nd_;
        stats[1] = nl;
        stats[2] = sc;
        stats[3] = nh;
    });
}

int lh_hmat_entry(lh_ctx *ctx, const lh_hmat *h, int64_t i, int64_t j, double *out) {
    return guard(ctx, [&] {
        const HMat &H = resident(ctx, h);
        LH_REQUIRE(i >= 0 && i < H.nrows && j >= 0 && j < H.ncols, LH_EINVAL, "entry outside the matrix");
        int32_t b = H.root;
        while (H.nodes[b].kind == K_HIER) {  // refined dense leaves keep their leaf kind
            const Node &nd = H.nodes[b];
            const int q = (i - nd.r0 >= nd.rs ? 2 : 0) + (j - nd.c0 >= nd.cs ? 1 : 0);
            b = nd.kid[q];
        }
        const Node &nd = H.nodes[b];
        LH_REQUIRE(nd.kind != K_FDENSE, LH_ETYPE, "cannot read an entry of an LU-factored leaf");
        cudaStream_t s = ctx->c.stream;
        const i64 li = i - nd.r0, lj = j - nd.c0;
        if (nd.kind == K_LR) {
            int32_t r = 0;
            LH_CUDA(cudaMemcpyAsync(&r, H.d_ranks + nd.rslot, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
            LH_CUDA(cudaStreamSynchronize(s));
            std::vector<double> u(std::max(r, 1)), v(std::max(r, 1));
            if (r > 0) {
                LH_CUDA(cudaMemcpy2DAsync(u.data(), sizeof(double), H.d_arena + nd.uoff + li,
                                          sizeof(double) * nd.m, sizeof(double), r, cudaMemcpyDeviceToHost, s));
                LH_CUDA(cudaMemcpy2DAsync(v.data(), sizeof(double), H.d_arena + nd.voff + lj,
                                          sizeof(double) * nd.n, sizeof(double), r, cudaMemcpyDeviceToHost, s));
                LH_CUDA(cudaStreamSynchronize(s));
            }
            double acc = 0.0;
            for (int c = 0; c < r; ++c) acc += u[c] * v[c];
            *out = acc;
        } else {
            LH_REQUIRE(nd.kind == K_DENSE, LH_ETYPE, "entry in a structurally zero block");
            LH_CUDA(cudaMemcpyAsync(out, H.d_arena + nd.doff + li + lj * nd.m, sizeof(double),
                                    cudaMemcpyDeviceToHost, s));
            LH_CUDA(cudaStreamSynchronize(s));
        }
    });
}

int lh_hmat_export_block(lh_ctx *ctx, const lh_hmat *h, int64_t block, double *a, double *b) {
    return guard(ctx, [&] {
        const HMat &H = resident(ctx, h);
        LH_REQUIRE(block >= 0 && block < (int64_t)H.leafblocks.size(), LH_EINVAL, "block index");
        const Node &nd = H.nodes[H.leafblocks[block]];
        cudaStream_t s = ctx->c.stream;
        if (nd.kind == K_LR) {
            const_cast<HMat &>(H).sync_ranks(s);
            int r = H.h_ranks[nd.rslot];
            if (a && r)
                LH_CUDA(cudaMemcpyAsync(a, H.d_arena + nd.uoff, sizeof(double) * nd.m * r,
                                        cudaMemcpyDeviceToHost, s));
            if (b && r)
                LH_CUDA(cudaMemcpyAsync(b, H.d_arena + nd.voff, sizeof(double) * nd.n * r,
                                        cudaMemcpyDeviceToHost, s));
        } else {
            if (a)
                LH_CUDA(cudaMemcpyAsync(a, H.d_arena + nd.doff, sizeof(double) * nd.m * nd.n,
                                        cudaMemcpyDeviceToHost, s));
            if (b && nd.kind == K_FDENSE) {
                std::vector<int32_t> p(nd.m);
                LH_CUDA(cudaMemcpyAsync(p.data(), H.d_perm + nd.poff, sizeof(int32_t) * nd.m,
                                        cudaMemcpyDeviceToHost, s));
                LH_CUDA(cudaStreamSynchronize(s));
                for (i64 i = 0; i < nd.m; ++i) b[i] = (double)p[i];
            }
        }
        LH_CUDA(cudaStreamSynchronize(s));
    });
}

int lh_hmat_layout(const lh_hmat *h, int64_t *recs, int64_t *sizes) {
    const HMat &H = h->h;
    if (sizes) {
        sizes[0] = H.arena_len;
        sizes[1] = H.nslots;
        sizes[2] = H.perm_len;
    }
    if (recs)
        for (size_t k = 0; k < H.leafblocks.size(); ++k) {
            const Node &n = H.nodes[H.leafblocks[k]];
            int64_t *r = recs + 11 * k;
            r[0] = n.r0;
            r[1] = n.r0 + n.m;
            r[2] = n.c0;
            r[3] = n.c0 + n.n;
            r[4] = n.kind;
            r[5] = n.doff;
            r[6] = n.uoff;
            r[7] = n.voff;
            r[8] = n.kcap;
            r[9] = n.rslot;
            r[10] = n.poff;
        }
    return LH_OK;
}

int lh_hmat_export_arena(lh_ctx *ctx, const lh_hmat *h, double *arena, int32_t *ranks,
                         int32_t *perm) {
    return guard(ctx, [&] {
        const HMat &H = resident(ctx, h);
        cudaStream_t s = ctx->c.stream;
        if (arena && H.arena_len)
            LH_CUDA(cudaMemcpyAsync(arena, H.d_arena, sizeof(double) * H.arena_len,
                                    cudaMemcpyDeviceToHost, s));
        if (ranks && H.nslots)
            LH_CUDA(cudaMemcpyAsync(ranks, H.d_ranks, sizeof(int32_t) * H.nslots,
                                    cudaMemcpyDeviceToHost, s));
        if (perm && H.perm_len)
            LH_CUDA(cudaMemcpyAsync(perm, H.d_perm, sizeof(int32_t) * H.perm_len,
                                    cudaMemcpyDeviceToHost, s));
        LH_CUDA(cudaStreamSynchronize(s));
        if (perm && H.perm_len) {
            // a refined leaf factored as 64-row halves: its net permutation is the halves'
            // permutations, each offset by the half's first row in the leaf
            for (int32_t b : H.leafblocks) {
                const Node &nd = H.nodes[b];
                if (nd.kind != K_FDENSE || nd.kid[0] < 0) continue;
                std::vector<int32_t> st{b};
                while (!st.empty()) {
                    const Node &q = H.nodes[st.back()];
                    st.pop_back();
                    if (q.kid[0] >= 0) {
                        st.push_back(q.kid[3]);
                        st.push_back(q.kid[0]);
                    } else if (q.r0 > nd.r0) {
                        for (i64 i = 0; i < q.m; ++i) perm[q.poff + i] += (int32_t)(q.r0 - nd.r0);
                    }
                }
            }
        }
    });
}

int lh_hmat_matvec(lh_ctx *ctx, const lh_hmat *h, const double *x, int64_t ldx, double *y,
                   int64_t ldy, int32_t nrhs) {
    return guard(ctx, [&] { matvec(ctx->c, resident(ctx, h), x, ldx, y, ldy, nrhs); });
}

int lh_hlu(lh_ctx *ctx, lh_hmat *h, double eps2) {
    return guard(ctx, [&] { hlu(ctx->c, resident(ctx, h), eps2); });
}

int lh_solve(lh_ctx *ctx, lh_hmat *f, double *b, int64_t ldb, int32_t nrhs, int32_t method) {
    return guard(ctx, [&] { solve(ctx->c, f->h, b, ldb, nrhs, method); });
}

int lh_prepare_inverse(lh_ctx *ctx, lh_hmat *f, double eps2) {
    return guard(ctx, [&] { prepare_inverse(ctx->c, f->h, eps2); });
}

int lh_prepare_propagator(lh_ctx *ctx, lh_hmat *f, double eps2) {
    return guard(ctx, [&] { prepare_propagator(ctx->c, f->h, eps2); });
}

int lh_propagator_stats(lh_hmat *f, double *out) {
    return guard(nullptr, [&] { propagator_stats(f->h, out); });
}

int32_t lh_step_graph_kernels(lh_hmat *f) { return step_graph_kernels(f->h); }

int lh_cn_last_path(lh_hmat *f, int32_t *out) {
    return guard(nullptr, [&] { cn_last_path(f->h, out); });
}

int lh_trisolve_dense(lh_ctx *ctx, lh_hmat *t, int32_t mode, int32_t unit, double *b, int64_t ldb,
                      int32_t nrhs) {
    return guard(ctx, [&] { trisolve_dense(ctx->c, resident(ctx, t), mode, unit != 0, b, ldb, nrhs); });
}

int lh_trisolve_block(lh_ctx *ctx, lh_hmat *t, const lh_hmat *b, int32_t mode, int32_t unit, double eps2,
                      lh_hmat **out) {
    lh_hmat *o = nullptr;
    int rc = guard(ctx, [&] {
        LH_REQUIRE(mode == 0 || mode == 2, LH_EINVAL, "block right-hand sides: mode 0 (L X = B) or 2 (X U = B)");
        LH_REQUIRE(!(mode == 2 && unit), LH_EINVAL, "unit_diagonal right solves are not supported on blocks");
        LH_REQUIRE(!b->h.factored, LH_EINVAL, "right-hand side must not be LU-factored");
        LH_REQUIRE(b->h.nrows == t->h.nrows && b->h.ncols == t->h.ncols && b->h.rt == t->h.rt &&
                       b->h.ct == t->h.ct,
                   LH_EINVAL, "block right-hand side must share the triangle's cluster trees");
        o = new lh_hmat();
        derive(ctx->c, resident(ctx, b), o->h, nullptr, 1.0, 32);  // deep copy (hops.py:294, :307)
        trisolve_block(ctx->c, resident(ctx, t), o->h, mode, unit != 0, eps2);
    });
    if (rc != LH_OK) {
        delete o;
        o = nullptr;
    }
    *out = o;
    return rc;
}

int lh_lowrank_add_recompress(lh_ctx *ctx, int64_t m, int64_t n, const double *u1, const double *v1,
                              int32_t r1, const double *u2, const double *v2, int32_t r2,
                              double eps2, double *u_out, double *v_out, int32_t *r_out) {
    return guard(ctx, [&] {
        *r_out = lowrank_add_recompress(ctx->c, m, n, u1, v1, r1, u2, v2, r2, eps2, u_out, v_out);
    });
}

int lh_cn_steps(lh_ctx *ctx, const lh_hmat *hm, lh_hmat *f, double *u, int64_t ldu, int32_t nrhs,
                int32_t nsteps, int32_t method) {
    return guard(ctx, [&] {
        cn_steps(ctx->c, const_cast<HMat &>(hm->h), f->h, u, ldu, nrhs, nsteps, method);
    });
}

int lh_cn_step_host(lh_ctx *ctx, const lh_hmat *hm, lh_hmat *f, const double *u_in_host,
                    double *u_out_host, int32_t method) {
    return guard(ctx, [&] {
        LH_REQUIRE(u_in_host && u_out_host, LH_EINVAL, "cn_step_host: null vector");
        cn_step_host(ctx->c, const_cast<HMat &>(hm->h), f->h, u_in_host, u_out_host, method);
    });
}

int lh_step_profile(lh_ctx *ctx, const lh_hmat *hm, lh_hmat *f, double *u, int32_t iters,
                    int32_t method, double *out) {
    return guard(ctx, [&] {
        step_profile(ctx->c, const_cast<HMat &>(hm->h), f->h, u, iters, method, out);
    });
}

int lh_hlu_stats(const lh_hmat *f, double *out) {
    for (int k = 0; k < 5; ++k) out[k] = f->h.lu_stats[k];
    out[5] = f->h.lu_stats[6];
    out[6] = f->h.lu_stats[7];
    return LH_OK;
}

int lh_hmat_save(lh_ctx *ctx, const lh_hmat *h, double eps2, const char *path) {
    return guard(ctx, [&] {
        LH_REQUIRE(h != nullptr && path != nullptr, LH_EINVAL, "save: null argument");
        save_hmat(ctx->c, resident(ctx, h), eps2, path);
    });
}

int lh_hmat_load(lh_ctx *ctx, const char *path, lh_tree **rt_out, lh_tree **ct_out, lh_hmat **out,
                 int32_t *factored, double *eps2) {
    lh_hmat *o = nullptr;
    lh_tree *r = nullptr, *c = nullptr;
    int rc = guard(ctx, [&] {
        LH_REQUIRE(path != nullptr, LH_EINVAL, "load: null path");
        o = new lh_hmat();
        r = new lh_tree();
        c = new lh_tree();
        double e = 0;
        load_hmat(ctx->c, path, o->h, r->t, c->t, e);
        *factored = o->h.factored ? 1 : 0;
        *eps2 = e;
        start_background_plans(o->h);  // no-op for a factor
    });
    if (rc != LH_OK) {
        delete o;
        delete r;
        delete c;
        o = nullptr;
        r = c = nullptr;
    }
    *out = o;
    *rt_out = r;
    *ct_out = c;
    return rc;
}

int lh_tree_points(const lh_tree *t, double *pts_host) {
    const Tree &T = *t->t;
    if (pts_host) std::memcpy(pts_host, T.pts.data(), sizeof(double) * T.pts.size());
    return T.dim;
}

static KOp resolve_op(const lh_operator *op) {
    KOp k;
    if (!op) return k;
    k.kind = op->kind;
    k.h = op->hmat ? &op->hmat->h : nullptr;
    k.method = op->method;
    k.a = op->a_dev;
    k.lda = op->lda;
    k.fn = op->fn;
    k.user = op->user;
    return k;
}

int lh_pcg(lh_ctx *ctx, const lh_operator *A, const lh_operator *Minv, const double *b, int64_t n,
           double tol, int32_t max_iter, double *x, double *res, int32_t *iters, int32_t *conv) {
    return guard(ctx, [&] {
        LH_REQUIRE(A != nullptr, LH_EINVAL, "pcg: null operator");
        LH_REQUIRE(n >= 0 && max_iter >= 0, LH_EINVAL, "pcg: negative size or iteration count");
        int it = 0, cv = 0;
        try {
            pcg(ctx->c, resolve_op(A), resolve_op(Minv), b, n, tol, max_iter, x, res, &it, &cv);
        } catch (...) {
            *iters = it;
            *conv = cv;
            throw;
        }
        *iters = it;
        *conv = cv;
    });
}

int lh_gmres_restarted(lh_ctx *ctx, const lh_operator *A, const lh_operator *Minv, const double *b,
                       int64_t n, double tol, int32_t restart, int32_t max_iter, double *x,
                       double *res, int32_t *iters, int32_t *conv) {
    return guard(ctx, [&] {
        LH_REQUIRE(A != nullptr, LH_EINVAL, "gmres: null operator");
        LH_REQUIRE(n >= 0 && max_iter >= 0, LH_EINVAL, "gmres: negative size or iteration count");
        int it = 0, cv = 0;
        gmres(ctx->c, resolve_op(A), resolve_op(Minv), b, n, tol, restart, max_iter, x, res, &it, &cv);
        *iters = it;
        *conv = cv;
    });
}

int lh_dense_gemv(lh_ctx *ctx, const double *a, int64_t lda, int64_t m, int64_t n, const double *x,
                  double *y) {
    return guard(ctx, [&] {
        LH_REQUIRE(m >= 0 && n >= 0 && lda >= n, LH_EINVAL, "dense_gemv: bad shape");
        dense_gemv(ctx->c, a, lda, m, n, x, y);
    });
}

int lh_cn_symbol(lh_ctx *ctx, const lh_measure *nu, const lh_cn_params *p, double *tA, double *tP,
                 double *tM, double *sums_host) {
    return guard(ctx, [&] { cn_symbol(ctx->c, *nu, *p, tA, tP, tM, sums_host); });
}

int lh_frac_apply_1d(lh_ctx *ctx, const lh_measure *nu, double h, int64_t M, int64_t K, double rho_r,
                     double tail, double m2, const double *u_dev, const double *far_dev, int32_t part,
                     double *out_dev, double *sums_host) {
    return guard(ctx, [&] {
        LH_REQUIRE(nu && u_dev && out_dev, LH_EINVAL, "null argument");
        frac_apply_1d(ctx->c, *nu, h, M, K, rho_r, tail, m2, u_dev, far_dev, part, out_dev, sums_host);
    });
}

int lh_frac_apply_2d(lh_ctx *ctx, double c, double s, const double *table_dev, double h, int64_t M,
                     int64_t K, double rho_r, double tail, double m2, const double *u_dev,
                     const double *far_dev, double *out_dev, double *sums_host) {
    return guard(ctx, [&] {
        LH_REQUIRE(u_dev && out_dev, LH_EINVAL, "null argument");
        frac_apply_2d(ctx->c, c, s, table_dev, h, M, K, rho_r, tail, m2, u_dev, far_dev, out_dev, sums_host);
    });
}

int lh_assemble_variable_order(lh_ctx *ctx, int32_t n, int64_t m, const int32_t *cells_host,
                               const double *s_host, double L_W, double rho_r, const double *gl16_host,
                               const double *gl64_host, double *A_dev, double *rowinfo_host) {
    return guard(ctx, [&] {
        LH_REQUIRE(cells_host && s_host && gl16_host && gl64_host && A_dev, LH_EINVAL, "null argument");
        assemble_variable_order(ctx->c, n, m, cells_host, s_host, L_W, rho_r, gl16_host, gl64_host, A_dev,
                                rowinfo_host);
    });
}

}  // extern "C"
