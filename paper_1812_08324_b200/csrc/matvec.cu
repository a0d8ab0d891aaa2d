// H-matvec y = H x (hops.py:50-70) as a two-phase HBM-streaming kernel pair.
//
// Phase 1: for every low-rank block b, partial products t_b = V_b^T x over
//          fixed column chunks (deterministic; no atomics).
// Phase 2: one CTA per row segment (<= 64 rows of a leaf cluster) accumulates
//          every dense piece D x and every low-rank piece U_b[seg,:] t_b that
//          covers the segment, and writes y[seg] once.
// The same plan type serves the CN operator H-, and the triangular-inverse
// factors of the fast solve.
#include <algorithm>
#include <map>

#include "core.h"
#include "dev.cuh"
#include "matvec.h"

namespace lh {

using dev::KC_MAX;
using dev::NT;

constexpr int SEG = 64;         // rows per segment
constexpr int GRP = NT / SEG;   // thread groups per segment
constexpr i64 VCHUNK = 4096;    // rows of V per phase-1 chunk

__global__ void __launch_bounds__(NT) vtx_kernel(const VChunk *chunks, int nch, const double *arena,
                                                 const int *ranks, const double *x, double *part,
                                                 double beta_unused) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int q = blockIdx.x; q < nch; q += gridDim.x) {
        VChunk C = chunks[q];
        int r = ranks[C.slot];
        const double *V = arena + C.voff;
        const double *xx = x + C.xc0;
        for (int c = w; c < r; c += dev::NW) {
            const double *v = V + (i64)c * C.ld;
            double s0 = 0.0, s1 = 0.0;
            int i = lane;
            for (; i + 32 < C.len; i += 64) {
                s0 += v[i] * xx[i];
                s1 += v[i + 32] * xx[i + 32];
            }
            if (i < C.len) s0 += v[i] * xx[i];
            s0 = dev::warp_sum(s0 + s1);
            if (lane == 0) part[(i64)q * KC_MAX + c] = s0;
        }
    }
}

__global__ void __launch_bounds__(NT) seg_kernel(const SegDesc *segs, int nseg, const MvDense *dp,
                                                 const MvLr *lp, const double *arena,
                                                 const int *ranks, const double *part,
                                                 const double *x, double *y, double alpha,
                                                 double beta) {
    __shared__ double tb[KC_MAX];
    __shared__ double acc_s[GRP][SEG];
    const int row = threadIdx.x % SEG, g = threadIdx.x / SEG;
    for (int s = blockIdx.x; s < nseg; s += gridDim.x) {
        SegDesc S = segs[s];
        double acc = 0.0;
        // dense pieces: D[row, j] x[j], columns split over the GRP groups
        for (int p = S.dbeg; p < S.dend; ++p) {
            MvDense P = dp[p];
            if (row < S.rows) {
                const double *D = arena + P.off + row;
                const double *xx = x + P.xc0;
                double a0 = 0.0, a1 = 0.0;
                int j = g;
                for (; j + GRP < P.ncols; j += 2 * GRP) {
                    a0 += D[(i64)j * P.ld] * xx[j];
                    a1 += D[(i64)(j + GRP) * P.ld] * xx[j + GRP];
                }
                if (j < P.ncols) a0 += D[(i64)j * P.ld] * xx[j];
                acc += a0 + a1;
            }
        }
        // low-rank pieces: U[row, :] t_b with t_b = sum of the block's chunk partials
        for (int p = S.lbeg; p < S.lend; ++p) {
            MvLr P = lp[p];
            int r = ranks[P.slot];
            __syncthreads();
            if (threadIdx.x < r) {
                double t = 0.0;
                for (int c = P.cbeg; c < P.cend; ++c) t += part[(i64)c * KC_MAX + threadIdx.x];
                tb[threadIdx.x] = t;
            }
            __syncthreads();
            if (row < S.rows) {
                const double *U = arena + P.off + row;
                for (int c = g; c < r; c += GRP) acc += U[(i64)c * P.ld] * tb[c];
            }
        }
        acc_s[g][row] = acc;
        __syncthreads();
        if (g == 0 && row < S.rows) {
            double v = acc_s[0][row];
            for (int k = 1; k < GRP; ++k) v += acc_s[k][row];
            double *yy = y + S.y0 + row;
            *yy = (beta == 0.0 ? 0.0 : beta * *yy) + alpha * v;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// plan construction
// ---------------------------------------------------------------------------
// Builds a plan over the given leaf blocks (default: all of H).  Row segments are
// the leaf clusters of the row tree split into <= SEG rows.
std::shared_ptr<MvPlan> build_mv_plan(const HMat &H, const std::vector<int32_t> &blocks,
                                      cudaStream_t s) {
    auto P = std::make_shared<MvPlan>();
    const Tree &rt = *H.rt;
    // segments
    std::vector<i64> seg_start;
    for (int32_t lc : rt.leaves) {
        const Cluster &c = rt.nodes[lc];
        for (i64 a = c.lo; a < c.hi; a += SEG) seg_start.push_back(a);
    }
    seg_start.push_back(rt.n);
    int nseg = (int)seg_start.size() - 1;
    auto seg_of = [&](i64 row) {
        return (int)(std::upper_bound(seg_start.begin(), seg_start.end(), row) - seg_start.begin()) - 1;
    };
    std::vector<std::vector<MvDense>> dps(nseg);
    std::vector<std::vector<MvLr>> lps(nseg);
    std::vector<VChunk> chunks;
    for (int32_t b : blocks) {
        const Node &nd = H.nodes[b];
        if (nd.kind == K_DENSE || nd.kind == K_FDENSE) {
            for (int sg = seg_of(nd.r0); sg < nseg && seg_start[sg] < nd.r0 + nd.m; ++sg) {
                i64 a = std::max(seg_start[sg], nd.r0), e = std::min(seg_start[sg + 1], nd.r0 + nd.m);
                LH_REQUIRE(a == seg_start[sg] && e == seg_start[sg + 1], LH_EINTERNAL,
                           "dense block not aligned with row segments");
                dps[sg].push_back({nd.doff + (a - nd.r0), nd.m, nd.c0, (int32_t)nd.n});
            }
        } else if (nd.kind == K_LR) {
            int cb = (int)chunks.size();
            for (i64 a = 0; a < nd.n; a += VCHUNK) {
                int len = (int)std::min(VCHUNK, nd.n - a);
                chunks.push_back({nd.voff + a, nd.n, nd.c0 + a, len, nd.rslot});
            }
            int ce = (int)chunks.size();
            for (int sg = seg_of(nd.r0); sg < nseg && seg_start[sg] < nd.r0 + nd.m; ++sg) {
                i64 a = std::max(seg_start[sg], nd.r0), e = std::min(seg_start[sg + 1], nd.r0 + nd.m);
                LH_REQUIRE(a == seg_start[sg] && e == seg_start[sg + 1], LH_EINTERNAL,
                           "low-rank block not aligned with row segments");
                lps[sg].push_back({nd.uoff + (a - nd.r0), nd.m, nd.rslot, cb, ce});
            }
        }
    }
    std::vector<SegDesc> segs(nseg);
    std::vector<MvDense> dall;
    std::vector<MvLr> lall;
    for (int sg = 0; sg < nseg; ++sg) {
        SegDesc &S = segs[sg];
        S.y0 = seg_start[sg];
        S.rows = (int32_t)(seg_start[sg + 1] - seg_start[sg]);
        S.dbeg = (int32_t)dall.size();
        dall.insert(dall.end(), dps[sg].begin(), dps[sg].end());
        S.dend = (int32_t)dall.size();
        S.lbeg = (int32_t)lall.size();
        lall.insert(lall.end(), lps[sg].begin(), lps[sg].end());
        S.lend = (int32_t)lall.size();
    }
    P->nseg = nseg;
    P->nch = (int)chunks.size();
    P->segs = dupload(segs, s);
    P->dp = dupload(dall, s);
    P->lp = dupload(lall, s);
    P->chunks = dupload(chunks, s);
    P->part = dalloc<double>((i64)std::max(P->nch, 1) * KC_MAX);
    P->n_dpieces = (i64)dall.size();
    P->n_lpieces = (i64)lall.size();
    LH_CUDA(cudaStreamSynchronize(s));
    return P;
}

MvPlan::~MvPlan() {
    cudaFree(segs);
    cudaFree(dp);
    cudaFree(lp);
    cudaFree(chunks);
    cudaFree(part);
}

void mv_vtx_launch(const MvPlan &P, const HMat &H, const double *x, int grid, cudaStream_t s) {
    vtx_kernel<<<grid, NT, 0, s>>>(P.chunks, P.nch, H.d_arena, H.d_ranks, x, P.part, 0.0);
}

void mv_seg_launch(const MvPlan &P, const HMat &H, const double *x, double *y, double alpha,
                   double beta, cudaStream_t s, int num_sms) {
    int g2 = std::min(P.nseg, num_sms * 32);
    seg_kernel<<<g2, NT, 0, s>>>(P.segs, P.nseg, P.dp, P.lp, H.d_arena, H.d_ranks, P.part, x, y,
                                 alpha, beta);
}

// y = alpha * H x + beta * y  for one right-hand side
void mv_run(const MvPlan &P, const HMat &H, const double *x, double *y, double alpha, double beta,
            cudaStream_t s, int num_sms) {
    if (P.nch > 0) {
        int g1 = std::min(P.nch, num_sms * 16);
        vtx_kernel<<<g1, NT, 0, s>>>(P.chunks, P.nch, H.d_arena, H.d_ranks, x, P.part, 0.0);
    }
    int g2 = std::min(P.nseg, num_sms * 32);
    seg_kernel<<<g2, NT, 0, s>>>(P.segs, P.nseg, P.dp, P.lp, H.d_arena, H.d_ranks, P.part, x, y,
                                 alpha, beta);
    LH_CUDA(cudaGetLastError());
}

MvPlan &get_mv_plan(HMat &H, cudaStream_t s) {
    if (!H.mv_plan) {
        auto p = build_mv_plan(H, H.leafblocks, s);
        H.mv_plan = std::static_pointer_cast<void>(p);
    }
    return *static_cast<MvPlan *>(H.mv_plan.get());
}

void matvec(Ctx &ctx, HMat &H, const double *x, i64 ldx, double *y, i64 ldy, int nrhs) {
    LH_REQUIRE(!H.factored, LH_EINVAL, "matvec of an LU-factored H-matrix is not defined");
    MvPlan &P = get_mv_plan(H, ctx.stream);
    for (int q = 0; q < nrhs; ++q)
        mv_run(P, H, x + (i64)q * ldx, y + (i64)q * ldy, 1.0, 0.0, ctx.stream, ctx.num_sms);
}

}  // namespace lh
