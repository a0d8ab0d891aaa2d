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
constexpr i64 VCHUNK = 1024;    // rows of V per phase-1 chunk (one warp)
#ifndef SEG_MIN_BLOCKS
#define SEG_MIN_BLOCKS 4        // CTAs per SM for the segment kernel (5-6 spill and lose ~10%)
#endif

// Phase 1: each CTA owns one chunk of rows of one V_b; every thread accumulates all
// r columns for its rows (x[i] read once, r independent coalesced loads per row),
// then a CTA reduction writes the chunk's r partial sums.
template <int RB>
__device__ __forceinline__ void vtx_warp(const VChunk &C, int r, const double *arena, const double *x,
                                         double *out, int lane) {
    const double *V = arena + C.voff;
    const double *xx = x + C.xc0;
    double acc[RB];
#pragma unroll
    for (int c = 0; c < RB; ++c) acc[c] = 0.0;
    int i = lane;
    // two rows per iteration: 2 (r + 1) independent loads in flight before the FMAs
    for (; i + 32 < C.len; i += 64) {
        const double x0 = xx[i], x1 = xx[i + 32];
        double v0[RB], v1[RB];
#pragma unroll
        for (int c = 0; c < RB; ++c) {
            v0[c] = c < r ? V[i + (i64)c * C.ld] : 0.0;
            v1[c] = c < r ? V[i + 32 + (i64)c * C.ld] : 0.0;
        }
#pragma unroll
        for (int c = 0; c < RB; ++c) acc[c] += v0[c] * x0 + v1[c] * x1;
    }
    if (i < C.len) {
        const double xi = xx[i];
#pragma unroll
        for (int c = 0; c < RB; ++c)
            if (c < r) acc[c] += V[i + (i64)c * C.ld] * xi;
    }
#pragma unroll
    for (int c = 0; c < RB; ++c)
        if (c < r) {
            const double v = dev::warp_sum(acc[c]);
            if (lane == 0) out[c] = v;
        }
    // ranks above RB (stale plan or rare large ranks): remaining columns one at a time
    for (int c = RB; c < r; ++c) {
        const double *v = V + (i64)c * C.ld;
        double s = 0.0;
        for (int i = lane; i < C.len; i += 32) s += v[i] * xx[i];
        s = dev::warp_sum(s);
        if (lane == 0) out[c] = s;
    }
}

// Phase 1: one warp per chunk (<= VCHUNK rows of one V_b); each lane accumulates all r
// columns for its rows (x[i] read once, r independent coalesced loads per row), then
// warp shuffles reduce: no block barriers, so small blocks cost little.
// The plan splits chunks by the rank seen at plan time: RB = 8 (32-register kernel, 8 CTAs
// per SM) or RB = 16.  A chunk that covers its whole block writes t_b directly (C.out >= 0);
// chunks of multi-chunk blocks write partials, reduced by treduce_kernel.
template <int RB>
__global__ void __launch_bounds__(NT, (RB <= 8 ? 6 : 4))
    vtx_kernel(const VChunk *chunks, int nch, const double *arena, const int *ranks,
               const double *x, double *part, double *tvec) {
    const int lane = threadIdx.x & 31;
    for (int q = blockIdx.x * dev::NW + (threadIdx.x >> 5); q < nch; q += gridDim.x * dev::NW) {
        const VChunk C = chunks[q];
        const int r = ranks[C.slot];
        double *out = C.tout >= 0 ? tvec + C.tout : part + (i64)C.pidx * KC_MAX;
        vtx_warp<RB>(C, r, arena, x, out, lane);
    }
}

// t_b[c] = sum of the chunk partials of a multi-chunk block b (one warp per block,
// fixed order: deterministic)
__global__ void treduce_kernel(const TJob *jobs, int njobs, const int *ranks, const double *part,
                               double *tvec) {
    const int lane = threadIdx.x & 31;
    for (int j = blockIdx.x * dev::NW + (threadIdx.x >> 5); j < njobs; j += gridDim.x * dev::NW) {
        const TJob J = jobs[j];
        const int r = ranks[J.slot];
        for (int c = 0; c < r; ++c) {
            double t = 0.0;
            for (int k = J.cbeg + lane; k < J.cend; k += 32) t += part[(i64)k * KC_MAX + c];
            t = dev::warp_sum(t);
            if (lane == 0) tvec[(i64)J.slot * KC_MAX + c] = t;
        }
    }
}

__global__ void __launch_bounds__(NT, SEG_MIN_BLOCKS) seg_kernel(const SegDesc *segs, int nseg, const MvDense *dp,
                                                 const MvLr *lp, const double *arena,
                                                 const int *ranks, const double *tvec,
                                                 const double *x, double *y, double alpha,
                                                 double beta, const double *z) {
    __shared__ double acc_s[GRP][SEG];
    const int row = threadIdx.x % SEG, g = threadIdx.x / SEG;
    for (int s = blockIdx.x; s < nseg; s += gridDim.x) {
        const SegDesc S = segs[s];
        double acc = 0.0;
        if (row < S.rows) {
            // dense pieces: D[row, j] x[j], columns split over the GRP groups; a full
            // 64-column piece issues its 16 loads per thread before any FMA
            for (int p = S.dbeg; p < S.dend; ++p) {
                const MvDense P = dp[p];
                const double *D = arena + P.off + row;
                const double *xx = x + P.xc0;
                if (P.ncols == 64) {
                    double d[16], xv[16];
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        d[q] = D[(i64)(g + GRP * q) * P.ld];
                        xv[q] = xx[g + GRP * q];
                    }
                    double a0 = 0.0, a1 = 0.0;
#pragma unroll
                    for (int q = 0; q < 16; q += 2) {
                        a0 += d[q] * xv[q];
                        a1 += d[q + 1] * xv[q + 1];
                    }
                    acc += a0 + a1;
                } else {
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
            // low-rank pieces: U[row, :] t_b (t_b precomputed, read through L1); four
            // pieces at a time so their descriptor -> rank -> U load chains overlap
            int p = S.lbeg;
            for (; p + 4 <= S.lend; p += 4) {
                MvLr Q[4];
                int r[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) Q[k] = lp[p + k];
#pragma unroll
                for (int k = 0; k < 4; ++k) r[k] = ranks[Q[k].slot];
                double u0[4], u1[4], t0[4], t1[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double *U = arena + Q[k].off + row;
                    const double *tb = tvec + (i64)Q[k].slot * KC_MAX;
                    u0[k] = g < r[k] ? U[(i64)g * Q[k].ld] : 0.0;
                    t0[k] = g < r[k] ? tb[g] : 0.0;
                    u1[k] = g + GRP < r[k] ? U[(i64)(g + GRP) * Q[k].ld] : 0.0;
                    t1[k] = g + GRP < r[k] ? tb[g + GRP] : 0.0;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) acc += u0[k] * t0[k] + u1[k] * t1[k];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double *U = arena + Q[k].off + row;
                    const double *tb = tvec + (i64)Q[k].slot * KC_MAX;
                    for (int c = g + 2 * GRP; c < r[k]; c += GRP) acc += U[(i64)c * Q[k].ld] * tb[c];
                }
            }
            for (; p < S.lend; ++p) {
                const MvLr P = lp[p];
                const int r = ranks[P.slot];
                const double *U = arena + P.off + row;
                const double *tb = tvec + (i64)P.slot * KC_MAX;
                for (int c = g; c < r; c += GRP) acc += U[(i64)c * P.ld] * tb[c];
            }
        }
        acc_s[g][row] = acc;
        __syncthreads();
        if (g == 0 && row < S.rows) {
            double v = acc_s[0][row];
            for (int k = 1; k < GRP; ++k) v += acc_s[k][row];
            const i64 i = S.y0 + row;
            y[i] = (beta == 0.0 ? 0.0 : beta * z[i]) + alpha * v;
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
    std::vector<VChunk> chunks, chunks16;
    std::vector<TJob> tjobs;
    int32_t max_slot = -1;
    int npart = 0;
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
            const bool big_rank = nd.rslot < (int32_t)H.h_ranks.size() ? H.h_ranks[nd.rslot] > 8 : true;
            std::vector<VChunk> &dst = big_rank ? chunks16 : chunks;
            if (nd.n <= VCHUNK) {
                dst.push_back({nd.voff, nd.n, nd.c0, (int32_t)nd.n, nd.rslot,
                               (i64)nd.rslot * KC_MAX, -1, 0});
            } else {
                int cb = npart;
                for (i64 a = 0; a < nd.n; a += VCHUNK) {
                    int len = (int)std::min(VCHUNK, nd.n - a);
                    dst.push_back({nd.voff + a, nd.n, nd.c0 + a, len, nd.rslot, -1, npart++, 0});
                }
                tjobs.push_back({nd.rslot, cb, npart});
            }
            max_slot = std::max(max_slot, nd.rslot);
            for (int sg = seg_of(nd.r0); sg < nseg && seg_start[sg] < nd.r0 + nd.m; ++sg) {
                i64 a = std::max(seg_start[sg], nd.r0), e = std::min(seg_start[sg + 1], nd.r0 + nd.m);
                LH_REQUIRE(a == seg_start[sg] && e == seg_start[sg + 1], LH_EINTERNAL,
                           "low-rank block not aligned with row segments");
                lps[sg].push_back({nd.uoff + (a - nd.r0), nd.m, nd.rslot, 0, 0});
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
    P->nch16 = (int)chunks16.size();
    P->segs = dupload(segs, s);
    P->dp = dupload(dall, s);
    P->lp = dupload(lall, s);
    P->chunks = dupload(chunks, s);
    P->chunks16 = dupload(chunks16, s);
    P->part = dalloc<double>((i64)std::max(npart, 1) * KC_MAX);
    P->ntj = (int)tjobs.size();
    P->tjobs = dupload(tjobs, s);
    P->tvec = dalloc<double>((i64)(max_slot + 1 > 0 ? max_slot + 1 : 1) * KC_MAX);
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
    cudaFree(chunks16);
    cudaFree(part);
    cudaFree(tjobs);
    cudaFree(tvec);
}

// phase 1 (V^T x partials) + t_b reduction
void mv_vtx_launch(const MvPlan &P, const HMat &H, const double *x, int grid, cudaStream_t s) {
    if (P.nch > 0) {
        int g = std::max(1, std::min(grid, (P.nch + dev::NW - 1) / dev::NW));
        vtx_kernel<8><<<g, NT, 0, s>>>(P.chunks, P.nch, H.d_arena, H.d_ranks, x, P.part, P.tvec);
    }
    if (P.nch16 > 0) {
        int g = std::max(1, std::min(grid, (P.nch16 + dev::NW - 1) / dev::NW));
        vtx_kernel<16><<<g, NT, 0, s>>>(P.chunks16, P.nch16, H.d_arena, H.d_ranks, x, P.part, P.tvec);
    }
    if (P.ntj > 0) {
        int g = std::max(1, std::min(148 * 8, (P.ntj + dev::NW - 1) / dev::NW));
        treduce_kernel<<<g, NT, 0, s>>>(P.tjobs, P.ntj, H.d_ranks, P.part, P.tvec);
    }
}

void mv_seg_launch(const MvPlan &P, const HMat &H, const double *x, double *y, double alpha,
                   double beta, cudaStream_t s, int num_sms, const double *z) {
    // (A one-warp-per-32-rows variant without shared memory measured slower on B200:
    // 370 vs 384 steps/s at 128 registers, 331 when capped to 64 with spills.)
    int g2 = std::min(P.nseg, num_sms * 32);
    seg_kernel<<<g2, NT, 0, s>>>(P.segs, P.nseg, P.dp, P.lp, H.d_arena, H.d_ranks, P.tvec, x, y,
                                 alpha, beta, z ? z : y);
}

// y = alpha * H x + beta * z (z = y when null) for one right-hand side
void mv_run(const MvPlan &P, const HMat &H, const double *x, double *y, double alpha, double beta,
            cudaStream_t s, int num_sms, const double *z) {
    mv_vtx_launch(P, H, x, num_sms * 16, s);
    mv_seg_launch(P, H, x, y, alpha, beta, s, num_sms, z);
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
