// Shared leaf bases for the propagator Z.
//
// After coarsening, every off-diagonal block b of Z is low-rank, U_b V_b^T.  For a row leaf t
// (a 64-row segment) the U rows of all blocks covering t span the row space of the whole
// off-diagonal row block Z(t, t^c); that space is small (rank 7-11 at 1e-12 for cfg3, while
// the blocks covering t carry ~150 columns).  So each row leaf gets one orthonormal basis Q_t
// and each column leaf one basis P_s, and a block is stored by small coefficient matrices:
//     U_b(t rows) ~ Q_t C_{t,b},   V_b(s rows) ~ P_s E_{s,b}.
// A matvec then streams the dense diagonal leaves, Q_t and P_s once, plus the coefficients:
//     x_hat_s = P_s^T x_s                         (V^T x kernel, P_s as a 64-row "V chunk")
//     t_b     = sum_{s in cols b} E_{s,b}^T x_hat_s   (coupling, this file)
//     y_hat_t = sum_{b covering t} C_{t,b} t_b       (coupling, this file)
//     y_t     = D_t x_t + Q_t y_hat_t              (segment kernel, Q_t as one low-rank piece)
// The bases come from a truncated column-pivoted Householder QR of the gathered, weighted
// factor rows (one CTA per leaf): U_b(t) columns weighted by the norms of the matching V_b
// columns (and vice versa), so the Frobenius residual of the gathered matrix bounds the error
// of every block's product, and it is truncated at eps relative to the leaf's row block.
#include <algorithm>
#include <cmath>
#include <numeric>

#include "core.h"
#include "dev.cuh"
#include "matvec.h"

namespace lh {

Coupling::~Coupling() {
    cudaFree(chunks);
    cudaFree(xidx);
    cudaFree(rows);
    cudaFree(tidx);
    cudaFree(xg);
    cudaFree(tg);
    cudaFree(tjobs);
    cudaFree(ebuf);
    cudaFree(cbuf);
    cudaFree(tb);
    cudaFree(part);
}

namespace {

using dev::NT;
using dev::NW;
using dev::KC_MAX;
constexpr int KQ = 32;     // basis capacity per leaf (the low-rank column capacity)
constexpr int LR = 64;     // leaf rows
constexpr int MAXC = 368;  // gathered columns per leaf (shared memory)

struct GPiece {  // gathered columns [col0, col0 + r): src[off + i + c * ld] * wts[woff + c]
    i64 off, ld, woff;
    int32_t r, col0;
};
struct BJob {  // one leaf: rows, pieces [p0, p1), total columns
    int32_t rows, p0, p1, ncol;
    i64 qout, cout;  // Q (rows x KQ, ld rows) and coefficients (KQ x ncol, ld KQ) in temp
};
struct CopyJob {  // dst[d0 + i * dsi + c * dsc] = src[s0 + i * ssi + c * ssc], i < ni, c < nc
    i64 s0, ssi, ssc, d0, dsi, dsc;
    int32_t ni, nc;
};

constexpr size_t BASIS_SMEM = sizeof(double) * ((size_t)LR * MAXC + MAXC + LR * KQ + KQ + 2 * NW + 8);

// column norms of every low-rank block's U and V (the weights)
__global__ void colnorm_kernel(const i64 *off, const i64 *len, int n, const double *arena, double *out) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (i64 j = (i64)blockIdx.x * NW + w; j < n; j += (i64)gridDim.x * NW) {
        const double *p = arena + off[j];
        double s = 0.0;
        for (i64 i = lane; i < len[j]; i += 32) s += p[i] * p[i];
        s = dev::warp_sum(s);
        if (lane == 0) out[j] = sqrt(s);
    }
}

__global__ void __launch_bounds__(NT) basis_kernel(const BJob *jobs, int njobs, const GPiece *pieces,
                                                   const double *arena, const double *wts, double eps,
                                                   int *kout, double *Qt, double *Ct) {
    extern __shared__ double4 smem_raw[];
    double *M = reinterpret_cast<double *>(smem_raw);  // LR x MAXC, ld LR
    double *res = M + (size_t)LR * MAXC;                // column residual norms^2
    double *Vr = res + MAXC;                            // reflectors, LR x KQ
    double *beta = Vr + LR * KQ;
    double *red = beta + KQ;
    __shared__ int s_p;
    __shared__ double s_v;
    for (int jb = blockIdx.x; jb < njobs; jb += gridDim.x) {
        const BJob J = jobs[jb];
        const int nc = J.ncol, rows = J.rows;
        for (int e = threadIdx.x; e < LR * nc; e += NT) M[e] = 0.0;
        for (int e = threadIdx.x; e < LR * KQ; e += NT) Vr[e] = 0.0;
        __syncthreads();
        for (int p = J.p0; p < J.p1; ++p) {
            const GPiece G = pieces[p];
            for (int e = threadIdx.x; e < rows * G.r; e += NT) {
                const int i = e % rows, c = e / rows;
                M[i + (G.col0 + c) * LR] = arena[G.off + i + (i64)c * G.ld] * wts[G.woff + c];
            }
        }
        __syncthreads();
        double tot = 0.0;
        for (int e = threadIdx.x; e < LR * nc; e += NT) tot += M[e] * M[e];
        tot = dev::block_sum(tot, red);
        int k = 0;
        for (; k < KQ && k < rows; ++k) {
            // residual column norms over rows k..rows-1
            double rem = 0.0;
            for (int j = threadIdx.x; j < nc; j += NT) {
                double s = 0.0;
                for (int i = k; i < rows; ++i) s += M[i + j * LR] * M[i + j * LR];
                res[j] = s;
                rem += s;
            }
            rem = dev::block_sum(rem, red);
            if (!(rem > eps * eps * tot)) break;
            // pivot: largest residual column (first on ties)
            if (threadIdx.x < 32) {
                double best = -1.0;
                int bi = 0;
                for (int j = threadIdx.x; j < nc; j += 32)
                    if (res[j] > best) {
                        best = res[j];
                        bi = j;
                    }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                    if (ob > best || (ob == best && oi < bi)) {
                        best = ob;
                        bi = oi;
                    }
                }
                if (threadIdx.x == 0) {
                    s_p = bi;
                    s_v = best;
                }
            }
            __syncthreads();
            const int p = s_p;
            const double nx = sqrt(s_v), x0 = M[k + p * LR];
            const double alpha = x0 >= 0.0 ? -nx : nx;
            // v = x - alpha e_k (rows k..), beta = 2 / v^T v
            double *v = Vr + k * LR;
            for (int i = k + threadIdx.x; i < rows; i += NT) v[i] = M[i + p * LR] - (i == k ? alpha : 0.0);
            const double vv = s_v - x0 * x0 + (x0 - alpha) * (x0 - alpha);
            const double b = vv > 0.0 ? 2.0 / vv : 0.0;
            if (threadIdx.x == 0) beta[k] = b;
            __syncthreads();
            for (int j = threadIdx.x; j < nc; j += NT) {
                double w = 0.0;
                for (int i = k; i < rows; ++i) w += v[i] * M[i + j * LR];
                w *= b;
                for (int i = k; i < rows; ++i) M[i + j * LR] -= w * v[i];
            }
            __syncthreads();
        }
        // coefficients: the first k rows of H M, unweighted
        for (int e = threadIdx.x; e < k * nc; e += NT) {
            const int i = e % k, j = e / k;
            Ct[J.cout + i + (i64)j * KQ] = M[i + j * LR];
        }
        __syncthreads();
        for (int p = J.p0; p < J.p1; ++p) {
            const GPiece G = pieces[p];
            for (int e = threadIdx.x; e < k * G.r; e += NT) {
                const int i = e % k, c = e / k;
                const double w = wts[G.woff + c];
                double *dst = Ct + J.cout + i + (i64)(G.col0 + c) * KQ;
                *dst = w > 0.0 ? *dst / w : 0.0;
            }
        }
        // Q = H_0 ... H_{k-1} [I; 0] (reuse M)
        for (int e = threadIdx.x; e < LR * k; e += NT) M[e] = ((e % LR) == (e / LR)) ? 1.0 : 0.0;
        __syncthreads();
        for (int t = k - 1; t >= 0; --t) {
            const double *v = Vr + t * LR;
            const double b = beta[t];
            for (int c = threadIdx.x; c < k; c += NT) {
                double w = 0.0;
                for (int i = t; i < rows; ++i) w += v[i] * M[i + c * LR];
                w *= b;
                for (int i = t; i < rows; ++i) M[i + c * LR] -= w * v[i];
            }
            __syncthreads();
        }
        for (int e = threadIdx.x; e < rows * k; e += NT) {
            const int i = e % rows, c = e / rows;
            Qt[J.qout + i + (i64)c * rows] = M[i + c * LR];
        }
        if (threadIdx.x == 0) kout[jb] = k;
        __syncthreads();
    }
}

__global__ void copy_kernel(const CopyJob *jobs, int njobs, const double *src, double *dst) {
    for (int j = blockIdx.x; j < njobs; j += gridDim.x) {
        const CopyJob J = jobs[j];
        const i64 n = (i64)J.ni * J.nc;
        for (i64 e = threadIdx.x; e < n; e += NT) {
            const i64 i = e % J.ni, c = e / J.ni;
            dst[J.d0 + i * J.dsi + c * J.dsc] = src[J.s0 + i * J.ssi + c * J.ssc];
        }
    }
}

// Both coupling products are flattened: a chunk's coefficients are one contiguous array whose
// element e belongs to output column e % w (w = r for t_b, k for y_hat).  Lane layout
// lane = c + w * g (G = 32 / w groups): each lane streams rows g, g + G, ... of its column
// with four independent loads in flight, then the groups are summed through shared memory.
__device__ __forceinline__ double group_sum(double acc, int lane, int w, int G, double *sm) {
    sm[lane] = acc;
    __syncwarp();
    double s = 0.0;
    if (lane < w)
        for (int g = 0; g < G; ++g) s += sm[lane + g * w];
    __syncwarp();
    return s;
}

__global__ void gather_kernel(const int32_t *idx, i64 n, const double *src, double *dst) {
    for (i64 e = (i64)blockIdx.x * NT + threadIdx.x; e < n; e += (i64)gridDim.x * NT) dst[e] = src[idx[e]];
}

__global__ void __launch_bounds__(NT) tcouple_kernel(const CplChunk *chunks, int n, const double *xg,
                                                     const double *ebuf, double *tb, double *part) {
    __shared__ double sm[NW][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int q = blockIdx.x * NW + w; q < n; q += gridDim.x * NW) {
        const CplChunk C = chunks[q];
        const int G = 32 / C.r, c = lane % C.r, g = lane / C.r;
        double acc = 0.0;
        if (g < G) {
            const double *E = ebuf + C.e0 + c;
            const double *x = xg + C.x0;
            int row = g;
            for (; row + 3 * G < C.nrow; row += 4 * G) {
                const double e0 = E[(i64)row * C.r], e1 = E[(i64)(row + G) * C.r];
                const double e2 = E[(i64)(row + 2 * G) * C.r], e3 = E[(i64)(row + 3 * G) * C.r];
                const double x0 = x[row], x1 = x[row + G], x2 = x[row + 2 * G], x3 = x[row + 3 * G];
                acc = fma(e0, x0, acc);
                acc = fma(e1, x1, acc);
                acc = fma(e2, x2, acc);
                acc = fma(e3, x3, acc);
            }
            for (; row < C.nrow; row += G) acc = fma(E[(i64)row * C.r], x[row], acc);
        }
        const double s = group_sum(g < G ? acc : 0.0, lane, C.r, G, sm[w]);
        if (lane < C.r) {
            if (C.out >= 0) part[(i64)C.out * KC_MAX + lane] = s;
            else tb[(i64)(-1 - C.out) * KC_MAX + lane] = s;
        }
    }
}

__global__ void __launch_bounds__(NT) ycouple_kernel(const CplRow *rows, int n, const double *tg,
                                                     const double *cbuf, double *tvec) {
    __shared__ double sm[NW][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int q = blockIdx.x * NW + w; q < n; q += gridDim.x * NW) {
        const CplRow R = rows[q];
        const int G = 32 / R.k, i = lane % R.k, g = lane / R.k;
        double acc = 0.0;
        if (g < G) {
            const double *Cm = cbuf + R.e0 + i;
            const double *t = tg + R.t0;
            int col = g;
            for (; col + 3 * G < R.ncol; col += 4 * G) {
                const double c0 = Cm[(i64)col * R.k], c1 = Cm[(i64)(col + G) * R.k];
                const double c2 = Cm[(i64)(col + 2 * G) * R.k], c3 = Cm[(i64)(col + 3 * G) * R.k];
                const double t0 = t[col], t1 = t[col + G], t2 = t[col + 2 * G], t3 = t[col + 3 * G];
                acc = fma(c0, t0, acc);
                acc = fma(c1, t1, acc);
                acc = fma(c2, t2, acc);
                acc = fma(c3, t3, acc);
            }
            for (; col < R.ncol; col += G) acc = fma(Cm[(i64)col * R.k], t[col], acc);
        }
        const double s = group_sum(g < G ? acc : 0.0, lane, R.k, G, sm[w]);
        if (lane < R.k) tvec[(i64)R.blk * KC_MAX + lane] = s;
    }
}

}  // namespace

using dev::KC_MAX;

void coupling_launch(const Coupling &C, const double *tvec_in, double *tvec_out, cudaStream_t s) {
    auto grid = [](i64 n, int per) { return (int)std::max<i64>(1, std::min<i64>(148 * 16, (n + per - 1) / per)); };
    if (C.nchunk > 0) {
        gather_kernel<<<grid(C.nx, NT), NT, 0, s>>>(C.xidx, C.nx, tvec_in, C.xg);
        tcouple_kernel<<<grid(C.nchunk, NW), NT, 0, s>>>(C.chunks, C.nchunk, C.xg, C.ebuf, C.tb, C.part);
    }
    treduce_launch(C.tjobs, C.ntj, C.part, C.tb, s);
    if (C.nrow > 0) {
        gather_kernel<<<grid(C.nt, NT), NT, 0, s>>>(C.tidx, C.nt, C.tb, C.tg);
        ycouple_kernel<<<grid(C.nrow, NW), NT, 0, s>>>(C.rows, C.nrow, C.tg, C.cbuf, tvec_out);
    }
    LH_CUDA(cudaGetLastError());
}

// Builds the shared-basis form ZS of Z (dense leaves copied, one row-basis node per row leaf,
// one column-basis node per column leaf) and its matvec plan with the coupling attached.
// Returns false (ZS untouched) when Z does not qualify: leaves above 64 rows, a leaf whose
// gathered factors exceed the shared-memory capacity, or a basis above KQ columns.
bool build_shared_basis(Ctx &ctx, HMat &Z, double eps, HMat &ZS, std::shared_ptr<MvPlan> &plan,
                        double *stats) {
    const cudaStream_t st = ctx.stream;
    Z.sync_ranks(st);
    const Tree &rt = *Z.rt, &ct = *Z.ct;
    auto leaf_starts = [](const Tree &T, std::vector<i64> &lo) {
        lo.clear();
        for (int32_t lc : T.leaves) {
            const Cluster &c = T.nodes[lc];
            if (c.hi - c.lo > LR) return false;
            lo.push_back(c.lo);
        }
        lo.push_back(T.n);
        return true;
    };
    std::vector<i64> rlo, clo;
    if (!leaf_starts(rt, rlo) || !leaf_starts(ct, clo)) return false;
    const int nrl = (int)rlo.size() - 1, ncl = (int)clo.size() - 1;
    auto leaf_of = [](const std::vector<i64> &lo, i64 x) {
        return (int)(std::upper_bound(lo.begin(), lo.end(), x) - lo.begin()) - 1;
    };
    // low-rank blocks and their covering leaves
    std::vector<int32_t> lr;
    for (int32_t b : Z.leafblocks)
        if (Z.nodes[b].kind == K_LR && Z.h_ranks[Z.nodes[b].rslot] > 0) lr.push_back(b);
    const int nb = (int)lr.size();
    if (nb == 0) return false;
    // weights: column norms of U (for the V side) and V (for the U side)
    std::vector<i64> woff(nb), noff, nlen;
    i64 nw = 0;
    for (int q = 0; q < nb; ++q) {
        const Node &nd = Z.nodes[lr[q]];
        const int r = Z.h_ranks[nd.rslot];
        woff[q] = nw;
        for (int c = 0; c < r; ++c) {  // U columns then V columns
            noff.push_back(nd.uoff + (i64)c * nd.m);
            nlen.push_back(nd.m);
        }
        for (int c = 0; c < r; ++c) {
            noff.push_back(nd.voff + (i64)c * nd.n);
            nlen.push_back(nd.n);
        }
        nw += 2 * r;
    }
    double *dw = dalloc<double>(std::max<i64>(nw, 1));
    {
        i64 *doff = dupload(noff, st), *dlen = dupload(nlen, st);
        colnorm_kernel<<<(int)std::min<i64>(148 * 16, (nw + NW - 1) / NW), NT, 0, st>>>(doff, dlen, (int)nw,
                                                                                     Z.d_arena, dw);
        LH_CUDA(cudaGetLastError());
        LH_CUDA(cudaStreamSynchronize(st));
        cudaFree(doff);
        cudaFree(dlen);
    }
    // gather lists: row side (U slices weighted by V norms), column side (V slices by U norms)
    struct Side {
        std::vector<std::vector<std::pair<int, int>>> cover;  // leaf -> (block q, column offset)
        std::vector<int> ncol;
    } side[2];
    for (int sd = 0; sd < 2; ++sd) {
        side[sd].cover.assign(sd ? ncl : nrl, {});
        side[sd].ncol.assign(sd ? ncl : nrl, 0);
    }
    for (int q = 0; q < nb; ++q) {
        const Node &nd = Z.nodes[lr[q]];
        const int r = Z.h_ranks[nd.rslot];
        for (int sd = 0; sd < 2; ++sd) {
            const std::vector<i64> &lo = sd ? clo : rlo;
            const i64 a = sd ? nd.c0 : nd.r0, len = sd ? nd.n : nd.m;
            for (int l = leaf_of(lo, a); l < (int)lo.size() - 1 && lo[l] < a + len; ++l) {
                if (lo[l] < a || lo[l + 1] > a + len) {
                    cudaFree(dw);
                    return false;  // block not aligned with the leaves
                }
                side[sd].cover[l].push_back({q, side[sd].ncol[l]});
                side[sd].ncol[l] += r;
            }
        }
    }
    for (int sd = 0; sd < 2; ++sd)
        for (int c : side[sd].ncol)
            if (c > MAXC) {
                cudaFree(dw);
                return false;
            }
    // basis computations (both sides in one launch)
    std::vector<BJob> jobs;
    std::vector<GPiece> pieces;
    i64 qlen = 0, clen = 0;
    for (int sd = 0; sd < 2; ++sd) {
        const std::vector<i64> &lo = sd ? clo : rlo;
        for (int l = 0; l < (int)lo.size() - 1; ++l) {
            BJob J{(int32_t)(lo[l + 1] - lo[l]), (int32_t)pieces.size(), 0, side[sd].ncol[l], qlen, clen};
            for (auto &pc : side[sd].cover[l]) {
                const Node &nd = Z.nodes[lr[pc.first]];
                const int r = Z.h_ranks[nd.rslot];
                if (sd == 0)
                    pieces.push_back({nd.uoff + (lo[l] - nd.r0), nd.m, woff[pc.first] + r, r, pc.second});
                else
                    pieces.push_back({nd.voff + (lo[l] - nd.c0), nd.n, woff[pc.first], r, pc.second});
            }
            J.p1 = (int32_t)pieces.size();
            qlen += (i64)J.rows * KQ;
            clen += (i64)KQ * std::max(J.ncol, 1);
            jobs.push_back(J);
        }
    }
    const int njobs = (int)jobs.size();
    double *Qt = dalloc<double>(qlen), *Ct = dalloc<double>(clen);
    int *dk = dalloc<int>(njobs);
    {
        BJob *dj = dupload(jobs, st);
        GPiece *dp = dupload(pieces, st);
        LH_CUDA(cudaFuncSetAttribute((const void *)basis_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)BASIS_SMEM));
        basis_kernel<<<std::min(njobs, ctx.num_sms), NT, BASIS_SMEM, st>>>(dj, njobs, dp, Z.d_arena, dw, eps, dk,
                                                                          Qt, Ct);
        LH_CUDA(cudaGetLastError());
        LH_CUDA(cudaStreamSynchronize(st));
        cudaFree(dj);
        cudaFree(dp);
    }
    cudaFree(dw);
    std::vector<int> k(njobs);
    LH_CUDA(cudaMemcpy(k.data(), dk, sizeof(int) * njobs, cudaMemcpyDeviceToHost));
    cudaFree(dk);
    // ---- ZS: dense leaves of Z, then row-basis nodes, then column-basis nodes
    ZS.rt = Z.rt;
    ZS.ct = Z.ct;
    ZS.rt_hold = Z.rt_hold;
    ZS.ct_hold = Z.ct_hold;
    ZS.nrows = Z.nrows;
    ZS.ncols = Z.ncols;
    ZS.nodes.clear();
    ZS.leafblocks.clear();
    std::vector<CopyJob> cj;
    i64 aoff = 0;
    for (int32_t b : Z.leafblocks) {
        const Node &s = Z.nodes[b];
        if (s.kind != K_DENSE && s.kind != K_FDENSE) continue;
        Node d = s;
        d.kind = K_DENSE;
        d.doff = aoff;
        for (int t = 0; t < 4; ++t) d.kid[t] = -1;
        d.vpar = -1;
        cj.push_back({s.doff, 1, s.m, aoff, 1, s.m, (int32_t)s.m, (int32_t)s.n});
        aoff += s.m * s.n;
        ZS.leafblocks.push_back((int32_t)ZS.nodes.size());
        ZS.nodes.push_back(d);
    }
    std::vector<int32_t> ranks;
    std::vector<int32_t> node_of_job(njobs, -1);
    for (int j = 0; j < njobs; ++j) {
        if (k[j] == 0) continue;
        const bool col = j >= nrl;
        const int l = col ? j - nrl : j;
        Node d{};
        d.kind = K_LR;
        d.rcl = d.ccl = -1;
        d.r0 = col ? 0 : rlo[l];
        d.m = col ? 0 : rlo[l + 1] - rlo[l];
        d.c0 = col ? clo[l] : 0;
        d.n = col ? clo[l + 1] - clo[l] : 0;
        for (int t = 0; t < 4; ++t) d.kid[t] = -1;
        d.kcap = k[j];
        d.rslot = (int32_t)ranks.size();
        ranks.push_back(k[j]);
        const i64 rows = jobs[j].rows;
        d.uoff = aoff;
        d.voff = aoff;
        d.doff = -1;
        d.vpar = -1;
        aoff += rows * k[j];  // Q / P, copied from the temp buffer below
        node_of_job[j] = (int32_t)ZS.nodes.size();
        ZS.leafblocks.push_back((int32_t)ZS.nodes.size());
        ZS.nodes.push_back(d);
    }
    ZS.root = 0;
    ZS.arena_len = aoff;
    ZS.d_arena = dalloc<double>(std::max<i64>(aoff, 1));
    ZS.nslots = (int32_t)ranks.size();
    ZS.d_ranks = dupload(ranks, st);
    ZS.h_ranks = ranks;
    {
        CopyJob *d = dupload(cj, st);
        copy_kernel<<<(int)std::min<size_t>(cj.size(), 148 * 16), NT, 0, st>>>(d, (int)cj.size(), Z.d_arena, ZS.d_arena);
        LH_CUDA(cudaGetLastError());
        LH_CUDA(cudaStreamSynchronize(st));
        cudaFree(d);
    }
    // Q and P come from the temp buffer, not Z's arena: redo those copies from Qt
    {
        std::vector<CopyJob> qj;
        for (int j = 0; j < njobs; ++j) {
            if (node_of_job[j] < 0) continue;
            const Node &d = ZS.nodes[node_of_job[j]];
            const i64 rows = jobs[j].rows;
            qj.push_back({jobs[j].qout, 1, rows, d.voff, 1, rows, (int32_t)rows, k[j]});
        }
        if (!qj.empty()) {
            CopyJob *d = dupload(qj, st);
            copy_kernel<<<(int)std::min<size_t>(qj.size(), 148 * 16), NT, 0, st>>>(d, (int)qj.size(), Qt, ZS.d_arena);
            LH_CUDA(cudaGetLastError());
            LH_CUDA(cudaStreamSynchronize(st));
            cudaFree(d);
        }
    }
    plan = build_mv_plan(ZS, ZS.leafblocks, st);
    // ---- coupling data
    auto C = std::make_shared<Coupling>();
    C->nb = nb;
    std::vector<CopyJob> ej, cjb;
    std::vector<int32_t> xidx, tidx;
    std::vector<CplChunk> chunks;
    std::vector<TJob> tjobs;
    i64 elen = 0, cl = 0;
    int npart = 0;
    // E_{s,b}: per block b its column leaves in order; row-major (k_s x r_b), contiguous per b
    std::vector<std::vector<std::pair<int, int>>> bcols(nb);  // block -> (column leaf, col offset)
    std::vector<std::vector<std::pair<int, int>>> brows(nb);
    for (int l = 0; l < ncl; ++l)
        for (auto &pc : side[1].cover[l]) bcols[pc.first].push_back({l, pc.second});
    for (int l = 0; l < nrl; ++l)
        for (auto &pc : side[0].cover[l]) brows[pc.first].push_back({l, pc.second});
    const int CHROWS = 192;  // E rows per chunk (one warp)
    for (int q = 0; q < nb; ++q) {
        const Node &nd = Z.nodes[lr[q]];
        const int r = Z.h_ranks[nd.rslot];
        const i64 e_beg = elen;
        const int x_beg = (int)xidx.size();
        for (auto &cs : bcols[q]) {
            const int j = nrl + cs.first;
            if (k[j] == 0) continue;
            // element (l, c) at ebuf[elen + l * r + c] <- Ct[cout + l + (col0 + c) * KQ]
            ej.push_back({jobs[j].cout + (i64)cs.second * KQ, 1, KQ, elen, r, 1, k[j], r});
            const int xb = plan->blk_of_node[node_of_job[j]];
            for (int l = 0; l < k[j]; ++l) xidx.push_back(xb * KC_MAX + l);
            elen += (i64)k[j] * r;
        }
        const int nrows_b = (int)xidx.size() - x_beg;
        if (nrows_b <= CHROWS) {
            chunks.push_back({e_beg, nrows_b, r, -1 - q, x_beg});
        } else {
            const int cb = npart;
            for (int a = 0; a < nrows_b; a += CHROWS)
                chunks.push_back({e_beg + (i64)a * r, std::min(CHROWS, nrows_b - a), r, npart++, x_beg + a});
            tjobs.push_back({q, r, cb, npart});
        }
    }
    std::vector<CplRow> rowsv;
    {
        std::vector<std::vector<std::pair<int, int>>> rcov(nrl);  // row leaf -> (block, col offset)
        for (int q = 0; q < nb; ++q)
            for (auto &rs : brows[q]) rcov[rs.first].push_back({q, rs.second});
        for (int l = 0; l < nrl; ++l) {
            if (k[l] == 0) continue;
            CplRow R{cl, 0, k[l], plan->blk_of_node[node_of_job[l]], (int32_t)tidx.size()};
            for (auto &pc : rcov[l]) {
                const Node &nd = Z.nodes[lr[pc.first]];
                const int r = Z.h_ranks[nd.rslot];
                // col-major (k_t x r_b) at cbuf[cl] <- Ct[cout + i + (col0 + c) * KQ]
                cjb.push_back({jobs[l].cout + (i64)pc.second * KQ, 1, KQ, cl, 1, k[l], k[l], r});
                for (int c = 0; c < r; ++c) tidx.push_back(pc.first * KC_MAX + c);
                cl += (i64)k[l] * r;
                R.ncol += r;
            }
            rowsv.push_back(R);
        }
    }
    C->ebuf = dalloc<double>(std::max<i64>(elen, 1));
    C->cbuf = dalloc<double>(std::max<i64>(cl, 1));
    for (int pass = 0; pass < 2; ++pass) {
        std::vector<CopyJob> &v = pass ? cjb : ej;
        if (v.empty()) continue;
        CopyJob *d = dupload(v, st);
        copy_kernel<<<(int)std::min<size_t>(v.size(), 148 * 16), NT, 0, st>>>(d, (int)v.size(), Ct,
                                                                              pass ? C->cbuf : C->ebuf);
        LH_CUDA(cudaGetLastError());
        LH_CUDA(cudaStreamSynchronize(st));
        cudaFree(d);
    }
    cudaFree(Qt);
    cudaFree(Ct);
    C->nchunk = (int)chunks.size();
    C->nrow = (int)rowsv.size();
    C->ntj = (int)tjobs.size();
    C->chunks = dupload(chunks, st);
    C->xidx = dupload(xidx, st);
    C->nx = (i64)xidx.size();
    C->xg = dalloc<double>(std::max<i64>(C->nx, 1));
    C->rows = dupload(rowsv, st);
    C->tidx = dupload(tidx, st);
    C->nt = (i64)tidx.size();
    C->tg = dalloc<double>(std::max<i64>(C->nt, 1));
    C->tjobs = dupload(tjobs, st);
    C->tb = dalloc<double>((i64)nb * KC_MAX);
    C->part = dalloc<double>((i64)std::max(npart, 1) * KC_MAX);
    C->bytes = 8 * (elen + cl) + 4 * (i64)(xidx.size() + tidx.size());
    LH_CUDA(cudaStreamSynchronize(st));
    plan->cpl = C;
    if (stats) {
        double ks = 0;
        for (int j = 0; j < njobs; ++j) ks += k[j];
        stats[0] = ks / std::max(njobs, 1);   // mean basis size
        stats[1] = (double)(elen + cl);       // coupling scalars
        stats[2] = (double)aoff;              // dense + bases scalars
    }
    return true;
}

}  // namespace lh
