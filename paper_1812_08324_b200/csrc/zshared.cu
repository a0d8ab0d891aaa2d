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
#include <functional>
#include <cmath>
#include <numeric>

#include "core.h"
#include "dev.cuh"
#include "matvec.h"
#include "h2step.h"

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

struct GPiece {  // M[row0 + i, col0 + c] = src[off + i + c * ld] * wts[woff + c], i < nr, c < r
    i64 off, ld, woff;
    int32_t r, col0;
    int32_t row0, nr;  // row0 > 0 only for the second child's rows of a nested (H2) basis
};
struct BJob {  // one leaf: rows, pieces [p0, p1), total columns
    int32_t rows, p0, p1, ncol;
    i64 qout, cout;  // Q (rows x KQ, ld rows) and coefficients (KQ x ncol, ld KQ) in temp
};
struct CopyJob {  // dst[d0 + i * dsi + c * dsc] = src[s0 + i * ssi + c * ssc], i < ni, c < nc
    i64 s0, ssi, ssc, d0, dsi, dsc;
    int32_t ni, nc;
};

constexpr size_t BASIS_SMEM = sizeof(double) * ((size_t)LR * MAXC + 2 * MAXC + LR * KQ + KQ + 2 * NW + 8);

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

// kout[j] = basis size, or -1 when KQ columns do not reach the tolerance
__global__ void __launch_bounds__(NT) basis_kernel(const BJob *jobs, int njobs, const GPiece *pieces,
                                                   const double *arena, const double *wts, double eps,
                                                   int *kout, double *Qt, double *Ct) {
    extern __shared__ double4 smem_raw[];
    double *M = reinterpret_cast<double *>(smem_raw);  // LR x MAXC, ld LR
    double *res = M + (size_t)LR * MAXC;                // column residual norms^2
    double *wcol = res + MAXC;                          // weight of every gathered column
    double *Vr = wcol + MAXC;                           // reflectors, LR x KQ
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
            for (int e = threadIdx.x; e < G.nr * G.r; e += NT) {
                const int i = e % G.nr, c = e / G.nr;
                M[G.row0 + i + (G.col0 + c) * LR] = arena[G.off + i + (i64)c * G.ld] * wts[G.woff + c];
            }
            if (G.row0 == 0)
                for (int c = threadIdx.x; c < G.r; c += NT) wcol[G.col0 + c] = wts[G.woff + c];
        }
        __syncthreads();
        double tot = 0.0;
        for (int e = threadIdx.x; e < LR * nc; e += NT) tot += M[e] * M[e];
        tot = dev::block_sum(tot, red);
        int k = 0;
        bool fail = false;
        for (;; ++k) {
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
            if (k == KQ || k == rows) {
                fail = k < rows;
                break;
            }
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
            const double w = wcol[j];
            Ct[J.cout + i + (i64)j * KQ] = w > 0.0 ? M[i + j * LR] / w : 0.0;
        }
        __syncthreads();
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
        if (threadIdx.x == 0) kout[jb] = fail ? -1 : k;
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
                const int32_t nr = (int32_t)(lo[l + 1] - lo[l]);
                if (sd == 0)
                    pieces.push_back({nd.uoff + (lo[l] - nd.r0), nd.m, woff[pc.first] + r, r, pc.second, 0, nr});
                else
                    pieces.push_back({nd.voff + (lo[l] - nd.c0), nd.n, woff[pc.first], r, pc.second, 0, nr});
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
    if (std::any_of(k.begin(), k.end(), [](int v) { return v < 0; })) {
        cudaFree(Qt);
        cudaFree(Ct);
        return false;  // a basis above KQ columns
    }
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
    ZS.d_arena = dalloc<double>(std::max<i64>(aoff, 1) + 4);  // + bulk-copy tail slack
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


// ===========================================================================
// Nested (H2) cluster bases (matvec.h: H2).  The leaf bases above become the bottom level of a
// nested basis: an internal cluster tau's basis is [Q_c1 0; 0 Q_c2] T_tau, with T_tau from the same
// truncated column-pivoted QR applied to the stacked child coefficients [C_{c1,b}; C_{c2,b}] of
// every block b covering tau (weighted as at the leaves).  A block b = (rho, sigma) is then the
// small coupling S_b = C_{rho,b} E_{sigma,b}^T, so a matvec streams the dense diagonal leaves,
// the leaf bases, the transfer matrices and the couplings: no per-leaf coefficient of a large
// block is stored any more.
// ===========================================================================
H2::~H2() {
    for (void *p : {(void *)leaves, (void *)ups, (void *)dns, (void *)cpls, (void *)up_lv, (void *)cnt, (void *)up_sub, (void *)dn_sub, (void *)dn_path, (void *)dn_pbeg,
                    (void *)dn_lv, (void *)pb, (void *)tu, (void *)td, (void *)sb, (void *)xh, (void *)wg,
                    (void *)crec, (void *)up_chain, (void *)up_cbeg, (void *)up_xcnt, (void *)dn_ycnt,
                    (void *)qleaf, (void *)dn_qbeg, (void *)yd})
        cudaFree(p);
}

namespace {

constexpr int H2_MAXP = 24;     // path length (top clusters above a row subtree)
constexpr unsigned FULL = 0xffffffffu;

// x_hat of one column leaf: lanes hold rows lane and lane + 32, one warp sum per basis column
__device__ __forceinline__ double h2_leaf(const H2Leaf &L, const double *pb, const double *x, int lane) {
    const double *P = pb + L.poff;
    const double x0 = lane < L.rows ? x[L.x0 + lane] : 0.0;
    const double x1 = lane + 32 < L.rows ? x[L.x0 + lane + 32] : 0.0;
    double mine = 0.0;
    // 8 basis columns per round trip: 16 columns (one trip for most leaves) measured slower,
    // 30.9 vs 24.4 us, the register cost halves the resident warps
    for (int c = 0; c < L.k; c += 8) {
        double p[8], q[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const bool ok = c + u < L.k;
            p[u] = ok ? P[lane + 64 * (c + u)] : 0.0;
            q[u] = ok ? P[lane + 32 + 64 * (c + u)] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double v = dev::warp_sum(fma(p[u], x0, q[u] * x1));
            if (lane == c + u) mine = v;
        }
    }
    return mine;  // lane j < L.k holds x_hat[j]
}

// y[j] = sum_i T[i * ldi + j * ldj] v[i], i < n, for lane j (act); v[i] held by lane i; T in shared memory
__device__ __forceinline__ double h2_apply_s(const double *T, int ldi, int n, double v, bool act) {
    double a0 = 0.0, a1 = 0.0;
    int i = 0;
    for (; i + 1 < n; i += 2) {
        const double t0 = act ? T[i * ldi] : 0.0, t1 = act ? T[(i + 1) * ldi] : 0.0;
        a0 = fma(t0, __shfl_sync(FULL, v, i), a0);
        a1 = fma(t1, __shfl_sync(FULL, v, i + 1), a1);
    }
    if (i < n) a0 = fma(act ? T[i * ldi] : 0.0, __shfl_sync(FULL, v, i), a0);
    return a0 + a1;
}
// the same with T in global memory: all loads issued before the first FMA
__device__ __forceinline__ double h2_apply_g(const double *T, i64 ldi, int n, double v, bool act) {
    double t[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) t[i] = (act && i < n) ? T[i * ldi] : 0.0;
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
        a0 = fma(t[i], __shfl_sync(FULL, v, i), a0);
        a1 = fma(t[i + 1], __shfl_sync(FULL, v, i + 1), a1);
    }
    return a0 + a1;
}

// two independent products, r1 = T1 v1 (n1 terms) and r2 = T2 v2 (n2 terms), all loads in flight
// together: one memory round trip for both
__device__ __forceinline__ void h2_apply_g2(const double *T1, i64 ld1, int n1, double v1, bool act1,
                                            const double *T2, i64 ld2, int n2, double v2, bool act2, double &r1,
                                            double &r2) {
    double a1 = 0.0, a2 = 0.0;
    const int n = max(n1, n2);
    for (int b = 0; b < n; b += 16) {  // one batch (one round trip) for k <= 16
        double t1[16], t2[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            t1[i] = (act1 && b + i < n1) ? T1[(b + i) * ld1] : 0.0;
            t2[i] = (act2 && b + i < n2) ? T2[(b + i) * ld2] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            a1 = fma(t1[i], __shfl_sync(FULL, v1, (b + i) & 31), a1);
            a2 = fma(t2[i], __shfl_sync(FULL, v2, (b + i) & 31), a2);
        }
    }
    r1 = a1;
    r2 = a2;
}

// couplings of one row cluster, w[i] = sum_e S_e x_hat_e, lane i < k
__device__ __forceinline__ double h2_couple(const H2Down &D, const H2Cpl *cpls, const double *sb,
                                            const double *xh, int lane) {
    double acc = 0.0;
    for (int e = D.c0; e < D.c1; ++e) {
        const H2Cpl C = cpls[e];
        const double xv = lane < C.kc ? __ldcg(xh + C.xoff + lane) : 0.0;
        acc += h2_apply_g(sb + C.soff + lane, C.kr, C.kc, xv, lane < D.k);
    }
    return acc;
}

// Programmatic dependent launch: a walk kernel stages its static operands (descriptors,
// transfer / coupling prefetches) while the previous kernel drains, then waits for its results.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// global -> shared copy by the whole CTA with every load of a thread in flight at once
template <class T>
__device__ __forceinline__ void h2_copy_in(T *dst, const T *src, int n) {
    constexpr int U = 8;
    for (int b = 0; b < n; b += U * NT) {
        T v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = b + u * NT + threadIdx.x;
            v[u] = i < n ? src[i] : T();
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = b + u * NT + threadIdx.x;
            if (i < n) dst[i] = v[u];
        }
    }
}

// x_hat of every column leaf: one warp per leaf, all CTAs resident (bandwidth-bound: P streams once)
__global__ void __launch_bounds__(NT) h2_leaf_kernel(const H2Leaf *leaves, int n, const double *pb, const double *x,
                                                    double *xh, i64 nx, double *xpad) {
    const int lane = threadIdx.x & 31;
    pdl_trigger();
    if (xpad)
        for (i64 i = (i64)blockIdx.x * NT + threadIdx.x; i < nx + 2; i += (i64)gridDim.x * NT)
            xpad[i] = i < nx ? x[i] : 0.0;  // the segment kernel's aligned, padded copy of x
    for (int l = blockIdx.x * NW + (threadIdx.x >> 5); l < n; l += gridDim.x * NW) {
        const H2Leaf L = leaves[l];
        const double v = h2_leaf(L, pb, x, lane);
        if (lane < L.k) xh[L.xoff + lane] = v;
    }
}

// Column walk above the leaves: one CTA per subtree (x_hat of its nodes kept in shared memory,
// levels by height, one memory round trip per level), then the top of the tree by
// last-arrival climbing: the second child to finish computes the parent (warp 0 only).
constexpr int H2_MAXN = 256;  // staged node descriptors per subtree
#ifndef H2_UP_MINB
#define H2_UP_MINB 2  // walk CTAs per SM by registers: room for the co-resident dense-leaf kernel
#endif
__global__ void __launch_bounds__(NT, H2_UP_MINB) h2_up_kernel(const H2Up *ups, const int32_t *up_lv, const int32_t *up_chain,
                                                      const int32_t *up_cbeg, const H2Sub *sub, const int32_t *up_xcnt,
                                                      int32_t *cnt, int maxh, const double *tu, double *xh, int dbg) {
    extern __shared__ __align__(16) double h2s[];
    double *xs = h2s;
    __shared__ H2Up su[H2_MAXN];
    __shared__ H2Up sc[H2_MAXP];
    const int s = blockIdx.x, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const H2Sub SB = sub[s];
    const int32_t *lv = up_lv + (i64)s * (maxh + 1);
    const int u0 = lv[0], nu = lv[maxh] - u0, c0 = up_cbeg[s], nc = up_cbeg[s + 1] - c0;
    {  // descriptors (subtree + climb chain) and x_hat slots to shared memory; transfers to L2
        pdl_trigger();
        constexpr int W = (int)(sizeof(H2Up) / 4);
        h2_copy_in(reinterpret_cast<int32_t *>(su), reinterpret_cast<const int32_t *>(ups + u0), nu * W);
        for (int i = threadIdx.x; i < nc * W; i += NT)
            reinterpret_cast<int32_t *>(sc)[i] = reinterpret_cast<const int32_t *>(ups + up_chain[c0 + i / W])[i % W];
        const char *t = reinterpret_cast<const char *>(tu + SB.tbeg);
        for (i64 o = 128 * (i64)threadIdx.x; o < 8 * (i64)SB.tlen; o += 128 * NT)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(t + o));
        pdl_wait();  // the leaves' x_hat
        h2_copy_in(xs, xh + SB.base, up_xcnt[s]);
    }
    __syncthreads();
    for (int q = w; q < nc; q += NW) {  // the climb's transfers to L2
        const char *t = reinterpret_cast<const char *>(tu + sc[q].toff);
        const int bytes = 8 * (sc[q].k1 + sc[q].k2) * sc[q].k;
        for (int o = 128 * lane; o < bytes; o += 128 * 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(t + o));
    }
    for (int hh = 0; hh < ((dbg & 2) ? 0 : maxh); ++hh) {
        const int a = lv[hh] - u0, b = lv[hh + 1] - u0;
        if (a == b) continue;
        for (int u = a + w; u < b; u += NW) {
            const H2Up &U = su[u];
            const double *T = tu + U.toff + lane;
            const double xa = lane < U.k1 ? xs[U.xoff1 - SB.base + lane] : 0.0;
            const double xb = lane < U.k2 ? xs[U.xoff2 - SB.base + lane] : 0.0;
            const bool act = lane < U.k;
            double v1, v2;
            h2_apply_g2(T, U.k, U.k1, xa, act, T + (i64)U.k1 * U.k, U.k, U.k2, xb, act, v1, v2);
            const double v = v1 + v2;
            if (act) {
                xh[U.xoff + lane] = v;
                xs[U.xoff - SB.base + lane] = v;
            }
        }
        __syncthreads();
    }
    if (w != 0 || (dbg & 1)) return;
    for (int q = 0; q < nc; ++q) {
        const int p = up_chain[c0 + q];
        const H2Up &U = sc[q];
        __syncwarp();
        int old = 0;
        if (lane == 0) {
            int32_t *c = cnt + p;
            asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;" : "=r"(old) : "l"(c), "r"(1) : "memory");
        }
        old = __shfl_sync(FULL, old, 0);
        if (old == 0) return;
        if (lane == 0) cnt[p] = 0;  // ready for the next application
        const double xa = lane < U.k1 ? __ldcg(xh + U.xoff1 + lane) : 0.0;
        const double xb = lane < U.k2 ? __ldcg(xh + U.xoff2 + lane) : 0.0;
        const bool act = lane < U.k;
        const double *T = tu + U.toff + lane;
        double v1, v2;
        h2_apply_g2(T, U.k, U.k1, xa, act, T + (i64)U.k1 * U.k, U.k, U.k2, xb, act, v1, v2);
        if (act) xh[U.xoff + lane] = v1 + v2;
    }
}

// couplings of every row cluster: w[yoff + i] = sum_e S_e x_hat_e (one warp per cluster)
__device__ __forceinline__ double h2_apply_g16(const double *T, i64 ldi, int n, double v, bool act) {
    double a0 = 0.0, a1 = 0.0;
    for (int b = 0; b < n; b += 16) {
        double t[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) t[i] = (act && b + i < n) ? T[(b + i) * ldi] : 0.0;
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            a0 = fma(t[i], __shfl_sync(FULL, v, (b + i) & 31), a0);
            a1 = fma(t[i + 1], __shfl_sync(FULL, v, (b + i + 1) & 31), a1);
        }
    }
    return a0 + a1;
}
__global__ void __launch_bounds__(NT, 4) h2_couple_kernel(const H2CRec *crec, int n, const H2Cpl *cpls,
                                                         const double *sb, const double *xh, double *wg) {
    const int lane = threadIdx.x & 31;
    pdl_trigger();
    for (int q = blockIdx.x * NW + (threadIdx.x >> 5); q < n; q += gridDim.x * NW) {  // couplings -> L2
        const H2CRec R = crec[q];
        const char *t = reinterpret_cast<const char *>(sb + R.soff);
        for (int o = 128 * lane; o < 8 * R.kr * R.kc; o += 128 * 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(t + o));
    }
    pdl_wait();  // x_hat of every column cluster
    for (int q = blockIdx.x * NW + (threadIdx.x >> 5); q < n; q += gridDim.x * NW) {
        const H2CRec R = crec[q];
        const double xv = lane < R.kc ? __ldcg(xh + R.xoff + lane) : 0.0;
        double acc = h2_apply_g16(sb + R.soff + lane, R.kr, R.kc, xv, lane < R.kr);
        for (int e = R.c0 + 1; e < R.c1; ++e) {  // further couplings of the same cluster (rare)
            const H2Cpl C = cpls[e];
            const double x2 = lane < C.kc ? __ldcg(xh + C.xoff + lane) : 0.0;
            acc += h2_apply_g16(sb + C.soff + lane, C.kr, C.kc, x2, lane < R.kr);
        }
        if (lane < R.kr) wg[R.yoff + lane] = acc;
    }
}

// Row walk: one CTA per subtree.  The transfers down the path above the subtree (one warp),
// then the subtree's levels (y_hat kept in shared memory, one round trip per level).
struct H2Fuse {  // the fused step's row-basis phase (FUSED = true)
    const H2QLeaf *ql;
    const int32_t *qbeg;
    const double *zar, *yd, *z;
    double *y;
    double alpha, beta;
};
template <bool FUSED>
__global__ void __launch_bounds__(NT, H2_UP_MINB) h2_down_kernel(const H2Down *dns, const int32_t *dn_path,
                                                        const int32_t *dn_pbeg, const int32_t *dn_lv,
                                                        const H2Sub *sub, const int32_t *dn_ycnt, int maxh, int ymax,
                                                        const double *td, const double *wg, double *tcol, int dbg,
                                                        H2Fuse fz) {
    extern __shared__ __align__(16) double h2s[];
    double *ws = h2s, *ys = ws + ymax;
    __shared__ double pw[H2_MAXP][KC_MAX];
    __shared__ H2Down pd[H2_MAXP];
    const int s = blockIdx.x, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const H2Sub SB = sub[s];
    const int pa = dn_pbeg[s], np = dn_pbeg[s + 1] - pa;
    const int32_t *lv = dn_lv + (i64)s * (maxh + 2);
    __shared__ H2Down sd[H2_MAXN];
    const int n0 = lv[0], nn = lv[maxh + 1] - n0;
    {
        h2_copy_in(reinterpret_cast<int32_t *>(sd), reinterpret_cast<const int32_t *>(dns + n0),
                   nn * (int)(sizeof(H2Down) / 4));
        for (int q = w; q < np; q += NW)
            if (lane == 0) pd[q] = dns[dn_path[pa + q]];
        const char *t = reinterpret_cast<const char *>(td + SB.tbeg);
        for (i64 o = 128 * (i64)threadIdx.x; o < 8 * (i64)SB.tlen; o += 128 * NT)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(t + o));
        pdl_wait();  // the couplings w
        h2_copy_in(ws, wg + SB.base, dn_ycnt[s]);
        __syncthreads();
        for (int q = w; q < np; q += NW)
            if (lane < pd[q].k) pw[q][lane] = wg[pd[q].yoff + lane];
    }
    __syncthreads();
    if (w == 0 && np > 1 && !(dbg & 4)) {  // transfers down the path
        for (int q = 1; q < np; ++q) {
            const H2Down &D = pd[q];
            const double yv = lane < D.kp ? pw[q - 1][lane] : 0.0;
            const double v = h2_apply_g(td + D.toff + D.roff + lane, D.ldt, D.kp, yv, lane < D.k);
            if (lane < D.k) pw[q][lane] += v;
            __syncwarp();
        }
    }
    __syncthreads();
    for (int d = 0; d <= ((dbg & 8) ? -1 : maxh); ++d) {
        const int a = lv[d] - n0, b = lv[d + 1] - n0;
        if (a == b) continue;
        for (int u = a + w; u < b; u += 2 * NW) {  // two nodes per warp and round trip
            const bool two = u + NW < b;
            const H2Down &D1 = sd[u];
            const H2Down &D2 = sd[two ? u + NW : u];
            auto parent_y = [&](const H2Down &D) {
                return lane < D.kp ? (D.yoffp >= 0 ? ys[D.yoffp - SB.base + lane] : pw[np - 1][lane]) : 0.0;
            };
            const bool act1 = lane < D1.k, act2 = two && lane < D2.k;
            double r1, r2;
            h2_apply_g2(td + D1.toff + D1.roff + lane, D1.ldt, D1.kp, parent_y(D1), act1, td + D2.toff + D2.roff + lane,
                        D2.ldt, D2.kp, parent_y(D2), act2, r1, r2);
            if (act1) {
                const double v = ws[D1.yoff - SB.base + lane] + r1;
                ys[D1.yoff - SB.base + lane] = v;
                if (!FUSED && D1.out >= 0) tcol[D1.out + lane] = v;
            }
            if (act2) {
                const double v = ws[D2.yoff - SB.base + lane] + r2;
                ys[D2.yoff - SB.base + lane] = v;
                if (!FUSED && D2.out >= 0) tcol[D2.out + lane] = v;
            }
        }
        __syncthreads();
    }
    if (!FUSED) return;
    // row-basis phase: y_t = alpha (yd_t + Q_t y_hat_t) + beta z_t for this subtree's row leaves
    // (one warp per leaf, lanes on rows lane and lane + 32, 8 basis columns per round trip)
    const int qa = fz.qbeg[s], qb = fz.qbeg[s + 1];
    for (int l = qa + w; l < qb; l += NW) {
        const H2QLeaf Q = fz.ql[l];
        const bool in0 = lane < Q.rows, in1 = lane + 32 < Q.rows;
        const i64 r0 = Q.r0 + lane, r1 = r0 + 32;
        const double d0 = in0 ? __ldcg(fz.yd + r0) : 0.0, d1 = in1 ? __ldcg(fz.yd + r1) : 0.0;
        const double z0 = (in0 && fz.beta != 0.0) ? fz.z[r0] : 0.0, z1 = (in1 && fz.beta != 0.0) ? fz.z[r1] : 0.0;
        const double *q = fz.zar + Q.qoff;
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
        for (int c = 0; c < Q.k; c += 8) {
            double p[8], pp[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const bool ok = c + u < Q.k;
                p[u] = (ok && in0) ? q[lane + (i64)(c + u) * Q.rows] : 0.0;
                pp[u] = (ok && in1) ? q[lane + 32 + (i64)(c + u) * Q.rows] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; u += 2) {
                const double y0 = c + u < Q.k ? ys[Q.yloc + c + u] : 0.0;
                const double y1 = c + u + 1 < Q.k ? ys[Q.yloc + c + u + 1] : 0.0;
                a0 = fma(p[u], y0, a0);
                b0 = fma(p[u + 1], y1, b0);
                a1 = fma(pp[u], y0, a1);
                b1 = fma(pp[u + 1], y1, b1);
            }
        }
        if (in0) fz.y[r0] = fz.alpha * (d0 + (a0 + b0)) + fz.beta * z0;
        if (in1) fz.y[r1] = fz.alpha * (d1 + (a1 + b1)) + fz.beta * z1;
    }
}

// S_b = Cr (kr x r, ld KQ) Cc^T (r x kc, ld KQ) -> sb[soff + i + j kr]; one warp per block
struct SJob {
    i64 cr, cc, soff;
    int32_t kr, kc, r, pad;
};
__global__ void spro_kernel(const SJob *jobs, int n, const double *Cr, const double *Cc, double *sb) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int q = blockIdx.x * NW + w; q < n; q += gridDim.x * NW) {
        const SJob J = jobs[q];
        for (int e = lane; e < J.kr * J.kc; e += 32) {
            const int i = e % J.kr, j = e / J.kr;
            double acc = 0.0;
            for (int c = 0; c < J.r; ++c) acc = fma(Cr[J.cr + i + (i64)c * KQ], Cc[J.cc + j + (i64)c * KQ], acc);
            sb[J.soff + e] = acc;
        }
    }
}

struct DevFrees {  // frees build temporaries on every exit path
    std::vector<void *> p;
    template <class T>
    T *add(T *q) {
        p.push_back((void *)q);
        return q;
    }
    ~DevFrees() {
        for (void *q : p) cudaFree(q);
    }
};

}  // namespace

// x_hat of the column leaves [l0, l1) (the host pipeline runs this per arrived x piece)
void h2_leaf_launch(const H2 &h, int l0, int l1, const double *x, cudaStream_t s) {
    if (l1 <= l0) return;
    const int g = (int)std::max<i64>(1, std::min<i64>(148 * 8, (l1 - l0 + NW - 1) / NW));
    h2_leaf_kernel<<<g, NT, 0, s>>>(h.leaves + l0, l1 - l0, h.pb, x, h.xh, 0, nullptr);
}

static void h2_smem_attrs() {
    static bool done = false;
    if (done) return;
    done = true;
    const int big = 160 * 1024;
    LH_CUDA(cudaFuncSetAttribute((const void *)h2_up_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    LH_CUDA(cudaFuncSetAttribute((const void *)h2_down_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    LH_CUDA(cudaFuncSetAttribute((const void *)h2_down_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
}

void h2_launch(const H2 &h, const double *x, double *tcol, double *xpad, i64 nx, cudaStream_t s, bool leaves) {
    h2_smem_attrs();
    const int dbg = getenv("LEVYH_H2_DBG") ? atoi(getenv("LEVYH_H2_DBG")) : 0;  // timing experiments only
    auto grid = [](i64 n, int per_sm) { return (int)std::max<i64>(1, std::min<i64>(148 * per_sm, (n + NW - 1) / NW)); };
    if (leaves) h2_leaf_kernel<<<grid(h.nleaf, 8), NT, 0, s>>>(h.leaves, h.nleaf, h.pb, x, h.xh, nx, xpad);
    else if (nx > 0) h2_leaf_kernel<<<grid(nx / 256 + 1, 8), NT, 0, s>>>(h.leaves, 0, h.pb, x, h.xh, nx, xpad);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    auto cfg = [&](int g, size_t smem) {
        cudaLaunchConfig_t c = {};
        c.gridDim = dim3(g);
        c.blockDim = dim3(NT);
        c.dynamicSmemBytes = smem;
        c.stream = s;
        c.attrs = at;
        c.numAttrs = 1;
        return c;
    };
    cudaLaunchConfig_t cu = cfg(h.nsub_up, 8 * (size_t)h.up_xmax), cc = cfg(grid(h.ncnode, 4), 0),
                       cd = cfg(h.nsub_dn, 16 * (size_t)h.dn_ymax);
    LH_CUDA(cudaLaunchKernelEx(&cu, h2_up_kernel, (const H2Up *)h.ups, (const int32_t *)h.up_lv,
                               (const int32_t *)h.up_chain, (const int32_t *)h.up_cbeg, (const H2Sub *)h.up_sub,
                               (const int32_t *)h.up_xcnt, h.cnt, h.maxh_up, (const double *)h.tu, h.xh, dbg));
    LH_CUDA(cudaLaunchKernelEx(&cc, h2_couple_kernel, (const H2CRec *)h.crec, h.ncnode, (const H2Cpl *)h.cpls,
                               (const double *)h.sb, (const double *)h.xh, h.wg));
    LH_CUDA(cudaLaunchKernelEx(&cd, h2_down_kernel<false>, (const H2Down *)h.dns, (const int32_t *)h.dn_path,
                               (const int32_t *)h.dn_pbeg, (const int32_t *)h.dn_lv, (const H2Sub *)h.dn_sub,
                               (const int32_t *)h.dn_ycnt, h.maxh_dn, h.dn_ymax, (const double *)h.td,
                               (const double *)h.wg, tcol, dbg, H2Fuse{}));
    LH_CUDA(cudaGetLastError());
}

void h2_launch_fused(const H2 &h, const double *x, double *y, double alpha, double beta, const double *z,
                     cudaStream_t s, cudaEvent_t dense_done) {
    h2_smem_attrs();
    const int dbg = getenv("LEVYH_H2_DBG") ? atoi(getenv("LEVYH_H2_DBG")) : 0;  // timing experiments only
    static int prio_hi = 0;
    static bool init = false;
    if (!init) {  // the walk is the critical path: highest priority over the dense stream
        int lo = 0, hi = 0;
        LH_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        prio_hi = getenv("LEVYH_H2_NOPRIO") ? lo : hi;
        init = true;
    }
    auto grid = [](i64 n, int per_sm) { return (int)std::max<i64>(1, std::min<i64>(148 * per_sm, (n + NW - 1) / NW)); };
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributePriority;
    at[0].val.priority = prio_hi;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    auto cfg = [&](int g, size_t smem, bool pdl) {
        cudaLaunchConfig_t c = {};
        c.gridDim = dim3(g);
        c.blockDim = dim3(NT);
        c.dynamicSmemBytes = smem;
        c.stream = s;
        c.attrs = at;
        c.numAttrs = pdl ? 2 : 1;
        return c;
    };
    const int fdbg = getenv("LEVYH_FUSE_DBG") ? atoi(getenv("LEVYH_FUSE_DBG")) : 0;  // timing only
    if (fdbg & 2) {  // dense branch alone
        LH_CUDA(cudaStreamWaitEvent(s, dense_done, 0));
        return;
    }
    // the walk's grids are bounded so that each SM keeps room for the co-resident dense-leaf
    // segment kernel (LEVYH_H2F_LEAF / LEVYH_H2F_CPL: CTAs per SM)
    const int gl = getenv("LEVYH_H2F_LEAF") ? atoi(getenv("LEVYH_H2F_LEAF")) : 2;
    const int gc = getenv("LEVYH_H2F_CPL") ? atoi(getenv("LEVYH_H2F_CPL")) : 2;
    cudaLaunchConfig_t cl = cfg(grid(h.nleaf, gl), 0, false), cu = cfg(h.nsub_up, 8 * (size_t)h.up_xmax, true),
                       cc = cfg(grid(h.ncnode, gc), 0, true), cd = cfg(h.nsub_dn, 16 * (size_t)h.dn_ymax, false);
    LH_CUDA(cudaLaunchKernelEx(&cl, h2_leaf_kernel, (const H2Leaf *)h.leaves, h.nleaf, (const double *)h.pb, x, h.xh,
                               (i64)0, (double *)nullptr));
    LH_CUDA(cudaLaunchKernelEx(&cu, h2_up_kernel, (const H2Up *)h.ups, (const int32_t *)h.up_lv,
                               (const int32_t *)h.up_chain, (const int32_t *)h.up_cbeg, (const H2Sub *)h.up_sub,
                               (const int32_t *)h.up_xcnt, h.cnt, h.maxh_up, (const double *)h.tu, h.xh, dbg));
    LH_CUDA(cudaLaunchKernelEx(&cc, h2_couple_kernel, (const H2CRec *)h.crec, h.ncnode, (const H2Cpl *)h.cpls,
                               (const double *)h.sb, (const double *)h.xh, h.wg));
    LH_CUDA(cudaStreamWaitEvent(s, dense_done, 0));
    LH_CUDA(cudaLaunchKernelEx(&cd, h2_down_kernel<true>, (const H2Down *)h.dns, (const int32_t *)h.dn_path,
                               (const int32_t *)h.dn_pbeg, (const int32_t *)h.dn_lv, (const H2Sub *)h.dn_sub,
                               (const int32_t *)h.dn_ycnt, h.maxh_dn, h.dn_ymax, (const double *)h.td,
                               (const double *)h.wg, (double *)nullptr, dbg,
                               H2Fuse{h.qleaf, h.dn_qbeg, h.zarena, h.yd, z, y, alpha, beta}));
    LH_CUDA(cudaGetLastError());
}

// Builds the nested-basis form of Z: ZS holds the dense leaves and one row-basis node Q_t per row
// leaf (the segment kernel's operands), the plan carries the H2 walk.  Returns false (nothing
// changed) when Z does not qualify: leaves above 64 rows, a cluster whose gathered factors exceed
// the shared-memory capacity, a basis above KQ columns, or a path deeper than H2_MAXP.
// A copy of T whose leaves above 64 points are split (at 64 points from the start, again while
// a part exceeds 64: the 64-row segments of the matvec plans); existing node ids are kept, the
// new children appended.  Lets the nested bases of a leaf-128 operator (cfg5) use 64-row leaf
// bases: its blocks keep their clusters, which are now internal nodes of the copy.
std::shared_ptr<Tree> refine_tree_leaves(const Tree &T, int maxleaf) {
    auto R = std::make_shared<Tree>(T);
    std::vector<int32_t> todo(R->leaves.begin(), R->leaves.end());
    auto bbox = [&](Cluster &c) {
        for (int d = 0; d < R->dim; ++d) {
            double lo = 0, hi = 0;
            for (i64 k = c.lo; k < c.hi; ++k) {
                const double v = R->pts[R->order[k] * R->dim + d];
                if (k == c.lo || v < lo) lo = v;
                if (k == c.lo || v > hi) hi = v;
            }
            c.blo[d] = lo;
            c.bhi[d] = hi;
        }
    };
    while (!todo.empty()) {
        const int32_t c = todo.back();
        todo.pop_back();
        if (R->nodes[c].size() <= maxleaf) continue;
        const Cluster p = R->nodes[c];
        Cluster a = p, b = p;
        a.hi = p.lo + maxleaf;
        b.lo = a.hi;
        a.depth = b.depth = p.depth + 1;
        a.kid[0] = a.kid[1] = b.kid[0] = b.kid[1] = -1;
        bbox(a);
        bbox(b);
        const int32_t ia = (int32_t)R->nodes.size();
        R->nodes.push_back(a);
        R->nodes.push_back(b);
        R->nodes[c].kid[0] = ia;
        R->nodes[c].kid[1] = ia + 1;
        todo.push_back(ia);
        todo.push_back(ia + 1);
    }
    R->leaves.clear();  // depth-first leaf order
    std::vector<int32_t> stk{0};
    while (!stk.empty()) {
        const int32_t c = stk.back();
        stk.pop_back();
        const Cluster &cl = R->nodes[c];
        if (cl.leaf()) R->leaves.push_back(c);
        else {
            stk.push_back(cl.kid[1]);
            stk.push_back(cl.kid[0]);
        }
    }
    return R;
}

static bool h2_fail(const char *why) {
    if (getenv("LEVYH_PLAN_VERBOSE")) fprintf(stderr, "[levyh] H2 form not built: %s\n", why);
    return false;
}

bool build_h2(Ctx &ctx, HMat &Z, double eps, int split, HMat &ZS, std::shared_ptr<MvPlan> &plan,
              double *stats) {
    const cudaStream_t st = ctx.stream;
    Z.sync_ranks(st);
    const Tree *trees[2] = {Z.rt, Z.ct};
    for (int sd = 0; sd < 2; ++sd)
        for (int32_t lc : trees[sd]->leaves)
            if (trees[sd]->nodes[lc].size() > LR) return h2_fail("leaf above 64 rows");
    std::vector<int32_t> lr;
    for (int32_t b : Z.leafblocks)
        if (Z.nodes[b].kind == K_LR && Z.h_ranks[Z.nodes[b].rslot] > 0) lr.push_back(b);
    const int nb = (int)lr.size();
    if (nb == 0) return h2_fail("no low-rank blocks");
    DevFrees tmp;
    // weights: column norms of U (for the V side) and V (for the U side)
    std::vector<i64> woff(nb), noff, nlen;
    i64 nw = 0;
    for (int q = 0; q < nb; ++q) {
        const Node &nd = Z.nodes[lr[q]];
        const int r = Z.h_ranks[nd.rslot];
        woff[q] = nw;
        for (int c = 0; c < r; ++c) {
            noff.push_back(nd.uoff + (i64)c * nd.m);
            nlen.push_back(nd.m);
        }
        for (int c = 0; c < r; ++c) {
            noff.push_back(nd.voff + (i64)c * nd.n);
            nlen.push_back(nd.n);
        }
        nw += 2 * r;
    }
    double *dw = tmp.add(dalloc<double>(std::max<i64>(nw, 1)));
    {
        i64 *doff = tmp.add(dupload(noff, st)), *dlen = tmp.add(dupload(nlen, st));
        colnorm_kernel<<<(int)std::min<i64>(148 * 16, (nw + NW - 1) / NW), NT, 0, st>>>(doff, dlen, (int)nw,
                                                                                     Z.d_arena, dw);
        LH_CUDA(cudaGetLastError());
    }
    LH_CUDA(cudaFuncSetAttribute((const void *)basis_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)BASIS_SMEM));
    // ---- bases, bottom-up per side (0: rows / U, 1: columns / V)
    struct Side {
        std::vector<std::vector<std::pair<int, int>>> cover;  // cluster -> (block q, column offset)
        std::vector<int> ncol, k, height, parent, rows;
        std::vector<char> has;
        std::vector<i64> cout, qout;
        double *Ct = nullptr, *Qt = nullptr;
        int maxh = 0;
    } S[2];
    auto col0_in = [](const std::vector<std::pair<int, int>> &cv, int q) {
        auto it = std::lower_bound(cv.begin(), cv.end(), std::make_pair(q, -1));
        return it != cv.end() && it->first == q ? it->second : -1;
    };
    for (int sd = 0; sd < 2; ++sd) {
        Side &D = S[sd];
        const Tree &T = *trees[sd];
        const int nn = (int)T.nodes.size();
        D.cover.assign(nn, {});
        D.ncol.assign(nn, 0);
        D.k.assign(nn, 0);
        D.height.assign(nn, 0);
        D.parent.assign(nn, -1);
        D.rows.assign(nn, 0);
        D.has.assign(nn, 0);
        D.cout.assign(nn, -1);
        D.qout.assign(nn, -1);
        std::vector<int32_t> order;  // preorder
        {
            std::vector<int32_t> stk{0};
            while (!stk.empty()) {
                const int32_t c = stk.back();
                stk.pop_back();
                order.push_back(c);
                const Cluster &cl = T.nodes[c];
                if (!cl.leaf())
                    for (int t = 1; t >= 0; --t) {
                        D.parent[cl.kid[t]] = c;
                        stk.push_back(cl.kid[t]);
                    }
            }
        }
        for (auto it = order.rbegin(); it != order.rend(); ++it) {
            const Cluster &cl = T.nodes[*it];
            if (!cl.leaf()) D.height[*it] = 1 + std::max(D.height[cl.kid[0]], D.height[cl.kid[1]]);
        }
        for (int q = 0; q < nb; ++q) {
            const Node &nd = Z.nodes[lr[q]];
            const int r = Z.h_ranks[nd.rslot];
            std::vector<int32_t> stk{sd ? nd.ccl : nd.rcl};
            while (!stk.empty()) {
                const int32_t c = stk.back();
                stk.pop_back();
                D.cover[c].push_back({q, D.ncol[c]});
                D.ncol[c] += r;
                D.has[c] = 1;
                const Cluster &cl = T.nodes[c];
                if (!cl.leaf()) {
                    stk.push_back(cl.kid[0]);
                    stk.push_back(cl.kid[1]);
                }
            }
        }
        i64 clen = 0, qlen = 0;
        for (int c = 0; c < nn; ++c) {
            if (!D.has[c]) continue;
            if (D.ncol[c] > MAXC) return h2_fail("gathered factor columns above MAXC");
            D.maxh = std::max(D.maxh, D.height[c]);
            D.cout[c] = clen;
            clen += (i64)KQ * D.ncol[c];
            D.qout[c] = qlen;
            qlen += (i64)(T.nodes[c].leaf() ? T.nodes[c].size() : LR) * KQ;
        }
        D.Ct = tmp.add(dalloc<double>(std::max<i64>(clen, 1)));
        D.Qt = tmp.add(dalloc<double>(std::max<i64>(qlen, 1)));
        for (int hh = 0; hh <= D.maxh; ++hh) {
            std::vector<BJob> jobs;
            std::vector<GPiece> pieces;
            std::vector<int32_t> who;
            for (int c = 0; c < nn; ++c) {
                if (!D.has[c] || D.height[c] != hh) continue;
                const Cluster &cl = T.nodes[c];
                BJob J{0, (int32_t)pieces.size(), 0, D.ncol[c], D.qout[c], D.cout[c]};
                if (cl.leaf()) {
                    J.rows = (int32_t)cl.size();
                    for (auto &pc : D.cover[c]) {
                        const Node &nd = Z.nodes[lr[pc.first]];
                        const int r = Z.h_ranks[nd.rslot];
                        if (sd == 0)
                            pieces.push_back({nd.uoff + (cl.lo - nd.r0), nd.m, woff[pc.first] + r, r, pc.second, 0,
                                              J.rows});
                        else
                            pieces.push_back({nd.voff + (cl.lo - nd.c0), nd.n, woff[pc.first], r, pc.second, 0,
                                              J.rows});
                    }
                } else {
                    const int c1 = cl.kid[0], c2 = cl.kid[1], k1 = D.k[c1], k2 = D.k[c2];
                    J.rows = k1 + k2;
                    if (J.rows == 0) continue;  // k = 0
                    for (auto &pc : D.cover[c]) {
                        const Node &nd = Z.nodes[lr[pc.first]];
                        const int r = Z.h_ranks[nd.rslot];
                        const i64 wo = woff[pc.first] + (sd == 0 ? r : 0);
                        const int a1 = col0_in(D.cover[c1], pc.first), a2 = col0_in(D.cover[c2], pc.first);
                        if (k1 > 0) pieces.push_back({D.cout[c1] + (i64)a1 * KQ, KQ, wo, r, pc.second, 0, k1});
                        if (k2 > 0) pieces.push_back({D.cout[c2] + (i64)a2 * KQ, KQ, wo, r, pc.second, k1, k2});
                    }
                }
                D.rows[c] = J.rows;
                J.p1 = (int32_t)pieces.size();
                jobs.push_back(J);
                who.push_back(c);
            }
            if (jobs.empty()) continue;
            const int nj = (int)jobs.size();
            BJob *dj = dupload(jobs, st);
            GPiece *dp = dupload(pieces, st);
            int *dk = dalloc<int>(nj);
            basis_kernel<<<std::min(nj, ctx.num_sms), NT, BASIS_SMEM, st>>>(dj, nj, dp, hh == 0 ? Z.d_arena : D.Ct,
                                                                           dw, eps, dk, D.Qt, D.Ct);
            LH_CUDA(cudaGetLastError());
            std::vector<int> kk(nj);
            LH_CUDA(cudaMemcpyAsync(kk.data(), dk, sizeof(int) * nj, cudaMemcpyDeviceToHost, st));
            LH_CUDA(cudaStreamSynchronize(st));
            cudaFree(dj);
            cudaFree(dp);
            cudaFree(dk);
            for (int j = 0; j < nj; ++j) {
                if (kk[j] < 0) return h2_fail("basis above KQ columns");
                D.k[who[j]] = kk[j];
            }
        }
    }
    const Tree &RT = *trees[0], &CT = *trees[1];
    if (getenv("LEVYH_H2_CHECK")) {  // host check: U_b ~ Qnest_rho C_{rho,b}, V_b ~ Pnest_sigma E_{sigma,b}
        LH_CUDA(cudaStreamSynchronize(st));
        std::vector<double> arena(Z.arena_len);
        LH_CUDA(cudaMemcpy(arena.data(), Z.d_arena, 8 * Z.arena_len, cudaMemcpyDeviceToHost));
        for (int sd = 0; sd < 2; ++sd) {
            const Side &D = S[sd];
            const Tree &T = *trees[sd];
            i64 ql = 0, cl = 0;
            for (size_t c = 0; c < T.nodes.size(); ++c)
                if (D.has[c]) {
                    ql = std::max<i64>(ql, D.qout[c] + (i64)(T.nodes[c].leaf() ? T.nodes[c].size() : LR) * KQ);
                    cl = std::max<i64>(cl, D.cout[c] + (i64)KQ * D.ncol[c]);
                }
            std::vector<double> Qh(ql), Ch(cl);
            LH_CUDA(cudaMemcpy(Qh.data(), D.Qt, 8 * ql, cudaMemcpyDeviceToHost));
            LH_CUDA(cudaMemcpy(Ch.data(), D.Ct, 8 * cl, cudaMemcpyDeviceToHost));
            // explicit nested basis of cluster c: size x k, column-major
            std::function<std::vector<double>(int)> basis = [&](int c) {
                const Cluster &cc = T.nodes[c];
                const int k = D.k[c];
                const i64 m = cc.size();
                std::vector<double> B(m * k, 0.0);
                if (cc.leaf()) {
                    for (i64 e = 0; e < m * k; ++e) B[e] = Qh[D.qout[c] + e];
                    return B;
                }
                const int c1 = cc.kid[0], c2 = cc.kid[1], k1 = D.k[c1], rows = D.rows[c];
                const i64 m1 = T.nodes[c1].size();
                auto B1 = basis(c1), B2 = basis(c2);
                for (int j = 0; j < k; ++j)
                    for (i64 i = 0; i < m; ++i) {
                        double v = 0.0;
                        if (i < m1)
                            for (int a = 0; a < k1; ++a) v += B1[i + a * m1] * Qh[D.qout[c] + a + (i64)j * rows];
                        else
                            for (int a = 0; a < D.k[c2]; ++a)
                                v += B2[(i - m1) + a * (m - m1)] * Qh[D.qout[c] + k1 + a + (i64)j * rows];
                        B[i + j * m] = v;
                    }
                return B;
            };
            double worst = 0.0;
            int wq = -1;
            for (int q = 0; q < nb; ++q) {
                const Node &nd = Z.nodes[lr[q]];
                const int r = Z.h_ranks[nd.rslot], c = sd ? nd.ccl : nd.rcl, k = D.k[c];
                const i64 m = sd ? nd.n : nd.m, off = sd ? nd.voff : nd.uoff;
                auto B = basis(c);
                int a = col0_in(D.cover[c], q);
                double num = 0.0, den = 0.0;
                for (int cc = 0; cc < r; ++cc)
                    for (i64 i = 0; i < m; ++i) {
                        double v = 0.0;
                        for (int t = 0; t < k; ++t) v += B[i + t * m] * Ch[D.cout[c] + t + (i64)(a + cc) * KQ];
                        const double u = arena[off + i + cc * m];
                        num += (u - v) * (u - v);
                        den += u * u;
                    }
                const double e = std::sqrt(num / std::max(den, 1e-300));
                if (e > worst) worst = e, wq = q;
            }
            fprintf(stderr, "[levyh] H2 check side %d: worst factor relative error %.3e (block %d, height %d)\n", sd,
                    worst, wq, wq >= 0 ? D.height[sd ? Z.nodes[lr[wq]].ccl : Z.nodes[lr[wq]].rcl] : -1);
        }
    }
    // ---- ZS: dense leaves of Z, then one basis node Q_t per row leaf
    ZS.rt = Z.rt;
    ZS.ct = Z.ct;
    ZS.rt_hold = Z.rt_hold;
    ZS.ct_hold = Z.ct_hold;
    ZS.nrows = Z.nrows;
    ZS.ncols = Z.ncols;
    ZS.nodes.clear();
    ZS.leafblocks.clear();
    std::vector<CopyJob> cj, qj;
    i64 aoff = 0;
    for (int32_t b : Z.leafblocks) {
        const Node &sn = Z.nodes[b];
        if (sn.kind != K_DENSE && sn.kind != K_FDENSE) continue;
        Node d = sn;
        d.kind = K_DENSE;
        d.doff = aoff;
        for (int t = 0; t < 4; ++t) d.kid[t] = -1;
        d.vpar = -1;
        cj.push_back({sn.doff, 1, sn.m, aoff, 1, sn.m, (int32_t)sn.m, (int32_t)sn.n});
        aoff += sn.m * sn.n;
        ZS.leafblocks.push_back((int32_t)ZS.nodes.size());
        ZS.nodes.push_back(d);
    }
    std::vector<int32_t> ranks, qnode(RT.nodes.size(), -1);
    for (int32_t lc : RT.leaves) {
        const int kq = S[0].k[lc];
        if (!S[0].has[lc] || kq == 0) continue;
        const Cluster &cl = RT.nodes[lc];
        Node d{};
        d.kind = K_LR;
        d.rcl = lc;
        d.ccl = -1;
        d.r0 = cl.lo;
        d.m = cl.size();
        d.c0 = 0;
        d.n = 0;
        for (int t = 0; t < 4; ++t) d.kid[t] = -1;
        d.kcap = kq;
        d.rslot = (int32_t)ranks.size();
        ranks.push_back(kq);
        d.uoff = d.voff = aoff;
        d.doff = -1;
        d.vpar = -1;
        qj.push_back({S[0].qout[lc], 1, d.m, aoff, 1, d.m, (int32_t)d.m, kq});
        aoff += d.m * kq;
        qnode[lc] = (int32_t)ZS.nodes.size();
        ZS.leafblocks.push_back((int32_t)ZS.nodes.size());
        ZS.nodes.push_back(d);
    }
    ZS.root = 0;
    ZS.arena_len = aoff;
    ZS.d_arena = dalloc<double>(std::max<i64>(aoff, 1) + 4);  // + bulk-copy tail slack
    ZS.nslots = (int32_t)ranks.size();
    ZS.d_ranks = dupload(ranks, st);
    ZS.h_ranks = ranks;
    auto run_copies = [&](const std::vector<CopyJob> &v, const double *src, double *dst) {
        if (v.empty()) return;
        CopyJob *d = dupload(v, st);
        copy_kernel<<<(int)std::min<size_t>(v.size(), 148 * 16), NT, 0, st>>>(d, (int)v.size(), src, dst);
        LH_CUDA(cudaGetLastError());
        LH_CUDA(cudaStreamSynchronize(st));
        cudaFree(d);
    };
    run_copies(cj, Z.d_arena, ZS.d_arena);
    run_copies(qj, S[0].Qt, ZS.d_arena);
    // LEVYH_H2_SPLIT_DENSE=1: row-basis pieces here, dense leaves in a lean plan of their own
    // streamed on a forked stream beside the walk.  Measured slower at N = 2^20 (the row-basis
    // pass alone is per-segment latency bound, 74 us, and the two branches barely overlap), so
    // the combined plan (dense leaf + row basis in one ring slot) is the default.
    if (getenv("LEVYH_H2_SPLIT_DENSE")) {
        std::vector<int32_t> dense_ids, q_ids;
        for (int32_t b : ZS.leafblocks) (ZS.nodes[b].kind == K_DENSE ? dense_ids : q_ids).push_back(b);
        plan = build_mv_plan(ZS, q_ids, st);
        plan->dense = build_mv_plan(ZS, dense_ids, st);
        plan->dense->lean = true;
        LH_CUDA(cudaStreamCreateWithFlags(&plan->fork, cudaStreamNonBlocking));
        for (cudaEvent_t &e : plan->fev) LH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    } else {
        plan = build_mv_plan(ZS, ZS.leafblocks, st);
    }
    auto h = std::make_shared<H2>();
    const Side &C = S[1], &R = S[0];
    // subtrees of height <= split; the split is the largest (<= 6) whose subtrees' transfer
    // matrices fit the shared-memory stage on both sides
    auto is_root = [&](const Side &D, int c, int sp) {
        const int p = D.parent[c];
        return D.has[c] && D.height[c] <= sp && (p < 0 || !D.has[p] || D.height[p] > sp);
    };
    auto subtree = [](const Tree &T, int r0) {  // preorder
        std::vector<int32_t> out, stk{r0};
        while (!stk.empty()) {
            const int32_t c = stk.back();
            stk.pop_back();
            out.push_back(c);
            const Cluster &cl = T.nodes[c];
            if (!cl.leaf()) {
                stk.push_back(cl.kid[1]);
                stk.push_back(cl.kid[0]);
            }
        }
        return out;
    };
    auto roots = [&](const Tree &T, const Side &D, int sp) {
        std::vector<int32_t> r;
        for (size_t c = 0; c < T.nodes.size(); ++c)
            if (is_root(D, (int)c, sp)) r.push_back((int32_t)c);
        std::sort(r.begin(), r.end(), [&](int x, int y) { return T.nodes[x].lo < T.nodes[y].lo; });
        return r;
    };
    if (split < 0) {  // the smallest split whose subtrees fit one wave (two CTAs per SM)
        split = 0;
        while (split < 12 && (int)std::max(roots(CT, C, split).size(), roots(RT, R, split).size()) > 2 * ctx.num_sms)
            ++split;
        // subtrees of at most 127 clusters: larger ones do not fit a CTA's shared memory (their
        // descriptors and x_hat slots); more subtrees then run as more CTAs (h2step.cu)
        split = std::min(split, 6);
    }
    auto even = [](i64 v) { return (v + 1) & ~(i64)1; };
    // ---- column side: x_hat slots per subtree, leaves (P_s, ld 64), transfers transposed
    std::vector<int32_t> xoff(CT.nodes.size(), -1);
    std::vector<H2Leaf> leaves;
    std::vector<H2Up> ups;
    std::vector<H2Sub> up_sub;
    std::vector<int32_t> up_lv, upidx(CT.nodes.size(), -1), up_xcnt, dn_ycnt;
    std::vector<CopyJob> pj, tj;
    i64 plen = 0, tulen = 0;
    int32_t nxh = 0;
    int up_tmax = 0, up_xmax = 0;
    const std::vector<int32_t> subs_up = roots(CT, C, split);
    int maxh_up = 0;
    for (int32_t r0 : subs_up) maxh_up = std::max(maxh_up, C.height[r0]);
    std::vector<int> up_h;  // height of every ups entry (multi-RHS walk)
    auto make_up = [&](int c) {
        const Cluster &cl = CT.nodes[c];
        up_h.push_back(C.height[c]);
        H2Up U{tulen, C.k[c], C.k[cl.kid[0]], C.k[cl.kid[1]], xoff[c], xoff[cl.kid[0]], xoff[cl.kid[1]], -1, 0};
        if (C.k[c] > 0 && C.rows[c] > 0)
            tj.push_back({C.qout[c], 1, C.rows[c], tulen, C.k[c], 1, C.rows[c], C.k[c]});
        tulen += (i64)C.rows[c] * C.k[c];
        return U;
    };
    std::vector<int32_t> up_leaf_beg;
    for (int32_t r0 : subs_up) {
        const std::vector<int32_t> nodes = subtree(CT, r0);
        const int32_t xb = nxh;
        up_leaf_beg.push_back((int32_t)leaves.size());
        for (int32_t c : nodes) {
            xoff[c] = nxh;
            nxh += C.k[c];
        }
        up_xmax = std::max(up_xmax, (int)(nxh - xb));
        up_xcnt.push_back(nxh - xb);
        for (int32_t c : nodes) {
            const Cluster &cl = CT.nodes[c];
            if (!cl.leaf() || C.k[c] == 0) continue;
            leaves.push_back({plen, cl.lo, (int32_t)cl.size(), C.k[c], xoff[c], 0});
            pj.push_back({C.qout[c], 1, cl.size(), plen, 1, LR, (int32_t)cl.size(), C.k[c]});
            plen += (i64)LR * C.k[c];
        }
        tulen = even(tulen);
        const i64 tb = tulen;
        up_lv.push_back((int32_t)ups.size());
        for (int hh = 1; hh <= maxh_up; ++hh) {
            for (int32_t c : nodes)
                if (!CT.nodes[c].leaf() && C.height[c] == hh) {
                    upidx[c] = (int32_t)ups.size();
                    ups.push_back(make_up(c));
                }
            up_lv.push_back((int32_t)ups.size());
        }
        tulen = even(tulen);
        up_sub.push_back({tb, (int32_t)(tulen - tb), xb});
        up_tmax = std::max(up_tmax, (int)(tulen - tb));
    }
    for (size_t c = 0; c < CT.nodes.size(); ++c)  // the top: clusters above the subtrees
        if (C.has[c] && C.height[c] > split) {
            xoff[c] = nxh;
            nxh += C.k[c];
        }
    for (size_t c = 0; c < CT.nodes.size(); ++c)
        if (C.has[c] && C.height[c] > split) {
            upidx[c] = (int32_t)ups.size();
            ups.push_back(make_up((int)c));
        }
    for (size_t c = 0; c < CT.nodes.size(); ++c)
        if (C.has[c] && C.height[c] > split) {
            const int p = C.parent[c];
            ups[upidx[c]].parent = (p >= 0 && C.has[p]) ? upidx[p] : -1;
        }
    // ---- row side: transfers per subtree (staged), y_hat slots, paths, couplings
    const std::vector<int32_t> subs_dn = roots(RT, R, split);
    std::vector<int32_t> yoff(RT.nodes.size(), -1), dnidx(RT.nodes.size(), -1), insub(RT.nodes.size(), -1);
    std::vector<i64> tdoff(RT.nodes.size(), -1);
    std::vector<CopyJob> dj2;
    std::vector<H2Sub> dn_sub;
    i64 tdlen = 0, sblen = 0;
    int dn_tmax = 0, dn_ymax = 0;
    int32_t nyh = 0;
    auto add_td = [&](int c) {
        if (R.has[c] && !RT.nodes[c].leaf() && R.rows[c] > 0 && R.k[c] > 0) {
            tdoff[c] = tdlen;
            dj2.push_back({R.qout[c], 1, R.rows[c], tdlen, 1, R.rows[c], R.rows[c], R.k[c]});
            tdlen += (i64)R.rows[c] * R.k[c];
        }
    };
    for (size_t q = 0; q < subs_dn.size(); ++q) {
        const std::vector<int32_t> nodes = subtree(RT, subs_dn[q]);
        tdlen = even(tdlen);
        const i64 tb = tdlen;
        const int32_t yb = nyh;
        for (int32_t c : nodes) {
            insub[c] = (int32_t)q;
            add_td(c);
            yoff[c] = nyh;
            nyh += R.k[c];
        }
        tdlen = even(tdlen);
        dn_sub.push_back({tb, (int32_t)(tdlen - tb), yb});
        dn_tmax = std::max(dn_tmax, (int)(tdlen - tb));
        dn_ymax = std::max(dn_ymax, (int)(nyh - yb));
        dn_ycnt.push_back(nyh - yb);
    }
    for (size_t c = 0; c < RT.nodes.size(); ++c)  // w slots of the top clusters
        if (R.has[c] && R.height[c] > split) {
            yoff[c] = nyh;
            nyh += R.k[c];
        }
    for (size_t c = 0; c < RT.nodes.size(); ++c)
        if (R.has[c] && R.height[c] > split) add_td((int)c);
    // tcol position of every tvec entry (the segment kernel's batch-ordered coefficients)
    std::vector<int32_t> tmap(plan->tcol_len);
    LH_CUDA(cudaMemcpy(tmap.data(), plan->tmap, sizeof(int32_t) * plan->tcol_len, cudaMemcpyDeviceToHost));
    std::vector<i64> tpos((i64)plan->nblk * KC_MAX + 1, -1);
    for (i64 e = 0; e < plan->tcol_len; ++e)
        if (tmap[e] >= 0) tpos[tmap[e]] = e;
    bool tcol_ok = plan->tcol_len < (i64)INT32_MAX;
    std::vector<H2Down> dns;
    std::vector<H2Cpl> cpls;
    std::vector<SJob> sj;
    std::vector<int32_t> dn_path, dn_pbeg{0}, dn_lv;
    std::vector<std::vector<int>> blocks_of(RT.nodes.size());
    for (int q = 0; q < nb; ++q) blocks_of[Z.nodes[lr[q]].rcl].push_back(q);
    std::vector<int32_t> dn_cl;  // row cluster of every dns entry (multi-RHS walk)
    auto make_dn = [&](int c) {
        const Cluster &cl = RT.nodes[c];
        dn_cl.push_back(c);
        H2Down D{0, 0, 0, 0, R.k[c], yoff[c], -1, (int32_t)cpls.size(), 0, -1, 0};
        const int p = R.parent[c];
        if (p >= 0 && R.has[p] && R.k[p] > 0 && tdoff[p] >= 0) {
            D.toff = tdoff[p];
            D.ldt = R.rows[p];
            D.roff = RT.nodes[p].kid[0] == c ? 0 : R.k[RT.nodes[p].kid[0]];
            D.kp = R.k[p];
            if (insub[c] >= 0 && insub[p] == insub[c]) D.yoffp = yoff[p];
        }
        for (int q : blocks_of[c]) {
            const Node &nd = Z.nodes[lr[q]];
            const int kr = R.k[c], kc = C.k[nd.ccl];
            if (kr == 0 || kc == 0) continue;
            const int ar = col0_in(R.cover[c], q), ac = col0_in(C.cover[nd.ccl], q);
            sj.push_back({R.cout[c] + (i64)ar * KQ, C.cout[nd.ccl] + (i64)ac * KQ, sblen, kr, kc,
                          Z.h_ranks[nd.rslot], 0});
            cpls.push_back({sblen, kr, kc, xoff[nd.ccl], 0});
            sblen += (i64)kr * kc;
        }
        D.c1 = (int32_t)cpls.size();
        if (insub[c] >= 0 && cl.leaf() && qnode[c] >= 0) {
            const i64 t0 = tpos[(i64)plan->blk_of_node[qnode[c]] * KC_MAX];
            for (int i = 0; i < R.k[c]; ++i)
                if (t0 < 0 || tpos[(i64)plan->blk_of_node[qnode[c]] * KC_MAX + i] != t0 + i) tcol_ok = false;
            D.out = (int32_t)t0;
        }
        return D;
    };
    int maxh_dn = 0, maxpath = 0;
    for (int32_t r0 : subs_dn) maxh_dn = std::max(maxh_dn, R.height[r0]);
    for (int32_t r0 : subs_dn) {  // subtree nodes by depth (contiguous per subtree)
        std::vector<int32_t> cur{r0};
        dn_lv.push_back((int32_t)dns.size());
        for (int d = 0; d <= maxh_dn; ++d) {
            std::vector<int32_t> nxt;
            for (int32_t c : cur) {
                dnidx[c] = (int32_t)dns.size();
                dns.push_back(make_dn(c));
                const Cluster &cl = RT.nodes[c];
                if (!cl.leaf())
                    for (int t = 0; t < 2; ++t)
                        if (R.has[cl.kid[t]]) nxt.push_back(cl.kid[t]);
            }
            dn_lv.push_back((int32_t)dns.size());
            cur.swap(nxt);
        }
    }
    for (size_t c = 0; c < RT.nodes.size(); ++c)  // the top clusters (path nodes)
        if (R.has[c] && R.height[c] > split) {
            dnidx[c] = (int32_t)dns.size();
            dns.push_back(make_dn((int)c));
        }
    for (int32_t r0 : subs_dn) {
        std::vector<int32_t> path;
        for (int p = R.parent[r0]; p >= 0 && R.has[p]; p = R.parent[p]) path.push_back(dnidx[p]);
        if ((int)path.size() > H2_MAXP) return h2_fail("row path deeper than H2_MAXP");
        maxpath = std::max(maxpath, (int)path.size());
        std::reverse(path.begin(), path.end());
        dn_path.insert(dn_path.end(), path.begin(), path.end());
        dn_pbeg.push_back((int32_t)dn_path.size());
    }
    if (!tcol_ok) return h2_fail("row-leaf coefficients not contiguous in tcol");
    LH_CUDA(cudaMemsetAsync(plan->tcol, 0, sizeof(double) * plan->tcol_len, st));  // padding stays zero
    // ---- device data
    h->split = split;
    h->nsub_up = (int)subs_up.size();
    h->nsub_dn = (int)subs_dn.size();
    h->maxh_up = maxh_up;
    h->maxh_dn = maxh_dn;
    h->maxpath = maxpath;
    h->up_tmax = up_tmax;
    h->up_xmax = (up_xmax + 1) & ~1;
    h->dn_tmax = dn_tmax;
    h->dn_ymax = (dn_ymax + 1) & ~1;
    std::vector<H2CRec> crec;
    for (size_t q = 0; q < dns.size(); ++q)
        if (dns[q].c1 > dns[q].c0 && dns[q].k > 0) {
            const H2Cpl &E = cpls[dns[q].c0];
            crec.push_back({E.soff, E.kr, E.kc, E.xoff, dns[q].yoff, dns[q].c0, dns[q].c1});
        }
    std::vector<int32_t> up_chain, up_cbeg{0};
    for (int32_t r0 : subs_up) {
        for (int p = C.parent[r0]; p >= 0 && C.has[p]; p = C.parent[p]) up_chain.push_back(upidx[p]);
        if ((int)(up_chain.size() - up_cbeg.back()) > H2_MAXP) return h2_fail("column climb deeper than H2_MAXP");
        up_cbeg.push_back((int32_t)up_chain.size());
    }
    // subtrees above H2_MAXN nodes only rule out the five-launch walk (its per-subtree staging);
    // the two-kernel step cuts its own chunk lists and is checked when it is built
    const char *big_subtree = nullptr;
    for (size_t q = 0; q + 1 < up_lv.size(); q += (size_t)maxh_up + 1)
        if (up_lv[q + maxh_up] - up_lv[q] > H2_MAXN) big_subtree = "column subtree above H2_MAXN nodes";
    for (size_t q = 0; q + 1 < dn_lv.size(); q += (size_t)maxh_dn + 2)
        if (dn_lv[q + maxh_dn + 1] - dn_lv[q] > H2_MAXN) big_subtree = "row subtree above H2_MAXN nodes";
    h->up_chain = dupload(up_chain, st);
    h->up_cbeg = dupload(up_cbeg, st);
    h->crec = dupload(crec, st);
    h->nleaf = (int)leaves.size();
    for (size_t l = 0; l < leaves.size(); ++l) {
        if (l > 0 && leaves[l].x0 < leaves[l - 1].x0) return h2_fail("column leaves out of row order");  // row order (host pipeline)
        h->leaf_end.push_back(leaves[l].x0 + leaves[l].rows);
    }
    h->ncnode = (int)crec.size();
    h->up_xcnt = dupload(up_xcnt, st);
    h->dn_ycnt = dupload(dn_ycnt, st);
    h->wg = dalloc<double>(std::max<i64>(nyh, 1));
    h->leaves = dupload(leaves, st);
    h->ups = dupload(ups, st);
    h->dns = dupload(dns, st);
    h->cpls = dupload(cpls, st);
    h->up_lv = dupload(up_lv, st);
    h->up_sub = dupload(up_sub, st);
    h->dn_sub = dupload(dn_sub, st);
    h->cnt = dalloc<int32_t>(std::max<size_t>(ups.size(), 1));
    LH_CUDA(cudaMemsetAsync(h->cnt, 0, sizeof(int32_t) * std::max<size_t>(ups.size(), 1), st));
    h->dn_path = dupload(dn_path, st);
    h->dn_pbeg = dupload(dn_pbeg, st);
    h->dn_lv = dupload(dn_lv, st);
    h->pb = dalloc<double>(std::max<i64>(plen, 1) + 4);  // + 4: bulk-copy tail slack
    LH_CUDA(cudaMemsetAsync(h->pb, 0, sizeof(double) * (std::max<i64>(plen, 1) + 4), st));
    h->tu = dalloc<double>(std::max<i64>(tulen, 2) + 4);
    h->td = dalloc<double>(std::max<i64>(tdlen, 2) + 4);
    h->sb = dalloc<double>(std::max<i64>(sblen, 1) + 4);
    h->xh = dalloc<double>(std::max<i64>(nxh, 1));
    run_copies(pj, C.Qt, h->pb);
    run_copies(tj, C.Qt, h->tu);
    run_copies(dj2, R.Qt, h->td);
    if (!sj.empty()) {
        SJob *d = dupload(sj, st);
        spro_kernel<<<(int)std::min<size_t>((sj.size() + NW - 1) / NW, 148 * 16), NT, 0, st>>>(d, (int)sj.size(), R.Ct,
                                                                                            C.Ct, h->sb);
        LH_CUDA(cudaGetLastError());
        LH_CUDA(cudaStreamSynchronize(st));
        cudaFree(d);
    }
    LH_CUDA(cudaStreamSynchronize(st));
    h->bytes = 8 * (plen + tulen + tdlen + sblen) + 8 * (i64)Z.ncols;
    {  // multi-RHS walk (h2mm.cu): Yh rows of row leaves with a basis are the ZS plan's T rows
        H2MMInput mi;
        mi.leaves = &leaves;
        mi.ups = &ups;
        mi.up_height = up_h;
        mi.dns = &dns;
        mi.cpls = &cpls;
        const i64 tbase = (i64)plan->nblk * KC_MAX;
        std::vector<int32_t> yrow(RT.nodes.size(), -1);
        for (size_t c = 0; c < RT.nodes.size(); ++c)
            if (yoff[c] >= 0)
                yrow[c] = (RT.nodes[c].leaf() && qnode[c] >= 0) ? plan->blk_of_node[qnode[c]] * KC_MAX
                                                                 : (int32_t)(tbase + yoff[c]);
        for (size_t d = 0; d < dns.size(); ++d) {
            const int c = dn_cl[d], p = R.parent[c];
            mi.dn_depth.push_back(RT.nodes[c].depth);
            mi.dn_row.push_back(yrow[c]);
            mi.dn_prow.push_back(dns[d].kp > 0 && p >= 0 ? yrow[p] : -1);
        }
        mi.nxh = nxh;
        mi.nyrows = tbase + nyh;
        mi.pb = h->pb;
        mi.tu = h->tu;
        mi.td = h->td;
        mi.sb = h->sb;
        h->mm = build_h2mm(mi, st);
    }
    // fused single-RHS step (default; LEVYH_H2_NOFUSE keeps the combined segment pass): the
    // dense leaves get a plan of their own for the co-resident segment kernel, and every row
    // leaf is assigned to a row-subtree CTA that finishes its rows (leaves without a basis
    // round-robin)
    if (!getenv("LEVYH_H2_NOFUSE") && !getenv("LEVYH_H2_SPLIT_DENSE") && !subs_dn.empty()) {
        std::vector<std::vector<H2QLeaf>> per(subs_dn.size());
        size_t rr = 0;
        for (int32_t lc : RT.leaves) {
            const Cluster &cl = RT.nodes[lc];
            if (cl.size() > 64) return h2_fail("row leaf above 64 rows");
            H2QLeaf q{0, cl.lo, (int32_t)cl.size(), 0, 0, 0};
            int sub = -1;
            if (qnode[lc] >= 0 && insub[lc] >= 0) {
                const Node &nd = ZS.nodes[qnode[lc]];
                q.qoff = nd.uoff;
                q.k = nd.kcap;
                sub = insub[lc];
                q.yloc = yoff[lc] - dn_sub[sub].base;
            } else if (qnode[lc] >= 0) {
                return false;  // a basis outside every row subtree (not produced by the builder)
            } else {
                sub = (int)(rr++ % subs_dn.size());
            }
            per[sub].push_back(q);
        }
        std::vector<H2QLeaf> ql;
        std::vector<int32_t> qb{0};
        for (auto &v : per) {
            ql.insert(ql.end(), v.begin(), v.end());
            qb.push_back((int32_t)ql.size());
        }
        std::vector<int32_t> dense_ids;
        for (int32_t b : ZS.leafblocks)
            if (ZS.nodes[b].kind == K_DENSE) dense_ids.push_back(b);
        const int fgrid = getenv("LEVYH_H2_DENSE_GRID") ? atoi(getenv("LEVYH_H2_DENSE_GRID")) : 0;
        auto fd = build_mv_plan(ZS, dense_ids, st, fgrid);
        fd->lean = getenv("LEVYH_H2_DENSE_CFG") ? atoi(getenv("LEVYH_H2_DENSE_CFG")) : 2;
        // the two-kernel step (h2step.cu): the same pieces cut into per-CTA chunk lists
        {
            H2SInput in;
            in.n = Z.nrows;
            in.leaves = &leaves;
            in.up_leaf_beg = up_leaf_beg;
            in.up_leaf_beg.push_back((int32_t)leaves.size());
            in.ups = &ups;
            in.up_lv = &up_lv;
            in.up_sub = &up_sub;
            in.up_xcnt = &up_xcnt;
            in.maxh_up = maxh_up;
            in.nsub_up = (int)subs_up.size();
            in.dns = &dns;
            in.dn_lv = &dn_lv;
            in.dn_sub = &dn_sub;
            in.dn_ycnt = &dn_ycnt;
            in.dn_path = &dn_path;
            in.dn_pbeg = &dn_pbeg;
            in.cpls = &cpls;
            for (int32_t r0 : subs_dn) in.dn_rows.push_back({RT.nodes[r0].lo, RT.nodes[r0].hi});
            in.maxh_dn = maxh_dn;
            in.nsub_dn = (int)subs_dn.size();
            for (int32_t lc : RT.leaves) {
                const Cluster &cl = RT.nodes[lc];
                H2SInput::RLeaf r{cl.lo, cl.size(), 0, 0, -1, -1};
                if (qnode[lc] >= 0 && insub[lc] >= 0) {
                    const Node &nd = ZS.nodes[qnode[lc]];
                    r.k = nd.kcap;
                    r.qoff = nd.uoff;
                    r.sub = insub[lc];
                    r.yloc = yoff[lc] - dn_sub[insub[lc]].base;
                }
                in.rleaf.push_back(r);
            }
            in.pb = h->pb;
            in.tu = h->tu;
            in.td = h->td;
            in.sb = h->sb;
            in.zarena = ZS.d_arena;
            in.segs.resize(fd->nseg);
            in.batches.resize(fd->nbatch);
            LH_CUDA(cudaMemcpy(in.segs.data(), fd->segs, sizeof(SegDesc) * fd->nseg, cudaMemcpyDeviceToHost));
            LH_CUDA(cudaMemcpy(in.batches.data(), fd->batches, sizeof(SBatch) * fd->nbatch, cudaMemcpyDeviceToHost));
            in.pbuf = fd->pbuf;
            if (!build_h2s(in, *h, ctx.num_sms, st) && getenv("LEVYH_PLAN_VERBOSE"))
                fprintf(stderr, "[levyh] H2 step kernels: not built (previous fused step in use)\n");
        }
        h->qleaf = dupload(ql, st);
        h->dn_qbeg = dupload(qb, st);
        h->zarena = ZS.d_arena;
        h->yd = dalloc<double>(std::max<i64>(Z.nrows, 1));
        plan->fdense = fd;
        if (!plan->fork) {
            int lo = 0, hi = 0;
            LH_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            LH_CUDA(cudaStreamCreateWithPriority(&plan->fork, cudaStreamNonBlocking, lo));
            for (cudaEvent_t &e : plan->fev) LH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
    }
    if (big_subtree && !h->step2) return h2_fail(big_subtree);
    plan->h2 = h;
    if (stats) {
        double ks = 0, nl = 0;
        for (int32_t lc : RT.leaves) ks += R.k[lc], nl += 1;
        for (int32_t lc : CT.leaves) ks += C.k[lc], nl += 1;
        stats[0] = ks / std::max(nl, 1.0);                  // mean leaf basis size
        stats[1] = (double)(plen + tulen + tdlen + sblen);  // column bases + transfers + couplings
        stats[2] = (double)aoff;                            // dense + row bases scalars
    }
    if (getenv("LEVYH_PLAN_VERBOSE"))
        fprintf(stderr, "[levyh] H2: %d/%d subtrees (split %d), path <= %d, P %.1f M, Tc %.1f M, Tr %.1f M, "
                        "S %.1f M, dense + Q %.1f M scalars, max height %d/%d, stage %d/%d doubles\n", h->nsub_up,
                h->nsub_dn, split, maxpath, plen * 1e-6, tulen * 1e-6, tdlen * 1e-6, sblen * 1e-6, aoff * 1e-6,
                R.maxh, C.maxh, up_tmax, dn_tmax);
    return true;
}

}  // namespace lh
