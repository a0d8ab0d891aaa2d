// H-matvec y = alpha H x + beta z (hops.py:50-70) as a two-phase HBM-streaming kernel pair.
//
// Phase 1 (vtx_kernel): for every low-rank block b, t_b = V_b^T x, one warp per <= 1024-row
//          chunk of V_b (chunk partials reduced by treduce_kernel; deterministic, no atomics);
//          tscatter_kernel then copies t_b once per row segment the block covers,
//          segment-ordered (tseg), so a segment's t values are contiguous.
// Phase 2: every row segment (<= 64 rows of a leaf cluster) accumulates its dense pieces D x
//          and its low-rank pieces U_b[seg, :] t_b and writes y[seg] once.
//          seg_tma_kernel: persistent, one CTA per SM over a byte-balanced contiguous range
//          of segments; a producer lane streams piece-aligned batches (<= 32 KB) of the
//          packed operands with cp.async.bulk into a 5-stage shared-memory ring (full/empty
//          mbarriers), together with each batch's piece descriptors, t_b span and x slice;
//          eight consumer warps compute from shared memory.
//          seg_kernel: the same per-segment work with direct loads (LEVYH_SEG_DIRECT=1).
// The operands are gathered once per plan into a packed buffer in streaming order.
#include <algorithm>
#include <map>

#include "core.h"
#include "dev.cuh"
#include "matvec.h"
#include "h2step.h"

namespace lh {

using dev::KC_MAX;
using dev::NT;

constexpr int SEG = 64;         // rows per segment
constexpr int GRP = NT / SEG;   // thread groups per segment
constexpr i64 VCHUNK_DEFAULT = 1024;  // rows of V per phase-1 chunk (one warp)
static i64 vchunk_rows() {
    static const i64 v = getenv("LEVYH_VCHUNK") ? std::max(64, atoi(getenv("LEVYH_VCHUNK"))) : VCHUNK_DEFAULT;
    return v;
}
#ifndef SEG_MIN_BLOCKS
#define SEG_MIN_BLOCKS 4        // CTAs per SM for the direct-load segment kernel
#endif
constexpr int SLOT_D = 5120;    // doubles of operand data per ring slot (40 KB: a 64 x 64 dense leaf plus a basis of <= 16 columns)
constexpr int SLOT_A = 1024;    // doubles of aux (descriptors, t_b span, x slice) per slot
constexpr int DESC_D = 64;      // aux doubles reserved for piece descriptors (32 x 16 B)
constexpr int MAX_PIECES = 32;  // pieces per batch

// ---------------------------------------------------------------------------
// phase 1
// ---------------------------------------------------------------------------
// Sum RB per-lane values over the warp, column c ending in lane group c (see vtx_warp).
template <int RB>
__device__ __forceinline__ void warp_transpose_reduce(double (&acc)[RB], int lane) {
#pragma unroll
    for (int o = 16, h = RB / 2; h >= 1; o >>= 1, h >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int k = 0; k < h; ++k) {
            const double send = up ? acc[k] : acc[k + h];
            const double keep = up ? acc[k + h] : acc[k];
            acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    constexpr int LOW = 32 / RB;
#pragma unroll
    for (int o = LOW / 2; o >= 1; o >>= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], o);
}

// one warp per chunk: each lane accumulates all r columns for its rows (x[i] read once,
// r coalesced loads per row), then warp shuffles reduce.  Every iteration issues all of its
// RB * ROWS loads before the first FMA (one memory round trip per iteration); RB * ROWS = 16
// loaded values + RB accumulators fit the 64-register budget of 4 CTAs per SM without spills.
template <int RB, int ROWS>
__device__ __forceinline__ void vtx_warp(const VChunk &C, const double *pbuf, const double *x,
                                         double *out, int lane) {
    const int r = vc_rank(C);
    const int len = C.len;
    const double *V = pbuf + C.voff;
    const double *xx = x + C.xc0;
    const int ld = len;
    double acc[RB];
#pragma unroll
    for (int c = 0; c < RB; ++c) acc[c] = 0.0;
    int i = lane;
    for (; i + 32 * (ROWS - 1) < len; i += 32 * ROWS) {
        double xv[ROWS], v[ROWS][RB];
#pragma unroll
        for (int q = 0; q < ROWS; ++q) xv[q] = __ldg(xx + i + 32 * q);
        const double *p = V + i;
#pragma unroll
        for (int c = 0; c < RB; ++c) {
#pragma unroll
            for (int q = 0; q < ROWS; ++q) v[q][c] = c < r ? __ldcs(p + 32 * q) : 0.0;
            p += ld;
        }
#pragma unroll
        for (int c = 0; c < RB; ++c)
#pragma unroll
            for (int q = 0; q < ROWS; ++q) acc[c] = fma(v[q][c], xv[q], acc[c]);
    }
    for (; i < len; i += 32) {
        const double xi = xx[i];
        const double *p = V + i;
#pragma unroll
        for (int c = 0; c < RB; ++c) {
            if (c < r) acc[c] = fma(__ldcs(p), xi, acc[c]);
            p += ld;
        }
    }
    // transpose-reduce: each butterfly level halves the columns a lane carries (send the half
    // the partner keeps), so RB columns cost RB/2 + RB/4 + ... + 1 + 2 shuffles instead of
    // 5 RB; afterwards lane l holds the full sum of column col(l) (bits 4.. of l, MSB first)
    warp_transpose_reduce<RB>(acc, lane);
    {
        int c = 0;
#pragma unroll
        for (int o = 16, h = RB / 2; h >= 1; o >>= 1, h >>= 1) c = 2 * c + ((lane & o) ? 1 : 0);
        constexpr int LOW = 32 / RB;  // lanes sharing one column after the exchange levels
        if ((lane & (LOW - 1)) == 0 && c < r) out[c] = acc[0];
    }
    // ranks above RB: remaining columns one at a time
    for (int c = RB; c < r; ++c) {
        const double *v = V + (i64)c * ld;
        double t = 0.0;
        for (int q = lane; q < len; q += 32) t += v[q] * xx[q];
        t = dev::warp_sum(t);
        if (lane == 0) out[c] = t;
    }
}

#ifndef VTX_MIN_BLOCKS
#define VTX_MIN_BLOCKS 3
#endif
template <int RB>
__global__ void __launch_bounds__(NT, VTX_MIN_BLOCKS)
    vtx_kernel(const VChunk *chunks, int nch, const double *pbuf, const double *x, double *part,
               double *tvec) {
    const int lane = threadIdx.x & 31;
    const int stride = gridDim.x * dev::NW;
    int q = blockIdx.x * dev::NW + (threadIdx.x >> 5);
    if (q >= nch) return;
    // the next chunk's descriptor is loaded while this chunk streams (one fewer dependent
    // memory round trip per chunk), spread one 32-bit word per lane so that it holds a single
    // register through the streaming loop
    static_assert(sizeof(VChunk) == 32, "VChunk is 8 words");
    auto word = [&](int qq) {
        return lane < 8 ? __ldg(reinterpret_cast<const int32_t *>(chunks + qq) + lane) : 0;
    };
    auto unpack = [&](int32_t w) {
        VChunk C;
        int32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __shfl_sync(0xffffffffu, w, k);
        C.voff = (i64)(((unsigned long long)(uint32_t)v[1] << 32) | (uint32_t)v[0]);
        C.xc0 = (i64)(((unsigned long long)(uint32_t)v[3] << 32) | (uint32_t)v[2]);
        C.len = v[4];
        C.r = v[5];
        C.blk = v[6];
        C.pidx = v[7];
        return C;
    };
    int32_t w = word(q);
    while (true) {
        const VChunk C = unpack(w);
        const int qn = q + stride;
        if (qn < nch) w = word(qn);
        double *out = (C.pidx >= 0 ? part + (i64)C.pidx * KC_MAX : tvec + (i64)C.blk * KC_MAX) +
                      vc_col0(C);
        vtx_warp<RB, 16 / RB>(C, pbuf, x, out, lane);
        if (qn >= nch) break;
        q = qn;
    }
}

// t_b[c] = sum of the chunk partials of a multi-chunk block: one CTA per block, warp w sums
// the chunks w, w + 8, ... (lane = column, four loads in flight), then warp 0 adds the eight
// warp sums in order (deterministic)
__global__ void treduce_kernel(const TJob *jobs, int njobs, const double *part, double *tvec) {
    __shared__ double sm[dev::NW][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int j = blockIdx.x; j < njobs; j += gridDim.x) {
        const TJob J = jobs[j];
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        if (lane < J.r) {
            const double *p = part + lane;
            int k = J.cbeg + w;
            for (; k + 3 * dev::NW < J.cend; k += 4 * dev::NW) {
                a0 += p[(i64)k * KC_MAX];
                a1 += p[(i64)(k + dev::NW) * KC_MAX];
                a2 += p[(i64)(k + 2 * dev::NW) * KC_MAX];
                a3 += p[(i64)(k + 3 * dev::NW) * KC_MAX];
            }
            for (; k < J.cend; k += dev::NW) a0 += p[(i64)k * KC_MAX];
        }
        sm[w][lane] = (a0 + a1) + (a2 + a3);
        __syncthreads();
        if (w == 0 && lane < J.r) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < dev::NW; ++q) s += sm[q][lane];
            tvec[(i64)J.blk * KC_MAX + lane] = s;
        }
        __syncthreads();
    }
}

// TMA kernel inputs: batch-ordered low-rank coefficients tcol[e] = tvec[tmap[e]], and x
// copied into an aligned buffer with two doubles of zero padding (16-byte bulk copies)
__global__ void tgather_kernel(const int32_t *tmap, i64 n, const double *tvec, double *tcol,
                               const double *x, i64 nx, double *xpad) {
    for (i64 e = (i64)blockIdx.x * NT + threadIdx.x; e < n + nx + 2; e += (i64)gridDim.x * NT) {
        if (e < n) {
            const int32_t m = tmap[e];
            tcol[e] = m >= 0 ? tvec[m] : 0.0;
        } else {
            const i64 i = e - n;
            xpad[i] = i < nx ? x[i] : 0.0;
        }
    }
}

// ---------------------------------------------------------------------------
// phase 2, direct loads
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT, SEG_MIN_BLOCKS)
    seg_kernel(const SegDesc *segs, int nseg, const MvDense *dp, const MvLr *lp, const double *pbuf,
               const double *tvec, const double *x, double *y, double alpha, double beta,
               const double *z) {
    __shared__ double acc_s[GRP][SEG];
    const int row = threadIdx.x % SEG, g = threadIdx.x / SEG;
    for (int s = blockIdx.x; s < nseg; s += gridDim.x) {
        const SegDesc S = segs[s];
        const i64 ld = S.ld;
        double acc = 0.0;
        if (row < S.rows) {
            // dense pieces: columns split over the GRP groups; a full 64-column piece issues
            // its 16 loads per thread before any FMA
            for (int p = S.dbeg; p < S.dend; ++p) {
                const MvDense P = dp[p];
                const double *D = pbuf + P.off + row;
                const double *xx = x + P.xc0;
                if (P.ncols == 64) {
                    double d[16], xv[16];
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        d[q] = D[(g + GRP * q) * ld];
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
                        a0 += D[j * ld] * xx[j];
                        a1 += D[(j + GRP) * ld] * xx[j + GRP];
                    }
                    if (j < P.ncols) a0 += D[j * ld] * xx[j];
                    acc += a0 + a1;
                }
            }
            // low-rank pieces, four at a time so their descriptor -> U load chains overlap
            int p = S.lbeg;
            for (; p + 4 <= S.lend; p += 4) {
                MvLr Q[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) Q[k] = lp[p + k];
                double u0[4], u1[4], t0[4], t1[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double *U = pbuf + Q[k].off + row;
                    const double *tb = tvec + (i64)Q[k].blk * KC_MAX;
                    u0[k] = g < Q[k].r ? U[g * ld] : 0.0;
                    t0[k] = g < Q[k].r ? tb[g] : 0.0;
                    u1[k] = g + GRP < Q[k].r ? U[(g + GRP) * ld] : 0.0;
                    t1[k] = g + GRP < Q[k].r ? tb[g + GRP] : 0.0;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) acc += u0[k] * t0[k] + u1[k] * t1[k];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double *U = pbuf + Q[k].off + row;
                    const double *tb = tvec + (i64)Q[k].blk * KC_MAX;
                    for (int c = g + 2 * GRP; c < Q[k].r; c += GRP) acc += U[c * ld] * tb[c];
                }
            }
            for (; p < S.lend; ++p) {
                const MvLr P = lp[p];
                const double *U = pbuf + P.off + row;
                const double *tb = tvec + (i64)P.blk * KC_MAX;
                for (int c = g; c < P.r; c += GRP) acc += U[c * ld] * tb[c];
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
// phase 2, bulk-copy (TMA) pipeline
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
template <int CONS>
__device__ __forceinline__ void consumer_sync() {  // the consumer warps only
    asm volatile("bar.sync 1, %0;" ::"n"(CONS) : "memory");
}

constexpr int XOFF = 0;    // aux: x slice (<= 66 doubles)
constexpr int TOFF = 128;  // aux: low-rank coefficients (<= MAXK)
constexpr int MAXK = 128;  // columns per batch (segments of < 32 rows would allow more)

// ST ring stages, CONS consumer threads (64 rows x CONS / 64 column groups).  The full
// configuration (5 stages, 16 consumer warps) owns an SM; the lean one (3 stages, 8 consumer
// warps: 128 KB, ~28 K registers) leaves room for the H2 walk CTAs that run beside it.
template <int ST, int CONS>
struct TmaSmem {
    double data[ST][SLOT_D];
    double aux[ST][TOFF + MAXK];
    double red[2][CONS / SEG][SEG];  // double-buffered: one consumer barrier per segment
    uint64_t full[ST], empty[ST];
    int32_t hdr[ST][4];  // K, kd, xadj
};
template <int ST, int CONS>
constexpr size_t tma_smem() { return sizeof(TmaSmem<ST, CONS>) + 128; }

template <int ST, int CONS>
__global__ void __launch_bounds__(CONS + 32, 1)
    seg_tma_kernel(const SegDesc *segs, const int32_t *cta_seg, const SBatch *batches,
                   const double *pbuf, const double *tcol, const double *x, double *y,
                   double alpha, double beta, const double *z) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int TMA_STAGES = ST, TMA_CONS = CONS, TGRP = CONS / SEG;
    TmaSmem<ST, CONS> &S = *reinterpret_cast<TmaSmem<ST, CONS> *>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < TMA_STAGES; ++i) {
            mbar_init(&S.full[i], 1);
            mbar_init(&S.empty[i], TMA_CONS / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int s0 = cta_seg[blockIdx.x], s1 = cta_seg[blockIdx.x + 1];
    if (warp == 0) {
        // producer: lane 0 walks this CTA's batches with a 4-deep register queue of
        // descriptors (loads in flight ahead of use) and issues the bulk copies,
        // TMA_STAGES slots ahead of the consumers
        if (lane == 0 && s0 < s1) {
            const int b0 = segs[s0].bbeg, b1 = segs[s1 - 1].bend;
            int stage = 0;
            uint32_t phase = 0;
            SBatch q0 = batches[b0];
            SBatch q1 = b0 + 1 < b1 ? batches[b0 + 1] : q0;
            SBatch q2 = b0 + 2 < b1 ? batches[b0 + 2] : q0;
            SBatch q3 = b0 + 3 < b1 ? batches[b0 + 3] : q0;
            for (int b = b0; b < b1; ++b) {
                const SBatch B = q0;
                q0 = q1;
                q1 = q2;
                q2 = q3;
                if (b + 4 < b1) q3 = batches[b + 4];
                mbar_wait(&S.empty[stage], phase ^ 1);
                S.hdr[stage][0] = B.K;
                S.hdr[stage][1] = B.kd;
                S.hdr[stage][2] = B.xadj;
                mbar_expect_tx(&S.full[stage], (uint32_t)B.total);
                const uint32_t tb = (uint32_t)(8 * ((B.K - B.kd + 1) & ~1));
                const uint32_t xb = B.kd ? (uint32_t)(8 * ((B.xadj + B.kd + 1) & ~1)) : 0u;
                bulk_g2s(S.data[stage], pbuf + B.src, (uint32_t)B.total - tb - xb, &S.full[stage]);
                if (tb) bulk_g2s(S.aux[stage] + TOFF, tcol + B.tsrc, tb, &S.full[stage]);
                if (xb) bulk_g2s(S.aux[stage] + XOFF, x + B.xsrc, xb, &S.full[stage]);
                if (++stage == TMA_STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        return;
    }
    // consumers: 64 rows x 8 column groups; group g takes columns g, g + 8, ... of each batch
    const int tid = threadIdx.x - 32, row = tid % SEG, g = tid / SEG;
    int stage = 0;
    uint32_t phase = 0;
    SegDesc sd = s0 < s1 ? segs[s0] : SegDesc{};
    for (int s = s0; s < s1; ++s) {
        const SegDesc cur = sd;
        // z row issued now, consumed after the batches: its latency hides behind them
        const double zv = (g == 0 && beta != 0.0 && row < cur.rows) ? z[cur.y0 + row] : 0.0;
        if (s + 1 < s1) sd = segs[s + 1];  // prefetch
        const int ld = cur.ld;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        for (int b = cur.bbeg; b < cur.bend; ++b) {
            mbar_wait(&S.full[stage], phase);
            const int K = S.hdr[stage][0], kd = S.hdr[stage][1], xadj = S.hdr[stage][2];
            const double *col = S.data[stage] + row;
            // dense columns [0, kd) against the x slice, low-rank columns [kd, K) against t
            {
                const double *cf = S.aux[stage] + XOFF + xadj;
                int k = g;
                for (; k + 3 * TGRP < kd; k += 4 * TGRP) {
                    const double c0 = cf[k], c1 = cf[k + TGRP], c2 = cf[k + 2 * TGRP], c3 = cf[k + 3 * TGRP];
                    const double m0 = col[k * ld], m1 = col[(k + TGRP) * ld];
                    const double m2 = col[(k + 2 * TGRP) * ld], m3 = col[(k + 3 * TGRP) * ld];
                    a0 += m0 * c0;
                    a1 += m1 * c1;
                    a2 += m2 * c2;
                    a3 += m3 * c3;
                }
                for (; k < kd; k += TGRP) a0 += col[k * ld] * cf[k];
            }
            {
                const double *cf = S.aux[stage] + TOFF - kd;
                int k = kd + g;
                for (; k + 3 * TGRP < K; k += 4 * TGRP) {
                    const double c0 = cf[k], c1 = cf[k + TGRP], c2 = cf[k + 2 * TGRP], c3 = cf[k + 3 * TGRP];
                    const double m0 = col[k * ld], m1 = col[(k + TGRP) * ld];
                    const double m2 = col[(k + 2 * TGRP) * ld], m3 = col[(k + 3 * TGRP) * ld];
                    a0 += m0 * c0;
                    a1 += m1 * c1;
                    a2 += m2 * c2;
                    a3 += m3 * c3;
                }
                for (; k < K; k += TGRP) a1 += col[k * ld] * cf[k];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.empty[stage]);
            if (++stage == TMA_STAGES) {
                stage = 0;
                phase ^= 1;
            }
        }
        double(*red)[SEG] = S.red[(s - s0) & 1];
        red[g][row] = (a0 + a1) + (a2 + a3);
        consumer_sync<CONS>();
        if (g == 0 && row < cur.rows) {
            double v = red[0][row];
#pragma unroll
            for (int q = 1; q < TGRP; ++q) v += red[q][row];
            y[cur.y0 + row] = (beta == 0.0 ? 0.0 : beta * zv) + alpha * v;
        }
    }
}

// gather the operands into the packed buffer (once per plan)
__global__ void pack_kernel(const PackJob *jobs, int njobs, const double *arena, double *pbuf) {
    for (int j = blockIdx.x; j < njobs; j += gridDim.x) {
        const PackJob J = jobs[j];
        const i64 n = (i64)J.rows * J.cols;
        for (i64 e = threadIdx.x; e < n; e += NT) {
            const i64 c = e / J.rows, i = e - c * J.rows;
            pbuf[J.dst + i + c * J.ld] = arena[J.src + i + c * J.src_ld];
        }
    }
}

// ---------------------------------------------------------------------------
// plan construction
// ---------------------------------------------------------------------------
static i64 even(i64 v) { return (v + 1) & ~i64(1); }

// Builds a plan over the given leaf blocks (default: all of H).  Row segments are the leaf
// clusters of the row tree split into <= SEG rows.
std::shared_ptr<MvPlan> build_mv_plan(HMat &H, const std::vector<int32_t> &blocks, cudaStream_t s,
                                      int tma_grid) {
    auto P = std::make_shared<MvPlan>();
    H.sync_ranks(s);  // the packed layout is sized by the current ranks
    const Tree &rt = *H.rt;
    std::vector<i64> seg_start;
    for (int32_t lc : rt.leaves) {
        const Cluster &c = rt.nodes[lc];
        for (i64 a = c.lo; a < c.hi; a += SEG) seg_start.push_back(a);
    }
    seg_start.push_back(rt.n);
    const int nseg = (int)seg_start.size() - 1;
    auto seg_of = [&](i64 row) {
        return (int)(std::upper_bound(seg_start.begin(), seg_start.end(), row) - seg_start.begin()) - 1;
    };
    struct DRef {
        i64 src, ld, xc0;
        int32_t ncols;
    };
    struct LRef {
        i64 src, ld;
        int32_t r, blk;
    };
    std::vector<std::vector<DRef>> dps(nseg);
    std::vector<std::vector<LRef>> lps(nseg);
    std::vector<VChunk> chunks, chunks16;
    std::vector<i64> vld, vld16;  // source ld (block row count of V) per chunk
    std::vector<TJob> tjobs;
    int nblk = 0, npart = 0;
    P->blk_of_node.assign(H.nodes.size(), -1);
    for (int32_t b : blocks) {
        const Node &nd = H.nodes[b];
        if (nd.kind == K_DENSE || nd.kind == K_FDENSE) {
            for (int sg = seg_of(nd.r0); sg < nseg && seg_start[sg] < nd.r0 + nd.m; ++sg) {
                i64 a = std::max(seg_start[sg], nd.r0), e = std::min(seg_start[sg + 1], nd.r0 + nd.m);
                LH_REQUIRE(a == seg_start[sg] && e == seg_start[sg + 1], LH_EINTERNAL,
                           "dense block not aligned with row segments");
                // pieces of at most 64 columns (one ring slot with ld <= 64)
                for (i64 j0 = 0; j0 < nd.n; j0 += 64)
                    dps[sg].push_back({nd.doff + (a - nd.r0) + j0 * nd.m, nd.m, nd.c0 + j0,
                                       (int32_t)std::min<i64>(64, nd.n - j0)});
            }
        } else if (nd.kind == K_LR) {
            const int r = H.h_ranks[nd.rslot];
            LH_REQUIRE(r <= KC_MAX, LH_EINTERNAL, "rank above the matvec capacity");
            if (r == 0) continue;
            const int blk = nblk++;
            P->blk_of_node[b] = blk;
            // ranks above 8 are split into column groups of <= 8 (the rank-8 V^T x kernel
            // keeps twice the loads in flight per register of the rank-16 one)
            static const bool split = !getenv("LEVYH_VTX16");
            std::vector<VChunk> &dst = (r > 8 && !split) ? chunks16 : chunks;
            std::vector<i64> &dld = (r > 8 && !split) ? vld16 : vld;
            const int cg = split ? 8 : r;
            auto emit = [&](i64 a, int len, int pidx) {
                for (int c0 = 0; c0 < r; c0 += cg) {
                    const int rr = std::min(cg, r - c0);
                    dst.push_back({nd.voff + a + (i64)c0 * nd.n, nd.c0 + a, len, rr | (c0 << 16), blk, pidx});
                    dld.push_back(nd.n);
                }
            };
            const i64 VCHUNK = vchunk_rows();
            if (nd.n == 0) {
                // row-only node (shared row basis): t_b comes from the coupling kernels
            } else if (nd.n <= VCHUNK) {
                emit(0, (int)nd.n, -1);
            } else {
                int cb = npart;
                for (i64 a = 0; a < nd.n; a += VCHUNK) emit(a, (int)std::min(VCHUNK, nd.n - a), npart++);
                tjobs.push_back({blk, r, cb, npart});
            }
            for (int sg = seg_of(nd.r0); sg < nseg && seg_start[sg] < nd.r0 + nd.m; ++sg) {
                i64 a = std::max(seg_start[sg], nd.r0), e = std::min(seg_start[sg + 1], nd.r0 + nd.m);
                LH_REQUIRE(a == seg_start[sg] && e == seg_start[sg + 1], LH_EINTERNAL,
                           "low-rank block not aligned with row segments");
                lps[sg].push_back({nd.uoff + (a - nd.r0), nd.m, r, blk});
            }
        }
    }
    if (getenv("LEVYH_PLAN_VERBOSE")) {
        for (int k = 0; k < 2; ++k) {
            const std::vector<VChunk> &cv = k ? chunks16 : chunks;
            std::map<std::pair<int, int>, std::pair<i64, double>> h;  // (len class, r) -> count, MB
            for (const VChunk &c : cv) {
                int lc = 1;
                while (lc < c.len) lc *= 2;
                auto &e = h[{lc, vc_rank(c)}];
                e.first++;
                e.second += 8.0 * c.len * vc_rank(c) / 1e6;
            }
            fprintf(stderr, "[mv plan] %s chunks %zu:", k ? "rank>8" : "rank<=8", cv.size());
            for (auto &e : h)
                fprintf(stderr, " len<=%d,r=%d:%lld(%.0fMB)", e.first.first, e.first.second,
                        (long long)e.second.first, e.second.second);
            fprintf(stderr, "\n");
        }
    }
    // packed layout (columns of ld = even(rows)) + bulk-copy batches of <= SLOT_D doubles,
    // at most one dense piece per batch and only as its first columns
    std::vector<PackJob> jobs;
    std::vector<SegDesc> segs(nseg);
    std::vector<MvDense> dall;
    std::vector<MvLr> lall;
    std::vector<SBatch> batches;
    std::vector<int32_t> tmap;
    std::vector<i64> seg_bytes(nseg, 0);
    i64 poff = 0;
    std::vector<int32_t> colmap;
    for (int sg = 0; sg < nseg; ++sg) {
        SegDesc &S = segs[sg];
        S.y0 = seg_start[sg];
        S.rows = (int32_t)(seg_start[sg + 1] - seg_start[sg]);
        S.ld = (int32_t)even(S.rows);
        S.poff = poff;
        S.cmoff = (int32_t)colmap.size();
        const i64 ld = S.ld;
        const int kmax = (int)std::min<i64>(MAXK, SLOT_D / ld);
        S.dbeg = (int32_t)dall.size();
        S.lbeg = (int32_t)lall.size();
        S.bbeg = (int32_t)batches.size();
        SBatch B{};
        auto close = [&]() {
            if (B.K == 0) return;
            const i64 tb = 8 * even(B.K - B.kd), xb = B.kd ? 8 * even(B.xadj + B.kd) : 0;
            B.total = (int32_t)(8 * B.K * ld + tb + xb);
            batches.push_back(B);
            seg_bytes[sg] += B.total;
            B = SBatch{};
        };
        auto open = [&]() {
            B = SBatch{};
            B.src = poff;
            B.tsrc = (i64)tmap.size();
        };
        open();
        for (const DRef &d : dps[sg]) {
            if (B.K > 0) {  // a dense piece always starts a batch
                close();
                open();
            }
            jobs.push_back({d.src, d.ld, poff, S.rows, d.ncols, S.ld, 0});
            dall.push_back({poff, d.xc0, d.ncols, 0});
            B.K = B.kd = d.ncols;
            for (int j = 0; j < d.ncols; ++j) colmap.push_back((int32_t)(d.xc0 + j));
            B.xsrc = d.xc0 & ~i64(1);
            B.xadj = (int32_t)(d.xc0 - B.xsrc);
            poff += (i64)d.ncols * ld;
        }
        for (const LRef &l : lps[sg]) {
            if (B.K + l.r > kmax) {
                close();
                open();
            }
            jobs.push_back({l.src, l.ld, poff, S.rows, l.r, S.ld, 0});
            lall.push_back({poff, l.r, l.blk});
            for (int c = 0; c < l.r; ++c) {
                tmap.push_back(l.blk * KC_MAX + c);
                colmap.push_back(-(1 + l.blk * KC_MAX + c));
            }
            B.K += l.r;
            poff += (i64)l.r * ld;
        }
        close();
        S.ncol = (int32_t)(colmap.size() - S.cmoff);
        // every batch's coefficient span starts 16-byte aligned in tcol
        if (tmap.size() & 1) tmap.push_back(-1);
        S.dend = (int32_t)dall.size();
        S.lend = (int32_t)lall.size();
        S.bend = (int32_t)batches.size();
    }
    // batches opened mid-segment took tsrc before alignment padding of the previous segment
    // only at segment starts; within a segment they are contiguous: re-derive aligned spans
    {
        std::vector<int32_t> tm2;
        for (int sg = 0; sg < nseg; ++sg)
            for (int b = segs[sg].bbeg; b < segs[sg].bend; ++b) {
                SBatch &B = batches[b];
                const i64 nlr = B.K - B.kd;
                const i64 from = B.tsrc;
                B.tsrc = (i64)tm2.size();
                for (i64 e = 0; e < nlr; ++e) tm2.push_back(tmap[from + e]);
                if (tm2.size() & 1) tm2.push_back(-1);
            }
        tmap.swap(tm2);
    }
    for (int k = 0; k < 2; ++k) {
        std::vector<VChunk> &cv = k ? chunks16 : chunks;
        const std::vector<i64> &ld = k ? vld16 : vld;
        for (size_t q = 0; q < cv.size(); ++q) {
            VChunk &c = cv[q];
            jobs.push_back({c.voff, ld[q], poff, c.len, vc_rank(c), c.len, 0});
            c.voff = poff;
            poff += even((i64)c.len * vc_rank(c));
        }
        // largest chunks first: the grid-stride warps (and the hardware block scheduler behind
        // them) then finish on the small chunks instead of starting a 1024-row chunk last
        if (!getenv("LEVYH_VTX_NOSORT"))
            std::stable_sort(cv.begin(), cv.end(), [](const VChunk &a, const VChunk &b) {
                return (i64)a.len * vc_rank(a) > (i64)b.len * vc_rank(b);
            });
    }
    // TMA kernel: contiguous, byte-balanced segment ranges, one CTA per SM
    int dev_id = 0, num_sms = 148;
    cudaGetDevice(&dev_id);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev_id);
    const int G = std::max(1, std::min(tma_grid > 0 ? tma_grid : num_sms, nseg));
    std::vector<int32_t> cta_seg(G + 1, nseg);
    {
        i64 total = 0;
        for (i64 v : seg_bytes) total += v;
        cta_seg[0] = 0;
        i64 accb = 0;
        int c = 1;
        for (int sg = 0; sg < nseg && c < G; ++sg) {
            accb += seg_bytes[sg];
            while (c < G && accb * G >= total * c) cta_seg[c++] = sg + 1;
        }
        for (; c < G; ++c) cta_seg[c] = nseg;
        cta_seg[G] = nseg;
    }
    P->nseg = nseg;
    P->nch = (int)chunks.size();
    P->nch16 = (int)chunks16.size();
    P->ntj = (int)tjobs.size();
    P->nbatch = (int)batches.size();
    P->tma_grid = G;
    P->pbuf_len = poff;
    P->pbuf = dalloc<double>(std::max<i64>(poff, 2));
    LH_CUDA(cudaMemsetAsync(P->pbuf, 0, sizeof(double) * std::max<i64>(poff, 2), s));  // pad rows
    P->tcol_len = (i64)tmap.size();
    P->tcol = dalloc<double>(std::max<i64>(P->tcol_len, 2));
    P->tmap = dupload(tmap, s);
    P->tvec = dalloc<double>((i64)std::max(nblk, 1) * KC_MAX);
    P->nx = H.ncols;
    P->xpad = dalloc<double>(H.ncols + 2);
    P->segs = dupload(segs, s);
    P->dp = dupload(dall, s);
    P->lp = dupload(lall, s);
    P->chunks = dupload(chunks, s);
    P->chunks16 = dupload(chunks16, s);
    {  // multi-RHS: chunks over the same x rows grouped (<= 64 output rows per group), so the
       // DMMA V^T X kernel stages each X tile once for all of them (matmat.cu: vtx_mm_group)
        std::map<std::pair<i64, int>, std::vector<VChunk>> by;
        std::vector<std::pair<i64, int>> order;
        for (int k = 0; k < 2; ++k)
            for (const VChunk &c : (k ? chunks16 : chunks)) {
                auto key = std::make_pair(c.xc0, c.len);
                if (!by.count(key)) order.push_back(key);
                by[key].push_back(c);
            }
        std::vector<VChunk> gch;
        std::vector<VGroup> gr;
        for (auto &key : order) {
            VGroup g{key.first, key.second, (int32_t)gch.size(), (int32_t)gch.size(), 0, 0};
            for (const VChunk &c : by[key]) {
                if (g.m + vc_rank(c) > 64) {
                    gr.push_back(g);
                    g = VGroup{key.first, key.second, (int32_t)gch.size(), (int32_t)gch.size(), 0, 0};
                }
                gch.push_back(c);
                g.cend = (int32_t)gch.size();
                g.m += vc_rank(c);
            }
            gr.push_back(g);
        }
        // by x rows: the groups of every level that read the same rows of X run close together,
        // so X comes from HBM about once and from L2 for the other levels
        std::stable_sort(gr.begin(), gr.end(), [](const VGroup &a, const VGroup &b) {
            return a.xc0 != b.xc0 ? a.xc0 < b.xc0 : a.len > b.len;
        });
        P->ngroup = (int)gr.size();
        P->groups = dupload(gr, s);
        P->gchunks = dupload(gch, s);
    }
    P->tjobs = dupload(tjobs, s);
    P->part = dalloc<double>((i64)std::max(npart, 1) * KC_MAX);
    P->batches = dupload(batches, s);
    P->cta_seg = dupload(cta_seg, s);
    // host-buffer pipelining: piece-ordered chunk copies and per-piece segment ranges
    {
        int NP = 4;
        if (const char *e = getenv("LEVYH_PIPE_PIECES")) NP = std::max(1, atoi(e));
        NP = (int)std::max<i64>(1, std::min<i64>(NP, nseg));
        P->npiece = NP;
        P->xcut.resize(NP + 1);
        // only the first x piece and the last y piece are exposed (the copy engine runs ahead
        // of V^T x and behind the segments): make those 1/16 of the vector, the rest equal
        auto frac = [&](int p, bool first_small) {
            if (NP == 1) return (double)p;
            const double f = 1.0 / 16;
            if (first_small) return p == 0 ? 0.0 : f + (1.0 - f) * (p - 1) / (NP - 1);
            return p == NP ? 1.0 : (1.0 - f) * p / (NP - 1);
        };
        for (int p = 0; p <= NP; ++p)
            P->xcut[p] = std::min<i64>(H.ncols, ((i64)(H.ncols * frac(p, true)) + 1) & ~i64(1));
        P->xcut[0] = 0;
        P->xcut[NP] = H.ncols;
        auto piece_of = [&](const VChunk &c) {
            int p = (int)(std::upper_bound(P->xcut.begin(), P->xcut.end(), c.xc0 + c.len - 1) -
                          P->xcut.begin()) - 1;
            return std::min(std::max(p, 0), NP - 1);
        };
        for (int k = 0; k < 2; ++k) {
            const std::vector<VChunk> &cv = k ? chunks16 : chunks;
            std::vector<VChunk> cp(cv.begin(), cv.end());
            std::stable_sort(cp.begin(), cp.end(), [&](const VChunk &a, const VChunk &b) {
                return piece_of(a) < piece_of(b);
            });  // within a piece: still largest first
            std::vector<int32_t> &off = k ? P->pch16 : P->pch;
            off.assign(NP + 1, 0);
            for (const VChunk &c : cp) off[piece_of(c) + 1]++;
            for (int p = 0; p < NP; ++p) off[p + 1] += off[p];
            (k ? P->chunks16_pp : P->chunks_pp) = dupload(cp, s);
        }
        // segment pieces (segments are in row order)
        std::vector<int> ps(NP + 1, nseg);
        ps[0] = 0;
        for (int p = 1; p < NP; ++p) {
            const i64 target = (i64)(H.nrows * frac(p, false));
            int sg = ps[p - 1];
            while (sg < nseg && segs[sg].y0 < target) ++sg;
            ps[p] = sg;
        }
        P->ycut.resize(NP + 1);
        for (int p = 0; p <= NP; ++p) P->ycut[p] = ps[p] < nseg ? segs[ps[p]].y0 : H.nrows;
        std::vector<int32_t> csp((size_t)NP * (G + 1));
        for (int p = 0; p < NP; ++p) {
            int32_t *cs = csp.data() + (size_t)p * (G + 1);
            i64 total = 0;
            for (int sg = ps[p]; sg < ps[p + 1]; ++sg) total += seg_bytes[sg];
            for (int c = 0; c <= G; ++c) cs[c] = ps[p + 1];
            cs[0] = ps[p];
            i64 accb = 0;
            int c = 1;
            for (int sg = ps[p]; sg < ps[p + 1] && c < G; ++sg) {
                accb += seg_bytes[sg];
                while (c < G && accb * G >= total * c) cs[c++] = sg + 1;
            }
        }
        P->cta_seg_pp = dupload(csp, s);
        for (int sg = 1; sg < nseg; ++sg)
            LH_REQUIRE(segs[sg].y0 > segs[sg - 1].y0, LH_EINTERNAL, "segments out of row order");
    }
    P->n_dpieces = (i64)dall.size();
    P->n_lpieces = (i64)lall.size();
    P->colmap = dupload(colmap, s);
    P->ncolmap = (i64)colmap.size();
    P->nblk = nblk;
    P->npart = npart;
    if (!jobs.empty()) {
        PackJob *dj = dupload(jobs, s);
        pack_kernel<<<std::min<int>((int)jobs.size(), 148 * 16), NT, 0, s>>>(dj, (int)jobs.size(),
                                                                            H.d_arena, P->pbuf);
        LH_CUDA(cudaGetLastError());
        LH_CUDA(cudaStreamSynchronize(s));
        cudaFree(dj);
    }
    LH_CUDA(cudaStreamSynchronize(s));
    return P;
}

MvPlan::~MvPlan() {
    if (fork) cudaStreamDestroy(fork);
    for (cudaEvent_t e : fev)
        if (e) cudaEventDestroy(e);
    cudaFree(pbuf);
    cudaFree(tcol);
    cudaFree(tmap);
    cudaFree(xpad);
    cudaFree(colmap);
    cudaFree(segs);
    cudaFree(dp);
    cudaFree(lp);
    cudaFree(chunks);
    cudaFree(chunks16);
    cudaFree(groups);
    cudaFree(gchunks);
    cudaFree(tjobs);
    cudaFree(part);
    cudaFree(tvec);
    cudaFree(batches);
    cudaFree(cta_seg);
    cudaFree(chunks_pp);
    cudaFree(chunks16_pp);
    cudaFree(cta_seg_pp);
}

// phase 1 (V^T x per chunk) + t_b reduction of multi-chunk blocks
// grid of the grid-stride V^T x kernels: 32 CTAs per SM (about ten resident waves; the
// block scheduler then balances the largest-first chunk list), LEVYH_VTX_BPS overrides;
// measured at N = 2^20: one wave 0.261 ms, 32 per SM 0.257 ms (chunks sorted), unsorted 0.300
template <int RB>
static int vtx_grid(int num_sms) {
    static int bps = 0;
    if (!bps) {
        const char *e = getenv("LEVYH_VTX_BPS");
        bps = e ? atoi(e) : 32;
        if (bps <= 0) LH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, vtx_kernel<RB>, NT, 0));
        bps = std::max(bps, 1);
    }
    return num_sms * bps;
}

void mv_vtx_launch(const MvPlan &P, const HMat &H, const double *x, int num_sms, cudaStream_t s) {
    (void)H;
    if (P.nch > 0) {
        int g = std::max(1, std::min(vtx_grid<8>(num_sms), (P.nch + dev::NW - 1) / dev::NW));
        vtx_kernel<8><<<g, NT, 0, s>>>(P.chunks, P.nch, P.pbuf, x, P.part, P.tvec);
    }
    if (P.nch16 > 0) {
        int g = std::max(1, std::min(vtx_grid<16>(num_sms), (P.nch16 + dev::NW - 1) / dev::NW));
        vtx_kernel<16><<<g, NT, 0, s>>>(P.chunks16, P.nch16, P.pbuf, x, P.part, P.tvec);
    }
    if (P.ntj > 0) treduce_kernel<<<std::min(P.ntj, 148 * 16), NT, 0, s>>>(P.tjobs, P.ntj, P.part, P.tvec);
    if (P.cpl) coupling_launch(*P.cpl, P.tvec, P.tvec, s);
    if (P.h2) h2_launch(*P.h2, x, P.tcol, P.xpad, P.nx, s);
}

// one launch of the TMA segment kernel over the CTA ranges cta (full or lean configuration)
static void seg_tma_launch(const MvPlan &P, const int32_t *cta, double *y, double alpha, double beta,
                           const double *z, cudaStream_t s) {
    if (P.lean == 3) {
        static bool attr = false;
        if (!attr) {
            LH_CUDA(cudaFuncSetAttribute((const void *)seg_tma_kernel<2, 128>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tma_smem<2, 128>()));
            attr = true;
        }
        seg_tma_kernel<2, 128><<<P.tma_grid, 128 + 32, tma_smem<2, 128>(), s>>>(P.segs, cta, P.batches, P.pbuf, P.tcol,
                                                                             P.xpad, y, alpha, beta, z);
    } else if (P.lean == 2) {
        static bool attr = false;
        if (!attr) {
            LH_CUDA(cudaFuncSetAttribute((const void *)seg_tma_kernel<3, 128>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tma_smem<3, 128>()));
            attr = true;
        }
        seg_tma_kernel<3, 128><<<P.tma_grid, 128 + 32, tma_smem<3, 128>(), s>>>(P.segs, cta, P.batches, P.pbuf, P.tcol,
                                                                             P.xpad, y, alpha, beta, z);
    } else if (P.lean) {
        static bool attr = false;
        if (!attr) {
            LH_CUDA(cudaFuncSetAttribute((const void *)seg_tma_kernel<3, 256>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tma_smem<3, 256>()));
            attr = true;
        }
        seg_tma_kernel<3, 256><<<P.tma_grid, 256 + 32, tma_smem<3, 256>(), s>>>(P.segs, cta, P.batches, P.pbuf, P.tcol,
                                                                             P.xpad, y, alpha, beta, z);
    } else {
        static bool attr = false;
        if (!attr) {
            LH_CUDA(cudaFuncSetAttribute((const void *)seg_tma_kernel<5, 512>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tma_smem<5, 512>()));
            attr = true;
        }
        seg_tma_kernel<5, 512><<<P.tma_grid, 512 + 32, tma_smem<5, 512>(), s>>>(P.segs, cta, P.batches, P.pbuf, P.tcol,
                                                                             P.xpad, y, alpha, beta, z);
    }
}

void mv_seg_launch(const MvPlan &P, const HMat &H, const double *x, double *y, double alpha,
                   double beta, cudaStream_t s, int num_sms, const double *z) {
    (void)H;
    static const bool direct = getenv("LEVYH_SEG_DIRECT") != nullptr;
    if (P.dense) {  // split H2 plan, serial form: dense leaves, then the row-basis pieces
        const MvPlan &D = *P.dense;
        tgather_kernel<<<(int)std::min<i64>((D.nx + 2 + NT - 1) / NT, 148 * 8), NT, 0, s>>>(
            D.tmap, 0, D.tvec, D.tcol, x, D.nx, D.xpad);
        seg_tma_launch(D, D.cta_seg, y, alpha, beta, z ? z : y, s);
        seg_tma_launch(P, P.cta_seg, y, alpha, 1.0, y, s);
        return;
    }
    if (!direct && P.nbatch > 0) {
        const i64 n = P.tcol_len + P.nx + 2;
        int g = (int)std::min<i64>((n + NT - 1) / NT, 148 * 8);
        if (!P.h2) tgather_kernel<<<g, NT, 0, s>>>(P.tmap, P.tcol_len, P.tvec, P.tcol, x, P.nx, P.xpad);
        seg_tma_launch(P, P.cta_seg, y, alpha, beta, z ? z : y, s);
        return;
    }
    // (A one-warp-per-32-rows variant without shared memory measured slower on B200.)
    int g2 = std::min(P.nseg, num_sms * 32);
    seg_kernel<<<g2, NT, 0, s>>>(P.segs, P.nseg, P.dp, P.lp, P.pbuf, P.tvec, x, y, alpha, beta,
                                 z ? z : y);
}

// y = alpha * H x + beta * z (z = y when null) for one right-hand side
void mv_run(const MvPlan &P, const HMat &H, const double *x, double *y, double alpha, double beta,
            cudaStream_t s, int num_sms, const double *z) {
    if (P.h2 && P.h2->step2) {  // two-kernel fused step (h2step.cu)
        h2s_launch(*P.h2, x, y, alpha, beta, z ? z : y, s);
        return;
    }
    if (P.fdense && P.h2 && P.h2->qleaf) {
        // fused H2 step: the dense diagonal leaves stream into yd on the forked low-priority
        // stream (co-resident segment kernel) while the latency-bound walk runs on s; the row
        // walk then applies Q_t y_hat_t and writes y = alpha (yd + Q y_hat) + beta z
        const MvPlan &D = *P.fdense;
        const int fdbg = getenv("LEVYH_FUSE_DBG") ? atoi(getenv("LEVYH_FUSE_DBG")) : 0;  // timing only
        LH_CUDA(cudaEventRecord(P.fev[0], s));
        LH_CUDA(cudaStreamWaitEvent(P.fork, P.fev[0], 0));
        if (!(fdbg & 1)) {
            tgather_kernel<<<(int)std::min<i64>((D.nx + 2 + NT - 1) / NT, 148 * 8), NT, 0, P.fork>>>(
                D.tmap, 0, D.tvec, D.tcol, x, D.nx, D.xpad);
            seg_tma_launch(D, D.cta_seg, P.h2->yd, 1.0, 0.0, P.h2->yd, P.fork);
        }
        LH_CUDA(cudaEventRecord(P.fev[1], P.fork));
        h2_launch_fused(*P.h2, x, y, alpha, beta, z ? z : y, s, P.fev[1]);
        LH_CUDA(cudaGetLastError());
        return;
    }
    if (P.dense) {
        // split H2 plan: the dense diagonal leaves stream on a forked stream (lean segment
        // kernel) while the latency-bound H2 walk runs; the row-basis pieces add in after both
        const MvPlan &D = *P.dense;
        LH_CUDA(cudaEventRecord(P.fev[0], s));
        LH_CUDA(cudaStreamWaitEvent(P.fork, P.fev[0], 0));
        tgather_kernel<<<(int)std::min<i64>((D.nx + 2 + NT - 1) / NT, 148 * 8), NT, 0, P.fork>>>(
            D.tmap, 0, D.tvec, D.tcol, x, D.nx, D.xpad);
        seg_tma_launch(D, D.cta_seg, y, alpha, beta, z ? z : y, P.fork);
        LH_CUDA(cudaEventRecord(P.fev[1], P.fork));
        h2_launch(*P.h2, x, P.tcol, P.xpad, 0, s);
        LH_CUDA(cudaStreamWaitEvent(s, P.fev[1], 0));
        seg_tma_launch(P, P.cta_seg, y, alpha, 1.0, y, s);
        LH_CUDA(cudaGetLastError());
        return;
    }
    mv_vtx_launch(P, H, x, num_sms, s);
    mv_seg_launch(P, H, x, y, alpha, beta, s, num_sms, z);
    LH_CUDA(cudaGetLastError());
}

void mv_run_host(const MvPlan &P, const double *x_host, double *x_dev, double *y_dev,
                 double *y_host, double alpha, double beta, bool z_is_x, cudaStream_t s,
                 cudaStream_t side, cudaEvent_t *ev, int num_sms) {
    const int NP = P.npiece;
    LH_REQUIRE(NP >= 1 && P.nbatch > 0, LH_EINTERNAL, "matvec plan without pipelining data");
    cudaEvent_t fork = ev[2 * NP], join = ev[2 * NP + 1];
    LH_CUDA(cudaEventRecord(fork, s));
    LH_CUDA(cudaStreamWaitEvent(side, fork, 0));
    for (int p = 0; p < NP; ++p) {  // x pieces in order on the copy stream
        const i64 a = P.xcut[p], b = P.xcut[p + 1];
        LH_CUDA(cudaMemcpyAsync(x_dev + a, x_host + a, sizeof(double) * (b - a), cudaMemcpyHostToDevice,
                                side));
        LH_CUDA(cudaEventRecord(ev[p], side));
    }
    const double *z = z_is_x ? x_dev : y_dev;
    if (P.dense) {  // split H2 plan: dense leaves on the copy stream once x is in, beside the walk
        const MvPlan &D = *P.dense;
        tgather_kernel<<<(int)std::min<i64>((D.nx + 2 + NT - 1) / NT, 148 * 8), NT, 0, side>>>(
            D.tmap, 0, D.tvec, D.tcol, x_dev, D.nx, D.xpad);
        seg_tma_launch(D, D.cta_seg, y_dev, alpha, beta, z, side);
        LH_CUDA(cudaEventRecord(P.fev[1], side));
    }
    int hl = 0;  // H2: column leaves whose x rows have arrived
    for (int p = 0; p < NP; ++p) {  // V^T x of the chunks whose x rows have arrived
        LH_CUDA(cudaStreamWaitEvent(s, ev[p], 0));
        if (P.h2) {
            const H2 &h = *P.h2;
            int he = hl;
            while (he < h.nleaf && h.leaf_end[he] <= P.xcut[p + 1]) ++he;
            if (p == NP - 1) he = h.nleaf;
            h2_leaf_launch(h, hl, he, x_dev, s);
            hl = he;
        }
        const int n8 = P.pch[p + 1] - P.pch[p], n16 = P.pch16[p + 1] - P.pch16[p];
        if (n8 > 0) {
            int g = std::max(1, std::min(vtx_grid<8>(num_sms), (n8 + dev::NW - 1) / dev::NW));
            vtx_kernel<8><<<g, NT, 0, s>>>(P.chunks_pp + P.pch[p], n8, P.pbuf, x_dev, P.part, P.tvec);
        }
        if (n16 > 0) {
            int g = std::max(1, std::min(vtx_grid<16>(num_sms), (n16 + dev::NW - 1) / dev::NW));
            vtx_kernel<16><<<g, NT, 0, s>>>(P.chunks16_pp + P.pch16[p], n16, P.pbuf, x_dev, P.part,
                                            P.tvec);
        }
    }
    if (P.ntj > 0) treduce_kernel<<<std::min(P.ntj, 148 * 16), NT, 0, s>>>(P.tjobs, P.ntj, P.part, P.tvec);
    if (P.cpl) coupling_launch(*P.cpl, P.tvec, P.tvec, s);
    if (P.h2) h2_launch(*P.h2, x_dev, P.tcol, P.xpad, P.dense ? 0 : P.nx, s, false);
    const i64 n = P.tcol_len + P.nx + 2;
    int g = (int)std::min<i64>((n + NT - 1) / NT, 148 * 8);
    if (!P.h2) tgather_kernel<<<g, NT, 0, s>>>(P.tmap, P.tcol_len, P.tvec, P.tcol, x_dev, P.nx, P.xpad);
    if (P.dense) LH_CUDA(cudaStreamWaitEvent(s, P.fev[1], 0));
    for (int p = 0; p < NP; ++p) {  // y pieces leave as soon as their segments are done
        if (P.dense) seg_tma_launch(P, P.cta_seg_pp + (size_t)p * (P.tma_grid + 1), y_dev, alpha, 1.0, y_dev, s);
        else seg_tma_launch(P, P.cta_seg_pp + (size_t)p * (P.tma_grid + 1), y_dev, alpha, beta, z, s);
        LH_CUDA(cudaEventRecord(ev[NP + p], s));
        LH_CUDA(cudaStreamWaitEvent(side, ev[NP + p], 0));
        const i64 a = P.ycut[p], b = P.ycut[p + 1];
        LH_CUDA(cudaMemcpyAsync(y_host + a, y_dev + a, sizeof(double) * (b - a), cudaMemcpyDeviceToHost,
                                side));
    }
    LH_CUDA(cudaEventRecord(join, side));
    LH_CUDA(cudaStreamWaitEvent(s, join, 0));
    LH_CUDA(cudaGetLastError());
}

void treduce_launch(const TJob *jobs, int n, const double *part, double *out, cudaStream_t s) {
    if (n <= 0) return;
    treduce_kernel<<<std::min(n, 148 * 16), NT, 0, s>>>(jobs, n, part, out);
}

MvPlan &get_mv_plan(HMat &H, cudaStream_t s) {
    ensure_resident(H, s);
    if (!H.mv_plan) {
        auto p = build_mv_plan(H, H.leafblocks, s);
        H.mv_plan = std::static_pointer_cast<void>(p);
    }
    return *static_cast<MvPlan *>(H.mv_plan.get());
}

void matvec(Ctx &ctx, HMat &H, const double *x, i64 ldx, double *y, i64 ldy, int nrhs) {
    LH_REQUIRE(!H.factored, LH_EINVAL, "matvec of an LU-factored H-matrix is not defined");
    MvPlan &P = get_mv_plan(H, ctx.stream);
    if (nrhs >= mm_min_rhs()) {  // one pass over the operator on the FP64 tensor cores
        const i64 ldk = mm_pad(nrhs);
        double *Xr = ctx.mm[0].ensure(H.ncols * ldk);
        double *Yr = ctx.mm[1].ensure(H.nrows * ldk);
        MmBufs b = mm_bufs(ctx, P, ldk);
        mm_transpose(x, ldx, Xr, ldk, H.ncols, nrhs, true, ctx.stream);
        mm_run(P, Xr, Yr, ldk, 1.0, 0.0, nullptr, b.T, b.part, ctx.stream);
        mm_transpose(Yr, ldk, y, ldy, H.nrows, nrhs, false, ctx.stream);
        return;
    }
    for (int q = 0; q < nrhs; ++q)
        mv_run(P, H, x + (i64)q * ldx, y + (i64)q * ldy, 1.0, 0.0, ctx.stream, ctx.num_sms);
}

}  // namespace lh
