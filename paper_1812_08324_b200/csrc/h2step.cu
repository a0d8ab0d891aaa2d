// Two-kernel single-RHS step of the nested-basis (H2) propagator: see h2step.h.
#include <algorithm>
#include <cstring>

#include "dev.cuh"
#include "h2step.h"

namespace lh {

H2S::~H2S() {
    for (void *p : {(void *)lb1, (void *)ub1, (void *)nb2, (void *)eb2, (void *)pb2, (void *)db2, (void *)qb2})
        if (p) cudaFree(p);
    for (void *p : {(void *)c1, (void *)c2, (void *)cb1, (void *)cb2, (void *)sb1, (void *)sl1, (void *)leaf,
                    (void *)up, (void *)cn, (void *)ce, (void *)path, (void *)dn, (void *)q, (void *)xpad, (void *)yd, (void *)sb2, (void *)td2})
        if (p) cudaFree(p);
}

static_assert(sizeof(H2SChunk) % 16 == 0 && sizeof(H2SLeaf) % 16 == 0 && sizeof(H2SUp) % 16 == 0 &&
                  sizeof(H2SCplN) % 16 == 0 && sizeof(H2SCplE) % 16 == 0 && sizeof(H2SPath) % 16 == 0 &&
                  sizeof(H2SDn) % 16 == 0 && sizeof(H2SQ) % 16 == 0,
              "descriptor arrays are bulk-copied");

namespace {

using dev::NT;
constexpr unsigned FULL = 0xffffffffu;
constexpr int CONS_T = H2S_CONS * 32;  // consumer threads
constexpr int TGRP = CONS_T / 64;      // column groups of the dense-leaf consumers
constexpr int RING_HDR = 128;          // bytes before the ring: full[ST], empty[ST] mbarriers

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t *b, int c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            saddr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk(void *dst, uint64_t src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     saddr(dst)),
                 "l"(src), "r"(bytes), "r"(saddr(bar))
                 : "memory");
}
// streamed operands are read once per application: evict-first in L2, so the small vectors the
// kernels exchange through L2 (x_hat, yd, the staging copy of x) stay resident
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_ef(void *dst, uint64_t src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            saddr(dst)),
        "l"(src), "r"(bytes), "r"(saddr(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void cons_bar() { asm volatile("bar.sync 1, %0;" ::"n"(CONS_T) : "memory"); }

// producer: lane 0 of warp 0 streams the chunks [c0, c1) through the ring
__device__ __forceinline__ bool skipped(const H2SChunk &C, int skip) {
    return ((skip & 1) && C.type == C_DENSE) || ((skip & 2) && (C.type == C_LEAF || C.type == C_ULVL));
}
// wait_types: chunk types whose operands the previous kernel writes (programmatic dependent
// launch: griddepcontrol.wait before the first of them; the others stream ahead)
template <int ST = H2S_ST>
__device__ __forceinline__ void produce(const H2SChunk *ch, int nch, unsigned char *ring, uint64_t *full,
                                        uint64_t *empty, int skip = 0, int wait_types = 0, int slotb = H2S_SLOTB) {
    int stage = 0;
    uint32_t phase = 0;
    bool waited = wait_types == 0;
    const uint64_t pol = evict_first_policy();
    for (int c = 0; c < nch; ++c) {
        const H2SChunk &C = ch[c];
        if (skipped(C, skip)) continue;
        if (!waited && ((wait_types >> C.type) & 1)) {
            pdl_wait();
            waited = true;
        }
        mb_wait(&empty[stage], phase ^ 1);
        uint32_t tot = 0;
        for (int i = 0; i < C.ncopy; ++i) tot += (uint32_t)C.bytes[i];
        mb_expect(&full[stage], tot);
        unsigned char *slot = ring + (size_t)stage * slotb;
        for (int i = 0; i < C.ncopy; ++i) bulk_ef(slot + C.dst[i], C.src[i], (uint32_t)C.bytes[i], &full[stage], pol);
        if (++stage == ST) {
            stage = 0;
            phase ^= 1;
        }
    }
}

// the CTA's descriptor slices -> shared memory in one bulk phase (thread 0 issues, all wait)
struct DSlice {
    const void *g;
    int bytes;
};
template <int N>
__device__ __forceinline__ void preload(unsigned char *dst, const DSlice (&sl)[N], uint64_t *bar) {
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (int i = 0; i < N; ++i) tot += (uint32_t)sl[i].bytes;
        mb_expect(bar, tot);
        int off = 0;
        for (int i = 0; i < N; ++i) {
            if (sl[i].bytes > 0) bulk(dst + off, (uint64_t)(uintptr_t)sl[i].g, (uint32_t)sl[i].bytes, bar);
            off += sl[i].bytes;
        }
    }
    mb_wait(bar, 0);
}

// v[j] (j < 2W) partial sums held by every lane -> lane l ends with the warp total of column
// l & (2W - 1) (W = 16: all 32 lanes distinct; W = 8: lanes l and l + 16 hold the same column).
// Halving exchanges: at width w a lane keeps the half of its live slots selected by lane bit w and
// adds the partner's copy of that half (2W - 1 shuffles), then W = 8 folds the two half-warps.
template <int W>
__device__ __forceinline__ double transpose_reduce(double (&v)[32], int lane) {
#pragma unroll
    for (int w = W; w >= 1; w >>= 1) {
        const bool up = (lane & w) != 0;
#pragma unroll
        for (int i = 0; i < w; ++i) {
            const double send = up ? v[i] : v[i + w];
            const double keep = up ? v[i + w] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
        }
    }
    if (W == 8) v[0] += __shfl_xor_sync(0xffffffffu, v[0], 16);
    return v[0];
}


struct K1Args {
    const H2SChunk *ch;
    const int32_t *cb, *lb, *ub, *sb, *sl;
    const H2SLeaf *leaf;
    const H2SUp *up;
    double *xh, *yd;
    int xsmax;
    // the top of the column tree (zshared.cu H2 climb arrays)
    const H2Up *ups;
    const int32_t *up_chain, *up_cbeg;
    int32_t *cnt;
    const double *tu;
    int skip;  // timing experiments only: bit 0 skips the dense chunks, bit 1 the walk
    unsigned long long *trace;  // timing experiments only: per CTA [start, descriptors, per-type totals]
};
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// K1: producer warp 0, climber warp 1, consumer warps 2 .. 9
__global__ void __launch_bounds__(CONS_T + 64, 1) h2s_up_kernel(K1Args A) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm), *empty = full + H2S_ST, *dbar = empty + H2S_ST;
    unsigned char *ring = sm + RING_HDR;
    double *xs = reinterpret_cast<double *>(ring + (size_t)H2S_ST * H2S_SLOTB);
    double(*red)[TGRP][64] = reinterpret_cast<double(*)[TGRP][64]>(xs + A.xsmax);
    unsigned char *desc = reinterpret_cast<unsigned char *>(red + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, b = blockIdx.x;
    if (threadIdx.x == 0) {
        for (int i = 0; i < H2S_ST; ++i) {
            mb_init(&full[i], 1);
            mb_init(&empty[i], H2S_CONS);
        }
        mb_init(dbar, 1);
        reinterpret_cast<int *>(dbar + 1)[0] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int c0 = A.cb[b], nch = A.cb[b + 1] - c0, l0 = A.lb[b], nl = A.lb[b + 1] - l0, u0 = A.ub[b],
              nu = A.ub[b + 1] - u0;
    const H2SChunk *chs = reinterpret_cast<const H2SChunk *>(desc);
    const H2SLeaf *lfs = reinterpret_cast<const H2SLeaf *>(chs + nch);
    const H2SUp *ups = reinterpret_cast<const H2SUp *>(lfs + nl);
    const unsigned long long tstart = A.trace ? gtime() : 0;
    pdl_trigger();  // K2 may launch onto SMs this kernel frees (it waits for x_hat and yd itself)
    {
        const DSlice sl[3] = {{A.ch + c0, nch * (int)sizeof(H2SChunk)},
                              {A.leaf + l0, nl * (int)sizeof(H2SLeaf)},
                              {A.up + u0, nu * (int)sizeof(H2SUp)}};
        preload(desc, sl, dbar);
    }
    if (A.trace && threadIdx.x == 0) {
        A.trace[b * 8 + 0] = tstart;
        A.trace[b * 8 + 1] = gtime();
    }
    if (warp == 0) {
        if (lane == 0) produce(chs, nch, ring, full, empty, A.skip);
        return;
    }
    volatile int *sdone = reinterpret_cast<volatile int *>(dbar + 1);  // subtrees finished (consumers)
    if (warp == 1 && (A.skip & 6)) return;
    if (warp == 1) {  // climber: the top of the tree once this CTA's subtree roots are in xh
        const int s0 = A.sb[blockIdx.x], s1 = A.sb[blockIdx.x + 1];
        for (int si = s0; si < s1; ++si) {  // the climb's transfers to L2 first
            const int sub = A.sl[si];
            for (int q = A.up_cbeg[sub]; q < A.up_cbeg[sub + 1]; ++q) {
                const H2Up &U = A.ups[A.up_chain[q]];
                const char *t = reinterpret_cast<const char *>(A.tu + U.toff);
                const int bytes = 8 * (U.k1 + U.k2) * U.k;
                for (int o = 128 * lane; o < bytes; o += 128 * 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(t + o));
            }
        }
        for (int si = s0; si < s1; ++si) {
            while (*sdone <= si - s0) __nanosleep(64);
            __threadfence();
            const int sub = A.sl[si];
            for (int q = A.up_cbeg[sub]; q < A.up_cbeg[sub + 1]; ++q) {
                const int p = A.up_chain[q];
                const H2Up U = A.ups[p];
                int old = 0;
                if (lane == 0) {
                    __threadfence();
                    asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;" : "=r"(old) : "l"(A.cnt + p), "r"(1) : "memory");
                }
                old = __shfl_sync(FULL, old, 0);
                if (old == 0) break;  // the sibling's climber computes the parent
                if (lane == 0) A.cnt[p] = 0;  // ready for the next application
                // every load of the step in flight before the first FMA (the climb is a chain of
                // dependent steps running beside the dense stream: one memory latency per level)
                const double xa = lane < U.k1 ? __ldcg(A.xh + U.xoff1 + lane) : 0.0;
                const double xb = lane < U.k2 ? __ldcg(A.xh + U.xoff2 + lane) : 0.0;
                const double *T = A.tu + U.toff + lane;
                const bool act = lane < U.k;
                double ta[32], tb[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    ta[i] = (act && i < U.k1) ? T[(i64)i * U.k] : 0.0;
                    tb[i] = (act && i < U.k2) ? T[(i64)(U.k1 + i) * U.k] : 0.0;
                }
                double a0 = 0.0, a1 = 0.0;
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    a0 = fma(ta[i], __shfl_sync(FULL, xa, i), a0);
                    a1 = fma(tb[i], __shfl_sync(FULL, xb, i), a1);
                }
                if (act) A.xh[U.xoff + lane] = a0 + a1;
            }
        }
        if (A.trace && lane == 0) A.trace[b * 8 + 7] = gtime();
        return;
    }
    // consumers
    const int cw = warp - 2, ct = threadIdx.x - 64, row = ct & 63, g = ct >> 6;
    int stage = 0, nseg = 0;
    uint32_t phase = 0;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    unsigned long long tw[4] = {0, 0, 0, 0};
    for (int c = 0; c < nch; ++c) {
        const H2SChunk &C = chs[c];
        if (skipped(C, A.skip)) continue;
        const unsigned long long ta = A.trace ? gtime() : 0;
        if (C.flags & F_NEWLVL) cons_bar();
        mb_wait(&full[stage], phase);
        if (A.trace) tw[3] += gtime() - ta;
        const double *slot = reinterpret_cast<const double *>(ring + (size_t)stage * H2S_SLOTB);
        if (C.type == C_DENSE) {
            const int K = C.e0, ld = (C.b + 1) & ~1;
            const double *col = slot + row, *xv = slot + 5120 + C.e2;
            if (C.flags & F_SEGFIRST) a0 = a1 = a2 = a3 = 0.0;
            int k = g;
            for (; k + 3 * TGRP < K; k += 4 * TGRP) {
                a0 = fma(col[k * ld], xv[k], a0);
                a1 = fma(col[(k + TGRP) * ld], xv[k + TGRP], a1);
                a2 = fma(col[(k + 2 * TGRP) * ld], xv[k + 2 * TGRP], a2);
                a3 = fma(col[(k + 3 * TGRP) * ld], xv[k + 3 * TGRP], a3);
            }
            for (; k < K; k += TGRP) a0 = fma(col[k * ld], xv[k], a0);
            if (C.flags & F_SEGLAST) {
                double(*rd)[64] = red[nseg & 1];
                rd[g][row] = (a0 + a1) + (a2 + a3);
                cons_bar();
                if (g == 0 && row < C.b) {
                    double v = rd[0][row];
#pragma unroll
                    for (int q = 1; q < TGRP; ++q) v += rd[q][row];
                    A.yd[C.a + row] = v;
                }
                ++nseg;
            }
        } else if (C.type == C_LEAF) {
            for (int l = C.a + cw; l < C.b; l += H2S_CONS) {
                const H2SLeaf &L = lfs[l - l0];
                // x_hat = P^T x with the rows across the lanes (rows lane, lane + 32; P's rows
                // beyond `rows` are zero, ld 64; x beyond `rows` masked): per column a lane
                // partial, then one transpose reduction leaves column j's sum in lane j
                const double *P = slot + L.p + lane, *xv = slot + L.xsl;
                const double x0 = lane < L.rows ? xv[lane] : 0.0;
                const double x1 = lane + 32 < L.rows ? xv[lane + 32] : 0.0;
                double v[32];
                double r;
                if (L.k <= 16) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) v[j] = j < L.k ? fma(P[64 * j], x0, P[64 * j + 32] * x1) : 0.0;
                    r = transpose_reduce<8>(v, lane);
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = j < L.k ? fma(P[64 * j], x0, P[64 * j + 32] * x1) : 0.0;
                    r = transpose_reduce<16>(v, lane);
                }
                if (lane < L.k) {
                    xs[L.xs + lane] = r;
                    A.xh[L.xh + lane] = r;
                }
            }
        } else {  // C_ULVL
            for (int u = C.a + cw; u < C.b; u += H2S_CONS) {
                const H2SUp &U = ups[u - u0];
                if (lane < U.k) {
                    const double *T = slot + U.t + lane;
                    double s0 = 0.0, s1 = 0.0;
                    for (int i = 0; i < U.k1; ++i) s0 = fma(T[i * U.k], xs[U.xs1 + i], s0);
                    for (int i = 0; i < U.k2; ++i) s1 = fma(T[(U.k1 + i) * U.k], xs[U.xs2 + i], s1);
                    xs[U.xs + lane] = s0 + s1;
                    A.xh[U.xh + lane] = s0 + s1;
                }
            }
        }
        __syncwarp();
        if (lane == 0) mb_arrive(&empty[stage]);
        if (A.trace) tw[C.type == C_DENSE ? 2 : C.type] += gtime() - ta;
        if (C.flags & F_END) {  // this subtree's x_hat are in xh: hand over to the climber
            __threadfence();
            cons_bar();  // (the next subtree also reuses xs)
            if (ct == 0) *sdone = *sdone + 1;
        }
        if (++stage == H2S_ST) {
            stage = 0;
            phase ^= 1;
        }
    }
    if (A.trace && ct == 0) {
        for (int i = 0; i < 4; ++i) A.trace[b * 8 + 2 + i] = tw[i];
        A.trace[b * 8 + 6] = gtime();
    }
}

struct K2Args {
    const H2SChunk *ch;
    const int32_t *cb, *nb, *eb, *pb, *db, *qb;
    const H2SCplN *cn;
    const H2SCplE *ce;
    const H2SPath *path;
    const H2SDn *dn;
    const H2SQ *q;
    const double *xh;
    int wsmax, ysmax;
    const double *z;  // zmode 2
    double *y;
    double alpha, beta;
    int zmode;  // 0: beta = 0, 1: z = x (staged xpad slice), 2: z from global
    unsigned long long *trace;  // timing experiments only
    int skip;  // timing experiments only: bit 0 skips the coupling products, bit 1 the levels, bit 2 the rows
    int slotb;  // ring slot bytes
};

// K2: producer warp 0, consumer warps 1 .. 8
template <int ST>
__global__ void __launch_bounds__(CONS_T + 32, ST == 2 ? 2 : 1) h2s_down_kernel(K2Args A) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm), *empty = full + ST, *dbar = empty + ST;
    unsigned char *ring = sm + RING_HDR;
    double *ws = reinterpret_cast<double *>(ring + (size_t)ST * A.slotb);
    double *ys = ws + A.wsmax;
    double *py = ys + A.ysmax;  // [2][32] path chain state
    double *xgb = py + 64;      // [2][H2S_XG] gathered x_hat of the coupling chunks (double-buffered)
    unsigned char *desc = reinterpret_cast<unsigned char *>(xgb + 2 * H2S_XG);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, b = blockIdx.x;
    if (threadIdx.x == 0) {
        for (int i = 0; i < ST; ++i) {
            mb_init(&full[i], 1);
            mb_init(&empty[i], H2S_CONS);
        }
        mb_init(dbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int c0 = A.cb[b], nch = A.cb[b + 1] - c0;
    const int n0 = A.nb[b], nn = A.nb[b + 1] - n0, e0 = A.eb[b], ne = A.eb[b + 1] - e0;
    const int p0 = A.pb[b], npth = A.pb[b + 1] - p0, d0 = A.db[b], nd = A.db[b + 1] - d0;
    const int q0 = A.qb[b], nq = A.qb[b + 1] - q0;
    const H2SChunk *chs = reinterpret_cast<const H2SChunk *>(desc);
    const H2SCplN *cns = reinterpret_cast<const H2SCplN *>(chs + nch);
    const H2SCplE *ces = reinterpret_cast<const H2SCplE *>(cns + nn);
    const H2SPath *pts = reinterpret_cast<const H2SPath *>(ces + ne);
    const H2SDn *dns = reinterpret_cast<const H2SDn *>(pts + npth);
    const H2SQ *qs = reinterpret_cast<const H2SQ *>(dns + nd);
    {
        const DSlice sl[6] = {{A.ch + c0, nch * (int)sizeof(H2SChunk)}, {A.cn + n0, nn * (int)sizeof(H2SCplN)},
                              {A.ce + e0, ne * (int)sizeof(H2SCplE)},   {A.path + p0, npth * (int)sizeof(H2SPath)},
                              {A.dn + d0, nd * (int)sizeof(H2SDn)},     {A.q + q0, nq * (int)sizeof(H2SQ)}};
        preload(desc, sl, dbar);
    }
    if (warp == 0) {
        // the coupling matrices, transfers and row bases do not depend on K1: they stream while
        // K1 finishes; the row chunks carry yd (written by K1) and wait for it
        if (lane == 0) produce<ST>(chs, nch, ring, full, empty, 0, 1 << C_Q, A.slotb);
        return;
    }
    const int cw = warp - 1, ct = threadIdx.x - 32;
    pdl_wait();  // x_hat (K1) before the first coupling gather
    // the x_hat the couplings read were written by K1 early and have since been pushed out of
    // L2 by K1's dense stream: bring them back for the whole CTA at once (one DRAM latency
    // instead of one per chunk of coupling products)
    for (int e = ct; e < ne; e += CONS_T) {
        const H2SCplE &E = ces[e];
        const double *p = A.xh + E.xh;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p + E.kc - 1));
    }
    int stage = 0, pcur = 0, xpar = 0;
    bool pre = false;  // this coupling chunk's x_hat were gathered during the previous chunk
    uint32_t phase = 0;
    unsigned long long tw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const unsigned long long tstart = A.trace ? gtime() : 0;
    for (int c = 0; c < nch; ++c) {
        const H2SChunk &C = chs[c];
        const unsigned long long ta = A.trace ? gtime() : 0;
        if (C.flags & F_BEGIN) {  // a new subtree: clear its w slots (nodes without couplings)
            cons_bar();
            for (int i = ct; i < C.e0; i += CONS_T) ws[i] = 0.0;
            cons_bar();
        } else if (C.flags & F_NEWLVL) {
            cons_bar();
        }
        mb_wait(&full[stage], phase);
        if (A.trace) tw[7] += gtime() - ta;
        const double *slot = reinterpret_cast<const double *>(ring + (size_t)stage * A.slotb);
        // lookahead between consecutive coupling chunks: the next chunk's x_hat are requested
        // now and stored after this chunk's products, so their L2 round trip overlaps them
        const bool ahead = C.type == C_CPL && c + 1 < nch && chs[c + 1].type == C_CPL && chs[c + 1].b > chs[c + 1].a;
        double xr[8];
        int ncb = 0, nce = 0;
        if (ahead) {
            ncb = cns[chs[c + 1].a - n0].c0;
            nce = cns[chs[c + 1].b - 1 - n0].c1;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int q = ncb + cw + H2S_CONS * i;
                xr[i] = (q < nce && lane < ces[q - e0].kc) ? __ldcg(A.xh + ces[q - e0].xh + lane) : 0.0;
            }
        }
        if (C.type == C_CPL && (A.skip & 1)) {
        } else if (C.type == C_DLVL && (A.skip & 2)) {
        } else if (C.type == C_Q && (A.skip & 4)) {
        } else if (C.type == C_CPL) {
            // the chunk's coupling products as one batch: its x_hat slices are gathered into the
            // slot tail (slot[C.e1 ..], one L2 round trip for the chunk: warp per coupling, lane
            // per entry), then consumer thread t computes chunk row t (node row i of w = sum_e
            // S_e x_hat_e); C.e2 rows in all
            double *xg = xgb + xpar * H2S_XG;
            const int nn_c = C.b - C.a;
            const int cb = nn_c > 0 ? cns[C.a - n0].c0 : 0, ce = nn_c > 0 ? cns[C.b - 1 - n0].c1 : 0;
            if (!pre)
                for (int q = cb + cw; q < ce; q += H2S_CONS) {
                    const H2SCplE &E = ces[q - e0];
                    if (lane < E.kc) xg[E.xo + lane] = __ldcg(A.xh + E.xh + lane);
                }
            cons_bar();
            for (int t = ct; t < C.e2; t += CONS_T) {
                int lo = 0, hi = nn_c - 1;  // the node holding chunk row t: last with ro <= t
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if ((cns[C.a + mid - n0].kr_ro >> 8) <= t) lo = mid;
                    else hi = mid - 1;
                }
                const H2SCplN &N = cns[C.a + lo - n0];
                const int kr = N.kr_ro & 255, i = t - (N.kr_ro >> 8);
                double a0 = 0.0, a1 = 0.0;
                for (int e = N.c0; e < N.c1; ++e) {
                    const H2SCplE &E = ces[e - e0];
                    const double *S = slot + E.s + i, *xv = xg + E.xo;
                    int j = 0;
                    for (; j + 1 < E.kc; j += 2) {
                        a0 = fma(S[j * kr], xv[j], a0);
                        a1 = fma(S[(j + 1) * kr], xv[j + 1], a1);
                    }
                    if (j < E.kc) a0 = fma(S[j * kr], xv[j], a0);
                }
                ws[N.ws + i] = a0 + a1;
            }
            if (nn_c > 0) xpar ^= 1;
        } else if (C.type == C_PATH) {
            if (cw == 0) {  // the chain above the subtree, one warp
                for (int it = C.a; it < C.b; ++it) {
                    const H2SPath &Pt = pts[it - p0];
                    double v = lane < Pt.k ? ws[Pt.ws + lane] : 0.0;
                    if (Pt.kp > 0 && lane < Pt.k) {
                        const double *T = slot + Pt.t + Pt.roff + lane;
                        const double *yp = py + 32 * pcur;
                        for (int j = 0; j < Pt.kp; ++j) v = fma(T[j * Pt.ldt], yp[j], v);
                    }
                    __syncwarp();
                    if (lane < Pt.k) {
                        py[32 * (pcur ^ 1) + lane] = v;
                        if (Pt.out >= 0) ys[Pt.out + lane] = v;
                    }
                    pcur ^= 1;
                    __syncwarp();
                }
            }
        } else if (C.type == C_DLVL) {
            for (int it = C.a + cw; it < C.b; it += H2S_CONS) {
                const H2SDn &D = dns[it - d0];
                if (lane < D.k) {
                    double v = ws[D.ws + lane];
                    const double *T = slot + D.t + D.roff + lane;
                    for (int j = 0; j < D.kp; ++j) v = fma(T[j * D.ldt], ys[D.ysp + j], v);
                    ys[D.ys + lane] = v;
                }
            }
        } else {  // C_Q: the rows of a run of row leaves
            for (int it = C.a + cw; it < C.b; it += H2S_CONS) {
                const H2SQ &Q = qs[it - q0];
                const bool in0 = lane < Q.rows, in1 = lane + 32 < Q.rows;
                double s0 = 0.0, s1 = 0.0, t0 = 0.0, t1 = 0.0;
                const double *qm = slot + Q.q;
                for (int cc = 0; cc < Q.k; cc += 2) {
                    const double y0 = ys[Q.ys + cc], y1 = cc + 1 < Q.k ? ys[Q.ys + cc + 1] : 0.0;
                    const double *q0 = qm + cc * Q.rows, *q1 = q0 + Q.rows;
                    const bool two = cc + 1 < Q.k;
                    if (in0) {
                        s0 = fma(q0[lane], y0, s0);
                        if (two) t0 = fma(q1[lane], y1, t0);
                    }
                    if (in1) {
                        s1 = fma(q0[lane + 32], y0, s1);
                        if (two) t1 = fma(q1[lane + 32], y1, t1);
                    }
                }
                const double *ydv = slot + Q.yd, *zv = slot + Q.zs;
                if (in0) {
                    const double zz = A.zmode == 1 ? zv[lane] : A.zmode == 2 ? A.z[Q.r0 + lane] : 0.0;
                    A.y[Q.r0 + lane] = A.alpha * (ydv[lane] + (s0 + t0)) + A.beta * zz;
                }
                if (in1) {
                    const double zz = A.zmode == 1 ? zv[lane + 32] : A.zmode == 2 ? A.z[Q.r0 + lane + 32] : 0.0;
                    A.y[Q.r0 + lane + 32] = A.alpha * (ydv[lane + 32] + (s1 + t1)) + A.beta * zz;
                }
            }
        }
        if (ahead) {  // (every warp passed this chunk's barrier: the other buffer is free)
            double *xn = xgb + xpar * H2S_XG;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int q = ncb + cw + H2S_CONS * i;
                if (q < nce && lane < ces[q - e0].kc) xn[ces[q - e0].xo + lane] = xr[i];
            }
            for (int q = ncb + cw + 8 * H2S_CONS; q < nce; q += H2S_CONS)
                if (lane < ces[q - e0].kc) xn[ces[q - e0].xo + lane] = __ldcg(A.xh + ces[q - e0].xh + lane);
        }
        pre = ahead;
        __syncwarp();
        if (lane == 0) mb_arrive(&empty[stage]);
        if (A.trace) tw[C.type] += gtime() - ta;
        if (++stage == ST) {
            stage = 0;
            phase ^= 1;
        }
    }
    if (A.trace && ct == 0) {
        for (int i = 3; i < 8; ++i) A.trace[b * 8 + i - 3] = tw[i];
        A.trace[b * 8 + 5] = tstart;
        A.trace[b * 8 + 6] = gtime();
    }
}

__global__ void xpad_kernel(const double *x, i64 n, double *xpad) {
    for (i64 i = (i64)blockIdx.x * NT + threadIdx.x; i < n + 2; i += (i64)gridDim.x * NT) xpad[i] = i < n ? x[i] : 0.0;
}

// ------------------------------------------------------------------------------------------
// host: chunk lists
// ------------------------------------------------------------------------------------------
struct Cut {  // one chunk being filled
    H2SChunk c{};
    int used = 0;  // bytes used in the slot
};

i64 even(i64 v) { return (v + 1) & ~(i64)1; }

// a copy of [src, src + bytes) merges into the chunk's last copy when it starts inside or at
// the end of that copy's source range
bool merges(const Cut &k, uint64_t src) {
    if (k.c.ncopy == 0) return false;
    const int i = k.c.ncopy - 1;
    return k.c.dst[i] + k.c.bytes[i] == k.used && src >= k.c.src[i] && src <= k.c.src[i] + (uint64_t)k.c.bytes[i];
}
// room for `ncopy` more copies of `bytes` in total (16-byte alignment slack included)
thread_local i64 slot_limit = H2S_SLOTB;  // ring slot bytes of the list being cut (K2 two per SM: H2S_SLOTB2)
bool fits(const Cut &k, i64 bytes, int ncopy) {
    return k.c.ncopy + ncopy <= 4 && k.used + bytes + 32 * std::max(ncopy, 1) <= slot_limit;
}
// appends [src, src + bytes) (any 8-byte aligned source: the copy starts at the 16-byte boundary
// below it); returns the slot offset, in doubles, of src
int add_copy(Cut &k, const void *p, i64 bytes) {
    const uint64_t src = (uint64_t)(uintptr_t)p;
    if (merges(k, src)) {
        const int i = k.c.ncopy - 1;
        const uint64_t e0 = k.c.src[i] + (uint64_t)k.c.bytes[i];
        const uint64_t e1 = std::max<uint64_t>(e0, (src + (uint64_t)bytes + 15) & ~15ull);
        k.c.bytes[i] += (int32_t)(e1 - e0);
        k.used += (int)(e1 - e0);
        return (k.c.dst[i] + (int)(src - k.c.src[i])) / 8;
    }
    const uint64_t sa = src & ~15ull;
    const int nb = (int)(((src + (uint64_t)bytes + 15) & ~15ull) - sa);
    const int off = k.used;
    k.c.src[k.c.ncopy] = sa;
    k.c.bytes[k.c.ncopy] = nb;
    k.c.dst[k.c.ncopy] = off;
    k.c.ncopy++;
    k.used += nb;
    return (off + (int)(src - sa)) / 8;
}

struct CopyJob2 {
    i64 src, dst, len;  // doubles
};
__global__ void gather_copy_kernel(const CopyJob2 *jobs, int n, const double *src, double *dst) {
    for (int j = blockIdx.x; j < n; j += gridDim.x) {
        const CopyJob2 J = jobs[j];
        for (i64 e = threadIdx.x; e < J.len; e += NT) dst[J.dst + e] = src[J.src + e];
    }
}
void run_gather(const std::vector<CopyJob2> &jobs, const double *src, double *dst, cudaStream_t st) {
    if (jobs.empty()) return;
    CopyJob2 *d = dupload(jobs, st);
    gather_copy_kernel<<<(int)std::min<size_t>(jobs.size(), 148 * 16), NT, 0, st>>>(d, (int)jobs.size(), src, dst);
    LH_CUDA(cudaGetLastError());
    LH_CUDA(cudaStreamSynchronize(st));
    cudaFree(d);
}

}  // namespace

static bool h2s_fail(const char *why) {
    if (getenv("LEVYH_PLAN_VERBOSE")) fprintf(stderr, "[levyh] H2 step kernels not built: %s\n", why);
    return false;
}

static bool build_h2s_impl(const H2SInput &in, H2 &h, int num_sms, cudaStream_t st, int two_slot);
bool build_h2s(const H2SInput &in, H2 &h, int num_sms, cudaStream_t st) {
    // K2 with one CTA per row subtree, two per SM, on the largest two-stage ring that leaves room
    // for the subtree's walk slots and descriptors in half an SM's shared memory; else one per SM
    for (int slot : {H2S_SLOTB2, 28 * 1024, 24 * 1024, 20 * 1024})
        if (build_h2s_impl(in, h, num_sms, st, slot)) return true;
    return build_h2s_impl(in, h, num_sms, st, 0);
}

static bool build_h2s_impl(const H2SInput &in, H2 &h, int num_sms, cudaStream_t st, int two_slot) {
    const bool allow_two = two_slot > 0;
    if (getenv("LEVYH_H2_V1")) return false;
    auto S = std::make_shared<H2S>();
    // one CTA per SM; with more than two subtrees per SM (N = 2^22), whole waves of CTAs with
    // about one subtree each (a CTA's descriptors and walk slots must fit its shared memory)
    const int nsub = std::max(in.nsub_up, in.nsub_dn);
    const int G = nsub <= 2 * num_sms ? num_sms : num_sms * ((nsub + num_sms - 1) / num_sms);
    const i64 SLOT = H2S_SLOTB;
    S->G = G;
    S->n = in.n;
    S->xpad = dalloc<double>(in.n + 4);
    S->yd = dalloc<double>(in.n + 4);
    LH_CUDA(cudaMemsetAsync(S->xpad, 0, sizeof(double) * (in.n + 4), st));
    LH_CUDA(cudaMemsetAsync(S->yd, 0, sizeof(double) * (in.n + 4), st));
    auto start = [](Cut &k, int type, int a) {
        k = Cut{};
        k.c.type = type;
        k.c.a = k.c.b = a;
    };
    // ---------------- K1: column subtrees (leaves, levels), then the dense diagonal leaves
    std::vector<H2SLeaf> lf;
    std::vector<H2SUp> upv;
    std::vector<std::vector<H2SChunk>> k1walk(G);
    std::vector<i64> wbytes(G, 0);
    std::vector<std::vector<int>> k1subs(G);
    std::vector<int32_t> sb1{0}, sl1;
    const int nsu = in.nsub_up;
    int xsmax = 2;
    for (int s = 0; s < nsu; ++s) k1subs[(int)((i64)s * G / std::max(nsu, 1))].push_back(s);
    for (int b = 0; b < G; ++b) {
        auto &out = k1walk[b];
        auto push = [&](Cut &k) {
            out.push_back(k.c);
            wbytes[b] += k.used;
        };
        for (int s : k1subs[b]) {
            const H2Sub &SB = (*in.up_sub)[s];
            xsmax = std::max(xsmax, (*in.up_xcnt)[s]);
            const size_t first = out.size();
            // leaves: one copy of the run's P bases (contiguous in pb) + one of its x rows
            const int l0 = in.up_leaf_beg[s], l1 = in.up_leaf_beg[s + 1];
            int la = l0;
            while (la < l1) {
                int lb = la;
                i64 pb = 0;
                while (lb < l1) {
                    const H2Leaf &L = (*in.leaves)[lb];
                    const i64 pnew = pb + 8 * 64 * (i64)L.k;
                    const i64 xrows = L.x0 + L.rows - (*in.leaves)[la].x0;
                    if (pnew + 8 * xrows + 64 > SLOT) break;
                    pb = pnew;
                    ++lb;
                }
                if (lb == la) return h2s_fail("a leaf basis run above one ring slot");
                const H2Leaf &F = (*in.leaves)[la], &E = (*in.leaves)[lb - 1];
                Cut k;
                start(k, C_LEAF, (int)lf.size());
                const int pbase = add_copy(k, in.pb + F.poff, 8 * (E.poff + 64 * (i64)E.k - F.poff));
                const int xbase = add_copy(k, S->xpad + F.x0, 8 * (E.x0 + E.rows - F.x0));
                for (int l = la; l < lb; ++l) {
                    const H2Leaf &L = (*in.leaves)[l];
                    H2SLeaf q{};
                    q.p = pbase + (int)(L.poff - F.poff);
                    q.xsl = xbase + (int)(L.x0 - F.x0);
                    q.rows = L.rows;
                    q.k = L.k;
                    q.xs = L.xoff - SB.base;
                    q.xh = L.xoff;
                    lf.push_back(q);
                }
                k.c.b = (int)lf.size();
                push(k);
                la = lb;
            }
            // levels: the transfers of one height are contiguous in tu
            const int32_t *lv = in.up_lv->data() + (size_t)s * (in.maxh_up + 1);
            for (int hh = 0; hh < in.maxh_up; ++hh) {
                const int a = lv[hh], e = lv[hh + 1];
                if (a == e) continue;
                Cut k;
                start(k, C_ULVL, (int)upv.size());
                k.c.flags = F_NEWLVL;
                for (int u = a; u < e; ++u) {
                    const H2Up &U = (*in.ups)[u];
                    const i64 tb = 8 * (i64)(U.k1 + U.k2) * U.k;
                    if (tb + 32 > SLOT) return h2s_fail("a column transfer above one ring slot");
                    if (k.c.a < k.c.b && !fits(k, tb, merges(k, (uint64_t)(uintptr_t)(in.tu + U.toff)) ? 0 : 1)) {
                        push(k);
                        start(k, C_ULVL, (int)upv.size());
                    }
                    H2SUp q{};
                    q.t = add_copy(k, in.tu + U.toff, tb);
                    q.k = U.k;
                    q.k1 = U.k1;
                    q.k2 = U.k2;
                    q.xs = U.xoff - SB.base;
                    q.xs1 = U.xoff1 - SB.base;
                    q.xs2 = U.xoff2 - SB.base;
                    q.xh = U.xoff;
                    upv.push_back(q);
                    k.c.b = (int)upv.size();
                }
                push(k);
            }
            if (out.size() == first) {  // nothing streamed: an empty chunk carries the end flag
                H2SChunk e{};
                e.type = C_LEAF;
                out.push_back(e);
            }
            out.back().flags |= F_END;
            sl1.push_back(s);
        }
        sb1.push_back((int32_t)sl1.size());
    }
    // dense diagonal leaves: byte-balanced over the CTAs, the walk's bytes counted in
    std::vector<H2SChunk> ch1;
    std::vector<int32_t> cb1{0};
    i64 dtot = 0, wtot = 0;
    std::vector<i64> segb(in.segs.size(), 0);
    for (size_t sg = 0; sg < in.segs.size(); ++sg) {
        const SegDesc &D = in.segs[sg];
        for (int bb = D.bbeg; bb < D.bend; ++bb) segb[sg] += in.batches[bb].total;
        dtot += segb[sg];
    }
    for (i64 w : wbytes) wtot += w;
    const double target = (double)(dtot + wtot) / G;
    size_t sg = 0;
    double acc = 0.0;
    // one dense segment after every `mix` walk chunks keeps the ring streaming while the walk's
    // levels wait on their consumer barriers (LEVYH_H2S_MIX, 0 = walk first, then dense)
    const int mix = getenv("LEVYH_H2S_MIX") ? atoi(getenv("LEVYH_H2S_MIX")) : 2;
    std::vector<int32_t> lb1{0}, ub1{0};
    for (int b = 0; b < G; ++b) {  // items were appended CTA by CTA
        int lmax = lb1.back(), umax = ub1.back();
        for (const H2SChunk &c : k1walk[b]) {
            if (c.type == C_LEAF && c.b > c.a) lmax = std::max(lmax, c.b);
            if (c.type == C_ULVL && c.b > c.a) umax = std::max(umax, c.b);
        }
        lb1.push_back(lmax);
        ub1.push_back(umax);
    }
    for (int b = 0; b < G; ++b) {
        acc += (double)wbytes[b];
        size_t wi = 0;
        auto more_dense = [&]() { return sg < in.segs.size() && (acc < target * (b + 1) || b + 1 == G); };
        while (wi < k1walk[b].size() || more_dense()) {
            for (int t = 0; t < (mix > 0 ? mix : 1 << 30) && wi < k1walk[b].size(); ++t) ch1.push_back(k1walk[b][wi++]);
            if (!more_dense()) {
                while (wi < k1walk[b].size()) ch1.push_back(k1walk[b][wi++]);
                break;
            }
            const SegDesc &D = in.segs[sg];
            const int ld = D.ld;
            for (int bb = D.bbeg; bb < D.bend; ++bb) {
                const SBatch &B = in.batches[bb];
                if (B.K != B.kd) return h2s_fail("dense plan batch with low-rank columns");  // a dense-only plan is expected
                H2SChunk c{};
                c.type = C_DENSE;
                c.a = (int32_t)D.y0;
                c.b = D.rows;
                c.e0 = B.K;
                c.e1 = B.kd;
                c.e2 = B.xadj;
                c.flags = (bb == D.bbeg ? F_SEGFIRST : 0) | (bb + 1 == D.bend ? F_SEGLAST : 0);
                const i64 db = 8 * (i64)B.K * ld, xb = 8 * even(B.xadj + B.kd);
                if (db > 40960 || xb > 1024 || (B.src & 1) || (B.xsrc & 1)) return h2s_fail("dense batch above the slot layout");
                c.ncopy = 2;
                c.src[0] = (uint64_t)(uintptr_t)(in.pbuf + B.src);
                c.bytes[0] = (int32_t)((db + 15) & ~(i64)15);
                c.dst[0] = 0;
                c.src[1] = (uint64_t)(uintptr_t)(S->xpad + B.xsrc);
                c.bytes[1] = (int32_t)((xb + 15) & ~(i64)15);
                c.dst[1] = 40960;
                ch1.push_back(c);
            }
            acc += (double)segb[sg];
            ++sg;
        }
        cb1.push_back((int32_t)ch1.size());
    }
    // ---------------- K2 operands reordered per row subtree: couplings (path, then subtree
    // nodes) and the parent transfers of the path and of every level, each contiguous
    const int nsd = in.nsub_dn;
    // K2 is bound by each CTA's dependent chain (couplings -> path -> levels -> rows), so it runs
    // one CTA per row subtree with two CTAs resident per SM on two-stage rings: with between one
    // and two subtrees per SM instead of chaining two subtrees in half of the CTAs, and in the
    // wave mode (more than two subtrees per SM, about one per CTA already) two waves at a time
    const bool waves = G > num_sms;
    const bool two = allow_two && !getenv("LEVYH_H2S_ONE_PER_SM") &&
                     (waves || (nsd > num_sms && nsd <= 2 * num_sms));
    const int G2 = (two && !waves) ? nsd : G;
    S->G2 = G2;
    S->st2 = two ? 2 : H2S_ST;
    if (allow_two && !two) return false;  // nothing to cut per subtree: the caller's one-per-SM pass builds it
    const i64 SLOT2 = two ? two_slot : H2S_SLOTB;
    S->slot2 = (int)SLOT2;
    struct LimitGuard {
        LimitGuard(i64 v) { slot_limit = v; }
        ~LimitGuard() { slot_limit = H2S_SLOTB; }
    } limit_guard(SLOT2);
    std::vector<CopyJob2> sjobs, tjobs;
    std::vector<i64> s_of(in.cpls->size(), -1);  // not used across subtrees (path S is duplicated)
    (void)s_of;
    i64 sb2len = 0, td2len = 0;
    struct SubOps {
        std::vector<std::pair<int, i64>> cpl_nodes;  // (dns index, w slot)
        std::vector<i64> sbeg;                       // sb2 offset of every node's first S
        std::vector<i64> path_t;                     // td2 offset of the parent transfer of path item q
        std::vector<std::vector<i64>> lvl_t;         // per depth: td2 offset of every node's parent transfer
    };
    std::vector<SubOps> ops(nsd);
    for (int s = 0; s < nsd; ++s) {
        SubOps &O = ops[s];
        const H2Sub &SB = (*in.dn_sub)[s];
        const int pa = (*in.dn_pbeg)[s], np = (*in.dn_pbeg)[s + 1] - pa;
        const int pw0 = (int)even((*in.dn_ycnt)[s]);
        const int32_t *lv = in.dn_lv->data() + (size_t)s * (in.maxh_dn + 2);
        sb2len = even(sb2len);
        auto add_node = [&](int u, i64 wslot) {
            const H2Down &D = (*in.dns)[u];
            if (D.c1 <= D.c0 || D.k == 0) return;
            O.cpl_nodes.push_back({u, wslot});
            O.sbeg.push_back(sb2len);
            for (int e = D.c0; e < D.c1; ++e) {
                const H2Cpl &E = (*in.cpls)[e];
                const i64 len = (i64)E.kr * E.kc;
                sjobs.push_back({E.soff, sb2len, len});
                sb2len += len;
            }
        };
        for (int q = 0; q < np; ++q) add_node((*in.dn_path)[pa + q], pw0 + 32 * q);
        for (int u = lv[0]; u < lv[in.maxh_dn + 1]; ++u) add_node(u, (*in.dns)[u].yoff - SB.base);
        td2len = even(td2len);
        auto add_t = [&](const H2Down &D) {
            const i64 off = td2len, len = (i64)D.ldt * D.kp;
            tjobs.push_back({D.toff, off, len});
            td2len += len;
            return off;
        };
        for (int q = 0; q < np; ++q) {
            const H2Down &D = (*in.dns)[(*in.dn_path)[pa + q]];
            O.path_t.push_back(q > 0 && D.kp > 0 ? add_t(D) : -1);
        }
        const H2Down &R0 = (*in.dns)[lv[0]];
        O.path_t.push_back(np > 0 && R0.kp > 0 ? add_t(R0) : -1);
        O.lvl_t.resize(in.maxh_dn + 1);
        for (int d = 1; d <= in.maxh_dn; ++d) {
            i64 last_toff = -1, last = -1;
            for (int u = lv[d]; u < lv[d + 1]; ++u) {
                const H2Down &D = (*in.dns)[u];
                if (D.yoffp < 0 || D.kp == 0) {
                    O.lvl_t[d].push_back(-1);
                    continue;
                }
                if (D.toff != last_toff) {
                    last = add_t(D);
                    last_toff = D.toff;
                }
                O.lvl_t[d].push_back(last);
            }
        }
    }
    double *sb2 = dalloc<double>(sb2len + 4), *td2 = dalloc<double>(td2len + 4);
    S->sb2 = sb2;
    S->td2 = td2;
    run_gather(sjobs, in.sb, sb2, st);
    run_gather(tjobs, in.td, td2, st);
    // ---------------- K2 chunks
    std::vector<H2SCplN> cnv;
    std::vector<H2SCplE> cev;
    std::vector<H2SPath> pv;
    std::vector<H2SDn> dnv;
    std::vector<H2SQ> qv;
    int wsmax = 2, ysmax = 2;
    std::vector<std::vector<int>> k2subs(G2);
    for (int s = 0; s < nsd; ++s) k2subs[(int)((i64)s * G2 / std::max(nsd, 1))].push_back(s);
    std::vector<char> leaf_done(in.rleaf.size(), 0);
    std::vector<i64> k2bytes(G2, 0);
    i64 k2type[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // ring bytes by chunk type (diagnostics)
    std::vector<std::vector<H2SChunk>> k2c(G2);
    // the rows of row leaves [la, lb): one copy each of their Q bases (contiguous in the ZS
    // arena), yd rows and x rows
    auto q_chunks = [&](int b, size_t la, size_t lb, bool newlvl) {
        auto &out = k2c[b];
        bool firstc = true;
        size_t l = la;
        while (l < lb) {
            size_t e = l;
            i64 qb = 0;
            while (e < lb) {
                const H2SInput::RLeaf &R = in.rleaf[e];
                const i64 qn = qb + 8 * R.rows * R.k;
                const i64 rows = R.r0 + R.rows - in.rleaf[l].r0;
                if (qn + 16 * rows + 96 > SLOT2) break;
                qb = qn;
                ++e;
            }
            if (e == l) return h2s_fail("a row-leaf run above one ring slot");
            Cut k;
            start(k, C_Q, (int)qv.size());
            if (newlvl && firstc) k.c.flags = F_NEWLVL;
            firstc = false;
            i64 q0 = -1, qend = -1;
            for (size_t t = l; t < e; ++t)
                if (in.rleaf[t].k > 0) {
                    if (q0 < 0) q0 = in.rleaf[t].qoff;
                    if (qend >= 0 && in.rleaf[t].qoff != qend) return h2s_fail("row bases not contiguous");  // Q not contiguous
                    qend = in.rleaf[t].qoff + in.rleaf[t].rows * in.rleaf[t].k;
                }
            const int qbase = q0 >= 0 ? add_copy(k, in.zarena + q0, 8 * (qend - q0)) : 0;
            const i64 r0 = in.rleaf[l].r0, r1 = in.rleaf[e - 1].r0 + in.rleaf[e - 1].rows;
            const int ybase = add_copy(k, S->yd + r0, 8 * (r1 - r0));
            const int zbase = add_copy(k, S->xpad + r0, 8 * (r1 - r0));
            for (size_t t = l; t < e; ++t) {
                const H2SInput::RLeaf &R = in.rleaf[t];
                H2SQ q{};
                q.q = R.k > 0 ? qbase + (int)(R.qoff - q0) : 0;
                q.yd = ybase + (int)(R.r0 - r0);
                q.zs = zbase + (int)(R.r0 - r0);
                q.rows = (int32_t)R.rows;
                q.k = (int32_t)R.k;
                q.ys = (int32_t)R.yloc;
                q.r0 = R.r0;
                qv.push_back(q);
                leaf_done[t] = 1;
            }
            k.c.b = (int)qv.size();
            out.push_back(k.c);
            k2bytes[b] += k.used;
            k2type[C_Q] += k.used;
            l = e;
        }
        return true;
    };
    for (int b = 0; b < G2; ++b) {
        auto &out = k2c[b];
        auto push = [&](Cut &k) {
            out.push_back(k.c);
            k2bytes[b] += k.used;
            k2type[std::min<int>(k.c.type, 7)] += k.used;
        };
        for (int s : k2subs[b]) {
            const SubOps &O = ops[s];
            const H2Sub &SB = (*in.dn_sub)[s];
            const int ycnt = (*in.dn_ycnt)[s];
            const int pa = (*in.dn_pbeg)[s], np = (*in.dn_pbeg)[s + 1] - pa;
            const int pw0 = (int)even(ycnt);
            const int wsn = pw0 + 32 * np;
            wsmax = std::max(wsmax, wsn);
            ysmax = std::max(ysmax, ycnt);
            const int32_t *lv = in.dn_lv->data() + (size_t)s * (in.maxh_dn + 2);
            // couplings: a chunk carries its nodes' coupling matrices; its x_hat slices (<= H2S_XG
            // doubles) are gathered into a shared-memory buffer, e2 = rows of w it computes
            Cut k;
            i64 xcnt = 0, rows = 0;
            auto cpl_done = [&](Cut &kk) {
                kk.c.e2 = (int32_t)rows;
                xcnt = rows = 0;
            };
            start(k, C_CPL, (int)cnv.size());
            k.c.flags = F_BEGIN;
            k.c.e0 = wsn;
            for (size_t t = 0; t < O.cpl_nodes.size(); ++t) {
                const H2Down &D = (*in.dns)[O.cpl_nodes[t].first];
                i64 sbytes = 0, kcs = 0;
                for (int e = D.c0; e < D.c1; ++e) {
                    sbytes += 8 * (i64)(*in.cpls)[e].kr * (*in.cpls)[e].kc;
                    kcs += (*in.cpls)[e].kc;
                }
                if (sbytes + 32 > SLOT2 || D.k > 255) return h2s_fail("a coupling node above one slot");
                const double *src = sb2 + O.sbeg[t];
                const bool mg = merges(k, (uint64_t)(uintptr_t)src);
                if (kcs > H2S_XG) return h2s_fail("a coupling node's x_hat above the gather buffer");
                if (k.c.a < k.c.b && (!fits(k, sbytes, mg ? 0 : 1) || xcnt + kcs > H2S_XG)) {
                    cpl_done(k);
                    push(k);
                    start(k, C_CPL, (int)cnv.size());
                }
                const int base = add_copy(k, src, sbytes);
                H2SCplN N{(int32_t)O.cpl_nodes[t].second, D.k | (int32_t)(rows << 8), (int)cev.size(), 0};
                i64 off = 0;
                for (int e = D.c0; e < D.c1; ++e) {
                    const H2Cpl &E = (*in.cpls)[e];
                    H2SCplE q{};
                    q.s = base + (int)off;
                    q.kc = E.kc;
                    q.xo = (int32_t)xcnt;
                    q.xh = (int32_t)E.xoff;
                    cev.push_back(q);
                    off += (i64)E.kr * E.kc;
                    xcnt += E.kc;
                }
                rows += D.k;
                N.c1 = (int)cev.size();
                cnv.push_back(N);
                k.c.b = (int)cnv.size();
            }
            cpl_done(k);
            push(k);  // possibly without items: it clears the w slots (F_BEGIN)
            // path chain, ending in the subtree root
            start(k, C_PATH, (int)pv.size());
            k.c.flags = F_NEWLVL;
            for (int q = 0; q <= np; ++q) {
                const H2Down &D = q < np ? (*in.dns)[(*in.dn_path)[pa + q]] : (*in.dns)[lv[0]];
                H2SPath P{};
                P.ws = q < np ? pw0 + 32 * q : D.yoff - SB.base;
                P.k = D.k;
                P.out = q < np ? -1 : D.yoff - SB.base;
                const i64 t = O.path_t[q];
                if (t >= 0) {
                    const i64 tb = 8 * (i64)D.ldt * D.kp;
                    if (tb + 32 > SLOT2) return h2s_fail("a path transfer above one ring slot");
                    if (k.c.a < k.c.b && !fits(k, tb, merges(k, (uint64_t)(uintptr_t)(td2 + t)) ? 0 : 1)) {
                        push(k);
                        start(k, C_PATH, (int)pv.size());
                    }
                    P.t = add_copy(k, td2 + t, tb);
                    P.kp = D.kp;
                    P.ldt = D.ldt;
                    P.roff = D.roff;
                }
                pv.push_back(P);
                k.c.b = (int)pv.size();
            }
            push(k);
            // levels below the root
            for (int d = 1; d <= in.maxh_dn; ++d) {
                const int a = lv[d], e = lv[d + 1];
                if (a == e) continue;
                start(k, C_DLVL, (int)dnv.size());
                k.c.flags = F_NEWLVL;
                i64 last_t = -1;
                int last_off = 0;
                for (int u = a; u < e; ++u) {
                    const H2Down &D = (*in.dns)[u];
                    H2SDn q{};
                    q.ys = D.yoff - SB.base;
                    q.ws = q.ys;
                    q.k = D.k;
                    const i64 t = O.lvl_t[d][u - a];
                    if (t >= 0) {
                        const i64 tb = 8 * (i64)D.ldt * D.kp;
                        if (tb + 32 > SLOT2) return h2s_fail("a row transfer above one ring slot");
                        if (t != last_t) {
                            if (k.c.a < k.c.b && !fits(k, tb, merges(k, (uint64_t)(uintptr_t)(td2 + t)) ? 0 : 1)) {
                                push(k);
                                start(k, C_DLVL, (int)dnv.size());
                            }
                            last_off = add_copy(k, td2 + t, tb);
                            last_t = t;
                        }
                        q.t = last_off;
                        q.kp = D.kp;
                        q.ldt = D.ldt;
                        q.roff = D.roff;
                        q.ysp = D.yoffp - SB.base;
                    }
                    dnv.push_back(q);
                    k.c.b = (int)dnv.size();
                }
                push(k);
            }
            // the rows of the leaves under the subtree root
            const i64 lo = in.dn_rows[s].first, hi = in.dn_rows[s].second;
            size_t la = std::lower_bound(in.rleaf.begin(), in.rleaf.end(), lo,
                                         [](const H2SInput::RLeaf &r, i64 v) { return r.r0 < v; }) -
                        in.rleaf.begin();
            size_t lb = la;
            while (lb < in.rleaf.size() && in.rleaf[lb].r0 < hi) ++lb;
            for (size_t l = la; l < lb; ++l)
                if (in.rleaf[l].k > 0 && in.rleaf[l].sub != s) return h2s_fail("a row leaf outside its subtree");
            if (!q_chunks(b, la, lb, true)) return h2s_fail("row chunks");
        }
    }
    // row leaves outside every row subtree (no basis): to the least-loaded CTAs
    for (size_t l = 0; l < in.rleaf.size();) {
        if (leaf_done[l]) {
            ++l;
            continue;
        }
        if (in.rleaf[l].k > 0) return h2s_fail("a leftover row leaf with a basis");
        size_t e = l;
        while (e < in.rleaf.size() && !leaf_done[e] && e - l < 32) ++e;
        const int b = (int)(std::min_element(k2bytes.begin(), k2bytes.end()) - k2bytes.begin());
        if (!q_chunks(b, l, e, false)) return h2s_fail("leftover row chunks");
        l = e;
    }
    // K2 items are appended CTA by CTA except the leftover leaves' Q items (appended last):
    // renumber every CTA's items contiguously
    std::vector<H2SChunk> ch2;
    std::vector<int32_t> cb2{0}, nb2{0}, eb2{0}, pb2{0}, db2{0}, qb2{0};
    std::vector<H2SCplN> cn2;
    std::vector<H2SCplE> ce2;
    std::vector<H2SPath> pv2;
    std::vector<H2SDn> dn2;
    std::vector<H2SQ> q2;
    for (int b = 0; b < G2; ++b) {
        for (H2SChunk c : k2c[b]) {
            const int a = c.a, e = c.b;
            if (c.type == C_CPL) {
                c.a = (int)cn2.size();
                for (int t = a; t < e; ++t) {
                    H2SCplN N = cnv[t];
                    const int f0 = N.c0, f1 = N.c1;
                    N.c0 = (int)ce2.size();
                    for (int f = f0; f < f1; ++f) ce2.push_back(cev[f]);
                    N.c1 = (int)ce2.size();
                    cn2.push_back(N);
                }
                c.b = (int)cn2.size();
            } else if (c.type == C_PATH) {
                c.a = (int)pv2.size();
                for (int t = a; t < e; ++t) pv2.push_back(pv[t]);
                c.b = (int)pv2.size();
            } else if (c.type == C_DLVL) {
                c.a = (int)dn2.size();
                for (int t = a; t < e; ++t) dn2.push_back(dnv[t]);
                c.b = (int)dn2.size();
            } else {
                c.a = (int)q2.size();
                for (int t = a; t < e; ++t) q2.push_back(qv[t]);
                c.b = (int)q2.size();
            }
            ch2.push_back(c);
        }
        cb2.push_back((int32_t)ch2.size());
        nb2.push_back((int32_t)cn2.size());
        eb2.push_back((int32_t)ce2.size());
        pb2.push_back((int32_t)pv2.size());
        db2.push_back((int32_t)dn2.size());
        qb2.push_back((int32_t)q2.size());
    }
    cnv.swap(cn2);
    cev.swap(ce2);
    pv.swap(pv2);
    dnv.swap(dn2);
    qv.swap(q2);
    for (int b = 0; b < G; ++b)
        S->desc1 = std::max<int>(S->desc1, (int)((cb1[b + 1] - cb1[b]) * sizeof(H2SChunk) +
                                                  (lb1[b + 1] - lb1[b]) * sizeof(H2SLeaf) +
                                                  (ub1[b + 1] - ub1[b]) * sizeof(H2SUp)));
    for (int b = 0; b < G2; ++b) {
        S->desc2 = std::max<int>(S->desc2, (int)((cb2[b + 1] - cb2[b]) * sizeof(H2SChunk) +
                                                  (nb2[b + 1] - nb2[b]) * sizeof(H2SCplN) +
                                                  (eb2[b + 1] - eb2[b]) * sizeof(H2SCplE) +
                                                  (pb2[b + 1] - pb2[b]) * sizeof(H2SPath) +
                                                  (db2[b + 1] - db2[b]) * sizeof(H2SDn) +
                                                  (qb2[b + 1] - qb2[b]) * sizeof(H2SQ)));
    }
    for (i64 v : k2bytes) S->bytes2 += v;
    S->bytes1 = dtot + wtot;
    S->xsmax = (int)even(xsmax);
    S->wsmax = (int)even(wsmax);
    S->ysmax = (int)even(ysmax);
    S->smem1 = RING_HDR + H2S_ST * H2S_SLOTB + 8 * S->xsmax + 8 * 2 * TGRP * 64 + S->desc1;
    S->smem2 = RING_HDR + S->st2 * S->slot2 +
               8 * (S->wsmax + S->ysmax + 64 + 2 * H2S_XG) + S->desc2;
    if (S->st2 == 2 && S->smem2 > 113 * 1024 - 512) {
        if (getenv("LEVYH_PLAN_VERBOSE"))
            fprintf(stderr, "[levyh] K2 two per SM: smem %d B (w %d, y %d doubles, descriptors %d B)\n", S->smem2,
                    S->wsmax, S->ysmax, S->desc2);
        return h2s_fail("K2 per-subtree CTAs above half an SM's shared memory");
    }
    int maxsm = 0, dev_id = 0;
    cudaGetDevice(&dev_id);
    cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev_id);
    if (S->smem1 > maxsm || S->smem2 > maxsm) {
        if (getenv("LEVYH_PLAN_VERBOSE"))
            fprintf(stderr, "[levyh] H2 step smem %d / %d B (x_hat %d, w %d, y %d doubles; descriptors %d / %d B), limit %d\n",
                    S->smem1, S->smem2, S->xsmax, S->wsmax, S->ysmax, S->desc1, S->desc2, maxsm);
        return h2s_fail("shared memory above the opt-in limit");
    }
    S->c1 = dupload(ch1, st);
    S->c2 = dupload(ch2, st);
    S->cb1 = dupload(cb1, st);
    S->cb2 = dupload(cb2, st);
    S->lb1 = dupload(lb1, st);
    S->ub1 = dupload(ub1, st);
    S->nb2 = dupload(nb2, st);
    S->eb2 = dupload(eb2, st);
    S->pb2 = dupload(pb2, st);
    S->db2 = dupload(db2, st);
    S->qb2 = dupload(qb2, st);
    S->sb1 = dupload(sb1, st);
    S->sl1 = dupload(sl1, st);
    S->leaf = dupload(lf, st);
    S->up = dupload(upv, st);
    S->cn = dupload(cnv, st);
    S->ce = dupload(cev, st);
    S->path = dupload(pv, st);
    S->dn = dupload(dnv, st);
    S->q = dupload(qv, st);
    LH_CUDA(cudaStreamSynchronize(st));
    if (getenv("LEVYH_PLAN_VERBOSE"))
        fprintf(stderr, "[levyh] H2 step K2 ring bytes: couplings %.1f MB, path %.1f MB, levels %.1f MB, rows %.1f MB; "
                        "%zu coupling nodes, %zu couplings, %zu path steps, %zu level nodes, %zu row leaves\n",
                k2type[C_CPL] * 1e-6, k2type[C_PATH] * 1e-6, k2type[C_DLVL] * 1e-6, k2type[C_Q] * 1e-6, cnv.size(),
                cev.size(), pv.size(), dnv.size(), qv.size());
    if (getenv("LEVYH_PLAN_VERBOSE"))
        fprintf(stderr, "[levyh] H2 step kernels: K1 %zu chunks (%.1f MB walk + %.1f MB dense), K2 %zu chunks "
                        "(%.1f MB), smem %d / %d B (descriptors %d / %d B)\n", ch1.size(), wtot * 1e-6, dtot * 1e-6,
                ch2.size(), S->bytes2 * 1e-6, S->smem1, S->smem2, S->desc1, S->desc2);
    h.step2 = S;
    return true;
}

static void h2s_kernels(const H2 &h, double *y, double alpha, double beta, const double *z, int zmode,
                        cudaStream_t s, cudaEvent_t *ev = nullptr) {
    const H2S &S = *h.step2;
    static bool attr = false;
    if (!attr) {
        LH_CUDA(cudaFuncSetAttribute((const void *)h2s_up_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        LH_CUDA(cudaFuncSetAttribute((const void *)h2s_down_kernel<H2S_ST>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        LH_CUDA(cudaFuncSetAttribute((const void *)h2s_down_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     113 * 1024));
        attr = true;
    }
    const int dbg = getenv("LEVYH_FUSE_DBG") ? atoi(getenv("LEVYH_FUSE_DBG")) : 0;  // timing experiments only
    K1Args a1{S.c1, S.cb1, S.lb1, S.ub1, S.sb1, S.sl1, S.leaf, S.up, h.xh, S.yd, S.xsmax,
              h.ups, h.up_chain, h.up_cbeg, h.cnt, h.tu, (dbg >> 2) & 7, nullptr};
    static unsigned long long *trace = nullptr;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    LH_CUDA(cudaStreamIsCapturing(s, &cap));
    if (getenv("LEVYH_H2S_TRACE") && cap == cudaStreamCaptureStatusNone) {  // timing experiments only: per-CTA phase times
        if (!trace) trace = dalloc<unsigned long long>((i64)(S.G + S.G2) * 8);
        a1.trace = trace;
    }
    cudaEvent_t te[3] = {nullptr, nullptr, nullptr};
    if (a1.trace)
        for (auto &e : te) cudaEventCreate(&e);
    if (a1.trace) cudaEventRecord(te[0], s);
    if (ev) LH_CUDA(cudaEventRecord(ev[0], s));
    if (!(dbg & 1)) h2s_up_kernel<<<S.G, CONS_T + 64, S.smem1, s>>>(a1);
    if (ev) LH_CUDA(cudaEventRecord(ev[1], s));
    if (a1.trace) cudaEventRecord(te[1], s);
    K2Args a2{S.c2, S.cb2, S.nb2, S.eb2, S.pb2, S.db2, S.qb2, S.cn, S.ce, S.path, S.dn, S.q, h.xh,
              S.wsmax, S.ysmax, z, y, alpha, beta, zmode, a1.trace ? a1.trace + (size_t)S.G * 8 : nullptr,
              (dbg >> 5) & 15, S.slot2};
    if (!(dbg & 2)) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(S.G2);
        cfg.blockDim = dim3(CONS_T + 32);
        cfg.dynamicSmemBytes = S.smem2;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = getenv("LEVYH_NO_PDL") ? 0 : 1;
        if (S.st2 == 2) LH_CUDA(cudaLaunchKernelEx(&cfg, h2s_down_kernel<2>, a2));
        else LH_CUDA(cudaLaunchKernelEx(&cfg, h2s_down_kernel<H2S_ST>, a2));
    }
    if (ev) LH_CUDA(cudaEventRecord(ev[2], s));
    LH_CUDA(cudaGetLastError());
    if (a1.trace && !getenv("LEVYH_H2S_TRACE_DONE")) {
        std::vector<unsigned long long> t((size_t)(S.G + S.G2) * 8);
        cudaEventRecord(te[2], s);
        LH_CUDA(cudaStreamSynchronize(s));
        float m1 = 0, m2 = 0;
        cudaEventElapsedTime(&m1, te[0], te[1]);
        cudaEventElapsedTime(&m2, te[1], te[2]);
        fprintf(stderr, "[h2s trace] events: K1 %.1f us, K2 %.1f us\n", 1e3 * m1, 1e3 * m2);
        for (auto &e : te) cudaEventDestroy(e);
        LH_CUDA(cudaMemcpy(t.data(), a1.trace, sizeof(unsigned long long) * t.size(), cudaMemcpyDeviceToHost));
        unsigned long long t0 = ~0ull;
        for (int b = 0; b < S.G; ++b) t0 = std::min(t0, t[b * 8]);
        unsigned long long tmax = 0;
        for (int b = 0; b < S.G; ++b) tmax = std::max(tmax, std::max(t[b * 8 + 6], t[b * 8 + 7]));
        fprintf(stderr, "[h2s trace] CTA span %.1f us\n", (tmax - t0) * 1e-3);
        {
            const unsigned long long *u = t.data() + (size_t)S.G * 8;
            double mx[7] = {0, 0, 0, 0, 0, 0, 0}, mean[7] = {0, 0, 0, 0, 0, 0, 0};
            for (int b = 0; b < S.G2; ++b) {
                const double v[6] = {u[b * 8] * 1e-3, u[b * 8 + 1] * 1e-3, u[b * 8 + 2] * 1e-3, u[b * 8 + 3] * 1e-3,
                                     u[b * 8 + 4] * 1e-3, (u[b * 8 + 6] - u[b * 8 + 5]) * 1e-3};
                for (int i = 0; i < 6; ++i) {
                    mx[i] = std::max(mx[i], v[i]);
                    mean[i] += v[i] / S.G2;
                }
            }
            fprintf(stderr, "[h2s trace] K2 mean/max us: cpl %.1f/%.1f path %.1f/%.1f lvl %.1f/%.1f q %.1f/%.1f "
                            "wait %.1f/%.1f total %.1f/%.1f\n", mean[0], mx[0], mean[1], mx[1], mean[2], mx[2], mean[3],
                    mx[3], mean[4], mx[4], mean[5], mx[5]);
        }
        for (int b = 0; b < S.G; b += 8)
            fprintf(stderr, "[h2s trace] cta %3d start %6.1f desc %6.1f | leaf %6.1f lvl %6.1f dense %6.1f wait %6.1f | end %6.1f climb end %6.1f us\n",
                    b, (t[b * 8] - t0) * 1e-3, (t[b * 8 + 1] - t0) * 1e-3, t[b * 8 + 2] * 1e-3, t[b * 8 + 3] * 1e-3,
                    t[b * 8 + 4] * 1e-3, t[b * 8 + 5] * 1e-3, (t[b * 8 + 6] - t0) * 1e-3,
                    t[b * 8 + 7] > t0 ? (t[b * 8 + 7] - t0) * 1e-3 : -1.0);
    }
}

void h2s_launch(const H2 &h, const double *x, double *y, double alpha, double beta, const double *z,
                cudaStream_t s) {
    const H2S &S = *h.step2;
    xpad_kernel<<<(int)std::min<i64>((S.n + 2 + NT - 1) / NT, 148 * 8), NT, 0, s>>>(x, S.n, S.xpad);
    h2s_kernels(h, y, alpha, beta, z, beta == 0.0 ? 0 : (z == x ? 1 : 2), s);
}

void h2s_launch_timed(const H2 &h, const double *x, double *y, double alpha, double beta, const double *z,
                      cudaStream_t s, cudaEvent_t *ev) {
    const H2S &S = *h.step2;
    LH_CUDA(cudaEventRecord(ev[0], s));
    xpad_kernel<<<(int)std::min<i64>((S.n + 2 + NT - 1) / NT, 148 * 8), NT, 0, s>>>(x, S.n, S.xpad);
    h2s_kernels(h, y, alpha, beta, z, beta == 0.0 ? 0 : (z == x ? 1 : 2), s, ev + 1);
}

void h2s_load(const H2 &h, const double *x, cudaStream_t s) {
    const H2S &S = *h.step2;
    xpad_kernel<<<(int)std::min<i64>((S.n + 2 + NT - 1) / NT, 148 * 8), NT, 0, s>>>(x, S.n, S.xpad);
    LH_CUDA(cudaGetLastError());
}

void h2s_step_inplace(const H2 &h, double alpha, double beta, cudaStream_t s, cudaEvent_t *ev) {
    // K2 stages every z row it reads (its own rows, once) before it writes y there, and K1 of
    // the next step reads x only after K2 has finished: the staging copy holds the state
    h2s_kernels(h, h.step2->xpad, alpha, beta, nullptr, beta == 0.0 ? 0 : 1, s, ev);
}

void h2s_store(const H2 &h, double *y, cudaStream_t s) {
    const H2S &S = *h.step2;
    LH_CUDA(cudaMemcpyAsync(y, S.xpad, sizeof(double) * S.n, cudaMemcpyDeviceToDevice, s));
}

void h2s_launch_host(const H2 &h, const double *x_host, double *y_dev, double *y_host, double alpha, double beta,
                     cudaStream_t s) {
    const H2S &S = *h.step2;
    LH_CUDA(cudaMemcpyAsync(S.xpad, x_host, sizeof(double) * S.n, cudaMemcpyHostToDevice, s));
    h2s_kernels(h, y_dev, alpha, beta, nullptr, beta == 0.0 ? 0 : 1, s);
    LH_CUDA(cudaMemcpyAsync(y_host, y_dev, sizeof(double) * S.n, cudaMemcpyDeviceToHost, s));
}

}  // namespace lh
