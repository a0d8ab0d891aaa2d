// Multi-RHS H-matmat Y = alpha H X + beta Z (hops.py:73-85 mul_dense; cfg4's 256 right-hand
// sides) on the FP64 tensor cores (mma.sync m8n8k4 f64, DMMA).
//
// X, Y, Z are row-major N x K (K a multiple of 64, the RHS tile); the operator uses the
// packed column stream of the single-RHS plan (matvec.cu), so one plan serves both paths.
//   phase 1 vtx_mm_kernel:  T_b (r x K) = V_b^T X[cols of b]   per V chunk and 64-RHS tile
//           (chunk partials of multi-chunk blocks summed by treduce_mm_kernel)
//   phase 2 seg_mm_kernel:  Y_seg (64 x K) = A_seg B_seg        per segment and 64-RHS tile
//           A_seg = the segment's column stream (64 x ncol), B_seg row q = X[colmap[q]]
//           (dense column) or T[-1 - colmap[q]] (low-rank column).
// Operand tiles are staged in shared memory with padded strides; each warp owns a
// 16 x 32 (phase 2) or r x 8 (phase 1) accumulator block of 8x8 DMMA fragments.
#include <algorithm>
#include <cstdlib>

#include "core.h"
#include "dev.cuh"
#include "matvec.h"

namespace lh {

using dev::KC_MAX;
using dev::NT;

constexpr int MM_N = 64;       // right-hand sides per tile
constexpr int MM_KB = 32;      // inner-dimension block staged per step
constexpr int MM_STR = 68;     // padded smem stride (doubles)

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// phase 1: one CTA per (V chunk, 64-RHS tile); 8 warps = 8 column tiles of 8 RHS, each with
// ceil(r/8) row tiles.  Inner dimension = the chunk's rows, staged MM_KB at a time.
__global__ void __launch_bounds__(NT) vtx_mm_kernel(const VChunk *chunks, const double *pbuf,
                                                    const double *X, i64 ldk, double *T,
                                                    double *part) {
    __shared__ double Vs[KC_MAX * MM_STR];   // [c][i]: V^T rows
    __shared__ double Xs[MM_KB * MM_STR];    // [i][n]
    const VChunk C = chunks[blockIdx.x];
    const int kc = blockIdx.y * MM_N;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int r = vc_rank(C), mt = (r + 7) >> 3;
    const double *V = pbuf + C.voff;
    double acc[4][2] = {};
    for (int k0 = 0; k0 < C.len; k0 += MM_KB) {
        const int kb = min(MM_KB, C.len - k0);
        for (int e = threadIdx.x; e < r * MM_KB; e += NT) {
            const int c = e / MM_KB, i = e % MM_KB;
            Vs[c * MM_STR + i] = i < kb ? V[(i64)(k0 + i) + (i64)c * C.len] : 0.0;
        }
        for (int e = threadIdx.x; e < MM_KB * MM_N; e += NT) {
            const int i = e / MM_N, n = e % MM_N;
            Xs[i * MM_STR + n] = i < kb ? X[(C.xc0 + k0 + i) * ldk + kc + n] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < MM_KB; kk += 4) {
            const double b = Xs[(kk + (l & 3)) * MM_STR + w * 8 + (l >> 2)];
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (t < mt) {
                    const int c = t * 8 + (l >> 2);
                    const double a = c < r ? Vs[c * MM_STR + kk + (l & 3)] : 0.0;
                    dmma(acc[t][0], acc[t][1], a, b);
                }
        }
        __syncthreads();
    }
    double *out = (C.pidx >= 0 ? part + (i64)C.pidx * KC_MAX * ldk : T + (i64)C.blk * KC_MAX * ldk) +
                  (i64)vc_col0(C) * ldk;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int c = t * 8 + (l >> 2);
        if (t < mt && c < r) {
            const int n = kc + w * 8 + (l & 3) * 2;
            out[(i64)c * ldk + n] = acc[t][0];
            out[(i64)c * ldk + n + 1] = acc[t][1];
        }
    }
}

// phase 1, grouped: one CTA per (group of chunks over the same x rows, 64-RHS tile); the X tile
// of every inner step is staged once for all the group's chunks (<= 64 output rows: 8 row
// fragments per warp, warp w owns RHS w*8 .. +8)
__global__ void __launch_bounds__(NT) vtx_mm_group_kernel(const VGroup *groups, const VChunk *gch,
                                                          const double *pbuf, const double *X, i64 ldk,
                                                          double *T, double *part) {
    // two stages of (Vs [MM_KB][64] k-major, rows XOR-swizzled by 8 (k & 3) so both the staging
    // stores and the DMMA fragment loads touch every bank pair twice; Xs [MM_KB][MM_STR]); the
    // next inner step is loaded into registers while the current one is multiplied.  Warp w
    // owns output rows 16 (w % 4) .. +16 and RHS 32 (w / 4) .. +32 (2 x 4 fragments).
    extern __shared__ double dsm[];
    constexpr int VS = MM_KB * 64, XS = MM_KB * MM_STR;
    __shared__ int32_t rq[64], rc[64];  // output row -> (chunk, column)
    __shared__ i64 ro[64];              // output row -> pbuf offset of its V column
    const VGroup G = groups[blockIdx.x];
    const int kc = blockIdx.y * MM_N;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int r0 = (w & 3) * 16, n0 = (w >> 2) * 32;
    if (threadIdx.x == 0) {
        int row = 0;
        for (int q = G.cbeg; q < G.cend; ++q) {
            const VChunk C = gch[q];
            for (int c = 0; c < vc_rank(C); ++c, ++row) {
                rq[row] = q;
                rc[row] = c;
                ro[row] = C.voff + (i64)c * C.len;
            }
        }
    }
    __syncthreads();
    constexpr int PV = 64 * MM_KB / NT, PX = MM_KB * MM_N / NT;  // elements per thread
    double rv[PV], rx[PX];
    // V element of register u: lanes cover 8 rows x 4 consecutive k (32-byte sectors of V)
    auto vrow = [&](int u) { return (((threadIdx.x + u * NT) >> 5) >> 3) * 8 + (l >> 2); };
    auto vk = [&](int u) { return (((threadIdx.x + u * NT) >> 5) & 7) * 4 + (l & 3); };
    auto load = [&](int k0) {
        const int kb = min(MM_KB, G.len - k0);
#pragma unroll
        for (int u = 0; u < PV; ++u) {
            const int r = vrow(u), k = vk(u);
            rv[u] = (r < G.m && k < kb) ? pbuf[ro[r] + k0 + k] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < PX; ++u) {
            const int e = threadIdx.x + u * NT, i = e / MM_N, n = e % MM_N;
            rx[u] = i < kb ? X[(G.xc0 + k0 + i) * ldk + kc + n] : 0.0;
        }
    };
    auto store = [&](int st) {
        double *Vs = dsm + st * (VS + XS), *Xs = Vs + VS;
#pragma unroll
        for (int u = 0; u < PV; ++u) {
            const int r = vrow(u), k = vk(u);
            Vs[k * 64 + (r ^ (8 * (k & 3)))] = rv[u];
        }
#pragma unroll
        for (int u = 0; u < PX; ++u) {
            const int e = threadIdx.x + u * NT;
            Xs[(e / MM_N) * MM_STR + e % MM_N] = rx[u];
        }
    };
    const bool act = r0 < G.m;
    double acc[2][4][2] = {};
    load(0);
    store(0);
    __syncthreads();
    int st = 0;
    for (int k0 = 0; k0 < G.len; k0 += MM_KB) {
        const bool more = k0 + MM_KB < G.len;
        if (more) load(k0 + MM_KB);
        const double *Vs = dsm + st * (VS + XS), *Xs = Vs + VS;
        if (act) {
#pragma unroll
            for (int kk = 0; kk < MM_KB; kk += 4) {
                const int k = kk + (l & 3);
                double a[2], b[4];
#pragma unroll
                for (int i = 0; i < 2; ++i) a[i] = Vs[k * 64 + ((r0 + i * 8 + (l >> 2)) ^ (8 * (l & 3)))];
#pragma unroll
                for (int j = 0; j < 4; ++j) b[j] = Xs[k * MM_STR + n0 + j * 8 + (l >> 2)];
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
            }
        }
        if (more) store(st ^ 1);
        __syncthreads();
        st ^= 1;
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int r = r0 + i * 8 + (l >> 2);
        if (r >= G.m) continue;
        const VChunk &C = gch[rq[r]];
        double *out = (C.pidx >= 0 ? part + (i64)C.pidx * KC_MAX * ldk : T + (i64)C.blk * KC_MAX * ldk) +
                      (i64)(vc_col0(C) + rc[r]) * ldk;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = kc + n0 + j * 8 + (l & 3) * 2;
            out[n] = acc[i][j][0];
            out[n + 1] = acc[i][j][1];
        }
    }
}
constexpr int VTXG_SMEM = 2 * (MM_KB * 64 + MM_KB * MM_STR) * 8;

// T rows of multi-chunk blocks: sum of their chunk partials (fixed order)
__global__ void treduce_mm_kernel(const TJob *jobs, const double *part, i64 ldk, int K, double *T) {
    const TJob J = jobs[blockIdx.x];
    for (int e = threadIdx.x; e < J.r * K; e += NT) {
        const int c = e / K, n = e % K;
        double s = 0.0;
        for (int k = J.cbeg; k < J.cend; ++k) s += part[((i64)k * KC_MAX + c) * ldk + n];
        T[((i64)J.blk * KC_MAX + c) * ldk + n] = s;
    }
}

// phase 2: one CTA per (segment, 64-RHS tile); warp w owns rows 16 (w % 4) .. +16 and
// RHS 32 (w / 4) .. +32 of the 64 x 64 output tile (2 x 4 DMMA fragments)
__global__ void __launch_bounds__(NT) seg_mm_kernel(const SegDesc *segs, const int32_t *colmap,
                                                    const double *pbuf, const double *X,
                                                    const double *T, i64 ldk, double *Y,
                                                    double alpha, double beta, const double *Z) {
    // two stages of (As [MM_KB][MM_STR], Bs [MM_KB][MM_STR]), register-staged prefetch of the next
    // inner step during the current one's DMMA
    extern __shared__ double dsm[];
    constexpr int AS = MM_KB * MM_STR;
    const SegDesc S = segs[blockIdx.x];
    const int kc = blockIdx.y * MM_N;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int r0 = (w & 3) * 16, n0 = (w >> 2) * 32;
    double acc[2][4][2] = {};
    const double *A = pbuf + S.poff;
    constexpr int PA = MM_KB * 64 / NT, PB = MM_KB * MM_N / NT;
    double ra[PA], rb[PB];
    auto load = [&](int q0) {
        const int qb = min(MM_KB, S.ncol - q0);
#pragma unroll
        for (int u = 0; u < PA; ++u) {
            const int e = threadIdx.x + u * NT, q = e / 64, i = e % 64;
            ra[u] = (q < qb && i < S.ld) ? A[(i64)(q0 + q) * S.ld + i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < PB; ++u) {
            const int e = threadIdx.x + u * NT, q = e / MM_N, n = e % MM_N;
            double v = 0.0;
            if (q < qb) {
                const int32_t src = colmap[S.cmoff + q0 + q];
                v = src >= 0 ? X[(i64)src * ldk + kc + n] : T[(i64)(-1 - src) * ldk + kc + n];
            }
            rb[u] = v;
        }
    };
    auto store = [&](int st) {
        double *As = dsm + st * 2 * AS, *Bs = As + AS;
#pragma unroll
        for (int u = 0; u < PA; ++u) {
            const int e = threadIdx.x + u * NT;
            As[(e / 64) * MM_STR + e % 64] = ra[u];
        }
#pragma unroll
        for (int u = 0; u < PB; ++u) {
            const int e = threadIdx.x + u * NT;
            Bs[(e / MM_N) * MM_STR + e % MM_N] = rb[u];
        }
    };
    load(0);
    store(0);
    __syncthreads();
    int st = 0;
    for (int q0 = 0; q0 < S.ncol; q0 += MM_KB) {
        const bool more = q0 + MM_KB < S.ncol;
        if (more) load(q0 + MM_KB);
        const double *As = dsm + st * 2 * AS, *Bs = As + AS;
#pragma unroll
        for (int kk = 0; kk < MM_KB; kk += 4) {
            double a[2], b[4];
#pragma unroll
            for (int i = 0; i < 2; ++i) a[i] = As[(kk + (l & 3)) * MM_STR + r0 + i * 8 + (l >> 2)];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[(kk + (l & 3)) * MM_STR + n0 + j * 8 + (l >> 2)];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
        if (more) store(st ^ 1);
        __syncthreads();
        st ^= 1;
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int row = r0 + i * 8 + (l >> 2);
        if (row >= S.rows) continue;
        const i64 yr = (S.y0 + row) * ldk;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = kc + n0 + j * 8 + (l & 3) * 2;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double zv = beta == 0.0 ? 0.0 : beta * Z[yr + n + h];
                Y[yr + n + h] = zv + alpha * acc[i][j][h];
            }
        }
    }
}
constexpr int SEGMM_SMEM = 2 * 2 * MM_KB * MM_STR * 8;

// column-major (ld) <-> row-major (ldk) conversion of an n x k block, 32 x 32 tiles
__global__ void transpose_kernel(const double *src, i64 lds, double *dst, i64 ldd, i64 n, int k,
                                 int to_rowmajor) {
    __shared__ double tile[32][33];
    const i64 i0 = (i64)blockIdx.x * 32;
    const int j0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int y = ty; y < 32; y += 8) {
        if (to_rowmajor) {  // src column-major: element (i, j) at src[i + j * lds]
            const i64 i = i0 + tx;
            const int j = j0 + y;
            tile[y][tx] = (i < n && j < k) ? src[i + (i64)j * lds] : 0.0;
        } else {            // src row-major: element (i, j) at src[i * lds + j]
            const i64 i = i0 + y;
            const int j = j0 + tx;
            tile[y][tx] = (i < n && j < k) ? src[i * lds + j] : 0.0;
        }
    }
    __syncthreads();
    for (int y = ty; y < 32; y += 8) {
        if (to_rowmajor) {  // dst row-major: (i0 + y, j0 + tx) = tile[tx][y]
            const i64 i = i0 + y;
            const int j = j0 + tx;
            if (i < n && j < k) dst[i * ldd + j] = tile[tx][y];
        } else {            // dst column-major: (i0 + tx, j0 + y) = tile[tx][y]
            const i64 i = i0 + tx;
            const int j = j0 + y;
            if (i < n && j < k) dst[i + (i64)j * ldd] = tile[tx][y];
        }
    }
}

void mm_transpose(const double *src, i64 lds, double *dst, i64 ldd, i64 n, int k, bool to_rowmajor,
                  cudaStream_t s) {
    dim3 grid((unsigned)((n + 31) / 32), (unsigned)((k + 31) / 32));
    transpose_kernel<<<grid, NT, 0, s>>>(src, lds, dst, ldd, n, k, to_rowmajor ? 1 : 0);
    LH_CUDA(cudaGetLastError());
}

static void mm_attrs() {
    static bool done = false;
    if (done) return;
    LH_CUDA(cudaFuncSetAttribute((const void *)vtx_mm_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 VTXG_SMEM));
    LH_CUDA(cudaFuncSetAttribute((const void *)seg_mm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 SEGMM_SMEM));
    done = true;
}

i64 mm_pad(int k) { return ((i64)k + MM_N - 1) / MM_N * MM_N; }

// right-hand-side count from which the DMMA matmat replaces per-column matvecs
int mm_min_rhs() {
    static const int v = getenv("LEVYH_MM_MIN") ? std::max(1, atoi(getenv("LEVYH_MM_MIN"))) : 8;
    return v;
}

MmBufs mm_bufs(Ctx &ctx, const MvPlan &P, i64 ldk) {
    MmBufs b;
    b.T = ctx.mm[2].ensure((i64)std::max(P.nblk, 1) * KC_MAX * ldk);
    b.part = ctx.mm[3].ensure((i64)std::max(P.npart, 1) * KC_MAX * ldk);
    return b;
}

// Y = alpha H X + beta Z, all row-major with ldk = mm_pad(K) (columns >= K are don't-care)
void mm_run(const MvPlan &P, const double *X, double *Y, i64 ldk, double alpha, double beta,
            const double *Z, double *T, double *part, cudaStream_t s) {
    LH_REQUIRE(!P.cpl && !P.h2, LH_EINTERNAL, "the multi-RHS matmat runs on the H-form plan");
    const unsigned nk = (unsigned)(ldk / MM_N);
    static const bool ungrouped = getenv("LEVYH_MM_NOGROUP") != nullptr;  // timing experiments only
    if (!ungrouped && P.ngroup > 0) {
        mm_attrs();
        vtx_mm_group_kernel<<<dim3(P.ngroup, nk), NT, VTXG_SMEM, s>>>(P.groups, P.gchunks, P.pbuf, X, ldk, T, part);
    } else {
        if (P.nch > 0) vtx_mm_kernel<<<dim3(P.nch, nk), NT, 0, s>>>(P.chunks, P.pbuf, X, ldk, T, part);
        if (P.nch16 > 0)
            vtx_mm_kernel<<<dim3(P.nch16, nk), NT, 0, s>>>(P.chunks16, P.pbuf, X, ldk, T, part);
    }
    if (P.ntj > 0) treduce_mm_kernel<<<P.ntj, NT, 0, s>>>(P.tjobs, part, ldk, (int)ldk, T);
    mm_attrs();
    seg_mm_kernel<<<dim3(P.nseg, nk), NT, SEGMM_SMEM, s>>>(P.segs, P.colmap, P.pbuf, X, T, ldk, Y, alpha, beta,
                                                           Z ? Z : Y);
    LH_CUDA(cudaGetLastError());
}

void seg_mm_launch(const MvPlan &P, const double *X, const double *T, i64 ldk, double *Y, double alpha,
                   double beta, const double *Z, cudaStream_t s) {
    const unsigned nk = (unsigned)(ldk / MM_N);
    mm_attrs();
    seg_mm_kernel<<<dim3(P.nseg, nk), NT, SEGMM_SMEM, s>>>(P.segs, P.colmap, P.pbuf, X, T, ldk, Y, alpha, beta,
                                                           Z ? Z : Y);
    LH_CUDA(cudaGetLastError());
}

}  // namespace lh
