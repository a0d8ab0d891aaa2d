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
    __shared__ double As[MM_KB * MM_STR];  // [q][row]
    __shared__ double Bs[MM_KB * MM_STR];  // [q][n]
    const SegDesc S = segs[blockIdx.x];
    const int kc = blockIdx.y * MM_N;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int r0 = (w & 3) * 16, n0 = (w >> 2) * 32;
    double acc[2][4][2] = {};
    const double *A = pbuf + S.poff;
    for (int q0 = 0; q0 < S.ncol; q0 += MM_KB) {
        const int qb = min(MM_KB, S.ncol - q0);
        for (int e = threadIdx.x; e < MM_KB * 64; e += NT) {
            const int q = e / 64, i = e % 64;
            As[q * MM_STR + i] = (q < qb && i < S.ld) ? A[(i64)(q0 + q) * S.ld + i] : 0.0;
        }
        for (int e = threadIdx.x; e < MM_KB * MM_N; e += NT) {
            const int q = e / MM_N, n = e % MM_N;
            double v = 0.0;
            if (q < qb) {
                const int32_t src = colmap[S.cmoff + q0 + q];
                v = src >= 0 ? X[(i64)src * ldk + kc + n] : T[(i64)(-1 - src) * ldk + kc + n];
            }
            Bs[q * MM_STR + n] = v;
        }
        __syncthreads();
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
        __syncthreads();
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
    if (P.nch > 0) vtx_mm_kernel<<<dim3(P.nch, nk), NT, 0, s>>>(P.chunks, P.pbuf, X, ldk, T, part);
    if (P.nch16 > 0)
        vtx_mm_kernel<<<dim3(P.nch16, nk), NT, 0, s>>>(P.chunks16, P.pbuf, X, ldk, T, part);
    if (P.ntj > 0) treduce_mm_kernel<<<P.ntj, NT, 0, s>>>(P.tjobs, part, ldk, (int)ldk, T);
    seg_mm_kernel<<<dim3(P.nseg, nk), NT, 0, s>>>(P.segs, P.colmap, P.pbuf, X, T, ldk, Y, alpha, beta,
                                                  Z ? Z : Y);
    LH_CUDA(cudaGetLastError());
}

void seg_mm_launch(const MvPlan &P, const double *X, const double *T, i64 ldk, double *Y, double alpha,
                   double beta, const double *Z, cudaStream_t s) {
    const unsigned nk = (unsigned)(ldk / MM_N);
    seg_mm_kernel<<<dim3(P.nseg, nk), NT, 0, s>>>(P.segs, P.colmap, P.pbuf, X, T, ldk, Y, alpha, beta, Z ? Z : Y);
    LH_CUDA(cudaGetLastError());
}

}  // namespace lh
