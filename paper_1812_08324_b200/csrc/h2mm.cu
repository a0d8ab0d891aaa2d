// Multi-RHS application of the nested-basis (H2) propagator on the FP64 tensor cores:
// Y = alpha Z X + beta W for K right-hand sides (cfg4's 256), X row-major N x ldk.
// Reference semantics: hops.mul_dense (hops.py:73-85) of Z = (A+)^-1 in H2 form.
//
// The single-RHS walk of h2step.cu becomes a sequence of batched K-wide DMMA products
// (mma.sync m8n8k4 f64), one launch per tree level:
//   leaves     Xh_s    = P_s^T X_s                         (k_s x 64) (64 x K)
//   up levels  Xh_tau  = T_tau^T [Xh_c1; Xh_c2]            by height, leaves first
//   couplings  Yh_rho  = sum_b S_b Xh_sigma(b)            every row cluster (zero when none)
//   down       Yh_c   += T_c Yh_parent                     by depth, root first
//   rows       Y       = alpha (D X + Q_t Yh_t) + beta W   the segment matmat of the ZS plan
//                                                          (matmat.cu seg_mm_kernel; Yh_t of a
//                                                          row leaf is stored in the T rows its
//                                                          Q_t piece reads)
// A job computes C[crow .. crow + m, tile] (=|+=) A (m x kk) B, A(i, j) = abase[aoff + i sa +
// j sb], B = the concatenation of up to four row ranges of the source matrix.
#include <algorithm>
#include <cstdlib>

#include "core.h"
#include "dev.cuh"
#include "matvec.h"

namespace lh {

using dev::KC_MAX;
using dev::NT;

namespace {

constexpr int TN = 64;    // right-hand sides per CTA tile
constexpr int KB = 32;    // inner block staged per step
constexpr int ASTR = 33;  // As[k][i] stride (m <= 32)
constexpr int BSTR = 68;  // Bs[k][n] stride

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// one CTA per (job, 64-RHS tile); warp w owns RHS w*8 .. +8 of the tile and all four 8-row
// fragments of the (<= 32)-row output
__global__ void __launch_bounds__(NT) h2mm_kernel(const H2MMJob *jobs, const double *abase, const double *B,
                                                   double *C, i64 ldk, int accum) {
    __shared__ double As[KB * ASTR];
    __shared__ double Bs[KB * BSTR];
    const H2MMJob J = jobs[blockIdx.x];
    const int n0 = blockIdx.y * TN;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    double acc[4][2] = {};
    for (int k0 = 0; k0 < J.kk; k0 += KB) {
        const int kb = min(KB, J.kk - k0);
        for (int e = threadIdx.x; e < 32 * KB; e += NT) {
            const int i = e / KB, j = e % KB;
            As[j * ASTR + i] = (i < J.m && j < kb) ? abase[J.aoff + (i64)i * J.sa + (i64)(k0 + j) * J.sb] : 0.0;
        }
        for (int e = threadIdx.x; e < KB * TN; e += NT) {
            const int j = e / TN, n = e % TN;
            double v = 0.0;
            if (j < kb) {
                int q = k0 + j, r = 0;
                while (q >= J.n[r]) q -= J.n[r++];
                v = B[(i64)(J.b[r] + q) * ldk + n0 + n];
            }
            Bs[j * BSTR + n] = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < KB; kk += 4) {
            const double b = Bs[(kk + (l & 3)) * BSTR + w * 8 + (l >> 2)];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const double a = As[(kk + (l & 3)) * ASTR + t * 8 + (l >> 2)];
                dmma(acc[t][0], acc[t][1], a, b);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int row = t * 8 + (l >> 2);
        if (row >= J.m) continue;
        double *c = C + (i64)(J.crow + row) * ldk + n0 + w * 8 + (l & 3) * 2;
        if (accum) {
            c[0] += acc[t][0];
            c[1] += acc[t][1];
        } else {
            c[0] = acc[t][0];
            c[1] = acc[t][1];
        }
    }
}

}  // namespace

H2MM::~H2MM() {
    if (jobs) cudaFree(jobs);
}

std::shared_ptr<H2MM> build_h2mm(const H2MMInput &in, cudaStream_t st) {
    auto M = std::make_shared<H2MM>();
    std::vector<H2MMJob> jv;
    auto level = [&](int src, int abase, int dst, int accum) {
        H2MMLevel L{(int32_t)jv.size(), 0, src, abase, dst, accum};
        M->levels.push_back(L);
    };
    auto close = [&]() {
        M->levels.back().end = (int32_t)jv.size();
        if (M->levels.back().end == M->levels.back().beg) M->levels.pop_back();
    };
    // leaves: Xh_s = P_s^T X_s, P_s at pb[poff + i + 64 j] (i < rows, j < k)
    level(H2MM_X, H2MM_PB, H2MM_XH, 0);
    for (const H2Leaf &L : *in.leaves) {
        if (L.k <= 0) continue;
        LH_REQUIRE(L.k <= 32, LH_EINTERNAL, "H2 multi-RHS: leaf basis above 32 columns");
        H2MMJob J{};
        J.aoff = L.poff;
        J.m = L.k;
        J.kk = L.rows;
        J.sa = 64;
        J.sb = 1;
        J.crow = L.xoff;
        J.b[0] = (int32_t)L.x0;
        J.n[0] = L.rows;
        jv.push_back(J);
    }
    close();
    // up levels by height: Xh_tau = T^T [Xh_c1; Xh_c2], element (j, i) at tu[toff + i k + j]
    int hmax = 0;
    for (int h : in.up_height) hmax = std::max(hmax, h);
    for (int h = 1; h <= hmax; ++h) {
        level(H2MM_XH, H2MM_TU, H2MM_XH, 0);
        for (size_t u = 0; u < in.ups->size(); ++u) {
            const H2Up &U = (*in.ups)[u];
            if (in.up_height[u] != h || U.k <= 0) continue;
            LH_REQUIRE(U.k <= 32, LH_EINTERNAL, "H2 multi-RHS: basis above 32 columns");
            H2MMJob J{};
            J.aoff = U.toff;
            J.m = U.k;
            J.kk = U.k1 + U.k2;
            J.sa = 1;
            J.sb = U.k;
            J.crow = U.xoff;
            J.b[0] = U.xoff1;
            J.n[0] = U.k1;
            J.b[1] = U.xoff2;
            J.n[1] = U.k2;
            jv.push_back(J);
        }
        close();
    }
    // couplings: Yh_rho = [S_1 .. S_m] [Xh_1; ..; Xh_m] (S contiguous, column-major ld kr); a node
    // without couplings gets a zero job; more than four couplings continue in accumulate jobs
    std::vector<H2MMJob> extra;
    level(H2MM_XH, H2MM_SB, H2MM_YH, 0);
    for (size_t d = 0; d < in.dns->size(); ++d) {
        const H2Down &D = (*in.dns)[d];
        if (D.k <= 0) continue;
        LH_REQUIRE(D.k <= 32, LH_EINTERNAL, "H2 multi-RHS: basis above 32 columns");
        for (int e0 = D.c0; e0 < D.c1 || e0 == D.c0; e0 += 4) {
            H2MMJob J{};
            J.m = D.k;
            J.sa = 1;
            J.sb = D.k;
            J.crow = in.dn_row[d];
            J.aoff = e0 < D.c1 ? (*in.cpls)[e0].soff : 0;
            for (int r = 0; r < 4 && e0 + r < D.c1; ++r) {
                const H2Cpl &E = (*in.cpls)[e0 + r];
                J.b[r] = E.xoff;
                J.n[r] = E.kc;
                J.kk += E.kc;
            }
            (e0 == D.c0 ? jv : extra).push_back(J);
            if (e0 >= D.c1) break;
        }
    }
    close();
    if (!extra.empty()) {
        level(H2MM_XH, H2MM_SB, H2MM_YH, 1);
        jv.insert(jv.end(), extra.begin(), extra.end());
        close();
    }
    // down levels by depth: Yh_c += T_c Yh_parent, element (i, j) at td[toff + roff + i + j ldt]
    int dmax = 0;
    for (int d : in.dn_depth) dmax = std::max(dmax, d);
    for (int dep = 1; dep <= dmax; ++dep) {
        level(H2MM_YH, H2MM_TD, H2MM_YH, 1);
        for (size_t d = 0; d < in.dns->size(); ++d) {
            const H2Down &D = (*in.dns)[d];
            if (in.dn_depth[d] != dep || D.k <= 0 || D.kp <= 0 || in.dn_prow[d] < 0) continue;
            H2MMJob J{};
            J.aoff = D.toff + D.roff;
            J.m = D.k;
            J.kk = D.kp;
            J.sa = 1;
            J.sb = D.ldt;
            J.crow = in.dn_row[d];
            J.b[0] = in.dn_prow[d];
            J.n[0] = D.kp;
            jv.push_back(J);
        }
        close();
    }
    for (const H2MMJob &J : jv) {
        LH_REQUIRE(J.kk == J.n[0] + J.n[1] + J.n[2] + J.n[3], LH_EINTERNAL, "H2 multi-RHS job ranges");
        M->flops_per_rhs += 2.0 * J.m * J.kk;
    }
    M->jobs = dupload(jv, st);
    M->njobs = (int)jv.size();
    M->nxh = in.nxh;
    M->nyrows = in.nyrows;
    M->pb = in.pb;
    M->tu = in.tu;
    M->td = in.td;
    M->sb = in.sb;
    LH_CUDA(cudaStreamSynchronize(st));
    return M;
}

void h2mm_run(H2MM &M, const MvPlan &zs, const double *X, double *Y, i64 ldk, double alpha, double beta,
              const double *W, cudaStream_t s) {
    double *xh = M.xh.ensure(std::max<i64>(M.nxh, 1) * ldk);
    double *yh = M.yh.ensure(std::max<i64>(M.nyrows, 1) * ldk);
    const unsigned nk = (unsigned)(ldk / TN);
    for (const H2MMLevel &L : M.levels) {
        const double *src = L.src == H2MM_X ? X : L.src == H2MM_XH ? xh : yh;
        const double *ab = L.abase == H2MM_PB ? M.pb : L.abase == H2MM_TU ? M.tu : L.abase == H2MM_SB ? M.sb : M.td;
        double *dst = L.dst == H2MM_XH ? xh : yh;
        h2mm_kernel<<<dim3((unsigned)(L.end - L.beg), nk), NT, 0, s>>>(M.jobs + L.beg, ab, src, dst, ldk, L.accum);
    }
    LH_CUDA(cudaGetLastError());
    seg_mm_launch(zs, X, yh, ldk, Y, alpha, beta, W ? W : Y, s);
}

}  // namespace lh
