// Entry generation (Toeplitz symbol of the singular CN operator) and H-matrix
// construction: partition + batched ACA + QR/SVD recompression with the
// reference truncation rule, dense-leaf fill.
//
// Reference: fractional.py:78-86 (window), :108-127 (power density),
// :285-301 (_window_sums_1d), :362-405 (frac_stencil_1d / Poisson assembly),
// levy.py:169-206 (local band, A+-), hmatrix.py:294-340 (build_from_dense).
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <limits>
#include <algorithm>
#include <cmath>
#include <numeric>

#include "core.h"
#include "dev.cuh"
#include "measure.cuh"

namespace lh {

using dev::KA_MAX;
using dev::KC_MAX;
using dev::NT;

// ===========================================================================
// entry generation
// ===========================================================================
constexpr int SUM_CHUNK = 4096;

// per-CTA partial sums of kern, rho*y*kern, rho*y*y*kern over a fixed chunk of j
__global__ void window_sums_kernel(MeasureDev nu, double h, i64 M, double rho_r, double *partials) {
    __shared__ double red[dev::NW];
    i64 j0 = -M + (i64)blockIdx.x * SUM_CHUNK;
    i64 j1 = min(j0 + SUM_CHUNK, M + 1);
    double s0 = 0.0, sg = 0.0, sd = 0.0;
    for (i64 j = j0 + threadIdx.x; j < j1; j += NT) {
        double kern = kern_eval(nu, j, h, M);
        double y = (double)j * h;
        double rho = window_eval(y, rho_r);
        s0 += kern;
        sg += (rho * y) * kern;
        sd += ((rho * y) * y) * kern;
    }
    s0 = dev::block_sum(s0, red);
    sg = dev::block_sum(sg, red);
    sd = dev::block_sum(sd, red);
    if (threadIdx.x == 0) {
        partials[3 * blockIdx.x + 0] = s0;
        partials[3 * blockIdx.x + 1] = sg;
        partials[3 * blockIdx.x + 2] = sd;
    }
}

__global__ void reduce_partials_kernel(const double *partials, int nparts, double *sums) {
    __shared__ double red[dev::NW];
    for (int q = 0; q < 3; ++q) {
        double s = 0.0;
        for (int k = threadIdx.x; k < nparts; k += NT) s += partials[3 * k + q];
        s = dev::block_sum(s, red);
        if (threadIdx.x == 0) sums[q] = s;
    }
}

struct SymbolArgs {
    double h, tail, m2, a, b, c, dt;
    i64 N, M;
};

// tA[k + N - 1] = A[i, i + k]; tP/tM for A+- (fractional.py:375-387, levy.py:173-176, :201-205)
__global__ void symbol_fill_kernel(MeasureDev nu, SymbolArgs p, const double *sums, double *tA,
                                   double *tP, double *tM) {
    const double S0 = sums[0], Sg = sums[1], Sd = sums[2];
    const double h = p.h;
    const double h2 = h * h;
    const i64 N = p.N;
    const i64 kmax = min(N - 1, p.M);
    const double hd = 0.5 * p.dt;
    for (i64 idx = (i64)blockIdx.x * NT + threadIdx.x; idx < 2 * N - 1; idx += (i64)gridDim.x * NT) {
        i64 k = idx - (N - 1);
        double W = 0.0;
        if (k != 0 && (k <= kmax && k >= -kmax)) W = kern_eval(nu, k, h, p.M);
        if (k == 0) W = 0.0 + ((-S0 - p.tail) - (p.m2 - Sd) / h2);
        double cside = (p.m2 - Sd) / (2 * h2);
        if (k == 1) W += cside - Sg / (2 * h);
        if (k == -1) W += cside + Sg / (2 * h);
        double t = -W;
        if (k == 0) t += 2 * p.a / h2 - p.c;
        if (k == 1) t += -p.a / h2 - p.b / (2 * h);
        if (k == -1) t += -p.a / h2 + p.b / (2 * h);
        tA[idx] = t;
        if (tP) tP[idx] = (k == 0 ? 1.0 : 0.0) + hd * t;
        if (tM) tM[idx] = (k == 0 ? 1.0 : 0.0) - hd * t;
    }
}

void cn_symbol(Ctx &ctx, const lh_measure &m, const lh_cn_params &p, double *tA, double *tP,
               double *tM, double *sums_host) {
    LH_REQUIRE(p.N >= 1 && p.M >= 1, LH_EINVAL, "need N >= 1 and M >= 1");
    LH_REQUIRE(p.h > 0 && p.rho_r > 0, LH_EINVAL, "need h > 0 and rho_r > 0");
    MeasureDev nu = measure_to_dev(m, p.M);
    i64 cnt = 2 * p.M + 1;
    int nparts = (int)((cnt + SUM_CHUNK - 1) / SUM_CHUNK);
    double *buf = (double *)ctx.ensure_scratch(sizeof(double) * (3 * (size_t)nparts + 4));
    double *sums = buf + 3 * (size_t)nparts;
    window_sums_kernel<<<nparts, NT, 0, ctx.stream>>>(nu, p.h, p.M, p.rho_r, buf);
    reduce_partials_kernel<<<1, NT, 0, ctx.stream>>>(buf, nparts, sums);
    SymbolArgs a{p.h, p.tail, p.m2, p.a, p.b, p.c, p.dt, p.N, p.M};
    int grid = (int)std::min<i64>((2 * p.N - 1 + NT - 1) / NT, 148 * 16);
    symbol_fill_kernel<<<grid, NT, 0, ctx.stream>>>(nu, a, sums, tA, tP, tM);
    LH_CUDA(cudaGetLastError());
    if (sums_host) {
        LH_CUDA(cudaMemcpyAsync(sums_host, sums, 3 * sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
        LH_CUDA(cudaStreamSynchronize(ctx.stream));
    }
}

// ---------------------------------------------------------------------------
// smooth (Gaussian) jump density: nu(y) = scale e^{-eps_sq y^2} (levy.py:72-81)
// CN operator of levy.CNSystem (levy.py:169-206, assemble_cn_1d :249-263):
//   A[i, j] = -nu((j - i) h) h,  (i, i +- 1) += -a/h^2 -+ b/(2h),
//   A[i, i] = 2a/h^2 - c + lam h,  lam = sum_{j=1..n_off} nu(-jh) + nu(jh)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double gauss_nu(double eps_sq, double scale, double y) {
    return scale * exp(-eps_sq * (y * y));
}

__global__ void gauss_lam_kernel(double eps_sq, double scale, double h, i64 n_off, double *partials) {
    __shared__ double red[dev::NW];
    const i64 j0 = 1 + (i64)blockIdx.x * SUM_CHUNK;
    const i64 j1 = min(j0 + SUM_CHUNK, n_off + 1);
    double s = 0.0;
    for (i64 j = j0 + threadIdx.x; j < j1; j += NT) {
        const double y = (double)j * h;
        s += gauss_nu(eps_sq, scale, -y) + gauss_nu(eps_sq, scale, y);
    }
    s = dev::block_sum(s, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void reduce_one_kernel(const double *partials, int nparts, double *out) {
    __shared__ double red[dev::NW];
    double s = 0.0;
    for (int k = threadIdx.x; k < nparts; k += NT) s += partials[k];
    s = dev::block_sum(s, red);
    if (threadIdx.x == 0) out[0] = s;
}

__global__ void gauss_symbol_kernel(double eps_sq, double scale, double h, i64 N, double a,
                                    double b, double c, double dt, const double *lam, double *tA,
                                    double *tP, double *tM) {
    const double hd = 0.5 * dt;
    const double h2 = h * h;
    for (i64 idx = (i64)blockIdx.x * NT + threadIdx.x; idx < 2 * N - 1; idx += (i64)gridDim.x * NT) {
        const i64 k = idx - (N - 1);
        double t;
        if (k == 0) {
            t = 2 * a / h2 - c + lam[0] * h;
        } else {
            t = -gauss_nu(eps_sq, scale, (double)k * h) * h;
            if (k == 1) t += -a / h2 - b / (2 * h);
            if (k == -1) t += -a / h2 + b / (2 * h);
        }
        tA[idx] = t;
        if (tP) tP[idx] = (k == 0 ? 1.0 : 0.0) + hd * t;
        if (tM) tM[idx] = (k == 0 ? 1.0 : 0.0) - hd * t;
    }
}

// 2D CN operator on a tensor grid (levy.py:178-206 _entries_a_2d + entries(which)): entry (i, j)
// of A / A+ / A- for the points order[i], order[j] (row-major grid index k = iy nx + ix) in the
// order the caller's cluster tree gives; the same operations as numpy.
struct Cn2dSrc {
    const int64_t *order;
    int nx, which;
    double h, eps_sq, scale, a, b, c, lam, hdt;
    __device__ __forceinline__ double operator()(i64 i, i64 j) const {
        const double h2 = h * h;
        const i64 r = order[i], q = order[j];
        const double dx = (double)((q % nx) - (r % nx)) * h, dy = (double)((q / nx) - (r / nx)) * h;
        double E = -(scale * exp(-eps_sq * (dx * dx + dy * dy))) * h2;
        const bool ex = fabs(dx) < 1.5 * h && fabs(dy) < 0.5 * h;
        const bool ey = fabs(dy) < 1.5 * h && fabs(dx) < 0.5 * h;
        if (ex && dx > 0.5 * h) E += -a / h2 - b / (2 * h);
        if (ex && dx < -0.5 * h) E += -a / h2 + b / (2 * h);
        if (ey && fabs(dy) > 0.5 * h) E += -a / h2;
        if (ex && ey) E = 4 * a / h2 - c + lam * h2;
        const double eye = (r == q) ? 1.0 : 0.0;
        return which == 0 ? E : which == 1 ? eye + hdt * E : eye - hdt * E;
    }
};

// the whole operator, row-major (ld N)
__global__ void cn2d_dense_kernel(i64 N, Cn2dSrc src, double *out) {
    const i64 total = N * N;
    for (i64 e = (i64)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (i64)gridDim.x * blockDim.x)
        out[e] = src(e / N, e % N);
}

void cn2d_dense(Ctx &ctx, i64 N, int nx, double h, double eps_sq, double scale, double a, double b, double c,
                double lam, double dt, int which, const int64_t *order_host, double *out_dev) {
    LH_REQUIRE(which >= 0 && which <= 2, LH_EINVAL, "which must be 0 (A), 1 (plus) or 2 (minus)");
    LH_REQUIRE(nx > 0 && N % nx == 0, LH_EINVAL, "N must be a multiple of nx");
    std::vector<int64_t> ord(order_host, order_host + N);
    int64_t *d = dupload(ord, ctx.stream);
    const int grid = (int)std::min<i64>((N * N + NT - 1) / NT, (i64)ctx.num_sms * 32);
    cn2d_dense_kernel<<<grid, NT, 0, ctx.stream>>>(N, Cn2dSrc{d, nx, which, h, eps_sq, scale, a, b, c, lam, 0.5 * dt},
                                                   out_dev);
    LH_CUDA(cudaGetLastError());
    LH_CUDA(cudaStreamSynchronize(ctx.stream));
    cudaFree(d);
}

void gauss_cn_symbol(Ctx &ctx, i64 N, double h, double eps_sq, double scale, i64 n_off, double a,
                     double b, double c, double dt, double *tA, double *tP, double *tM,
                     double *lam_host) {
    LH_REQUIRE(N >= 1 && n_off >= 1 && h > 0, LH_EINVAL, "need N >= 1, n_off >= 1 and h > 0");
    LH_REQUIRE(eps_sq > 0 && scale >= 0, LH_EINVAL, "Gaussian density needs eps_sq > 0, scale >= 0");
    const int nparts = (int)((n_off + SUM_CHUNK - 1) / SUM_CHUNK);
    double *buf = (double *)ctx.ensure_scratch(sizeof(double) * ((size_t)nparts + 2));
    double *lam = buf + nparts;
    gauss_lam_kernel<<<nparts, NT, 0, ctx.stream>>>(eps_sq, scale, h, n_off, buf);
    reduce_one_kernel<<<1, NT, 0, ctx.stream>>>(buf, nparts, lam);
    const int grid = (int)std::min<i64>((2 * N - 1 + NT - 1) / NT, 148 * 16);
    gauss_symbol_kernel<<<grid, NT, 0, ctx.stream>>>(eps_sq, scale, h, N, a, b, c, dt, lam, tA, tP, tM);
    LH_CUDA(cudaGetLastError());
    if (lam_host) {
        LH_CUDA(cudaMemcpyAsync(lam_host, lam, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
        LH_CUDA(cudaStreamSynchronize(ctx.stream));
    }
}

// ===========================================================================
// entry sources
// ===========================================================================
struct ToepSrc {  // A[i, j] = t[(nrows - 1) + j - i]
    const double *t;
    i64 nrows;
    __device__ __forceinline__ double operator()(i64 i, i64 j) const { return t[nrows - 1 + j - i]; }
};
struct DenseSrc {  // row-major (numpy C order) or column-major
    const double *A;
    i64 lda;
    int row_major;
    __device__ __forceinline__ double operator()(i64 i, i64 j) const {
        return row_major ? A[i * lda + j] : A[i + j * lda];
    }
};

struct GaussSrc {  // expansion.kernel: scale e^{-eps_sq (x_i - y_j)^2} (hmatrix.py:174-176)
    const double *x, *y;
    double eps_sq, scale;
    __device__ __forceinline__ double operator()(i64 i, i64 j) const {
        const double d = x[i] - y[j];
        return scale * exp(-eps_sq * d * d);
    }
};

struct Gauss2Src {  // gaussian_expansion_2d's kernel: scale e^{-eps_sq |x_i - y_j|^2} (hmatrix.py:197-200)
    const double *x, *y;  // n x 2 row-major
    double eps_sq, scale;
    __device__ __forceinline__ double operator()(i64 i, i64 j) const {
        const double d0 = x[2 * i] - y[2 * j], d1 = x[2 * i + 1] - y[2 * j + 1];
        return scale * exp(-eps_sq * (d0 * d0 + d1 * d1));
    }
};

// ===========================================================================
// dense fill
// ===========================================================================
struct FillJob {
    i64 r0, c0, m, n, off;
};

template <class Src>
__global__ void dense_fill_kernel(Src src, const FillJob *jobs, int njobs, double *arena) {
    for (int b = blockIdx.x; b < njobs; b += gridDim.x) {
        FillJob J = jobs[b];
        double *D = arena + J.off;
        i64 tot = J.m * J.n;
        for (i64 e = threadIdx.x; e < tot; e += NT) {
            i64 i = e % J.m, j = e / J.m;
            D[e] = src(J.r0 + i, J.c0 + j);
        }
    }
}

// ===========================================================================
// ACA + recompression, one low-rank block per CTA (persistent, size-sorted)
// ===========================================================================
struct AcaJob {
    i64 r0, c0, m, n;
    i64 wu, wv;      // workspace offsets: U (m x KA), V (n x KA), column-major
    i64 fu, fv;      // final offsets in the arena (ld m / n)
    int32_t kcap;    // final capacity
    int32_t slot;    // rank slot
};

struct AcaSmem {
    dev::RecompSmem R;
    double ui[KA_MAX];
    double vj[KA_MAX];
    double hu[KA_MAX];
    double hv[KA_MAX];
    long long used[KA_MAX + 16];
    double redv[dev::NW];
    long long redi[dev::NW];
    double red[dev::NW];
    int nused;
};

// Adaptive cross approximation with partial pivoting on block (r0, c0, m, n).
// Returns the number of terms K; U[:, :K], V[:, :K] hold A ~= U V^T.
template <class Src>
__device__ int aca_block(const Src &src, i64 r0, i64 c0, i64 m, i64 n, double *U, double *V,
                         int KA, double tol, AcaSmem &S, int &converged) {
    int k = 0, fails = 0, conv = 0;
    double nS2 = 0.0;
    long long i = 0;
    if (threadIdx.x == 0) S.nused = 0;
    converged = 0;
    __syncthreads();
    while (k < KA) {
        for (int l = threadIdx.x; l < k; l += NT) S.ui[l] = U[i + (i64)l * m];
        __syncthreads();
        // residual row i -> V[:, k]
        double *vk = V + (i64)k * n;
        double best = -1.0;
        long long bj = 0;
        for (i64 j = threadIdx.x; j < n; j += NT) {
            double r = src(r0 + i, c0 + j);
            for (int l = 0; l < k; ++l) r -= S.ui[l] * V[j + (i64)l * n];
            vk[j] = r;
            double a = fabs(r);
            if (a > best) {
                best = a;
                bj = j;
            }
        }
        double amax;
        long long jstar;
        dev::block_argmax(best, bj, S.redv, S.redi, amax, jstar);
        if (threadIdx.x == 0 && S.nused < KA_MAX + 16) S.used[S.nused++] = i;
        __syncthreads();
        if (!(amax > 0.0)) {
            // row already represented exactly: try the next unused row
            if (++fails > 8 || S.nused >= m || S.nused >= KA_MAX + 16) {
                converged = 1;
                break;
            }
            long long cand = i;
            bool ok = false;
            for (int tries = 0; tries < KA_MAX + 16 && !ok; ++tries) {
                cand = (cand + 1) % m;
                ok = true;
                for (int q = 0; q < S.nused; ++q) ok = ok && (S.used[q] != cand);
            }
            i = cand;
            continue;
        }
        fails = 0;
        double delta = vk[jstar];
        double inv = 1.0 / delta;
        for (int l = threadIdx.x; l < k; l += NT) S.vj[l] = V[jstar + (i64)l * n];
        __syncthreads();
        for (i64 j = threadIdx.x; j < n; j += NT) vk[j] *= inv;
        // residual column jstar -> U[:, k]
        double *uk = U + (i64)k * m;
        for (i64 ii = threadIdx.x; ii < m; ii += NT) {
            double c = src(r0 + ii, c0 + jstar);
            for (int l = 0; l < k; ++l) c -= U[ii + (i64)l * m] * S.vj[l];
            uk[ii] = c;
        }
        __syncthreads();
        // |S_k|_F^2 update
        dev::col_dots(U, m, m, k, uk, S.hu);
        dev::col_dots(V, n, n, k, vk, S.hv);
        double su = 0.0, sv = 0.0;
        for (i64 ii = threadIdx.x; ii < m; ii += NT) su += uk[ii] * uk[ii];
        for (i64 j = threadIdx.x; j < n; j += NT) sv += vk[j] * vk[j];
        su = dev::block_sum(su, S.red);
        sv = dev::block_sum(sv, S.red);
        double cross = 0.0;
        for (int l = 0; l < k; ++l) cross += S.hu[l] * S.hv[l];
        nS2 += 2.0 * cross + su * sv;
        ++k;
        if (sqrt(su * sv) <= tol * sqrt(fabs(nS2))) {
            if (++conv >= 2) {
                converged = 1;
                break;
            }
        } else {
            conv = 0;
        }
        // next pivot row: argmax |U[:, k-1]| over unused rows
        best = -1.0;
        long long bi = 0;
        for (i64 ii = threadIdx.x; ii < m; ii += NT) {
            double a = fabs(uk[ii]);
            if (a > best) {
                bool fresh = true;
                for (int q = 0; q < S.nused; ++q) fresh = fresh && (S.used[q] != ii);
                if (fresh) {
                    best = a;
                    bi = ii;
                }
            }
        }
        double bmax;
        long long inext;
        dev::block_argmax(best, bi, S.redv, S.redi, bmax, inext);
        if (bmax < 0.0) {  // every row used
            converged = 1;
            break;
        }
        i = inext;
        __syncthreads();
    }
    __syncthreads();
    return k;
}

// Cross approximation with FULL pivoting for small blocks (m n <= ACA_FULL_MAX, 2D operators):
// the residual lives in shared memory, every step takes the entry of largest modulus and
// subtracts the rank-one cross exactly, and the stop test is exact: ||R||_F <= tol ||A||_F.
// Partial pivoting can stop early on the smooth 2D kernels (it never visits rows whose part of
// the block it has not yet seen), which shows up as ranks below the SVD's.
constexpr int ACA_FULL_MAX = 96 * 96;
template <class Src>
__device__ int aca_block_full(const Src &src, i64 r0, i64 c0, i64 m, i64 n, double *U, double *V, int KA,
                              double tol, AcaSmem &S, double *R, int &converged) {
    const i64 mn = m * n;
    double a2 = 0.0;
    for (i64 e = threadIdx.x; e < mn; e += NT) {
        const double v = src(r0 + e % m, c0 + e / m);
        R[e] = v;
        a2 += v * v;
    }
    a2 = dev::block_sum(a2, S.red);
    converged = 0;
    int k = 0;
    if (!(a2 > 0.0)) {
        converged = 1;
        return 0;
    }
    while (k < KA) {
        double best = -1.0, r2 = 0.0;
        long long be = 0;
        for (i64 e = threadIdx.x; e < mn; e += NT) {
            const double a = fabs(R[e]);
            r2 += R[e] * R[e];
            if (a > best) {
                best = a;
                be = e;
            }
        }
        r2 = dev::block_sum(r2, S.red);
        if (r2 <= tol * tol * a2) {
            converged = 1;
            break;
        }
        double amax;
        long long estar;
        dev::block_argmax(best, be, S.redv, S.redi, amax, estar);
        if (!(amax > 0.0)) {
            converged = 1;
            break;
        }
        const i64 is = estar % m, js = estar / m;
        const double inv = 1.0 / R[estar];
        double *uk = U + (i64)k * m, *vk = V + (i64)k * n;
        for (i64 i = threadIdx.x; i < m; i += NT) uk[i] = R[i + js * m];
        for (i64 j = threadIdx.x; j < n; j += NT) vk[j] = R[is + j * m] * inv;
        __syncthreads();
        for (i64 e = threadIdx.x; e < mn; e += NT) R[e] -= uk[e % m] * vk[e / m];
        __syncthreads();
        ++k;
    }
    if (!converged) {  // the cap reached: converged if the last update left the tolerance met
        double r2 = 0.0;
        for (i64 e = threadIdx.x; e < mn; e += NT) r2 += R[e] * R[e];
        r2 = dev::block_sum(r2, S.red);
        converged = r2 <= tol * tol * a2;
    }
    __syncthreads();
    return k;
}

// flags: 0 ok (low rank), 2 -> store dense (rank > min//2), 3 -> rank > kcap,
//        4 -> ACA hit max rank without converging
template <class Src>
__global__ void __launch_bounds__(NT) aca_kernel(Src src, const AcaJob *jobs, int njobs,
                                                 int *counter, double *work, double *arena,
                                                 int *ranks, int *flags, int KA, double tol,
                                                 double eps1, int full_pivot) {
    extern __shared__ double4 smem_raw[];
    AcaSmem &S = *reinterpret_cast<AcaSmem *>(smem_raw);
    double *Rres = reinterpret_cast<double *>(reinterpret_cast<char *>(smem_raw) + ((sizeof(AcaSmem) + 15) & ~15));
    __shared__ int s_job;
    while (true) {
        if (threadIdx.x == 0) s_job = atomicAdd(counter, 1);
        __syncthreads();
        int jb = s_job;
        __syncthreads();
        if (jb >= njobs) break;
        AcaJob J = jobs[jb];
        double *U = work + J.wu;
        double *V = work + J.wv;
        int conv = 0;
        int K = (full_pivot && J.m * J.n <= ACA_FULL_MAX)
                    ? aca_block_full(src, J.r0, J.c0, J.m, J.n, U, V, KA, tol, S, Rres, conv)
                    : aca_block(src, J.r0, J.c0, J.m, J.n, U, V, KA, tol, S, conv);
        i64 half = min(J.m, J.n) / 2;
        int rmax = (int)min((i64)min(J.kcap, KC_MAX), half);
        int r = dev::recompress(U, J.m, J.m, V, J.n, J.n, K, 0, eps1, arena + J.fu, J.m,
                                arena + J.fv, J.n, rmax, S.R);
        if (threadIdx.x == 0) {
            int f = 0;
            if (r > half) f = 2;
            else if (r > rmax) f = 3;
            else if (!conv) f = 4;
            ranks[J.slot] = (f == 0 || f == 4) ? r : 0;
            flags[jb] = f;
        }
        __syncthreads();
    }
}

// ===========================================================================
// host: build
// ===========================================================================
static void set_smem(const void *fn, size_t bytes) {
    LH_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

// storage layout: dense region then low-rank region; returns the low-rank leaves in ACA
// order (size-sorted, largest first)
static std::vector<int32_t> build_layout(Ctx &ctx, HMat &H, const lh_hconfig &cfg,
                                         const std::vector<int32_t> *cap_of = nullptr) {
    // column capacity: kept ranks stay <= KC_MAX; a capacity up to KA_MAX leaves room for the
    // H-LU's low-rank updates before each recompression (2D operators)
    const int kcap = std::min(std::max(cfg.kcap, 1), KA_MAX);
    i64 off = 0;
    int nslots = 0;
    std::vector<int32_t> lr;
    for (int32_t b : H.leafblocks) {
        Node &nd = H.nodes[b];
        if (nd.kind == K_DENSE) {
            nd.doff = off;
            off += nd.m * nd.n;
        }
    }
    for (int32_t b : H.leafblocks) {
        Node &nd = H.nodes[b];
        if (nd.kind == K_LR) {
            // capacity = stored rank + H-LU fill before recompression (<= KA_MAX); kept ranks
            // stay <= KC_MAX
            nd.kcap = cap_of ? std::min(std::max((*cap_of)[b], kcap), KA_MAX) : kcap;
            nd.rslot = nslots++;
            nd.uoff = off;
            off += nd.m * nd.kcap;
            nd.voff = off;
            off += nd.n * nd.kcap;
            lr.push_back(b);
        }
    }
    H.arena_len = off;
    H.d_arena = dalloc<double>(off);
    H.nslots = nslots;
    H.d_ranks = dalloc<int32_t>(std::max(nslots, 1));
    LH_CUDA(cudaMemsetAsync(H.d_ranks, 0, sizeof(int32_t) * std::max(nslots, 1), ctx.stream));
    std::sort(lr.begin(), lr.end(), [&](int32_t a, int32_t b) {
        i64 sa = H.nodes[a].m + H.nodes[a].n, sb = H.nodes[b].m + H.nodes[b].n;
        return sa != sb ? sa > sb : a < b;
    });
    return lr;
}

// ACA + recompression of the given low-rank leaves in size-sorted batches bounded by a
// workspace budget; returns the blocks whose rank exceeds min(m,n)//2 (to be stored dense)
template <class Src>
static std::vector<int32_t> run_aca(Ctx &ctx, HMat &H, Src src, const lh_hconfig &cfg,
                                    const std::vector<int32_t> &lr) {
    const int KA = std::min(std::max(cfg.max_aca_rank, 1), KA_MAX);
    const int kcap = std::min(std::max(cfg.kcap, 1), KC_MAX);
    const i64 budget = (i64)1 << 30;  // doubles (8 GiB)
    std::vector<int32_t> to_dense;
    // full pivoting on small blocks of 2D operators (the residual in shared memory)
    const int full = (H.rt && H.rt->dim == 2) ? 1 : 0;
    size_t smem = sizeof(AcaSmem);
    if (full) smem = ((sizeof(AcaSmem) + 15) & ~(size_t)15) + sizeof(double) * ACA_FULL_MAX;
    set_smem((const void *)aca_kernel<Src>, smem);
    size_t p = 0;
    double *work = nullptr;
    i64 work_len = 0;
    while (p < lr.size()) {
        std::vector<AcaJob> jobs;
        i64 w = 0;
        size_t q = p;
        while (q < lr.size()) {
            const Node &nd = H.nodes[lr[q]];
            i64 need = (nd.m + nd.n) * KA;
            if (!jobs.empty() && w + need > budget) break;
            AcaJob J{nd.r0, nd.c0, nd.m, nd.n, w, w + nd.m * KA, nd.uoff, nd.voff, nd.kcap, nd.rslot};
            jobs.push_back(J);
            w += need;
            ++q;
        }
        if (w > work_len) {
            if (work) cudaFree(work);
            work = dalloc<double>(w);
            work_len = w;
        }
        AcaJob *djobs = dupload(jobs, ctx.stream);
        int *dcnt = dalloc<int>(1 + (i64)jobs.size());
        int *dflags = dcnt + 1;
        LH_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(int) * (1 + jobs.size()), ctx.stream));
        int grid = std::min<int>((int)jobs.size(), ctx.num_sms * 2);
        aca_kernel<Src><<<grid, NT, smem, ctx.stream>>>(src, djobs, (int)jobs.size(), dcnt, work,
                                                        H.d_arena, H.d_ranks, dflags, KA,
                                                        cfg.aca_tol, cfg.eps1, full);
        LH_CUDA(cudaGetLastError());
        std::vector<int> flags(jobs.size());
        LH_CUDA(cudaMemcpyAsync(flags.data(), dflags, sizeof(int) * jobs.size(),
                                cudaMemcpyDeviceToHost, ctx.stream));
        LH_CUDA(cudaStreamSynchronize(ctx.stream));
        cudaFree(djobs);
        cudaFree(dcnt);
        for (size_t k = 0; k < jobs.size(); ++k) {
            const Node &nd = H.nodes[lr[p + k]];
            if (flags[k] == 2) to_dense.push_back(lr[p + k]);
            else if (flags[k] == 3)
                throw Error(LH_ERANK, "recompressed rank exceeds kcap=" + std::to_string(kcap) +
                                          " for block (" + std::to_string(nd.r0) + "," +
                                          std::to_string(nd.c0) + "," + std::to_string(nd.m) + "x" +
                                          std::to_string(nd.n) + ")");
            else if (flags[k] == 4)
                throw Error(LH_ERANK, "ACA did not converge within max_aca_rank=" +
                                          std::to_string(KA) + " for block (" +
                                          std::to_string(nd.r0) + "," + std::to_string(nd.c0) +
                                          "," + std::to_string(nd.m) + "x" + std::to_string(nd.n) +
                                          ")");
        }
        p = q;
    }
    if (work) cudaFree(work);
    return to_dense;
}

// blocks whose rank exceeds min(m,n)//2 are stored dense (hmatrix.py:301-302,331), appended
// in block order; then every dense leaf is filled from the entry source
template <class Src>
static void build_finalize(Ctx &ctx, HMat &H, Src src, std::vector<int32_t> to_dense) {
    std::sort(to_dense.begin(), to_dense.end());
    if (!to_dense.empty()) {
        i64 extra = 0;
        for (int32_t b : to_dense) extra += H.nodes[b].m * H.nodes[b].n;
        double *na = dalloc<double>(H.arena_len + extra);
        LH_CUDA(cudaMemcpyAsync(na, H.d_arena, sizeof(double) * H.arena_len, cudaMemcpyDeviceToDevice,
                                ctx.stream));
        LH_CUDA(cudaStreamSynchronize(ctx.stream));
        cudaFree(H.d_arena);
        H.d_arena = na;
        i64 o = H.arena_len;
        for (int32_t b : to_dense) {
            Node &nd = H.nodes[b];
            nd.kind = K_DENSE;
            nd.doff = o;
            o += nd.m * nd.n;
            nd.uoff = nd.voff = -1;
        }
        H.arena_len += extra;
    }
    std::vector<FillJob> fj;
    for (int32_t b : H.leafblocks) {
        const Node &nd = H.nodes[b];
        if (nd.kind == K_DENSE) fj.push_back({nd.r0, nd.c0, nd.m, nd.n, nd.doff});
    }
    if (!fj.empty()) {
        FillJob *d = dupload(fj, ctx.stream);
        int grid = (int)std::min<size_t>(fj.size(), (size_t)ctx.num_sms * 16);
        dense_fill_kernel<Src><<<grid, NT, 0, ctx.stream>>>(src, d, (int)fj.size(), H.d_arena);
        LH_CUDA(cudaGetLastError());
        LH_CUDA(cudaStreamSynchronize(ctx.stream));
        cudaFree(d);
    }
    H.sync_ranks(ctx.stream);
}

template <class Src>
static void run_build(Ctx &ctx, HMat &H, Src src, const lh_hconfig &cfg) {
    std::vector<int32_t> lr = build_layout(ctx, H, cfg);
    std::vector<int32_t> to_dense = run_aca(ctx, H, src, cfg, lr);
    build_finalize(ctx, H, src, to_dense);
}

// ---------------------------------------------------------------------------
// sharded assembly: admissible blocks are independent, so rank q of W
// compresses its share (longest-processing-time assignment by m + n over the size-sorted
// list, identical on every rank), packs its factors, and after an all-gather every rank
// unpacks the others' blocks and finalizes (dense conversions + local dense fill).
// ---------------------------------------------------------------------------
struct ShardState {
    int rank = 0, world = 1;
    std::vector<std::vector<int32_t>> owned;  // per rank, its blocks in ACA order
    std::vector<int32_t> to_dense;            // dense conversions seen so far
    const double *t = nullptr;                // Toeplitz symbol (kept alive by the caller)
    std::vector<double> pack_meta;            // this rank's packed metadata (host)
};

static std::vector<std::vector<int32_t>> lpt_assign(const HMat &H, const std::vector<int32_t> &lr,
                                                    int world) {
    std::vector<std::vector<int32_t>> own(world);
    std::vector<i64> load(world, 0);
    for (int32_t b : lr) {  // lr is size-sorted, largest first
        int q = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        own[q].push_back(b);
        load[q] += H.nodes[b].m + H.nodes[b].n;
    }
    return own;
}

void build_toeplitz_shard(Ctx &ctx, HMat &H, const double *t, const lh_hconfig &cfg, int rank,
                          int world) {
    LH_REQUIRE(world >= 1 && rank >= 0 && rank < world, LH_EINVAL, "invalid shard rank/world");
    std::vector<int32_t> lr = build_layout(ctx, H, cfg);
    auto st = std::make_shared<ShardState>();
    st->rank = rank;
    st->world = world;
    st->t = t;
    st->owned = lpt_assign(H, lr, world);
    ToepSrc s{t, H.nrows};
    st->to_dense = run_aca(ctx, H, s, cfg, st->owned[rank]);
    H.sync_ranks(ctx.stream);
    H.shard = st;
}

static ShardState &shard_of(HMat &H) {
    LH_REQUIRE(H.shard != nullptr, LH_EINVAL, "H-matrix is not a pending sharded build");
    return *static_cast<ShardState *>(H.shard.get());
}

struct GatherJob {
    i64 a, b;  // arena offset, packed offset
    i64 rows;
    int32_t cols, dir;  // dir 0: arena -> packed, 1: packed -> arena (ld = rows both sides)
};

__global__ void shard_copy_kernel(const GatherJob *jobs, int njobs, double *arena, double *packed) {
    for (int j = blockIdx.x; j < njobs; j += gridDim.x) {
        const GatherJob J = jobs[j];
        const i64 n = J.rows * J.cols;
        for (i64 e = threadIdx.x; e < n; e += NT) {
            if (J.dir == 0) packed[J.b + e] = arena[J.a + e];
            else arena[J.a + e] = packed[J.b + e];
        }
    }
}

static void run_jobs(Ctx &ctx, const std::vector<GatherJob> &jobs, double *arena, double *packed) {
    if (jobs.empty()) return;
    GatherJob *d = dupload(jobs, ctx.stream);
    int grid = (int)std::min<size_t>(jobs.size(), (size_t)ctx.num_sms * 16);
    shard_copy_kernel<<<grid, NT, 0, ctx.stream>>>(d, (int)jobs.size(), arena, packed);
    LH_CUDA(cudaGetLastError());
    LH_CUDA(cudaStreamSynchronize(ctx.stream));
    cudaFree(d);
}

// packed layout of rank q's share: [count][per block: rank, or -1 if stored dense] then
// U (m x r) and V (n x r) of every low-rank block, in the owner's ACA order
i64 shard_pack(Ctx &ctx, HMat &H, double *buf, i64 cap) {
    ShardState &st = shard_of(H);
    const auto &own = st.owned[st.rank];
    std::vector<char> dense(H.nodes.size(), 0);
    for (int32_t b : st.to_dense) dense[b] = 1;
    const i64 nmeta = 1 + (i64)own.size();
    i64 len = nmeta;
    for (int32_t b : own) {
        const Node &nd = H.nodes[b];
        if (!dense[b]) len += (nd.m + nd.n) * H.h_ranks[nd.rslot];
    }
    if (!buf) return len;
    LH_REQUIRE(cap >= len, LH_EINVAL, "shard pack buffer too small");
    std::vector<double> meta(nmeta);
    meta[0] = (double)own.size();
    std::vector<GatherJob> jobs;
    i64 o = nmeta;
    for (size_t k = 0; k < own.size(); ++k) {
        const Node &nd = H.nodes[own[k]];
        if (dense[own[k]]) {
            meta[1 + k] = -1.0;
            continue;
        }
        const int r = H.h_ranks[nd.rslot];
        meta[1 + k] = (double)r;
        jobs.push_back({nd.uoff, o, nd.m, r, 0});
        o += nd.m * r;
        jobs.push_back({nd.voff, o, nd.n, r, 0});
        o += nd.n * r;
    }
    LH_CUDA(cudaMemcpyAsync(buf, meta.data(), sizeof(double) * nmeta, cudaMemcpyHostToDevice, ctx.stream));
    run_jobs(ctx, jobs, H.d_arena, buf);
    return len;
}

void shard_unpack(Ctx &ctx, HMat &H, int src_rank, const double *buf, i64 len) {
    ShardState &st = shard_of(H);
    LH_REQUIRE(src_rank >= 0 && src_rank < st.world, LH_EINVAL, "invalid source rank");
    if (src_rank == st.rank) return;
    const auto &own = st.owned[src_rank];
    const i64 nmeta = 1 + (i64)own.size();
    LH_REQUIRE(len >= nmeta, LH_EINVAL, "shard buffer shorter than its metadata");
    std::vector<double> meta(nmeta);
    LH_CUDA(cudaMemcpyAsync(meta.data(), buf, sizeof(double) * nmeta, cudaMemcpyDeviceToHost, ctx.stream));
    LH_CUDA(cudaStreamSynchronize(ctx.stream));
    LH_REQUIRE((i64)meta[0] == (i64)own.size(), LH_EINVAL, "shard buffer from a different partition");
    std::vector<GatherJob> jobs;
    std::vector<int32_t> rk_slot, rk_val;
    i64 o = nmeta;
    for (size_t k = 0; k < own.size(); ++k) {
        const Node &nd = H.nodes[own[k]];
        const int r = (int)meta[1 + k];
        if (r < 0) {
            st.to_dense.push_back(own[k]);
            continue;
        }
        H.h_ranks[nd.rslot] = r;
        jobs.push_back({nd.uoff, o, nd.m, r, 1});
        o += nd.m * r;
        jobs.push_back({nd.voff, o, nd.n, r, 1});
        o += nd.n * r;
    }
    LH_REQUIRE(o <= len, LH_EINVAL, "shard buffer shorter than its factors");
    run_jobs(ctx, jobs, H.d_arena, const_cast<double *>(buf));
    LH_CUDA(cudaMemcpyAsync(H.d_ranks, H.h_ranks.data(), sizeof(int32_t) * H.nslots,
                            cudaMemcpyHostToDevice, ctx.stream));
    LH_CUDA(cudaStreamSynchronize(ctx.stream));
}

void shard_finalize(Ctx &ctx, HMat &H) {
    ShardState &st = shard_of(H);
    ToepSrc s{st.t, H.nrows};
    std::vector<int32_t> td = st.to_dense;
    H.shard.reset();
    build_finalize(ctx, H, s, td);
}

// ---------------------------------------------------------------------------
// sharded assembly over the context's NCCL communicator, with the
// exchange overlapped with the compression: every rank's share is cut into `stages` parts
// (identically on every rank); while stage s + 1 compresses on the context's stream, stage s's
// packed factors are all-gathered on the communication stream (lengths first, then one padded
// all-gather).  stats: compress s, host wait for the exchange s, finalize s, bytes sent, received.
// ---------------------------------------------------------------------------
static i64 pack_list(Ctx &ctx, HMat &H, const std::vector<int32_t> &blocks, const std::vector<char> &dense,
                     double *buf, cudaStream_t s) {
    const i64 nmeta = 1 + (i64)blocks.size();
    std::vector<double> meta(nmeta);
    meta[0] = (double)blocks.size();
    std::vector<GatherJob> jobs;
    i64 o = nmeta;
    for (size_t k = 0; k < blocks.size(); ++k) {
        const Node &nd = H.nodes[blocks[k]];
        if (dense[blocks[k]]) {
            meta[1 + k] = -1.0;
            continue;
        }
        const int r = H.h_ranks[nd.rslot];
        meta[1 + k] = (double)r;
        jobs.push_back({nd.uoff, o, nd.m, r, 0});
        o += nd.m * r;
        jobs.push_back({nd.voff, o, nd.n, r, 0});
        o += nd.n * r;
    }
    if (buf) {
        LH_CUDA(cudaMemcpyAsync(buf, meta.data(), sizeof(double) * nmeta, cudaMemcpyHostToDevice, s));
        if (!jobs.empty()) {
            GatherJob *d = dupload(jobs, s);
            int grid = (int)std::min<size_t>(jobs.size(), (size_t)ctx.num_sms * 16);
            shard_copy_kernel<<<grid, NT, 0, s>>>(d, (int)jobs.size(), H.d_arena, buf);
            LH_CUDA(cudaGetLastError());
            LH_CUDA(cudaStreamSynchronize(s));
            cudaFree(d);
        }
        LH_CUDA(cudaStreamSynchronize(s));
    }
    return o;
}

void build_toeplitz_nccl(Ctx &ctx, HMat &H, const double *t, const lh_hconfig &cfg, int stages, double *stats) {
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
    const int rank = nccl_rank(ctx), world = nccl_world(ctx);
    cudaStream_t cs = nccl_stream(ctx);
    stages = std::max(1, stages);
    std::vector<int32_t> lr = build_layout(ctx, H, cfg);
    const auto owned = lpt_assign(H, lr, world);
    auto part = [&](int q, int sidx) {  // stage sidx of rank q's share (in its ACA order)
        const auto &o = owned[q];
        const size_t a = o.size() * sidx / stages, b = o.size() * (sidx + 1) / stages;
        return std::vector<int32_t>(o.begin() + a, o.begin() + b);
    };
    auto cap_of = [&](int q, int sidx) {  // upper bound of a packed stage (capacity columns)
        i64 c = 1;
        for (int32_t b : part(q, sidx)) c += 1 + (H.nodes[b].m + H.nodes[b].n) * H.nodes[b].kcap;
        return c;
    };
    ToepSrc src{t, H.nrows};
    std::vector<char> dense(H.nodes.size(), 0);
    std::vector<int32_t> to_dense;
    struct Stage {
        double *send = nullptr, *recv = nullptr;
        int64_t *dlen = nullptr;
        std::vector<int64_t> lens;
        i64 maxlen = 0;
        cudaEvent_t packed = nullptr;
    };
    std::vector<Stage> stg(stages);
    double t_aca = 0, t_wait = 0, sent = 0, recvd = 0;
    auto cleanup = [&]() {
        for (Stage &S : stg) {
            if (S.send) cudaFree(S.send);
            if (S.recv) cudaFree(S.recv);
            if (S.dlen) cudaFree(S.dlen);
            if (S.packed) cudaEventDestroy(S.packed);
        }
    };
    try {
        for (int sidx = 0; sidx < stages; ++sidx) {
            Stage &S = stg[sidx];
            auto t0 = now();
            const std::vector<int32_t> mine = part(rank, sidx);
            std::vector<int32_t> td = run_aca(ctx, H, src, cfg, mine);
            H.sync_ranks(ctx.stream);
            t_aca += sec(t0, now());
            for (int32_t b : td) {
                dense[b] = 1;
                to_dense.push_back(b);
            }
            i64 bound = 0;
            for (int q = 0; q < world; ++q) bound = std::max(bound, cap_of(q, sidx));
            S.send = dalloc<double>(bound);
            S.dlen = dalloc<int64_t>(2 * (i64)world + 1);
            const i64 len = pack_list(ctx, H, mine, dense, S.send, ctx.stream);
            sent += 8.0 * len;
            LH_CUDA(cudaEventCreateWithFlags(&S.packed, cudaEventDisableTiming));
            LH_CUDA(cudaEventRecord(S.packed, ctx.stream));
            // lengths on the communication stream (it first finishes the previous stage's payload)
            auto tw = now();
            LH_CUDA(cudaStreamWaitEvent(cs, S.packed, 0));
            const int64_t mylen = len;
            LH_CUDA(cudaMemcpyAsync(S.dlen + world, &mylen, sizeof(int64_t), cudaMemcpyHostToDevice, cs));
            nccl_allgather_i64(ctx, S.dlen + world, S.dlen, 1, cs);
            S.lens.assign(world, 0);
            LH_CUDA(cudaMemcpyAsync(S.lens.data(), S.dlen, sizeof(int64_t) * world, cudaMemcpyDeviceToHost, cs));
            LH_CUDA(cudaStreamSynchronize(cs));
            t_wait += sec(tw, now());
            for (int64_t v : S.lens) S.maxlen = std::max<i64>(S.maxlen, v);
            LH_REQUIRE(S.maxlen <= bound, LH_EINTERNAL, "packed stage above its capacity bound");
            S.recv = dalloc<double>((i64)world * S.maxlen);
            nccl_allgather_f64(ctx, S.send, S.recv, (size_t)S.maxlen, cs);  // overlaps the next stage
        }
        auto tw = now();
        LH_CUDA(cudaStreamSynchronize(cs));
        t_wait += sec(tw, now());
        auto tf = now();
        // unpack every other rank's stages (their factors, ranks and dense decisions)
        for (int sidx = 0; sidx < stages; ++sidx) {
            Stage &S = stg[sidx];
            for (int q = 0; q < world; ++q) {
                recvd += 8.0 * S.lens[q];
                if (q == rank) continue;
                const std::vector<int32_t> theirs = part(q, sidx);
                const double *buf = S.recv + (i64)q * S.maxlen;
                const i64 nmeta = 1 + (i64)theirs.size();
                std::vector<double> meta(nmeta);
                LH_CUDA(cudaMemcpyAsync(meta.data(), buf, sizeof(double) * nmeta, cudaMemcpyDeviceToHost,
                                        ctx.stream));
                LH_CUDA(cudaStreamSynchronize(ctx.stream));
                LH_REQUIRE((i64)meta[0] == (i64)theirs.size(), LH_EINTERNAL, "stage from a different partition");
                std::vector<GatherJob> jobs;
                i64 o = nmeta;
                for (size_t k = 0; k < theirs.size(); ++k) {
                    const Node &nd = H.nodes[theirs[k]];
                    const int r = (int)meta[1 + k];
                    if (r < 0) {
                        to_dense.push_back(theirs[k]);
                        continue;
                    }
                    H.h_ranks[nd.rslot] = r;
                    jobs.push_back({nd.uoff, o, nd.m, r, 1});
                    o += nd.m * r;
                    jobs.push_back({nd.voff, o, nd.n, r, 1});
                    o += nd.n * r;
                }
                LH_REQUIRE(o <= S.lens[q], LH_EINTERNAL, "stage shorter than its factors");
                run_jobs(ctx, jobs, H.d_arena, const_cast<double *>(buf));
            }
        }
        LH_CUDA(cudaMemcpyAsync(H.d_ranks, H.h_ranks.data(), sizeof(int32_t) * H.nslots, cudaMemcpyHostToDevice,
                                ctx.stream));
        LH_CUDA(cudaStreamSynchronize(ctx.stream));
        cleanup();
        build_finalize(ctx, H, src, to_dense);
        if (stats) {
            stats[0] = t_aca;
            stats[1] = t_wait;
            stats[2] = sec(tf, now());
            stats[3] = sent;
            stats[4] = recvd;
        }
    } catch (...) {
        cleanup();
        throw;
    }
}

void build_toeplitz(Ctx &ctx, HMat &H, const double *t, const lh_hconfig &cfg) {
    ToepSrc s{t, H.nrows};
    run_build(ctx, H, s, cfg);
}

void build_dense(Ctx &ctx, HMat &H, const double *A, i64 lda, int row_major, const lh_hconfig &cfg) {
    DenseSrc s{A, lda, row_major};
    run_build(ctx, H, s, cfg);
}

// ===========================================================================
// series builder (hmatrix.py:243-291 build_from_expansion with the Gaussian family of
// gaussian_expansion_1d, :156-186): every admissible block with min(m, n) > n_min is
// low-rank with n_terms analytic columns around the ROW cluster centre c,
//   U[i, k] = scale (2 eps_sq s_i)^k e^{-eps_sq s_i^2} / k!   (s_i = x_i - c)
//   V[j, k] = t_j^k e^{-eps_sq t_j^2}                         (t_j = y_j - c)
// by the reference's column recurrence (col_k = col_{k-1} * base / k), one thread per
// row, one CTA per block; no dense fallback (the series rank is kept as is).
// ===========================================================================
struct SeriesJob {
    i64 r0, c0, m, n, uoff, voff;
    double centre;
    int32_t K, slot;
};

__global__ void series_kernel(const SeriesJob *jobs, int njobs, const double *xr, const double *yc,
                              double eps_sq, double scale, double *arena, int32_t *ranks) {
    for (int b = blockIdx.x; b < njobs; b += gridDim.x) {
        const SeriesJob J = jobs[b];
        for (i64 e = threadIdx.x; e < J.m + J.n; e += NT) {
            const bool row = e < J.m;
            const double t = row ? xr[J.r0 + e] - J.centre : yc[J.c0 + e - J.m] - J.centre;
            double *out = row ? arena + J.uoff + e : arena + J.voff + (e - J.m);
            const i64 ld = row ? J.m : J.n;
            double v = (row ? scale : 1.0) * exp(-eps_sq * t * t);
            const double base = row ? 2.0 * eps_sq * t : t;
            out[0] = v;
            for (int k = 1; k < J.K; ++k) {
                v = row ? v * base / (double)k : v * base;
                out[(i64)k * ld] = v;
            }
        }
        if (threadIdx.x == 0) ranks[J.slot] = J.K;
    }
}

// hmatrix.py:270-281 (rank_bound_gaussian) and :284-290 (_expansion_terms)
int gauss_series_terms(double eps_sq, double D, int fixed_rank, double delta) {
    if (!(delta > 0.0)) return fixed_rank;
    if (D <= 0.0) return 1;
    const double eps = std::sqrt(eps_sq);
    const double e2 = 2.0 * eps * eps * D * D;
    const double bound = std::max(e2 / std::log(2.0) - std::log2(delta) - 1.0, 6.0 * e2 - 1.0);
    return std::max(0, (int)std::floor(bound) + 1) + 1;
}

void build_gauss_series(Ctx &ctx, HMat &H, const double *t, const double *xr, const double *yc,
                        double eps_sq, double scale, int fixed_rank, double delta,
                        const lh_hconfig &cfg) {
    LH_REQUIRE(eps_sq > 0, LH_EINVAL, "series builder needs eps_sq > 0");
    LH_REQUIRE(delta > 0 || fixed_rank >= 1, LH_EINVAL, "fixed_rank must be >= 1");
    LH_REQUIRE(H.rt->dim == 1 && H.ct->dim == 1, LH_EINVAL, "the device series builder is 1D");
    // per-block series rank; blocks whose rank exceeds KC_MAX / 2 get the full recompression
    // width (rank + an H-LU update of up to the same order) as capacity
    std::vector<int32_t> terms(H.nodes.size(), 0), cap(H.nodes.size(), 0);
    for (int32_t b : H.leafblocks) {
        const Node &nd = H.nodes[b];
        if (nd.kind != K_LR) continue;
        terms[b] = gauss_series_terms(eps_sq, diameter(H.rt->nodes[nd.rcl], 1), fixed_rank, delta);
        cap[b] = 2 * terms[b] > KC_MAX ? KA_MAX : 0;
    }
    std::vector<int32_t> lr = build_layout(ctx, H, cfg, &cap);
    std::vector<SeriesJob> jobs;
    jobs.reserve(lr.size());
    for (int32_t b : lr) {
        const Node &nd = H.nodes[b];
        const Cluster &rc = H.rt->nodes[nd.rcl];
        const int K = terms[b];
        if (K > KC_MAX)
            throw Error(LH_ERANK, "series rank " + std::to_string(K) + " exceeds the stored-rank limit " +
                                      std::to_string(KC_MAX) + " for block (" +
                                      std::to_string(nd.r0) + "," + std::to_string(nd.c0) + "," +
                                      std::to_string(nd.m) + "x" + std::to_string(nd.n) + ")");
        jobs.push_back({nd.r0, nd.c0, nd.m, nd.n, nd.uoff, nd.voff, 0.5 * (rc.blo[0] + rc.bhi[0]), K,
                        nd.rslot});
    }
    if (!jobs.empty()) {
        SeriesJob *d = dupload(jobs, ctx.stream);
        const int grid = (int)std::min<size_t>(jobs.size(), (size_t)ctx.num_sms * 16);
        series_kernel<<<grid, NT, 0, ctx.stream>>>(d, (int)jobs.size(), xr, yc, eps_sq, scale,
                                                   H.d_arena, H.d_ranks);
        LH_CUDA(cudaGetLastError());
        LH_CUDA(cudaStreamSynchronize(ctx.stream));
        cudaFree(d);
    }
    if (t) build_finalize(ctx, H, ToepSrc{t, H.nrows}, {});
    else build_finalize(ctx, H, GaussSrc{xr, yc, eps_sq, scale}, {});
}

// 2D: gaussian_expansion_2d (hmatrix.py:189-216): the factor families are tensor products of the
// 1D ones, column a T + b = col_a(first coordinate) * col_b(second coordinate), T terms per
// dimension, block rank T^2; U's first-coordinate family carries `scale`.  Points are n x 2
// row-major device arrays in tree order; the centre is the row cluster's box centre.
constexpr int SERIES2D_TMAX = 5;  // T^2 <= KC_MAX
static_assert(SERIES2D_TMAX * SERIES2D_TMAX <= KC_MAX && (SERIES2D_TMAX + 1) * (SERIES2D_TMAX + 1) > KC_MAX,
              "2D series terms per dimension follow the stored-rank limit");
struct SeriesJob2 {
    i64 r0, c0, m, n, uoff, voff;
    double cx, cy;
    int32_t T, slot;
};

__global__ void series2d_kernel(const SeriesJob2 *jobs, int njobs, const double *xr, const double *yc,
                                double eps_sq, double scale, double *arena, int32_t *ranks) {
    for (int b = blockIdx.x; b < njobs; b += gridDim.x) {
        const SeriesJob2 J = jobs[b];
        for (i64 e = threadIdx.x; e < J.m + J.n; e += NT) {
            const bool row = e < J.m;
            const double *p = row ? xr + 2 * (J.r0 + e) : yc + 2 * (J.c0 + e - J.m);
            const double t0 = p[0] - J.cx, t1 = p[1] - J.cy;
            double *out = row ? arena + J.uoff + e : arena + J.voff + (e - J.m);
            const i64 ld = row ? J.m : J.n;
            double a1[SERIES2D_TMAX], a2[SERIES2D_TMAX];
            a1[0] = (row ? scale : 1.0) * exp(-eps_sq * t0 * t0);
            a2[0] = 1.0 * exp(-eps_sq * t1 * t1);
            const double b0 = row ? 2.0 * eps_sq * t0 : t0, b1 = row ? 2.0 * eps_sq * t1 : t1;
#pragma unroll
            for (int k = 1; k < SERIES2D_TMAX; ++k) {
                a1[k] = row ? a1[k - 1] * b0 / (double)k : a1[k - 1] * b0;
                a2[k] = row ? a2[k - 1] * b1 / (double)k : a2[k - 1] * b1;
            }
#pragma unroll
            for (int a = 0; a < SERIES2D_TMAX; ++a)
#pragma unroll
                for (int c = 0; c < SERIES2D_TMAX; ++c)
                    if (a < J.T && c < J.T) out[(i64)(a * J.T + c) * ld] = a1[a] * a2[c];
        }
        if (threadIdx.x == 0) ranks[J.slot] = J.T * J.T;
    }
}

void build_gauss_series_2d(Ctx &ctx, HMat &H, const double *xr, const double *yc, double eps_sq, double scale,
                           int fixed_rank, double delta, const lh_hconfig &cfg, const lh_cn2d_entries *ent) {
    LH_REQUIRE(eps_sq > 0, LH_EINVAL, "series builder needs eps_sq > 0");
    LH_REQUIRE(delta > 0 || fixed_rank >= 1, LH_EINVAL, "fixed_rank must be >= 1");
    LH_REQUIRE(H.rt->dim == 2 && H.ct->dim == 2, LH_EINVAL, "the 2D series builder needs 2D cluster trees");
    std::vector<int32_t> terms(H.nodes.size(), 0), cap(H.nodes.size(), 0);
    for (int32_t b : H.leafblocks) {
        const Node &nd = H.nodes[b];
        if (nd.kind != K_LR) continue;
        const int T = gauss_series_terms(eps_sq, diameter(H.rt->nodes[nd.rcl], 2), fixed_rank, delta);
        if (T > SERIES2D_TMAX)
            throw Error(LH_ERANK, "2D series rank " + std::to_string(T) + "^2 exceeds the stored-rank limit " +
                                      std::to_string(KC_MAX) + " for block (" + std::to_string(nd.r0) + "," +
                                      std::to_string(nd.c0) + "," + std::to_string(nd.m) + "x" +
                                      std::to_string(nd.n) + "): use at most " + std::to_string(SERIES2D_TMAX) +
                                      " terms per dimension, or build_from_dense");
        terms[b] = T;
        cap[b] = 2 * T * T > KC_MAX ? KA_MAX : 0;
    }
    std::vector<int32_t> lr = build_layout(ctx, H, cfg, &cap);
    std::vector<SeriesJob2> jobs;
    jobs.reserve(lr.size());
    for (int32_t b : lr) {
        const Node &nd = H.nodes[b];
        const Cluster &rc = H.rt->nodes[nd.rcl];
        jobs.push_back({nd.r0, nd.c0, nd.m, nd.n, nd.uoff, nd.voff, 0.5 * (rc.blo[0] + rc.bhi[0]),
                        0.5 * (rc.blo[1] + rc.bhi[1]), terms[b], nd.rslot});
    }
    if (!jobs.empty()) {
        SeriesJob2 *d = dupload(jobs, ctx.stream);
        const int grid = (int)std::min<size_t>(jobs.size(), (size_t)ctx.num_sms * 16);
        series2d_kernel<<<grid, NT, 0, ctx.stream>>>(d, (int)jobs.size(), xr, yc, eps_sq, scale, H.d_arena,
                                                     H.d_ranks);
        LH_CUDA(cudaGetLastError());
        LH_CUDA(cudaStreamSynchronize(ctx.stream));
        cudaFree(d);
    }
    if (ent) {
        LH_REQUIRE(ent->which >= 0 && ent->which <= 2, LH_EINVAL, "which must be 0 (A), 1 (plus) or 2 (minus)");
        LH_REQUIRE(ent->nx > 0 && H.nrows % ent->nx == 0 && H.nrows == H.ncols && ent->order_dev, LH_EINVAL,
                   "entry source: square operator on an nx x (N / nx) grid with its tree order");
        build_finalize(ctx, H,
                       Cn2dSrc{ent->order_dev, ent->nx, ent->which, ent->h, ent->eps_sq, ent->scale, ent->a,
                               ent->b, ent->c, ent->lam, 0.5 * ent->dt},
                       {});
    } else {
        build_finalize(ctx, H, Gauss2Src{xr, yc, eps_sq, scale}, {});
    }
}

// ===========================================================================
// derive: same partition/ranks, U scaled, dense refilled from a symbol
// ===========================================================================
struct CopyLrJob {
    i64 su, sv, du, dv, m, n;
    int32_t slot;
};

__global__ void copy_lr_kernel(const CopyLrJob *jobs, int njobs, const double *src, double *dst,
                               const int *ranks, double scale) {
    for (int b = blockIdx.x; b < njobs; b += gridDim.x) {
        CopyLrJob J = jobs[b];
        int r = ranks[J.slot];
        for (i64 e = threadIdx.x; e < J.m * r; e += NT) {
            i64 i = e % J.m, c = e / J.m;
            dst[J.du + i + c * J.m] = scale * src[J.su + i + c * J.m];
        }
        for (i64 e = threadIdx.x; e < J.n * r; e += NT) {
            i64 i = e % J.n, c = e / J.n;
            dst[J.dv + i + c * J.n] = src[J.sv + i + c * J.n];
        }
    }
}

__global__ void copy_dense_kernel(const FillJob *jobs, int njobs, const double *src, double *dst,
                                  const i64 *src_off) {
    for (int b = blockIdx.x; b < njobs; b += gridDim.x) {
        FillJob J = jobs[b];
        for (i64 e = threadIdx.x; e < J.m * J.n; e += NT) dst[J.off + e] = src[src_off[b] + e];
    }
}

// 64-bit tag unique across processes with overwhelming probability (checkpoints carry it)
static uint64_t fresh_pair_tag() {
    static std::atomic<uint64_t> ctr{0};
    uint64_t z = (uint64_t)std::chrono::steady_clock::now().time_since_epoch().count() ^
                 ((uint64_t)getpid() << 32) ^ (0x9E3779B97F4A7C15ull * (ctr.fetch_add(1) + 1));
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z ? z : 1;
}

// Counts dense entries of D that are not those of 2I - S: exact negatives off the diagonal,
// 2 - s within 8 ulp of 2 on it (1 +- dt/2 a_ii rounded separately).
__global__ void pair_check_kernel(const FillJob *jobs, int njobs, const double *src,
                                  const i64 *src_off, const double *dst, unsigned long long *bad) {
    for (int b = blockIdx.x; b < njobs; b += gridDim.x) {
        FillJob J = jobs[b];
        unsigned long long nb = 0;
        for (i64 e = threadIdx.x; e < J.m * J.n; e += NT) {
            const i64 i = e % J.m, j = e / J.m;
            const double sv = src[src_off[b] + e], dv = dst[J.off + e];
            if (J.r0 + i == J.c0 + j) nb += !(fabs(dv - (2.0 - sv)) <= 8.0 * 2.220446049250313e-16 * 2.0);
            else nb += !(dv == -sv);
        }
        if (nb) atomicAdd(bad, nb);
    }
}

// Copy of `S` with LR capacity kcap (<= 0: tight = rank), LR U scaled by `scale`.
// If t != nullptr dense blocks are refilled from the Toeplitz symbol, else copied.
void derive(Ctx &ctx, const HMat &S, HMat &D, const double *t, double scale, int kcap) {
    LH_REQUIRE(!S.factored, LH_EINVAL, "cannot derive from a factored H-matrix");
    D.cn_pair_tag = 0;
    D.pair_tag = 0;
    D.rt = S.rt;
    D.ct = S.ct;
    D.rt_hold = S.rt_hold;
    D.ct_hold = S.ct_hold;
    D.nrows = S.nrows;
    D.ncols = S.ncols;
    D.root = S.root;
    D.nodes = S.nodes;
    D.leafblocks = S.leafblocks;
    D.nslots = S.nslots;
    D.h_ranks = S.h_ranks;
    i64 off = 0;
    for (int32_t b : D.leafblocks) {
        Node &nd = D.nodes[b];
        if (nd.kind == K_DENSE) {
            nd.doff = off;
            off += nd.m * nd.n;
        }
    }
    std::vector<CopyLrJob> lj;
    for (int32_t b : D.leafblocks) {
        Node &nd = D.nodes[b];
        if (nd.kind == K_LR) {
            int r = S.h_ranks[nd.rslot];
            nd.kcap = kcap > 0 ? std::max(kcap, r) : r;
            LH_REQUIRE(nd.kcap <= KC_MAX, LH_ERANK, "kcap exceeds the compile-time maximum");
            nd.uoff = off;
            off += nd.m * nd.kcap;
            nd.voff = off;
            off += nd.n * nd.kcap;
            const Node &sn = S.nodes[b];
            lj.push_back({sn.uoff, sn.voff, nd.uoff, nd.voff, nd.m, nd.n, nd.rslot});
        }
    }
    D.arena_len = off;
    D.d_arena = dalloc<double>(off);
    D.d_ranks = dalloc<int32_t>(std::max(D.nslots, 1));
    LH_CUDA(cudaMemcpyAsync(D.d_ranks, S.d_ranks, sizeof(int32_t) * std::max(D.nslots, 1),
                            cudaMemcpyDeviceToDevice, ctx.stream));
    if (!lj.empty()) {
        CopyLrJob *d = dupload(lj, ctx.stream);
        int grid = (int)std::min<size_t>(lj.size(), (size_t)ctx.num_sms * 16);
        copy_lr_kernel<<<grid, NT, 0, ctx.stream>>>(d, (int)lj.size(), S.d_arena, D.d_arena,
                                                    D.d_ranks, scale);
        LH_CUDA(cudaGetLastError());
        LH_CUDA(cudaStreamSynchronize(ctx.stream));
        cudaFree(d);
    }
    std::vector<FillJob> fj;
    std::vector<i64> so;
    for (int32_t b : D.leafblocks) {
        const Node &nd = D.nodes[b];
        if (nd.kind == K_DENSE) {
            fj.push_back({nd.r0, nd.c0, nd.m, nd.n, nd.doff});
            so.push_back(S.nodes[b].doff);
        }
    }
    if (!fj.empty()) {
        FillJob *d = dupload(fj, ctx.stream);
        int grid = (int)std::min<size_t>(fj.size(), (size_t)ctx.num_sms * 16);
        if (t) {
            ToepSrc s{t, D.nrows};
            dense_fill_kernel<ToepSrc><<<grid, NT, 0, ctx.stream>>>(s, d, (int)fj.size(), D.d_arena);
            if (scale == -1.0) {
                // CN pair provenance (lh_cn_steps: u <- 2 Z u - u is exact only for A- = 2I - A+):
                // the low-rank blocks are (-U, V) by construction; check every dense entry
                i64 *dso = dupload(so, ctx.stream);
                unsigned long long *bad = dalloc<unsigned long long>(1);
                LH_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), ctx.stream));
                pair_check_kernel<<<grid, NT, 0, ctx.stream>>>(d, (int)fj.size(), S.d_arena, dso,
                                                               D.d_arena, bad);
                LH_CUDA(cudaGetLastError());
                unsigned long long nbad = 1;
                LH_CUDA(cudaMemcpyAsync(&nbad, bad, sizeof(nbad), cudaMemcpyDeviceToHost, ctx.stream));
                LH_CUDA(cudaStreamSynchronize(ctx.stream));
                cudaFree(bad);
                cudaFree(dso);
                if (nbad == 0) {
                    if (!S.pair_tag) S.pair_tag = fresh_pair_tag();
                    D.cn_pair_tag = S.pair_tag;
                }
            }
        } else {
            i64 *dso = dupload(so, ctx.stream);
            copy_dense_kernel<<<grid, NT, 0, ctx.stream>>>(d, (int)fj.size(), S.d_arena, D.d_arena, dso);
            LH_CUDA(cudaStreamSynchronize(ctx.stream));
            cudaFree(dso);
        }
        LH_CUDA(cudaGetLastError());
        LH_CUDA(cudaStreamSynchronize(ctx.stream));
        cudaFree(d);
    }
}

}  // namespace lh

// ===========================================================================
// Near-field compression of a computed H-matrix (the propagator Z = (LU)^-1):
// every dense leaf off the diagonal whose numerical rank at `eps` (Frobenius tail relative to
// the block, the hops.py:124-131 rule) is small is converted to a low-rank leaf in place
// (U then V inside the leaf's own m x n storage).  The block structure of the reference
// partition is kept; only the leaf's representation changes.  One CTA per block: ACA with
// partial pivoting on the stored entries, CGS2 QR of both factors, Jacobi SVD, truncation.
// ===========================================================================
namespace lh {
namespace {

struct NfJob {
    i64 m, n, doff, wu, wv;
};

__global__ void __launch_bounds__(NT) nf_compress_kernel(const NfJob *jobs, int njobs, int *counter,
                                                         double *work, double *arena, int *ranks_out,
                                                         int KA, double aca_tol, double eps) {
    extern __shared__ double4 smem_raw[];
    AcaSmem &S = *reinterpret_cast<AcaSmem *>(smem_raw);
    __shared__ int s_job;
    while (true) {
        if (threadIdx.x == 0) s_job = atomicAdd(counter, 1);
        __syncthreads();
        const int jb = s_job;
        __syncthreads();
        if (jb >= njobs) break;
        const NfJob J = jobs[jb];
        double *U = work + J.wu, *V = work + J.wv;
        double *D = arena + J.doff;
        DenseSrc src{D, J.m, 0};
        int conv = 0;
        const int K = aca_block(src, 0, 0, J.m, J.n, U, V, KA, aca_tol, S, conv);
        // keep only conversions that at least halve the storage
        const int rmax = (int)min((i64)KC_MAX, (J.m * J.n) / (2 * (J.m + J.n)));
        int r = conv ? dev::recompress(U, J.m, J.m, V, J.n, J.n, K, 1, eps, U, J.m, V, J.n, rmax, S.R)
                     : rmax + 1;
        const bool ok = conv && r <= rmax;
        if (ok) {  // every ACA read of D is done (recompress ends with a barrier)
            for (i64 e = threadIdx.x; e < J.m * r; e += NT) D[e] = U[e];
            for (i64 e = threadIdx.x; e < J.n * r; e += NT) D[J.m * r + e] = V[e];
        }
        if (threadIdx.x == 0) ranks_out[jb] = ok ? r : -1;
        __syncthreads();
    }
}

}  // namespace

// Returns the number of converted leaves.  Updates the node table and the rank slots; any
// matvec plan of H must be rebuilt afterwards.
i64 compress_near_field(Ctx &ctx, HMat &H, double eps) {
    std::vector<int32_t> cand;
    for (int32_t b : H.leafblocks) {
        const Node &nd = H.nodes[b];
        const bool off_diag = nd.r0 + nd.m <= nd.c0 || nd.c0 + nd.n <= nd.r0;
        if (nd.kind == K_DENSE && off_diag && nd.vpar < 0 && std::min(nd.m, nd.n) >= 16)
            cand.push_back(b);
    }
    if (cand.empty()) return 0;
    const int KA = KA_MAX;
    std::vector<NfJob> jobs;
    i64 w = 0;
    for (int32_t b : cand) {
        const Node &nd = H.nodes[b];
        jobs.push_back({nd.m, nd.n, nd.doff, w, w + nd.m * KA});
        w += (nd.m + nd.n) * KA;
    }
    double *work = dalloc<double>(w);
    NfJob *djobs = dupload(jobs, ctx.stream);
    int *dcnt = dalloc<int>(1 + (i64)jobs.size());
    int *dranks = dcnt + 1;
    LH_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(int), ctx.stream));
    const size_t smem = sizeof(AcaSmem);
    set_smem((const void *)nf_compress_kernel, smem);
    const int grid = (int)std::min<size_t>(jobs.size(), (size_t)ctx.num_sms * 2);
    nf_compress_kernel<<<grid, NT, smem, ctx.stream>>>(djobs, (int)jobs.size(), dcnt, work, H.d_arena,
                                                       dranks, KA, 0.1 * eps, eps);
    LH_CUDA(cudaGetLastError());
    std::vector<int> r(jobs.size());
    LH_CUDA(cudaMemcpyAsync(r.data(), dranks, sizeof(int) * r.size(), cudaMemcpyDeviceToHost, ctx.stream));
    LH_CUDA(cudaStreamSynchronize(ctx.stream));
    cudaFree(work);
    cudaFree(djobs);
    cudaFree(dcnt);
    // new rank slots for the converted leaves
    H.sync_ranks(ctx.stream);
    std::vector<int32_t> ranks = H.h_ranks;
    i64 nconv = 0;
    for (size_t k = 0; k < cand.size(); ++k) {
        if (r[k] < 0) continue;
        Node &nd = H.nodes[cand[k]];
        nd.kind = K_LR;
        nd.kcap = std::max(r[k], 1);
        nd.uoff = nd.doff;
        nd.voff = nd.doff + nd.m * r[k];
        nd.rslot = (int32_t)ranks.size();
        nd.doff = -1;
        for (int q = 0; q < 4; ++q) nd.kid[q] = -1;
        ranks.push_back(r[k]);
        ++nconv;
    }
    if (nconv) {
        int32_t *nr = dupload(ranks, ctx.stream);
        LH_CUDA(cudaStreamSynchronize(ctx.stream));
        cudaFree(H.d_ranks);
        H.d_ranks = nr;
        H.nslots = (int32_t)ranks.size();
        H.h_ranks = ranks;
    }
    return nconv;
}

}  // namespace lh

// ===========================================================================
// Coarsening of a computed H-matrix (the propagator Z): bottom-up, a 2 x 2
// hierarchical block off the diagonal whose four children are low-rank is replaced by one
// low-rank block when the recompressed sum of its children needs fewer scalars.  The
// embedded factors of the sum are block-structured (the U's of kids 11, 12 share the top
// rows, those of 21, 22 the bottom rows; the V's of 11, 21 the left columns, of 12, 22 the
// right ones), so their QR factorisations split into four independent half-height QRs
// (CGS2, one CTA each), the K x K core R_u R_v^T is formed from the four R's and
// SVD-truncated (Jacobi, the hops.py:124-131 Frobenius-tail rule at eps relative to the
// merged block) on one CTA, and the merged factors Q_side * coefficients are written
// row-parallel straight into the grown arena.
// ===========================================================================
namespace lh {
void walk_leaves(HMat &H);
namespace {

struct QrSide {        // [A | B]: rows x (ra + rb), from two kids' factors (ld = rows)
    i64 rows, srca, srcb, w;
    int32_t ra, rb;
};
struct CoreJob {       // merge k: sides 4k..4k+3 = top, bottom, left, right
    int32_t r11, r12, r21, r22;
    int32_t rmax, pad;
};
struct ApplyJob {      // out[row0 + i + c * ld] = sum_l Q[i + l * rows] * coef[coff + l + c * KA_MAX]
    i64 q, rows, out, ld, row0;
    int32_t K, r, coff, pad;
};

constexpr int QR_SMEM_D = KA_MAX * KA_MAX + KA_MAX + 2 * dev::NW;

__global__ void __launch_bounds__(NT) side_qr_kernel(const QrSide *sides, int nsides, int *counter,
                                                     const double *arena, double *work, double *Rout) {
    extern __shared__ double4 smem_raw[];
    double *R = reinterpret_cast<double *>(smem_raw);
    double *h = R + KA_MAX * KA_MAX;
    double *red = h + KA_MAX;
    __shared__ int s_job;
    while (true) {
        if (threadIdx.x == 0) s_job = atomicAdd(counter, 1);
        __syncthreads();
        const int jb = s_job;
        __syncthreads();
        if (jb >= nsides) break;
        const QrSide S = sides[jb];
        double *W = work + S.w;
        for (i64 e = threadIdx.x; e < S.rows * S.ra; e += NT) W[e] = arena[S.srca + e];
        for (i64 e = threadIdx.x; e < S.rows * S.rb; e += NT) W[S.rows * S.ra + e] = arena[S.srcb + e];
        __syncthreads();
        const int K = S.ra + S.rb;
        dev::cgs2(W, S.rows, S.rows, K, R, h, red);
        for (int e = threadIdx.x; e < KA_MAX * KA_MAX; e += NT)
            Rout[(i64)jb * KA_MAX * KA_MAX + e] = R[e];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(NT) core_kernel(const CoreJob *jobs, int njobs, int *counter,
                                                  const double *Rin, double *coef, int *ranks_out,
                                                  double eps) {
    extern __shared__ double4 smem_raw[];
    dev::RecompSmem &S = *reinterpret_cast<dev::RecompSmem *>(smem_raw);
    __shared__ int s_job;
    while (true) {
        if (threadIdx.x == 0) s_job = atomicAdd(counter, 1);
        __syncthreads();
        const int jb = s_job;
        __syncthreads();
        if (jb >= njobs) break;
        const CoreJob J = jobs[jb];
        const double *Rt = Rin + (i64)(4 * jb + 0) * KA_MAX * KA_MAX;
        const double *Rb = Rin + (i64)(4 * jb + 1) * KA_MAX * KA_MAX;
        const double *Rl = Rin + (i64)(4 * jb + 2) * KA_MAX * KA_MAX;
        const double *Rr = Rin + (i64)(4 * jb + 3) * KA_MAX * KA_MAX;
        const int Kt = J.r11 + J.r12, Kb = J.r21 + J.r22, Kl = J.r11 + J.r21, K = Kt + Kb;
        // R_u (K x K): diag(R_top, R_bot), columns ordered kids 11, 12, 21, 22
        // R_v (K x K): rows = left basis then right basis; columns 11, 12, 21, 22
        for (int e = threadIdx.x; e < KA_MAX * KA_MAX; e += NT) {
            S.Ru[e] = 0.0;
            S.Rv[e] = 0.0;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < K * K; e += NT) {
            const int i = e % K, j = e / K;
            if (i < Kt && j < Kt) S.Ru[i + j * KA_MAX] = Rt[i + j * KA_MAX];
            if (i >= Kt && j >= Kt) S.Ru[i + j * KA_MAX] = Rb[(i - Kt) + (j - Kt) * KA_MAX];
            // column j of V_big: kid and its column within the kid
            double v = 0.0;
            if (j < J.r11) {
                if (i < Kl) v = Rl[i + j * KA_MAX];
            } else if (j < Kt) {
                if (i >= Kl) v = Rr[(i - Kl) + (j - J.r11) * KA_MAX];
            } else if (j < Kt + J.r21) {
                if (i < Kl) v = Rl[i + (J.r11 + j - Kt) * KA_MAX];
            } else {
                if (i >= Kl) v = Rr[(i - Kl) + (J.r12 + j - Kt - J.r21) * KA_MAX];
            }
            S.Rv[i + j * KA_MAX] = v;
        }
        __syncthreads();
        // C = R_u R_v^T
        for (int e = threadIdx.x; e < K * K; e += NT) {
            const int i = e % K, j = e / K;
            double acc = 0.0;
            for (int l = 0; l < K; ++l) acc += S.Ru[i + l * KA_MAX] * S.Rv[j + l * KA_MAX];
            S.Cc[i + j * KA_MAX] = acc;
        }
        __syncthreads();
        dev::jacobi_svd(S.Cc, S.Rv, K, S.sigma, S.ord, S.red);
        const int r = dev::truncation_rank(S.sigma, S.ord, K, 1, eps);
        const bool ok = r <= J.rmax;
        if (ok) {  // coefficients: Cu[:, c] = (C Z)[:, ord[c]], Cv[:, c] = Z[:, ord[c]]
            double *cu = coef + (i64)(2 * jb) * KA_MAX * KC_MAX;
            double *cv = coef + (i64)(2 * jb + 1) * KA_MAX * KC_MAX;
            for (int e = threadIdx.x; e < K * r; e += NT) {
                const int l = e % K, c = e / K;
                cu[l + c * KA_MAX] = S.Cc[l + S.ord[c] * KA_MAX];
                cv[l + c * KA_MAX] = S.Rv[l + S.ord[c] * KA_MAX];
            }
        }
        if (threadIdx.x == 0) ranks_out[jb] = ok ? r : -1;
        __syncthreads();
    }
}

// row-parallel: one CTA per (job, 256-row tile), grid-stride over tiles
__global__ void __launch_bounds__(NT) apply_kernel(const ApplyJob *jobs, const i64 *tile0, int njobs,
                                                   i64 ntiles, const double *work, const double *coef,
                                                   double *arena) {
    for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int lo = 0, hi = njobs - 1;  // job of tile t: last j with tile0[j] <= t
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (tile0[mid] <= t) lo = mid;
            else hi = mid - 1;
        }
        const ApplyJob J = jobs[lo];
        const i64 i = (t - tile0[lo]) * NT + threadIdx.x;
        if (i >= J.rows) continue;
        const double *Q = work + J.q;
        const double *cf = coef + J.coff;
        double acc[KC_MAX];
#pragma unroll
        for (int c = 0; c < KC_MAX; ++c) acc[c] = 0.0;
        for (int l = 0; l < J.K; ++l) {
            const double q = Q[i + (i64)l * J.rows];
#pragma unroll
            for (int c = 0; c < KC_MAX; ++c)
                if (c < J.r) acc[c] += q * cf[l + c * KA_MAX];
        }
#pragma unroll
        for (int c = 0; c < KC_MAX; ++c)
            if (c < J.r) arena[J.out + J.row0 + i + (i64)c * J.ld] = acc[c];
    }
}

}  // namespace

i64 coarsen_hmat(Ctx &ctx, HMat &H, double eps) {
    std::vector<int> depth(H.nodes.size(), -1);
    std::vector<int32_t> st{H.root};
    depth[H.root] = 0;
    int maxd = 0;
    while (!st.empty()) {
        int32_t b = st.back();
        st.pop_back();
        const Node &nd = H.nodes[b];
        if (nd.kind == K_HIER)
            for (int k = 0; k < 4; ++k) {
                depth[nd.kid[k]] = depth[b] + 1;
                maxd = std::max(maxd, depth[b] + 1);
                st.push_back(nd.kid[k]);
            }
    }
    H.sync_ranks(ctx.stream);
    std::vector<int32_t> ranks = H.h_ranks;
    i64 merged = 0;
    i64 max_rows = std::numeric_limits<i64>::max();
    if (const char *e = getenv("LEVYH_COARSEN_MAXROWS")) max_rows = atoll(e);
    const size_t qr_smem = sizeof(double) * QR_SMEM_D, core_smem = sizeof(dev::RecompSmem);
    set_smem((const void *)side_qr_kernel, qr_smem);
    set_smem((const void *)core_kernel, core_smem);
    for (int d = maxd - 1; d >= 0; --d) {
        const auto tl = std::chrono::steady_clock::now();
        std::vector<int32_t> cand;
        std::vector<CoreJob> cores;
        std::vector<QrSide> sides;
        i64 w = 0;
        for (size_t b = 0; b < H.nodes.size(); ++b) {
            const Node &nd = H.nodes[b];
            if (depth[b] != d || nd.kind != K_HIER) continue;
            const bool off_diag = nd.r0 + nd.m <= nd.c0 || nd.c0 + nd.n <= nd.r0;
            if (!off_diag || std::max(nd.m, nd.n) > max_rows) continue;
            const Node *k[4];
            bool ok = true;
            int r[4];
            i64 store = 0;
            for (int q = 0; q < 4 && ok; ++q) {
                k[q] = &H.nodes[nd.kid[q]];
                ok = k[q]->kind == K_LR && k[q]->vpar < 0;
                if (ok) {
                    r[q] = ranks[k[q]->rslot];
                    store += (i64)r[q] * (k[q]->m + k[q]->n);
                }
            }
            if (!ok) continue;
            const int K = r[0] + r[1] + r[2] + r[3];
            if (K > KA_MAX || K == 0) continue;  // all-zero groups are left alone
            CoreJob J{r[0], r[1], r[2], r[3], (int32_t)std::min<i64>(KC_MAX, (store - 1) / (nd.m + nd.n)), 0};
            if (J.rmax < 0) continue;
            // sides: top = [U11 U12], bottom = [U21 U22], left = [V11 V21], right = [V12 V22]
            const QrSide sd[4] = {
                {k[0]->m, k[0]->uoff, k[1]->uoff, 0, r[0], r[1]},
                {k[2]->m, k[2]->uoff, k[3]->uoff, 0, r[2], r[3]},
                {k[0]->n, k[0]->voff, k[2]->voff, 0, r[0], r[2]},
                {k[1]->n, k[1]->voff, k[3]->voff, 0, r[1], r[3]}};
            for (int q = 0; q < 4; ++q) {
                QrSide S = sd[q];
                S.w = w;
                w += S.rows * std::max(S.ra + S.rb, 1);
                sides.push_back(S);
            }
            cores.push_back(J);
            cand.push_back((int32_t)b);
        }
        if (cores.empty()) continue;
        const int nc = (int)cores.size(), ns = (int)sides.size();
        double *work = dalloc<double>(std::max<i64>(w, 1));
        double *Rbuf = dalloc<double>((i64)ns * KA_MAX * KA_MAX);
        double *coef = dalloc<double>((i64)2 * nc * KA_MAX * KC_MAX);
        QrSide *dsides = dupload(sides, ctx.stream);
        CoreJob *dcores = dupload(cores, ctx.stream);
        int *dcnt = dalloc<int>(2 + (i64)nc);
        LH_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(int) * 2, ctx.stream));
        side_qr_kernel<<<(int)std::min<i64>(ns, (i64)ctx.num_sms * 2), NT, qr_smem, ctx.stream>>>(
            dsides, ns, dcnt, H.d_arena, work, Rbuf);
        LH_CUDA(cudaGetLastError());
        core_kernel<<<(int)std::min<i64>(nc, (i64)ctx.num_sms * 2), NT, core_smem, ctx.stream>>>(
            dcores, nc, dcnt + 1, Rbuf, coef, dcnt + 2, eps);
        LH_CUDA(cudaGetLastError());
        std::vector<int> rk(nc);
        LH_CUDA(cudaMemcpyAsync(rk.data(), dcnt + 2, sizeof(int) * nc, cudaMemcpyDeviceToHost, ctx.stream));
        LH_CUDA(cudaStreamSynchronize(ctx.stream));
        // grow the arena by the accepted factors and write them row-parallel
        i64 add = 0;
        std::vector<i64> uo(nc, -1), vo(nc, -1);
        std::vector<ApplyJob> aj;
        std::vector<i64> tile0;
        i64 ntiles = 0;
        for (int c = 0; c < nc; ++c) {
            if (rk[c] < 0) continue;
            const Node &nd = H.nodes[cand[c]];
            const int r = rk[c];
            uo[c] = H.arena_len + add;
            add += nd.m * r;
            vo[c] = H.arena_len + add;
            add += nd.n * r;
            if (r == 0) continue;
            const QrSide *sd = &sides[4 * c];
            const CoreJob &J = cores[c];
            const int Kt = J.r11 + J.r12, Kl = J.r11 + J.r21;
            const i64 cu = (i64)(2 * c) * KA_MAX * KC_MAX, cv = (i64)(2 * c + 1) * KA_MAX * KC_MAX;
            const ApplyJob jobs4[4] = {
                {sd[0].w, sd[0].rows, uo[c], nd.m, 0, Kt, r, (int32_t)0, 0},
                {sd[1].w, sd[1].rows, uo[c], nd.m, sd[0].rows, J.r21 + J.r22, r, (int32_t)Kt, 0},
                {sd[2].w, sd[2].rows, vo[c], nd.n, 0, Kl, r, (int32_t)0, 0},
                {sd[3].w, sd[3].rows, vo[c], nd.n, sd[2].rows, J.r12 + J.r22, r, (int32_t)Kl, 0}};
            for (int q = 0; q < 4; ++q) {
                ApplyJob A = jobs4[q];
                A.coff += (int32_t)(q < 2 ? cu : cv);  // absolute coefficient offset
                if (A.K == 0 || A.rows == 0) continue;
                tile0.push_back(ntiles);
                ntiles += (A.rows + NT - 1) / NT;
                aj.push_back(A);
            }
        }
        if (add > 0) {
            double *na = dalloc<double>(H.arena_len + add);
            LH_CUDA(cudaMemcpyAsync(na, H.d_arena, sizeof(double) * H.arena_len, cudaMemcpyDeviceToDevice,
                                    ctx.stream));
            LH_CUDA(cudaMemsetAsync(na + H.arena_len, 0, sizeof(double) * add, ctx.stream));
            if (!aj.empty()) {
                ApplyJob *daj = dupload(aj, ctx.stream);
                i64 *dt0 = dupload(tile0, ctx.stream);
                apply_kernel<<<(int)std::min<i64>(ntiles, (i64)ctx.num_sms * 16), NT, 0, ctx.stream>>>(
                    daj, dt0, (int)aj.size(), ntiles, work, coef, na);
                LH_CUDA(cudaGetLastError());
                LH_CUDA(cudaStreamSynchronize(ctx.stream));
                cudaFree(daj);
                cudaFree(dt0);
            }
            LH_CUDA(cudaStreamSynchronize(ctx.stream));
            cudaFree(H.d_arena);
            H.d_arena = na;
            for (int c = 0; c < nc; ++c) {
                if (rk[c] < 0) continue;
                Node &nd = H.nodes[cand[c]];
                nd.kind = K_LR;
                nd.uoff = uo[c];
                nd.voff = vo[c];
                nd.kcap = std::max(rk[c], 1);
                nd.rslot = (int32_t)ranks.size();
                ranks.push_back(rk[c]);
                for (int t = 0; t < 4; ++t) nd.kid[t] = -1;
                ++merged;
            }
            H.arena_len += add;
        }
        cudaFree(work);
        cudaFree(Rbuf);
        cudaFree(coef);
        cudaFree(dsides);
        cudaFree(dcores);
        cudaFree(dcnt);
        if (getenv("LEVYH_PLAN_VERBOSE")) {
            i64 acc = 0, bigM = 0;
            for (int c = 0; c < nc; ++c) {
                acc += rk[c] >= 0;
                bigM = std::max(bigM, H.nodes[cand[c]].m);
            }
            fprintf(stderr, "[levyh] coarsen depth %d: %d candidates, %lld merged, largest %lld rows, "
                            "workspace %.2f GB, %.3f s\n", d, nc, (long long)acc, (long long)bigM, 8e-9 * (double)w,
                    std::chrono::duration<double>(std::chrono::steady_clock::now() - tl).count());
        }
    }
    if (merged) {
        int32_t *nr = dupload(ranks, ctx.stream);
        LH_CUDA(cudaStreamSynchronize(ctx.stream));
        cudaFree(H.d_ranks);
        H.d_ranks = nr;
        H.nslots = (int32_t)ranks.size();
        H.h_ranks = ranks;
        walk_leaves(H);
    }
    return merged;
}

}  // namespace lh
