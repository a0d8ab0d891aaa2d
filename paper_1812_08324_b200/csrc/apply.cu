// Matrix-free evaluators of the singular generator and the variable-order L-shape assembly.
//
// Reference: fractional.py:285-361 (_window_sums_1d, eval_i1..i3, frac_apply_1d),
// :413-477 (_window_sums_2d, frac_apply_2d), :539-622 (assemble_variable_order).
//
// frac_apply_*: the windowed correlation conv[i] = sum_k u[i + k] kern[k] is the whole cost
// ((2K+1)(2M+1) fused multiply-adds in 1D, (2K+1)^2 (2M+1)^2 in 2D, FP64 compute bound); it
// runs as a register-tiled sliding-window product: a thread owns 8 consecutive outputs, keeps a
// 16-sample window of u in registers and consumes 8 taps per step (64 FMAs per eight 128-bit
// shared-memory loads), u and the taps staged through shared memory.  The window dimension is
// split across CTAs into partial sums that a finishing kernel adds in a fixed order together
// with the compensator terms (deterministic, no atomics).
//
// assemble_variable_order: one CTA per matrix row; offset tables (log r^2, trapezoid weights,
// window) are computed once, the row's kernel values, its six window sums, the graded
// Gauss-Legendre second moment and the tail mass on the device, and the dense row is written
// once (the matrix is the only HBM traffic: 8 m^2 bytes).
#include <algorithm>
#include <cmath>
#include <vector>

#include "core.h"
#include "dev.cuh"
#include "measure.cuh"

namespace lh {

using dev::NT;

namespace {

constexpr int AP_R = 8;            // outputs per thread
constexpr int AP_NT = 128;         // threads per CTA (1D, wide 2D rows); AP_NT_S for narrow 2D rows
constexpr int AP_NT_S = 32;
constexpr int AP_TILE = AP_R * AP_NT;  // outputs per CTA
constexpr int AP_WC = 512;         // taps staged per round

// shared-memory index of u sample x: one 16-byte pad per 16 doubles, so that the 128-bit loads
// of eight consecutive threads (64 bytes apart) fall into eight different 16-byte bank groups
__device__ __forceinline__ int upad(int x) { return x + 2 * (x >> 4); }
constexpr int AP_USMEM = AP_TILE + AP_WC + 2 * ((AP_TILE + AP_WC) / 16) + 16;

// acc[r] += sum_{k < ntaps} us[8 t + r + k] * ks[k]; ntaps a multiple of 8 (zero padded)
__device__ __forceinline__ void corr_accumulate(double (&acc)[AP_R], const double *us, const double *ks,
                                                int ntaps) {
    const int t = threadIdx.x;
    double w[2 * AP_R];
    {
        const double2 *p = reinterpret_cast<const double2 *>(us + upad(AP_R * t));
#pragma unroll
        for (int q = 0; q < AP_R / 2; ++q) {
            double2 v = p[q];
            w[2 * q] = v.x;
            w[2 * q + 1] = v.y;
        }
    }
    for (int k = 0; k < ntaps; k += AP_R) {
        const double2 *p = reinterpret_cast<const double2 *>(us + upad(AP_R * t + k + AP_R));
#pragma unroll
        for (int q = 0; q < AP_R / 2; ++q) {
            double2 v = p[q];
            w[AP_R + 2 * q] = v.x;
            w[AP_R + 2 * q + 1] = v.y;
        }
        double kk[AP_R];
        const double2 *pk = reinterpret_cast<const double2 *>(ks + k);
#pragma unroll
        for (int q = 0; q < AP_R / 2; ++q) {
            double2 v = pk[q];
            kk[2 * q] = v.x;
            kk[2 * q + 1] = v.y;
        }
#pragma unroll
        for (int j = 0; j < AP_R; ++j)
#pragma unroll
            for (int r = 0; r < AP_R; ++r) acc[r] = fma(w[r + j], kk[j], acc[r]);
#pragma unroll
        for (int r = 0; r < AP_R; ++r) w[r] = w[AP_R + r];
    }
}

// kern[j + M] = nu(j h) w_j (fractional.py:285-296)
__global__ void kern_table_kernel(MeasureDev nu, double h, i64 M, double *kern) {
    for (i64 idx = (i64)blockIdx.x * blockDim.x + threadIdx.x; idx < 2 * M + 1;
         idx += (i64)gridDim.x * blockDim.x)
        kern[idx] = kern_eval(nu, idx - M, h, M);
}

constexpr int SUM_CHUNK = 4096;

// per-CTA partial sums of kern, rho y kern, rho y^2 kern over a fixed chunk of the table
__global__ void sums1d_kernel(const double *kern, double h, i64 M, double rho_r, double *partials) {
    __shared__ double red[dev::NW];
    double s0 = 0.0, sg = 0.0, sd = 0.0;
    const i64 lo = (i64)blockIdx.x * SUM_CHUNK, hi = min(lo + SUM_CHUNK, 2 * M + 1);
    for (i64 idx = lo + threadIdx.x; idx < hi; idx += blockDim.x) {
        const double y = (double)(idx - M) * h, k = kern[idx];
        const double rho = window_eval(y, rho_r);
        s0 += k;
        sg += (rho * y) * k;
        sd += ((rho * y) * y) * k;
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

// sums[q] = sum over parts of partials[nq * part + q], one CTA, fixed order
__global__ void reduce_parts_kernel(const double *partials, int nparts, int nq, double *sums) {
    __shared__ double red[dev::NW];
    for (int q = 0; q < nq; ++q) {
        double v = 0.0;
        for (int k = threadIdx.x; k < nparts; k += blockDim.x) v += partials[nq * k + q];
        v = dev::block_sum(v, red);
        if (threadIdx.x == 0) sums[q] = v;
    }
}

// partial[part][i] = sum over the part's taps of u[i + k] kern[k]   (np.correlate 'valid')
__global__ void __launch_bounds__(AP_NT) corr1d_kernel(const double *__restrict__ u, const double *__restrict__ kern,
                                                       i64 nout, i64 ntap, i64 taps_per_part,
                                                       double *__restrict__ partial) {
    __shared__ __align__(16) double us[AP_USMEM];
    __shared__ __align__(16) double ks[AP_WC];
    const i64 i0 = (i64)blockIdx.x * AP_TILE;
    const i64 k_lo = (i64)blockIdx.y * taps_per_part;
    const i64 k_hi = min(k_lo + taps_per_part, ntap);
    const i64 ulen = nout + ntap - 1;
    double acc[AP_R];
#pragma unroll
    for (int r = 0; r < AP_R; ++r) acc[r] = 0.0;
    for (i64 k0 = k_lo; k0 < k_hi; k0 += AP_WC) {
        const int nt = (int)min((i64)AP_WC, k_hi - k0);
        const int nt8 = (nt + AP_R - 1) / AP_R * AP_R;
        __syncthreads();
        for (int x = threadIdx.x; x < AP_TILE + nt8 + AP_R; x += AP_NT) {
            const i64 g = i0 + k0 + x;
            us[upad(x)] = g < ulen ? u[g] : 0.0;
        }
        for (int x = threadIdx.x; x < nt8; x += AP_NT) ks[x] = x < nt ? kern[k0 + x] : 0.0;
        __syncthreads();
        corr_accumulate(acc, us, ks, nt8);
    }
    double *dst = partial + (i64)blockIdx.y * nout;
#pragma unroll
    for (int r = 0; r < AP_R; ++r) {
        const i64 i = i0 + AP_R * threadIdx.x + r;
        if (i < nout) dst[i] = acc[r];
    }
}

// frac_apply_1d's last lines (fractional.py:350-360); part 1: the near-field term I1 alone
__global__ void finish1d_kernel(const double *partial, int nparts, i64 nout, const double *u, i64 M, double h,
                                const double *sums, double tail, double m2, const double *far, int part,
                                double *out) {
    const double S0 = sums[0], Sg = sums[1], Sd = sums[2];
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < nout; i += (i64)gridDim.x * blockDim.x) {
        double conv = 0.0;
        for (int p = 0; p < nparts; ++p) conv += partial[(i64)p * nout + i];
        const double uc = u[M + i], ue = u[M + i + 1], uw = u[M + i - 1];
        const double d1 = (ue - uw) / (2 * h);
        const double d2 = (ue + uw - 2 * uc) / (2 * h * h);
        const double i1 = conv - uc * S0 - d1 * Sg - d2 * Sd;
        out[i] = part == 1 ? i1 : i1 + (far ? far[i] : 0.0) - uc * tail + d2 * m2;
    }
}

// ---- 2D ------------------------------------------------------------------------------------
// kern[jx, jy] = c (x^2 + y^2)^(-(2 + 2s)/2) w_jx w_jy, centre 0 (fractional.py:413-423); with a
// caller table (nu.density2 evaluated on the host) only the weights are applied here
__global__ void kern2d_kernel(double c, double s, const double *table, double h, i64 M, double *kern) {
    const i64 W = 2 * M + 1;
    for (i64 idx = (i64)blockIdx.x * blockDim.x + threadIdx.x; idx < W * W; idx += (i64)gridDim.x * blockDim.x) {
        const i64 jx = idx / W - M, jy = idx % W - M;
        const double x = (double)jx * h, y = (double)jy * h;
        const double wx = (jx == M || jx == -M) ? h / 2.0 : h, wy = (jy == M || jy == -M) ? h / 2.0 : h;
        double nu = 0.0;
        if (jx != 0 || jy != 0) nu = table ? table[idx] : c * pow(x * x + y * y, -(2.0 + 2.0 * s) / 2.0);
        kern[idx] = nu * (wx * wy);
    }
}

// per-CTA partials of S0, Sgx, Sgy, Sdxx, Sdyy, Sdxy (fractional.py:424-432) over a chunk of offsets
__global__ void sums2d_kernel(const double *kern, double h, i64 M, double rho_r, double *partials) {
    __shared__ double red[dev::NW];
    const i64 W = 2 * M + 1;
    const i64 lo = (i64)blockIdx.x * SUM_CHUNK, hi = min(lo + SUM_CHUNK, W * W);
    double a[6] = {0, 0, 0, 0, 0, 0};
    for (i64 idx = lo + threadIdx.x; idx < hi; idx += blockDim.x) {
        const double x = (double)(idx / W - M) * h, y = (double)(idx % W - M) * h, k = kern[idx];
        const double rho = window_eval(hypot(x, y), rho_r);
        a[0] += k;
        a[1] += (rho * x) * k;
        a[2] += (rho * y) * k;
        a[3] += ((rho * x) * x) * k;
        a[4] += ((rho * y) * y) * k;
        a[5] += ((rho * x) * y) * k;
    }
    for (int q = 0; q < 6; ++q) {
        const double v = dev::block_sum(a[q], red);
        if (threadIdx.x == 0) partials[6 * blockIdx.x + q] = v;
    }
}

// partial[z][ix, iy] = sum over the part's window rows jx and all jy of u[ix + jx, iy + jy] kern[jx, jy]:
// CTA = one output row ix, a tile of iy and a range of window rows, each row a 1D sliding-window
// product
template <int NTH>
__global__ void __launch_bounds__(NTH) corr2d_kernel(const double *__restrict__ u, const double *__restrict__ kern,
                                                     i64 nout, i64 W, i64 side, i64 rows_per_part,
                                                     double *__restrict__ partial) {
    constexpr int TILE = AP_R * NTH;
    __shared__ __align__(16) double us[TILE + AP_WC + 2 * ((TILE + AP_WC) / 16) + 16];
    __shared__ __align__(16) double ks[AP_WC];
    const i64 ix = blockIdx.y;
    const i64 i0 = (i64)blockIdx.x * TILE;
    const i64 jx_lo = (i64)blockIdx.z * rows_per_part, jx_hi = min(jx_lo + rows_per_part, W);
    double acc[AP_R];
#pragma unroll
    for (int r = 0; r < AP_R; ++r) acc[r] = 0.0;
    for (i64 jx = jx_lo; jx < jx_hi; ++jx) {
        const double *urow = u + (ix + jx) * side;
        const double *krow = kern + jx * W;
        for (i64 k0 = 0; k0 < W; k0 += AP_WC) {
            const int nt = (int)min((i64)AP_WC, W - k0);
            const int nt8 = (nt + AP_R - 1) / AP_R * AP_R;
            __syncthreads();
            for (int x = threadIdx.x; x < TILE + nt8 + AP_R; x += NTH) {
                const i64 g = i0 + k0 + x;
                us[upad(x)] = g < side ? urow[g] : 0.0;
            }
            for (int x = threadIdx.x; x < nt8; x += NTH) ks[x] = x < nt ? krow[k0 + x] : 0.0;
            __syncthreads();
            corr_accumulate(acc, us, ks, nt8);
        }
    }
    double *dst = partial + ((i64)blockIdx.z * nout + ix) * nout;
#pragma unroll
    for (int r = 0; r < AP_R; ++r) {
        const i64 iy = i0 + AP_R * threadIdx.x + r;
        if (iy < nout) dst[iy] = acc[r];
    }
}

// fractional.py:452-477
__global__ void finish2d_kernel(const double *partial, int nparts, i64 nout, const double *u, i64 M, i64 side,
                                double h, const double *sums, double tail, double m2, const double *far,
                                double *out) {
    const double h2 = h * h;
    for (i64 e = (i64)blockIdx.x * blockDim.x + threadIdx.x; e < nout * nout; e += (i64)gridDim.x * blockDim.x) {
        const i64 ix = e / nout + M, iy = e % nout + M;
        auto U = [&](i64 a, i64 b) { return u[a * side + b]; };
        const double uc = U(ix, iy);
        const double ux = (U(ix + 1, iy) - U(ix - 1, iy)) / (2 * h);
        const double uy = (U(ix, iy + 1) - U(ix, iy - 1)) / (2 * h);
        const double uxx = (U(ix + 1, iy) + U(ix - 1, iy) - 2 * uc) / h2;
        const double uyy = (U(ix, iy + 1) + U(ix, iy - 1) - 2 * uc) / h2;
        const double uxy = (U(ix + 1, iy + 1) + U(ix - 1, iy - 1) - U(ix + 1, iy - 1) - U(ix - 1, iy + 1)) / (4 * h2);
        double conv = 0.0;
        for (int p = 0; p < nparts; ++p) conv += partial[(i64)p * nout * nout + e];
        const double i1 = conv - uc * sums[0] - ux * sums[1] - uy * sums[2] - 0.5 * uxx * sums[3] -
                          0.5 * uyy * sums[4] - uxy * sums[5];
        out[e] = i1 + (far ? far[e] : 0.0) - uc * tail + 0.5 * (uxx + uyy) * m2;
    }
}

// ---- variable-order L-shape assembly ---------------------------------------------------------
struct VoTables {
    double *logr2, *w2, *rho;  // (2 Mw + 1)^2 each
};

// fractional.py:563-575: offset tables shared by every row
__global__ void vo_tables_kernel(int Mw, double h, double rho_r, VoTables T) {
    const int W = 2 * Mw + 1;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < W * W; idx += gridDim.x * blockDim.x) {
        const int ox = idx / W - Mw, oy = idx % W - Mw;
        const double dx = (double)ox * h, dy = (double)oy * h;
        double r2 = dx * dx + dy * dy;
        if (ox == 0 && oy == 0) r2 = 1.0;
        const double wx = (ox == Mw || ox == -Mw) ? h / 2.0 : h, wy = (oy == Mw || oy == -Mw) ? h / 2.0 : h;
        T.logr2[idx] = log(r2);
        T.w2[idx] = wx * wy;
        T.rho[idx] = window_eval(sqrt(r2), rho_r);
    }
}

__global__ void vo_cell_table_kernel(const int32_t *cells, i64 m, int n, int32_t *table) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (i64)gridDim.x * blockDim.x)
        table[(i64)cells[2 * i] * n + cells[2 * i + 1]] = (int32_t)i;
}

__constant__ double c_gl16_x[16], c_gl16_w[16], c_gl64_x[64], c_gl64_w[64];

// frac_kernel_constant(2, s) (fractional.py:89-105)
__device__ __forceinline__ double frac_const2(double s) {
    const double log_c = 2 * s * log(2.0) + lgamma(1.0 + s) - log(M_PI) - (lgamma(1.0 - s) - log(s));
    return exp(log_c);
}

// _graded_moment of f(r) = pi rho(r) c r^(-2-2s) r^3 on [0, radius] (fractional.py:200-246), one
// thread: 16-point Gauss-Legendre panels on dyadic intervals with geometric completion
__device__ double graded_m2(double c, double s, double radius, int *ok) {
    const double rel_tol = 1e-12;
    double total = 0.0, hi = radius, prev_part = 0.0, prev_val = 0.0;
    bool have_prev = false;
    for (int lev = 0; lev < 60; ++lev) {
        const double lo = hi / 2.0;
        const double mid = 0.5 * (lo + hi), rad = 0.5 * (hi - lo);
        double dot = 0.0;
        for (int q = 0; q < 16; ++q) {
            const double r = mid + rad * c_gl16_x[q];
            const double f = M_PI * window_eval(r, radius) * (c * pow(r, -2.0 - 2.0 * s)) * (r * r * r);
            dot += f * c_gl16_w[q];
        }
        const double part = rad * dot;
        total += part;
        double val = total;
        if (have_prev && 0 < fabs(part) && fabs(part) < fabs(prev_part)) {
            const double q = part / prev_part;
            if (0 < q && q < 1) val = total + part * q / (1.0 - q);
        }
        if (fabs(part) < rel_tol * fmax(fabs(val), 1e-300)) return val;
        if (have_prev && fabs(val - prev_val) <= rel_tol * fmax(fabs(val), 1e-300)) return val;
        prev_part = part;
        prev_val = val;
        have_prev = true;
        hi = lo;
    }
    *ok = 0;
    return total;
}

// tail_mass_square_2d (fractional.py:266-278)
__device__ double tail_square(double c, double s, double L_W) {
    double dot = 0.0;
    for (int q = 0; q < 64; ++q) {
        const double phi = (c_gl64_x[q] + 1.0) * (M_PI / 8.0);
        const double r0 = L_W / cos(phi);
        dot += (c * pow(r0, -2 * s) / (2 * s)) * c_gl64_w[q];
    }
    return 8.0 * (M_PI / 8.0) * dot;
}

// One CTA per row i (fractional.py:581-614, do_row).  rowinfo (optional, 8 per row): S0, sgx,
// sgy, sdxx, sdyy, sdxy, m2, tail.
__global__ void __launch_bounds__(NT) vo_rows_kernel(int n, i64 m, int Mw, double h, double L_W, double rho_r,
                                                     const int32_t *__restrict__ cells,
                                                     const double *__restrict__ sfield,
                                                     const int32_t *__restrict__ table, VoTables T,
                                                     double *__restrict__ A, double *rowinfo, int *status) {
    __shared__ double red[dev::NW];
    __shared__ double sh_m2, sh_tail;
    const int W = 2 * Mw + 1;
    for (i64 i = blockIdx.x; i < m; i += gridDim.x) {
        const double si = sfield[i];
        const double ci = frac_const2(si);
        const int gx = cells[2 * i], gy = cells[2 * i + 1];
        double *row = A + i * m;
        __syncthreads();
        if (Mw < n - 1)  // otherwise every column lies inside the window and is written below
            for (i64 j = threadIdx.x; j < m; j += NT) row[j] = 0.0;
        if (threadIdx.x == NT - 1) {
            int ok = 1;
            sh_m2 = graded_m2(ci, si, rho_r, &ok);
            sh_tail = tail_square(ci, si, L_W);
            if (!ok) atomicExch(status, 1);
        }
        __syncthreads();
        double a[6] = {0, 0, 0, 0, 0, 0};
        for (int idx = threadIdx.x; idx < W * W; idx += NT) {
            const int ox = idx / W - Mw, oy = idx % W - Mw;
            double k = ci * exp(-(1.0 + si) * T.logr2[idx]);
            if (ox == 0 && oy == 0) k = 0.0;
            const double kw = k * T.w2[idx];
            const double dx = (double)ox * h, dy = (double)oy * h, rho = T.rho[idx];
            a[0] += kw;
            a[1] += (rho * dx) * kw;
            a[2] += (rho * dy) * kw;
            a[3] += ((rho * dx) * dx) * kw;
            a[4] += ((rho * dy) * dy) * kw;
            a[5] += ((rho * dx) * dy) * kw;
            const int cx = gx + ox, cy = gy + oy;
            if (cx >= 0 && cx < n && cy >= 0 && cy < n) {
                const int32_t col = table[(i64)cx * n + cy];
                if (col >= 0) row[col] = (k * h) * h;
            }
        }
        for (int q = 0; q < 6; ++q) a[q] = dev::block_sum(a[q], red);
        __syncthreads();
        if (threadIdx.x == 0) {
            const double S0 = a[0], sgx = a[1], sgy = a[2], sdxx = a[3], sdyy = a[4], sdxy = a[5];
            const double m2 = sh_m2, tail = sh_tail, h2 = h * h;
            auto add = [&](int dx, int dy, double val) {
                const int cx = gx + dx, cy = gy + dy;
                if (cx >= 0 && cx < n && cy >= 0 && cy < n) {
                    const int32_t col = table[(i64)cx * n + cy];
                    if (col >= 0) row[col] += val;
                }
            };
            const double cxx = 0.5 * (m2 - sdxx) / h2, cyy = 0.5 * (m2 - sdyy) / h2;
            add(0, 0, -S0 - tail - 2 * cxx - 2 * cyy);
            add(1, 0, cxx - sgx / (2 * h));
            add(-1, 0, cxx + sgx / (2 * h));
            add(0, 1, cyy - sgy / (2 * h));
            add(0, -1, cyy + sgy / (2 * h));
            const double cxy = -sdxy / (4 * h2);
            add(1, 1, cxy);
            add(-1, -1, cxy);
            add(1, -1, -cxy);
            add(-1, 1, -cxy);
            if (rowinfo) {
                double *ri = rowinfo + 8 * i;
                ri[0] = S0, ri[1] = sgx, ri[2] = sgy, ri[3] = sdxx, ri[4] = sdyy, ri[5] = sdxy, ri[6] = m2,
                ri[7] = tail;
            }
        }
    }
}

int grid_for(i64 work, int per_cta, int cap) {
    return (int)std::max<i64>(1, std::min<i64>((work + per_cta - 1) / per_cta, cap));
}

}  // namespace

void frac_apply_1d(Ctx &ctx, const lh_measure &m, double h, i64 M, i64 K, double rho_r, double tail, double m2,
                   const double *u, const double *far, int part, double *out, double *sums_host) {
    LH_REQUIRE(M >= 1 && K >= 0 && h > 0 && rho_r > 0, LH_EINVAL, "need M >= 1, K >= 0, h > 0 and rho_r > 0");
    LH_REQUIRE(part == 0 || part == 1, LH_EINVAL, "part must be 0 (full) or 1 (I1 only)");
    MeasureDev nu = measure_to_dev(m, M);
    const i64 nout = 2 * K + 1, ntap = 2 * M + 1;
    const i64 tiles = (nout + AP_TILE - 1) / AP_TILE;
    // window split: about three CTAs per SM in flight, parts of at least AP_WC taps
    i64 nparts = std::max<i64>(1, std::min<i64>((3 * (i64)ctx.num_sms + tiles - 1) / tiles, (ntap + AP_WC - 1) / AP_WC));
    i64 per = ((ntap + nparts - 1) / nparts + AP_R - 1) / AP_R * AP_R;
    nparts = (ntap + per - 1) / per;
    const int nsum = (int)((ntap + SUM_CHUNK - 1) / SUM_CHUNK);
    double *buf = dalloc<double>(ntap + 4 + 3 * (i64)nsum + nparts * nout);
    double *kern = buf, *sums = buf + ntap, *sparts = sums + 4, *partial = sparts + 3 * (i64)nsum;
    kern_table_kernel<<<grid_for(ntap, 256, ctx.num_sms * 8), 256, 0, ctx.stream>>>(nu, h, M, kern);
    sums1d_kernel<<<nsum, NT, 0, ctx.stream>>>(kern, h, M, rho_r, sparts);
    reduce_parts_kernel<<<1, NT, 0, ctx.stream>>>(sparts, nsum, 3, sums);
    corr1d_kernel<<<dim3((unsigned)tiles, (unsigned)nparts), AP_NT, 0, ctx.stream>>>(u, kern, nout, ntap, per, partial);
    finish1d_kernel<<<grid_for(nout, 256, ctx.num_sms * 8), 256, 0, ctx.stream>>>(partial, (int)nparts, nout, u, M, h,
                                                                                 sums, tail, m2, far, part, out);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && sums_host)
        e = cudaMemcpyAsync(sums_host, sums, 3 * sizeof(double), cudaMemcpyDeviceToHost, ctx.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx.stream);
    cudaFree(buf);
    LH_CUDA(e);
}

void frac_apply_2d(Ctx &ctx, double c, double s, const double *table, double h, i64 M, i64 K, double rho_r,
                   double tail, double m2, const double *u, const double *far, double *out, double *sums_host) {
    LH_REQUIRE(M >= 1 && K >= 0 && h > 0 && rho_r > 0, LH_EINVAL, "need M >= 1, K >= 0, h > 0 and rho_r > 0");
    const i64 nout = 2 * K + 1, W = 2 * M + 1, side = 2 * (M + K) + 1;
    LH_REQUIRE(nout <= 65535, LH_EINVAL, "main grid too large for the 2D evaluator");
    // narrow rows take 32-thread CTAs (256 outputs); window rows split into parts until about
    // sixteen warps per SM are in flight
    const bool narrow = nout <= 2 * AP_R * AP_NT_S;
    const int nth = narrow ? AP_NT_S : AP_NT;
    const i64 tiles = (nout + AP_R * nth - 1) / (AP_R * nth);
    const i64 want = (16 * (i64)ctx.num_sms * 32 + tiles * nout * nth - 1) / (tiles * nout * nth);
    i64 nparts = std::max<i64>(1, std::min<i64>(std::min<i64>(want, W), 64));
    const i64 per = (W + nparts - 1) / nparts;
    nparts = (W + per - 1) / per;
    const int nsum = (int)((W * W + SUM_CHUNK - 1) / SUM_CHUNK);
    double *buf = dalloc<double>(W * W + 8 + 6 * (i64)nsum + nparts * nout * nout);
    double *kern = buf, *sums = buf + W * W, *sparts = sums + 8, *partial = sparts + 6 * (i64)nsum;
    kern2d_kernel<<<grid_for(W * W, 256, ctx.num_sms * 8), 256, 0, ctx.stream>>>(c, s, table, h, M, kern);
    sums2d_kernel<<<nsum, NT, 0, ctx.stream>>>(kern, h, M, rho_r, sparts);
    reduce_parts_kernel<<<1, NT, 0, ctx.stream>>>(sparts, nsum, 6, sums);
    const dim3 grid((unsigned)tiles, (unsigned)nout, (unsigned)nparts);
    if (narrow)
        corr2d_kernel<AP_NT_S><<<grid, AP_NT_S, 0, ctx.stream>>>(u, kern, nout, W, side, per, partial);
    else
        corr2d_kernel<AP_NT><<<grid, AP_NT, 0, ctx.stream>>>(u, kern, nout, W, side, per, partial);
    finish2d_kernel<<<grid_for(nout * nout, 256, ctx.num_sms * 8), 256, 0, ctx.stream>>>(
        partial, (int)nparts, nout, u, M, side, h, sums, tail, m2, far, out);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && sums_host)
        e = cudaMemcpyAsync(sums_host, sums, 6 * sizeof(double), cudaMemcpyDeviceToHost, ctx.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx.stream);
    cudaFree(buf);
    LH_CUDA(e);
}

void assemble_variable_order(Ctx &ctx, int n, i64 m, const int32_t *cells_host, const double *s_host, double L_W,
                             double rho_r, const double *gl16, const double *gl64, double *A, double *rowinfo_host) {
    LH_REQUIRE(n >= 2 && n % 2 == 0, LH_EINVAL, "n must be even for the L-shape grid");
    LH_REQUIRE(m >= 1 && m <= (i64)n * n, LH_EINVAL, "m must be within 1 .. n^2");
    LH_REQUIRE(L_W > 0 && rho_r > 0, LH_EINVAL, "need L_W > 0 and rho_r > 0");
    for (i64 i = 0; i < m; ++i) {
        LH_REQUIRE(s_host[i] > 0 && s_host[i] < 1, LH_EINVAL, "order field must map into (0, 1)");
        LH_REQUIRE(cells_host[2 * i] >= 0 && cells_host[2 * i] < n && cells_host[2 * i + 1] >= 0 &&
                       cells_host[2 * i + 1] < n,
                   LH_EINVAL, "cell coordinates out of range");
    }
    const double h = 2.0 / n;
    const int Mw = (int)std::llround(L_W / h);
    LH_REQUIRE(Mw >= 1 && Mw <= 16384, LH_EINVAL, "window offsets out of range");
    const i64 WW = (i64)(2 * Mw + 1) * (2 * Mw + 1);
    LH_CUDA(cudaMemcpyToSymbolAsync(c_gl16_x, gl16, 16 * sizeof(double), 0, cudaMemcpyHostToDevice, ctx.stream));
    LH_CUDA(cudaMemcpyToSymbolAsync(c_gl16_w, gl16 + 16, 16 * sizeof(double), 0, cudaMemcpyHostToDevice, ctx.stream));
    LH_CUDA(cudaMemcpyToSymbolAsync(c_gl64_x, gl64, 64 * sizeof(double), 0, cudaMemcpyHostToDevice, ctx.stream));
    LH_CUDA(cudaMemcpyToSymbolAsync(c_gl64_w, gl64 + 64, 64 * sizeof(double), 0, cudaMemcpyHostToDevice, ctx.stream));
    double *dbuf = dalloc<double>(3 * WW + m + (rowinfo_host ? 8 * m : 0));
    VoTables T{dbuf, dbuf + WW, dbuf + 2 * WW};
    double *sdev = dbuf + 3 * WW, *rinfo = rowinfo_host ? sdev + m : nullptr;
    int32_t *ibuf = dalloc<int32_t>(2 * m + (i64)n * n + 1);
    int32_t *cells = ibuf, *table = ibuf + 2 * m;
    int *status = (int *)(table + (i64)n * n);
    cudaError_t e = cudaMemcpyAsync(cells, cells_host, 2 * m * sizeof(int32_t), cudaMemcpyHostToDevice, ctx.stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(sdev, s_host, m * sizeof(double), cudaMemcpyHostToDevice, ctx.stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(table, 0xff, ((i64)n * n) * sizeof(int32_t), ctx.stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(status, 0, sizeof(int), ctx.stream);
    int st = 0;
    if (e == cudaSuccess) {
        vo_tables_kernel<<<grid_for(WW, 256, ctx.num_sms * 8), 256, 0, ctx.stream>>>(Mw, h, rho_r, T);
        vo_cell_table_kernel<<<grid_for(m, 256, ctx.num_sms * 8), 256, 0, ctx.stream>>>(cells, m, n, table);
        vo_rows_kernel<<<(int)std::min<i64>(m, (i64)ctx.num_sms * 8), NT, 0, ctx.stream>>>(n, m, Mw, h, L_W, rho_r, cells,
                                                                                        sdev, table, T, A, rinfo,
                                                                                        status);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(&st, status, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream);
    if (e == cudaSuccess && rowinfo_host)
        e = cudaMemcpyAsync(rowinfo_host, rinfo, 8 * m * sizeof(double), cudaMemcpyDeviceToHost, ctx.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx.stream);
    cudaFree(dbuf);
    cudaFree(ibuf);
    LH_CUDA(e);
    LH_REQUIRE(st == 0, LH_EINTERNAL, "graded quadrature did not converge within 60 levels");
}

}  // namespace lh
