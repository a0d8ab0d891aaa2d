// CTA-level fp64 primitives shared by the ACA builder and the H-LU executor.
// All routines are called by every thread of a 256-thread CTA.
#pragma once

#include <cstdint>

namespace lh {
namespace dev {

typedef long long i64;

constexpr int NT = 256;             // threads per CTA
constexpr int NW = NT / 32;         // warps per CTA
constexpr int KA_MAX = 48;          // max columns entering a recompression
constexpr int KC_MAX = 32;          // max rank kept after recompression

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// deterministic block sum; result broadcast to all threads.  red: >= NW doubles.
__device__ __forceinline__ double block_sum(double v, double *red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < NW; ++k) s += red[k];
    return s;
}

// argmax of a (>= 0) with the smallest index on ties; result broadcast.
__device__ __forceinline__ void block_argmax(double a, i64 idx, double *redv, i64 *redi,
                                             double &ba, i64 &bi) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double oa = __shfl_xor_sync(0xffffffffu, a, o);
        i64 oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (oa > a || (oa == a && oi < idx)) {
            a = oa;
            idx = oi;
        }
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) {
        redv[w] = a;
        redi[w] = idx;
    }
    __syncthreads();
    ba = redv[0];
    bi = redi[0];
    for (int k = 1; k < NW; ++k) {
        if (redv[k] > ba || (redv[k] == ba && redi[k] < bi)) {
            ba = redv[k];
            bi = redi[k];
        }
    }
}

// h[l] = sum_i Q[i,l] * u[i] for l < k (one warp per column l, lanes over rows).
__device__ __forceinline__ void col_dots(const double *Q, i64 ldq, i64 m, int k, const double *u,
                                         double *h) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int l = w; l < k; l += NW) {
        const double *q = Q + (i64)l * ldq;
        // 8 independent loads per lane per iteration: in-order issue would otherwise pay
        // one memory round trip per iteration on long columns
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        i64 i = lane;
        for (; i + 96 < m; i += 128) {
            const double q0 = q[i], q1 = q[i + 32], q2 = q[i + 64], q3 = q[i + 96];
            const double u0 = u[i], u1 = u[i + 32], u2 = u[i + 64], u3 = u[i + 96];
            s0 += q0 * u0;
            s1 += q1 * u1;
            s2 += q2 * u2;
            s3 += q3 * u3;
        }
        for (; i < m; i += 32) s0 += q[i] * u[i];
        s0 = warp_sum((s0 + s1) + (s2 + s3));
        if (lane == 0) h[l] = s0;
    }
}

// per-thread partial sum of squares over a strided column (4 independent loads in flight)
__device__ __forceinline__ double sumsq(const double *u, i64 m) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    i64 i = threadIdx.x;
    for (; i + 3 * NT < m; i += 4 * NT) {
        const double a = u[i], b = u[i + NT], c = u[i + 2 * NT], d = u[i + 3 * NT];
        s0 += a * a;
        s1 += b * b;
        s2 += c * c;
        s3 += d * d;
    }
    for (; i < m; i += NT) s0 += u[i] * u[i];
    return (s0 + s1) + (s2 + s3);
}

// Classical Gram-Schmidt with one reorthogonalisation (CGS2), in place:
// Q (m x K, column-major, ldq) becomes orthonormal columns, R (K x K, col-major,
// ld KA_MAX, shared) upper triangular with A = Q R.  Zero columns stay zero (R_kk = 0).
__device__ __noinline__ static void cgs2(double *Q, i64 ldq, i64 m, int K, double *R, double *h, double *red) {
    for (int k = 0; k < K; ++k) {
        double *u = Q + (i64)k * ldq;
        for (int l = threadIdx.x; l < KA_MAX; l += NT) R[l + k * KA_MAX] = 0.0;
        const double n0 = sqrt(block_sum(sumsq(u, m), red));
        for (int pass = 0; pass < 2; ++pass) {
            __syncthreads();
            col_dots(Q, ldq, m, k, u, h);
            __syncthreads();
            // four rows per iteration: 4k independent loads before the first use
            i64 i = threadIdx.x;
            for (; i + 3 * NT < m; i += 4 * NT) {
                double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
                int l = 0;
                for (; l + 4 <= k; l += 4) {  // 16 independent loads per batch
                    double a[4][4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const double *ql = Q + (i64)(l + j) * ldq + i;
                        a[j][0] = ql[0];
                        a[j][1] = ql[NT];
                        a[j][2] = ql[2 * NT];
                        a[j][3] = ql[3 * NT];
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const double hl = h[l + j];
                        s0 += a[j][0] * hl;
                        s1 += a[j][1] * hl;
                        s2 += a[j][2] * hl;
                        s3 += a[j][3] * hl;
                    }
                }
                for (; l < k; ++l) {
                    const double *ql = Q + (i64)l * ldq + i;
                    const double hl = h[l];
                    s0 += ql[0] * hl;
                    s1 += ql[NT] * hl;
                    s2 += ql[2 * NT] * hl;
                    s3 += ql[3 * NT] * hl;
                }
                const double a0 = u[i], a1 = u[i + NT], a2 = u[i + 2 * NT], a3 = u[i + 3 * NT];
                u[i] = a0 - s0;
                u[i + NT] = a1 - s1;
                u[i + 2 * NT] = a2 - s2;
                u[i + 3 * NT] = a3 - s3;
            }
            for (; i < m; i += NT) {
                double s = 0.0;
                for (int l = 0; l < k; ++l) s += Q[i + (i64)l * ldq] * h[l];
                u[i] -= s;
            }
            for (int l = threadIdx.x; l < k; l += NT) R[l + k * KA_MAX] += h[l];
        }
        __syncthreads();
        double nrm = sqrt(block_sum(sumsq(u, m), red));
        // a residual at rounding level after reorthogonalisation means the column is
        // numerically inside span(q_0..q_{k-1}): drop it (q_k = 0, R_kk = 0) so Q keeps
        // orthonormal columns (normalising noise would not be orthogonal to the span)
        if (!(nrm > 1e-13 * n0)) nrm = 0.0;
        double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
        {
            i64 i = threadIdx.x;
            for (; i + 3 * NT < m; i += 4 * NT) {
                const double a = u[i], b = u[i + NT], c = u[i + 2 * NT], d = u[i + 3 * NT];
                u[i] = a * inv;
                u[i + NT] = b * inv;
                u[i + 2 * NT] = c * inv;
                u[i + 3 * NT] = d * inv;
            }
            for (; i < m; i += NT) u[i] *= inv;
        }
        if (threadIdx.x == 0) R[k + k * KA_MAX] = nrm;
        __syncthreads();
    }
}

// One-sided Jacobi SVD (Hestenes) of C (K x K, col-major, ld KA_MAX, shared).
// On exit C <- C V (columns = sigma_i * w_i), V (K x K) orthogonal.  Then
// sigma[i] = ||C[:,i]|| and ord[] sorts them descending (stable by index).
// Round-robin ordering: each step rotates P/2 disjoint column pairs, one warp per pair
// (K <= 32: one row per lane; K <= 48: two).  The step is a latency chain (shared loads,
// three interleaved warp reductions, the rotation, one barrier), so the rotation uses two
// long-latency FP64 ops: h = hypot(d, g), then w = 1/sqrt((|d| + h)^2 + g^2), with
// d = ||b||^2 - ||a||^2, g = 2 <a, b>: c = (|d| + h) w, s = sign(d) g w (Rutishauser's
// t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = d / g, scaled by |d| + h).
__device__ __noinline__ static int jacobi_svd(double *C, double *V, int K, double *sigma, int *ord, double *red) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int e = threadIdx.x; e < K * KA_MAX; e += NT) {
        int i = e % KA_MAX, j = e / KA_MAX;
        V[e] = (i == j) ? 1.0 : 0.0;
    }
    __shared__ int s_rot;
    const int P = (K + 1) & ~1;  // even number of slots (one dummy if K odd)
    const int L = P - 1;
    const bool two = K > 32;
    const int i0 = lane, i1 = lane + 32;
    const bool h0 = i0 < K, h1 = two && i1 < K;
    int sweep = 0;
    for (; sweep < 40 && K > 1; ++sweep) {
        if (threadIdx.x == 0) s_rot = 0;
        __syncthreads();
        bool rot = false;
        for (int step = 0; step < L; ++step) {
            for (int pr = w; pr < P / 2; pr += NW) {
                // slot 0 fixed, the others rotate by one position per step
                int a = pr - 1 + step, b = L - 1 - pr + step;
                a = a >= L ? a - L : a;
                b = b >= L ? b - L : b;
                a = pr == 0 ? 0 : a + 1;
                b += 1;
                if (a >= K || b >= K) continue;
                if (a > b) {
                    const int t = a;
                    a = b;
                    b = t;
                }
                double *ca = C + a * KA_MAX, *cb = C + b * KA_MAX;
                double *va = V + a * KA_MAX, *vb = V + b * KA_MAX;
                const double x0 = h0 ? ca[i0] : 0.0, y0 = h0 ? cb[i0] : 0.0;
                const double x1 = h1 ? ca[i1] : 0.0, y1 = h1 ? cb[i1] : 0.0;
                const double p0 = h0 ? va[i0] : 0.0, q0 = h0 ? vb[i0] : 0.0;
                const double p1 = h1 ? va[i1] : 0.0, q1 = h1 ? vb[i1] : 0.0;
                double al = x0 * x0 + x1 * x1, be = y0 * y0 + y1 * y1, ga = x0 * y0 + x1 * y1;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    al += __shfl_xor_sync(0xffffffffu, al, o);
                    be += __shfl_xor_sync(0xffffffffu, be, o);
                    ga += __shfl_xor_sync(0xffffffffu, ga, o);
                }
                // |<a,b>| > 1e-15 ||a|| ||b||, squared (no square roots on the chain)
                if (ga != 0.0 && ga * ga > 1e-30 * (al * be)) {
                    const double d = be - al, g = 2.0 * ga;
                    const double u = fabs(d) + hypot(d, g);
                    const double wn = rsqrt(u * u + g * g);
                    const double c = u * wn, sn = (d >= 0.0 ? g : -g) * wn;
                    if (h0) {
                        ca[i0] = c * x0 - sn * y0;
                        cb[i0] = sn * x0 + c * y0;
                        va[i0] = c * p0 - sn * q0;
                        vb[i0] = sn * p0 + c * q0;
                    }
                    if (h1) {
                        ca[i1] = c * x1 - sn * y1;
                        cb[i1] = sn * x1 + c * y1;
                        va[i1] = c * p1 - sn * q1;
                        vb[i1] = sn * p1 + c * q1;
                    }
                    rot = true;
                }
            }
            __syncthreads();
        }
        if (rot && lane == 0) s_rot = 1;
        __syncthreads();
        const int any = s_rot;
        __syncthreads();
        if (!any) break;
    }
    // singular values and descending order
    for (int j = w; j < K; j += NW) {
        double s = 0.0;
        for (int i = lane; i < K; i += 32) s += C[i + j * KA_MAX] * C[i + j * KA_MAX];
        s = warp_sum(s);
        if (lane == 0) sigma[j] = sqrt(s);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i < K; ++i) ord[i] = i;
        for (int i = 1; i < K; ++i) {  // insertion sort, stable
            int x = ord[i];
            int j = i - 1;
            while (j >= 0 && sigma[ord[j]] < sigma[x]) {
                ord[j + 1] = ord[j];
                --j;
            }
            ord[j + 1] = x;
        }
    }
    __syncthreads();
    return sweep;
}

// rule 0: count sigma > eps * sigma_1 (hmatrix.py:297-300, build);
// rule 1: smallest r with ||s[r:]|| <= eps ||s|| (hops.py:124-131, H-arithmetic).
__device__ __forceinline__ int truncation_rank(const double *sigma, const int *ord, int K, int rule,
                                               double eps) {
    if (K == 0) return 0;
    if (rule == 0) {
        double s1 = sigma[ord[0]];
        if (s1 == 0.0) return 0;
        int r = 0;
        for (int i = 0; i < K; ++i) r += sigma[ord[i]] > eps * s1 ? 1 : 0;
        return r;
    }
    double tot = 0.0;
    for (int i = 0; i < K; ++i) tot += sigma[ord[i]] * sigma[ord[i]];
    tot = sqrt(tot);
    if (tot == 0.0) return 0;
    double tail = 0.0;
    int r = K;
    // tails from the end: tail_r = sqrt(sum_{i>=r} s_i^2); smallest r with tail_r <= eps*tot
    for (int i = K; i >= 0; --i) {
        if (i < K) tail += sigma[ord[i]] * sigma[ord[i]];
        if (sqrt(tail) <= eps * tot) r = i;
    }
    return r;
}

// out[i, c] = sum_l Q[i, l] * Cm[l, c] for c < r (row-wise; in place if out == Q is safe).
__device__ static void apply_coeffs(const double *Q, i64 ldq, i64 m, int K, const double *Cm, int ldc,
                             int r, double *out, i64 ldo) {
    for (i64 i = threadIdx.x; i < m; i += NT) {
        double acc[KC_MAX];
#pragma unroll
        for (int c = 0; c < KC_MAX; ++c) acc[c] = 0.0;
        for (int l0 = 0; l0 < K; l0 += 8) {
            // 8 independent loads of the row before they are consumed
            double q[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) q[j] = l0 + j < K ? Q[i + (i64)(l0 + j) * ldq] : 0.0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (l0 + j >= K) break;
#pragma unroll
                for (int c = 0; c < KC_MAX; ++c)
                    if (c < r) acc[c] += q[j] * Cm[l0 + j + c * ldc];
            }
        }
#pragma unroll
        for (int c = 0; c < KC_MAX; ++c)
            if (c < r) out[i + (i64)c * ldo] = acc[c];
    }
}

// Shared workspace of one recompression.
struct RecompSmem {
    double Ru[KA_MAX * KA_MAX];
    double Rv[KA_MAX * KA_MAX];
    double Cc[KA_MAX * KA_MAX];
    double sigma[KA_MAX];
    double h[KA_MAX];
    double red[2 * NW];
    i64 redi[NW];
    int ord[KA_MAX];
};

// Recompress U V^T (U: m x K, V: n x K, column-major) -> U' V'^T of rank r by
// QR(U), QR(V), SVD(Ru Rv^T), truncation `rule` at `eps`.  U and V are
// overwritten by their Q factors.  If r <= rmax, writes U' = Qu (W_r S_r) to uo and
// V' = Qv Z_r to vo (uo/vo may alias U/V).  Returns r (possibly > rmax: not written).
// Mirrors hops.py:134-144 (rule 1) and hmatrix.py:294-303 (rule 0).
__device__ static int recompress(double *U, i64 ldu, i64 m, double *V, i64 ldv, i64 n, int K, int rule,
                          double eps, double *uo, i64 ldo_u, double *vo, i64 ldo_v, int rmax,
                          RecompSmem &S) {
    if (K == 0) return 0;
    cgs2(U, ldu, m, K, S.Ru, S.h, S.red);
    cgs2(V, ldv, n, K, S.Rv, S.h, S.red);
    // C = Ru Rv^T (K x K)
    for (int e = threadIdx.x; e < K * K; e += NT) {
        int i = e % K, j = e / K;
        double s = 0.0;
        for (int l = 0; l < K; ++l) s += S.Ru[i + l * KA_MAX] * S.Rv[j + l * KA_MAX];
        S.Cc[i + j * KA_MAX] = s;
    }
    __syncthreads();
    // Jacobi: C <- C Z, Z accumulated in Rv (Rv no longer needed), Ru free for coeffs
    jacobi_svd(S.Cc, S.Rv, K, S.sigma, S.ord, S.red);
    int r = truncation_rank(S.sigma, S.ord, K, rule, eps);
    if (r > rmax) return r;
    // coefficient matrices: Cu[:, c] = (C Z)[:, ord[c]], Cv[:, c] = Z[:, ord[c]]
    for (int e = threadIdx.x; e < K * r; e += NT) {
        int l = e % K, c = e / K;
        S.Ru[l + c * KA_MAX] = S.Cc[l + S.ord[c] * KA_MAX];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < K * r; e += NT) {
        int l = e % K, c = e / K;
        S.Cc[l + c * KA_MAX] = S.Rv[l + S.ord[c] * KA_MAX];
    }
    __syncthreads();
    apply_coeffs(U, ldu, m, K, S.Ru, KA_MAX, r, uo, ldo_u);
    apply_coeffs(V, ldv, n, K, S.Cc, KA_MAX, r, vo, ldo_v);
    __syncthreads();
    return r;
}

}  // namespace dev
}  // namespace lh
