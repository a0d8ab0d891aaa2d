// Persistent dataflow executor for the static H-arithmetic DAG (plan.cpp) and
// the host drivers of H-LU (hops.py:392-421), solve (hops.py:424-432), the
// triangular-inverse factors of the fast solve, and the CN stepping loop
// (levy.py:309-330).
//
// One 256-thread CTA per SM claims tasks in the planner's (critical-path
// ordered, topological) order from a global counter, spins until every
// predecessor has published its completion flag, runs the task, then
// publishes its own flag with release semantics.  All CTAs are co-resident
// (cooperative launch), so the claim order guarantees progress.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <future>

#include "core.h"
#include "dev.cuh"
#include "matvec.h"
#include "h2step.h"
#include "plan_impl.h"

namespace lh {

using dev::KA_MAX;
using dev::KC_MAX;
using dev::NT;

struct ExecArgs {
    const DTask *tasks;
    int32_t ntasks;
    const int32_t *deps;
    const DPiece *pieces;
    int32_t *done;
    int32_t *heads;      // per bucket: next FIFO slot to take
    int32_t *tails;      // per bucket: next FIFO slot to fill
    int32_t *done_count; // finished tasks
    const int32_t *qoff; // per bucket: offset of its FIFO in `queue`
    int32_t *queue;      // ready FIFOs (task ids, -1 = not yet filled)
    int32_t *remaining;  // unfinished predecessors per task
    const int32_t *succ_beg, *succ;  // successor CSR, entries = task | bucket << SUCC_SHIFT
    int32_t *err;  // [0] code, [1] task, [2] path
    double *base[NBASE];
    int32_t *ranks;
    int32_t *perm;
    unsigned long long *times;  // optional: [2*t] start (deps met), [2*t+1] end (globaltimer ns)
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

constexpr int SMEM_BYTES = 168 * 1024;
constexpr unsigned POLL_NS_MAX = 128;
constexpr int SUCC_SHIFT = 28;
constexpr int SUCC_MASK = (1 << SUCC_SHIFT) - 1;

__device__ __forceinline__ double *vp(const ExecArgs &A, const DView &v) { return A.base[v.base] + v.off; }
__device__ __forceinline__ i64 vi(const DView &v, i64 i, i64 j) {
    return v.trans ? j + i * (i64)v.ld : i + j * (i64)v.ld;
}
__device__ __forceinline__ int vcols(const ExecArgs &A, const DView &v) {
    return v.wslot >= 0 ? A.ranks[v.wslot] : v.cols;
}
__device__ __forceinline__ void set_err(const ExecArgs &A, int code, int task, int path) {
    if (atomicCAS(&A.err[0], 0, code) == 0) {
        A.err[1] = task;
        A.err[2] = path;
    }
}
__device__ __forceinline__ int ld_acquire(const int32_t *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int32_t *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------------------
// GETRF fast path (m <= 64): right-looking LU with partial pivoting held in registers,
// thread (row tx = t % 64, columns ty + 4 q, q < 16); per column one warp-shuffle pivot search
// on the two warps owning the column, the pivot row / old row j / column j exchanged through
// shared memory, two barriers.  The arithmetic is LAPACK dgetf2's (reciprocal pivot scaling,
// rank-1 update).  Then the packed leaf inverse P = strict_lower(L^-1) + upper(U^-1) by a
// blocked inversion (8 x 8 diagonal blocks by substitution, then seven block diagonals),
// L^-1 and U^-1 concurrently on the two halves of the CTA.  The leaf is padded to 64 x 64
// with the identity.
// ---------------------------------------------------------------------------
constexpr int LD65 = 65;  // odd leading dimension: conflict-free column and row walks

__device__ void task_getrf64(const ExecArgs &A, const DTask &T, int tid, double *sm) {
    const DView &v = T.v[0];
    const int m = v.rows;
    double *G = vp(A, v);
    double *S = sm;                       // LU factors, 64 x 64 padded, ld 65
    double *Li = sm + 64 * LD65;          // L^-1 (unit lower)
    double *Ui = sm + 2 * 64 * LD65;      // U^-1 (upper)
    double *Tw = sm + 3 * 64 * LD65;      // block-product workspace, 2 x 512
    double *prow = Tw + 1024, *jrow = prow + 64, *colj = jrow + 64;
    int *piv = (int *)(colj + 64);
    __shared__ double s_cv[2];
    __shared__ int s_ci[2];
    const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
    const int lane = threadIdx.x & 31;
    // Speculative pass without row exchanges: partial pivoting keeps every diagonal pivot iff
    // |a_jj| >= |a_ij| (i > j) at every step, which is checked exactly on the values the
    // pivoted algorithm would compare; then the factors are bit-identical to it (same
    // operations in the same order).  No leaf of the SURVEY a16 operators pivots.  Layout:
    // row t >> 2, columns (t & 3) + 4 q, so a row's four threads are adjacent lanes and the
    // column-j value reaches them by one shuffle; one barrier per column.
    bool spec_ok;
    {
        const int tr = threadIdx.x >> 2, tc = threadIdx.x & 3;
        double b[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int c = tc + 4 * q;
            b[q] = (tr < m && c < m) ? G[tr + c * (i64)v.ld] : (tr == c ? 1.0 : 0.0);
        }
        // columns in groups of four share the register index q = j / 4, so with the group
        // loop unrolled every register index and column comparison is a compile-time
        // constant: a step is (16 - j/4) DFMAs fed by 128-bit shared loads of row j
        // (stored [thread column][q], i.e. each thread's 16 values contiguous)
        bool ok = true;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int j = 4 * k + jj;
                if (j < m) {
                    double *Pj = Tw + (j & 1) * 64;  // double-buffered row j
                    if (tr == j) {
#pragma unroll
                        for (int q = k; q < 16; q += 2)
                            *reinterpret_cast<double2 *>(Pj + tc * 16 + q - (q & 1)) =
                                make_double2((q & 1) ? b[q - 1] : b[q], (q & 1) ? b[q] : b[q + 1]);
                    }
                    __syncthreads();
                    const double lv = __shfl_sync(0xffffffffu, b[k], (lane & ~3) | jj);
                    if (tr > j && tr < m) {
                        const double d = Pj[jj * 16 + k];
                        ok = ok && (d != 0.0 ? fabs(lv) <= fabs(d) : lv == 0.0);
                        const double l = d != 0.0 ? lv * (1.0 / d) : lv;
                        // q == k: column tc + 4k, updated if tc > jj, the multiplier if tc == jj
                        const double pk = Pj[tc * 16 + k];
                        if (tc > jj) b[k] -= l * pk;
                        else if (tc == jj) b[k] = l;
#pragma unroll
                        for (int q = (k + 1) & ~1; q < 16; q += 2) {
                            const double2 pr = *reinterpret_cast<const double2 *>(Pj + tc * 16 + q);
                            if (q > k) b[q] -= l * pr.x;
                            b[q + 1] -= l * pr.y;
                        }
                    }
                }
            }
        }
        spec_ok = __syncthreads_and(ok);
        if (spec_ok) {
#pragma unroll
            for (int q = 0; q < 16; ++q) S[tr + (tc + 4 * q) * LD65] = b[q];
            if (threadIdx.x < 64) piv[threadIdx.x] = threadIdx.x;
        }
    }
    double a[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int c = ty + 4 * q;
        a[q] = (tx < m && c < m) ? G[tx + c * (i64)v.ld] : (tx == c ? 1.0 : 0.0);
    }
    for (int j = 0; j < m && !spec_ok; ++j) {
        const int jt = j & 3, jq = j >> 2;
        if (ty == jt) {  // idamax over rows j..m-1 of column j, first index on ties
            double best = -1.0;
            int bi = j;
#pragma unroll
            for (int q = 0; q < 16; ++q)
                if (q == jq && tx >= j && tx < m) {
                    best = fabs(a[q]);
                    bi = tx;
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
            if (lane == 0) {
                s_cv[tx >> 5] = best;
                s_ci[tx >> 5] = bi;
            }
        }
        __syncthreads();
        const int p = (s_cv[1] > s_cv[0] || (s_cv[1] == s_cv[0] && s_ci[1] < s_ci[0])) ? s_ci[1] : s_ci[0];
        if (tx == p) {
#pragma unroll
            for (int q = 0; q < 16; ++q) prow[ty + 4 * q] = a[q];
        }
        if (tx == j && p != j) {
#pragma unroll
            for (int q = 0; q < 16; ++q) jrow[ty + 4 * q] = a[q];
        }
        if (ty == jt) {
#pragma unroll
            for (int q = 0; q < 16; ++q)
                if (q == jq) colj[tx] = a[q];
        }
        __syncthreads();
        if (p != j) {  // swap rows j and p
            if (tx == j) {
#pragma unroll
                for (int q = 0; q < 16; ++q) a[q] = prow[ty + 4 * q];
            } else if (tx == p) {
#pragma unroll
                for (int q = 0; q < 16; ++q) a[q] = jrow[ty + 4 * q];
            }
        }
        if (tx > j && tx < m) {
            const double d = prow[j];
            const double lv = (tx == p) ? jrow[j] : colj[tx];
            const double l = d != 0.0 ? lv * (1.0 / d) : lv;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int c = ty + 4 * q;
                if (c > j) a[q] -= l * prow[c];
                else if (c == j) a[q] = l;
            }
        }
        if (threadIdx.x == 0) piv[j] = p;
    }
    if (!spec_ok) {
#pragma unroll
        for (int q = 0; q < 16; ++q) S[tx + (ty + 4 * q) * LD65] = a[q];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < m * m; e += NT) G[e % m + (e / m) * (i64)v.ld] = S[(e % m) + (e / m) * LD65];
    if (threadIdx.x == 0) {
        int32_t *pp = A.perm + T.aux;
        for (int i = 0; i < m; ++i) pp[i] = i;
        for (int i = 0; i < m; ++i) {
            int q = piv[i];
            if (q != i) {
                int t = pp[i];
                pp[i] = pp[q];
                pp[q] = t;
            }
        }
        for (int i = 0; i < m; ++i)
            if (S[i + i * LD65] == 0.0) {
                set_err(A, LH_ESINGULAR, tid, T.path);
                break;
            }
    }
    if (!(T.flags & 1)) return;
    // ---- blocked inverses of the padded factors: threads 0..127 L^-1, 128..255 U^-1
    const bool up = threadIdx.x >= 128;
    const int u = threadIdx.x & 127;
    double *X = up ? Ui : Li;
    double *Tp = Tw + (up ? 512 : 0);
    for (int e = u; e < 64 * 64; e += 128) X[(e & 63) + (e >> 6) * LD65] = 0.0;
    __syncthreads();
    if (u < 64) {  // diagonal 8 x 8 blocks: one column of one block per thread
        const int bi = u >> 3, cc = u & 7, o = 8 * bi;
        double x[8];
        if (!up) {  // unit lower: x[r] = e_cc[r] - sum_{s<r} L[r][s] x[s]
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                double t = (r == cc) ? 1.0 : 0.0;
#pragma unroll
                for (int s2 = 0; s2 < 8; ++s2)
                    if (s2 < r) t -= S[o + r + (o + s2) * LD65] * x[s2];
                x[r] = t;
            }
        } else {  // upper: x[r] = (e_cc[r] - sum_{s>r} U[r][s] x[s]) / U[r][r]
#pragma unroll
            for (int r = 7; r >= 0; --r) {
                double t = (r == cc) ? 1.0 : 0.0;
#pragma unroll
                for (int s2 = 0; s2 < 8; ++s2)
                    if (s2 > r) t -= S[o + r + (o + s2) * LD65] * x[s2];
                x[r] = t / S[o + r + (o + r) * LD65];
            }
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) X[o + r + (o + cc) * LD65] = x[r];
    }
    __syncthreads();
    for (int d = 1; d < 8; ++d) {
        const int nblk = 8 - d;  // blocks (i, i - d) of L^-1 / (i, i + d) of U^-1, i < nblk
        // T = sum_k F_ik X_kj over the d source blocks between the block's row and column
        for (int e = u; e < nblk * 64; e += 128) {
            const int bk = e >> 6, r = (e >> 3) & 7, c = e & 7;
            double t = 0.0;
            if (!up) {
                const int i = bk + d, j = bk;  // L: k = j .. i-1
                for (int k = j; k < i; ++k)
#pragma unroll
                    for (int s2 = 0; s2 < 8; ++s2)
                        t += S[8 * i + r + (8 * k + s2) * LD65] * X[8 * k + s2 + (8 * j + c) * LD65];
            } else {
                const int i = bk, j = bk + d;  // U: k = i+1 .. j
                for (int k = i + 1; k <= j; ++k)
#pragma unroll
                    for (int s2 = 0; s2 < 8; ++s2)
                        t += S[8 * i + r + (8 * k + s2) * LD65] * X[8 * k + s2 + (8 * j + c) * LD65];
            }
            Tp[e] = t;
        }
        __syncthreads();
        // X_ij = -X_ii T
        for (int e = u; e < nblk * 64; e += 128) {
            const int bk = e >> 6, r = (e >> 3) & 7, c = e & 7;
            const int i = up ? bk : bk + d, j = up ? bk + d : bk;
            double t = 0.0;
#pragma unroll
            for (int s2 = 0; s2 < 8; ++s2) t += X[8 * i + r + (8 * i + s2) * LD65] * Tp[(bk << 6) + (s2 << 3) + c];
            X[8 * i + r + (8 * j + c) * LD65] = -t;
        }
        __syncthreads();
    }
    double *Pg = A.base[T.v[1].base] + T.v[1].off;
    for (int e = threadIdx.x; e < m * m; e += NT) {
        int i = e % m, c = e / m;
        Pg[e] = (i > c) ? Li[i + c * LD65] : Ui[i + c * LD65];
    }
}

// ---------------------------------------------------------------------------
// Register-tiled small GEMM helpers: thread (row tx = t % 64, column group ty = t / 64)
// owns columns c0 + ty + 4q, q < NQ.  Operands stream through L1 (row-coalesced), no
// shared-memory staging and no barriers; NQ is picked from the column count.
// ---------------------------------------------------------------------------
struct Strided {  // element (i, j) at p[i * si + j * sj]
    const double *p;
    i64 si, sj;
};
__device__ __forceinline__ Strided strided(const ExecArgs &A, const DView &v) {
    Strided s;
    s.p = A.base[v.base] + v.off;
    s.si = v.trans ? v.ld : 1;
    s.sj = v.trans ? 1 : v.ld;
    return s;
}

// acc[q] += sum_{j in [j0, j1)} M(tx, j) * X(xrow(j), c0 + ty + 4q)
template <int NQ>
__device__ __forceinline__ void tile_fma(double (&acc)[NQ], const Strided &M, int tx, int j0, int j1,
                                         const Strided &X, const int32_t *xperm, int c0, int ty,
                                         int kc) {
    const double *mrow = M.p + tx * M.si;
    int cidx[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) cidx[q] = min(c0 + ty + 4 * q, c0 + kc - 1);  // clamp: always valid
    int j = j0;
    for (; j + 2 <= j1; j += 2) {
        const double a0 = mrow[j * M.sj], a1 = mrow[(j + 1) * M.sj];
        const i64 r0 = xperm ? xperm[j] : j, r1 = xperm ? xperm[j + 1] : j + 1;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const double x0 = X.p[r0 * X.si + cidx[q] * X.sj];
            const double x1 = X.p[r1 * X.si + cidx[q] * X.sj];
            acc[q] += a0 * x0 + a1 * x1;
        }
    }
    if (j < j1) {
        const double a0 = mrow[j * M.sj];
        const i64 r0 = xperm ? xperm[j] : j;
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] += a0 * X.p[r0 * X.si + cidx[q] * X.sj];
    }
}

// ---------------------------------------------------------------------------
// cp.async staging: copies carry no register result, so every copy of a tile issues
// back to back and the tile costs one memory round trip (a load->store loop would
// serialise one round trip per element).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp8(double *smem, const double *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// stage a (rows x cols) view into smem at dst[i + j * lds] (optionally row-permuted source)
__device__ __forceinline__ void stage_view(double *dst, int lds, const Strided &S, int rows, int cols,
                                           int col0, const int32_t *rperm) {
    for (int e = threadIdx.x; e < rows * cols; e += NT) {
        const int i = e % rows, j = e / rows;
        const i64 ri = rperm ? rperm[i] : i;
        cp8(dst + i + j * lds, S.p + ri * S.si + (i64)(col0 + j) * S.sj);
    }
}

// TRSM via the packed leaf inverse (m <= 64): P and B staged with cp.async, product from
// shared memory, written back in place (all reads of B precede the writes).
template <int NQ>
__device__ void trsm_inv_staged(const ExecArgs &A, const DTask &T, int k, double *sm) {
    const DView &bv = T.v[1];
    const DView &iv = T.v[2];
    const int m = iv.rows;
    const int mode = T.flags & 15;
    const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
    double *Ps = sm;               // m x m, ld 65
    double *Bs = sm + 64 * LD65;   // m x 64, ld 65
    const Strided Pg = strided(A, iv);
    const Strided Bg = strided(A, bv);
    const int32_t *perm = mode == 0 ? A.perm + T.aux : nullptr;
    double *Bw = vp(A, bv);
    stage_view(Ps, LD65, Pg, m, m, 0, nullptr);
    for (int c0 = 0; c0 < k; c0 += 4 * NQ) {
        const int kc = min(4 * NQ, k - c0);
        stage_view(Bs, LD65, Bg, m, kc, c0, perm);
        cp_commit();
        cp_wait<0>();
        __syncthreads();
        double acc[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
        int cq[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) cq[q] = min(ty + 4 * q, kc - 1) * LD65;
        if (tx < m) {
            if (mode == 0) {
                for (int l = 0; l < tx; ++l) {
                    const double a = Ps[tx + l * LD65];
#pragma unroll
                    for (int q = 0; q < NQ; ++q) acc[q] += a * Bs[l + cq[q]];
                }
#pragma unroll
                for (int q = 0; q < NQ; ++q) acc[q] += Bs[tx + cq[q]];
            } else if (mode == 1) {
                for (int l = tx; l < m; ++l) {
                    const double a = Ps[tx + l * LD65];
#pragma unroll
                    for (int q = 0; q < NQ; ++q) acc[q] += a * Bs[l + cq[q]];
                }
            } else {
                for (int l = 0; l <= tx; ++l) {
                    const double a = Ps[l + tx * LD65];
#pragma unroll
                    for (int q = 0; q < NQ; ++q) acc[q] += a * Bs[l + cq[q]];
                }
            }
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int c = ty + 4 * q;
                if (c < kc) Bw[vi(bv, tx, c0 + c)] = acc[q];
            }
        }
        __syncthreads();  // Bs reused by the next column chunk
    }
}

// TRSM via the packed leaf inverse, register-tiled: out = op(T^-1) P B (in place on B)
template <int NQ>
__device__ void trsm_inv_tiled(const ExecArgs &A, const DTask &T, int k) {
    const DView &bv = T.v[1];
    const DView &iv = T.v[2];
    const int m = iv.rows;
    const int mode = T.flags & 15;
    const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
    Strided Pm = strided(A, iv);
    if (mode == 2) {  // U^-T: M(i, l) = P(l, i)
        Pm.si = iv.ld;
        Pm.sj = 1;
    }
    const Strided B = strided(A, bv);
    const int32_t *perm = mode == 0 ? A.perm + T.aux : nullptr;
    double *Bw = vp(A, bv);
    for (int c0 = 0; c0 < k; c0 += 4 * NQ) {
        const int kc = min(4 * NQ, k - c0);
        double acc[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
        if (tx < m) {
            if (mode == 0) {
                tile_fma<NQ>(acc, Pm, tx, 0, tx, B, perm, c0, ty, kc);   // strict lower of L^-1
                const i64 rp = perm[tx];                                    // unit diagonal
#pragma unroll
                for (int q = 0; q < NQ; ++q)
                    acc[q] += B.p[rp * B.si + min(c0 + ty + 4 * q, c0 + kc - 1) * B.sj];
            } else if (mode == 1) {
                tile_fma<NQ>(acc, Pm, tx, tx, m, B, nullptr, c0, ty, kc);
            } else {
                tile_fma<NQ>(acc, Pm, tx, 0, tx + 1, B, nullptr, c0, ty, kc);
            }
        }
        __syncthreads();  // every read of this column chunk of B precedes the in-place write
        if (tx < m) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int c = ty + 4 * q;
                if (c < kc) Bw[vi(bv, tx, c0 + c)] = acc[q];
            }
        }
        __syncthreads();
    }
}

__device__ void task_trsm_fast(const ExecArgs &A, const DTask &T, double *sm) {
    const int k = vcols(A, T.v[1]);
    if (k <= 0) return;
    if (k <= 8) trsm_inv_staged<2>(A, T, k, sm);
    else if (k <= 16) trsm_inv_staged<4>(A, T, k, sm);
    else if (k <= 32) trsm_inv_staged<8>(A, T, k, sm);
    else trsm_inv_staged<16>(A, T, k, sm);
}

// TRSM through the packed leaf inverse: B <- op(T^-1) P B as a small GEMM
// (mode 0: L^-1 with the leaf permutation; 1: U^-1; 2: U^-T).
__device__ void task_trsm_inv(const ExecArgs &A, const DTask &T, double *sm) {
    const DView &bv = T.v[1];
    const DView &iv = T.v[2];
    const int m = iv.rows;
    const int mode = T.flags & 15;
    const double *Pg = A.base[iv.base] + iv.off;
    double *Bg = vp(A, bv);
    const int k = vcols(A, bv);
    if (k <= 0) return;
    double *Ps = sm;                 // m x m, ld 65
    double *Bs = sm + 64 * LD65;     // m x 64, ld 65
    const int32_t *perm = A.perm + T.aux;
    for (int e = threadIdx.x; e < m * m; e += NT) Ps[(e % m) + (e / m) * LD65] = Pg[e];
    const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
    for (int c0 = 0; c0 < k; c0 += 64) {
        const int kc = min(64, k - c0);
        __syncthreads();
        for (int e = threadIdx.x; e < m * kc; e += NT) {
            int i = e % m, c = e / m;
            int src = (mode == 0) ? perm[i] : i;
            Bs[i + c * LD65] = Bg[vi(bv, src, c0 + c)];
        }
        __syncthreads();
        double acc[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) acc[q] = 0.0;
        if (tx < m) {
            if (mode == 0) {
                for (int l = 0; l < tx; ++l) {
                    const double a = Ps[tx + l * LD65];
#pragma unroll
                    for (int q = 0; q < 16; ++q) acc[q] += a * Bs[l + (ty + 4 * q) * LD65];
                }
#pragma unroll
                for (int q = 0; q < 16; ++q) acc[q] += Bs[tx + (ty + 4 * q) * LD65];
            } else if (mode == 1) {
                for (int l = tx; l < m; ++l) {
                    const double a = Ps[tx + l * LD65];
#pragma unroll
                    for (int q = 0; q < 16; ++q) acc[q] += a * Bs[l + (ty + 4 * q) * LD65];
                }
            } else {
                for (int l = 0; l <= tx; ++l) {
                    const double a = Ps[l + tx * LD65];
#pragma unroll
                    for (int q = 0; q < 16; ++q) acc[q] += a * Bs[l + (ty + 4 * q) * LD65];
                }
            }
        }
        __syncthreads();
        if (tx < m) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int c = ty + 4 * q;
                if (c < kc) Bg[vi(bv, tx, c0 + c)] = acc[q];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// GETRF: partial pivoting LU of a dense m x m leaf (sla.lu_factor, hops.py:394)
// ---------------------------------------------------------------------------
__device__ void task_getrf(const ExecArgs &A, const DTask &T, int tid, double *sm) {
    const DView &v = T.v[0];
    const int m = v.rows;
    if (m <= 64 && !v.trans) {
        task_getrf64(A, T, tid, sm);
        return;
    }
    double *G = vp(A, v);
    double *S = sm;                       // m x m, column-major
    int *piv = (int *)(sm + m * m);
    __shared__ int s_p;
    for (int e = threadIdx.x; e < m * m; e += NT) S[e] = G[vi(v, e % m, e / m)];
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = 0; j < m; ++j) {
        // pivot: first index of max |A[i, j]|, i >= j (idamax)
        if (w == 0) {
            double best = -1.0;
            int bi = j;
            for (int i = j + lane; i < m; i += 32) {
                double a = fabs(S[i + j * m]);
                if (a > best) {
                    best = a;
                    bi = i;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                double ob = __shfl_xor_sync(0xffffffffu, best, o);
                int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) {
                    best = ob;
                    bi = oi;
                }
            }
            if (lane == 0) {
                s_p = bi;
                piv[j] = bi;
            }
        }
        __syncthreads();
        const int p = s_p;
        if (p != j)
            for (int c = threadIdx.x; c < m; c += NT) {
                double t = S[j + c * m];
                S[j + c * m] = S[p + c * m];
                S[p + c * m] = t;
            }
        __syncthreads();
        const double d = S[j + j * m];
        if (d != 0.0)
            for (int i = j + 1 + threadIdx.x; i < m; i += NT) S[i + j * m] /= d;
        __syncthreads();
        const int rem = m - j - 1;
        for (int e = threadIdx.x; e < rem * rem; e += NT) {
            int i = j + 1 + e % rem, c = j + 1 + e / rem;
            S[i + c * m] -= S[i + j * m] * S[j + c * m];
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < m * m; e += NT) G[vi(v, e % m, e / m)] = S[e];
    if (threadIdx.x == 0) {
        // net permutation P^T b == b[perm] (hops.py:171-177)
        int32_t *pp = A.perm + T.aux;
        for (int i = 0; i < m; ++i) pp[i] = i;
        for (int i = 0; i < m; ++i) {
            int q = piv[i];
            if (q != i) {
                int t = pp[i];
                pp[i] = pp[q];
                pp[q] = t;
            }
        }
        for (int i = 0; i < m; ++i)
            if (S[i + i * m] == 0.0) {
                set_err(A, LH_ESINGULAR, tid, T.path);
                break;
            }
    }
}

// ---------------------------------------------------------------------------
// TRSM with a factored leaf: mode 0 unit-L with the leaf permutation, 1 U, 2 U^T
// (dtrsm in _leaf_solve, hops.py:185-208)
// ---------------------------------------------------------------------------
// generic TRSM (any m whose triangle fits shared memory): flags = mode | unit << 4 |
// pivots << 5 | packed-inverse << 6 | check-diagonal << 7.  Mode 0 solves with the lower
// triangle (unit or not, leaf pivots applied to B for LU-factored leaves), 1 with the upper
// triangle, 2 with its transpose (_leaf_solve, hops.py:191-208).
__device__ void task_trsm(const ExecArgs &A, const DTask &T, int tid, double *sm) {
    if (T.flags & 64) {
        task_trsm_fast(A, T, sm);
        return;
    }
    const DView &tv = T.v[0];
    const DView &bv = T.v[1];
    const int m = tv.rows;
    const int mode = T.flags & 15;
    const double *Tg = vp(A, tv);
    double *Bg = vp(A, bv);
    const int k = vcols(A, bv);
    if (k <= 0) return;
    double *Ts = sm;
    double *Bs = sm + m * m;
    const bool unit = T.flags & 16, pivots = T.flags & 32;
    const int32_t *perm = A.perm + T.aux;
    for (int e = threadIdx.x; e < m * m; e += NT) Ts[e] = Tg[vi(tv, e % m, e / m)];
    if (T.flags & 128) {  // _check_triangular_leaf (hops.py:179-182): zero on the diagonal
        __shared__ int s_zero;
        if (threadIdx.x == 0) s_zero = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += NT)
            if (Ts[i + i * m] == 0.0) s_zero = 1;
        __syncthreads();
        if (s_zero) {
            if (threadIdx.x == 0) set_err(A, LH_ESINGULAR, tid, T.path);
            return;
        }
    }
    const int CW = 32;
    for (int c0 = 0; c0 < k; c0 += CW) {
        const int kc = min(CW, k - c0);
        __syncthreads();
        for (int e = threadIdx.x; e < m * kc; e += NT) {
            int i = e % m, c = e / m;
            int src = (mode == 0 && pivots) ? perm[i] : i;
            Bs[e] = Bg[vi(bv, src, c0 + c)];
        }
        __syncthreads();
        if (mode == 0) {
            for (int l = 0; l < m - 1 + (unit ? 0 : 1); ++l) {
                if (!unit) {
                    for (int c = threadIdx.x; c < kc; c += NT) Bs[l + c * m] /= Ts[l + l * m];
                    __syncthreads();
                }
                const int rem = m - l - 1;
                for (int e = threadIdx.x; e < rem * kc; e += NT) {
                    int i = l + 1 + e % rem, c = e / rem;
                    Bs[i + c * m] -= Ts[i + l * m] * Bs[l + c * m];
                }
                __syncthreads();
            }
        } else if (mode == 1) {
            for (int l = m - 1; l >= 0; --l) {
                if (!unit) {
                    for (int c = threadIdx.x; c < kc; c += NT) Bs[l + c * m] /= Ts[l + l * m];
                    __syncthreads();
                }
                for (int e = threadIdx.x; e < l * kc; e += NT) {
                    int i = e % l, c = e / l;
                    Bs[i + c * m] -= Ts[i + l * m] * Bs[l + c * m];
                }
                __syncthreads();
            }
        } else {
            for (int l = 0; l < m; ++l) {
                if (!unit) {
                    for (int c = threadIdx.x; c < kc; c += NT) Bs[l + c * m] /= Ts[l + l * m];
                    __syncthreads();
                }
                const int rem = m - l - 1;
                for (int e = threadIdx.x; e < rem * kc; e += NT) {
                    int i = l + 1 + e % rem, c = e / rem;
                    Bs[i + c * m] -= Ts[l + i * m] * Bs[l + c * m];
                }
                __syncthreads();
            }
        }
        for (int e = threadIdx.x; e < m * kc; e += NT) Bg[vi(bv, e % m, c0 + e / m)] = Bs[e];
    }
}

// ---------------------------------------------------------------------------
// SEGMUL: Y_seg = beta Y_seg + alpha * sum of pieces (mul_dense/tmul_dense rows)
// ---------------------------------------------------------------------------
// fast path: Y segment of <= 64 rows, no transposed operands; each piece's X rows (or
// W) staged in shared memory, the piece's rows streamed from global (coalesced), 16
// accumulators per thread (row t % 64, columns t / 64 + 4q).
__device__ void task_segmul_fast(const ExecArgs &A, const DTask &T, double *sm) {
    const DView &yv = T.v[0];
    const int s = yv.rows;
    const int k = vcols(A, yv);
    double *Yg = vp(A, yv);
    const bool overwrite = T.flags & 1;
    const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
    double *Xs = sm;
    for (int c0 = 0; c0 < k; c0 += 64) {
        const int kc = min(64, k - c0);
        double acc[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) acc[q] = 0.0;
        for (int p = T.pc_beg; p < T.pc_end; ++p) {
            const DPiece pc = A.pieces[p];
            const double *M = vp(A, pc.mat);
            const double *X = vp(A, pc.x);
            const int inner = pc.kind == 0 ? pc.mat.cols : vcols(A, pc.mat);
            if (inner == 0) continue;
            __syncthreads();
            for (int e = threadIdx.x; e < inner * kc; e += NT) {
                int j = e % inner, c = e / inner;
                Xs[e] = X[j + (i64)(c0 + c) * pc.x.ld];
            }
            __syncthreads();
            if (tx < s) {
                const double *Mr = M + tx;
                const i64 ldm = pc.mat.ld;
                for (int j = 0; j < inner; ++j) {
                    const double a = Mr[j * ldm];
                    const double *xr = Xs + j;
#pragma unroll
                    for (int q = 0; q < 16; ++q) acc[q] += a * xr[(ty + 4 * q) * inner];
                }
            }
        }
        if (tx < s) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int c = ty + 4 * q;
                if (c < kc) {
                    double &y = Yg[tx + (i64)(c0 + c) * yv.ld];
                    y = (overwrite ? 0.0 : y) + T.alpha * acc[q];
                }
            }
        }
    }
}

// SEGMUL for segments of <= 64 rows whose pieces have inner dimension <= 64: each piece's
// matrix rows and X rows are staged with cp.async, double-buffered so the copies of piece
// p+1 overlap the products of piece p.
template <int NQ>
__device__ void segmul_staged(const ExecArgs &A, const DTask &T, int k, double *sm) {
    const DView &yv = T.v[0];
    const int s = yv.rows;
    const bool overwrite = T.flags & 1;
    const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
    double *Yw = vp(A, yv);
    constexpr int BUF = 2 * 64 * LD65;  // M tile + X tile
    for (int c0 = 0; c0 < k; c0 += 4 * NQ) {
        const int kc = min(4 * NQ, k - c0);
        double acc[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
        int cq[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) cq[q] = min(ty + 4 * q, kc - 1) * LD65;
        auto stage = [&](int p, int buf) {
            const DPiece pc = A.pieces[p];
            const int inner = pc.kind == 0 ? pc.mat.cols : vcols(A, pc.mat);
            double *Ms = sm + buf * BUF;
            stage_view(Ms, LD65, strided(A, pc.mat), s, inner, 0, nullptr);
            stage_view(Ms + 64 * LD65, LD65, strided(A, pc.x), inner, kc, c0, nullptr);
            cp_commit();
        };
        if (T.pc_beg < T.pc_end) stage(T.pc_beg, 0);
        for (int p = T.pc_beg; p < T.pc_end; ++p) {
            const int buf = (p - T.pc_beg) & 1;
            if (p + 1 < T.pc_end) {
                stage(p + 1, buf ^ 1);
                cp_wait<1>();
            } else {
                cp_wait<0>();
            }
            __syncthreads();
            const DPiece &pc = A.pieces[p];
            const int inner = pc.kind == 0 ? pc.mat.cols : vcols(A, pc.mat);
            const double *Ms = sm + buf * BUF;
            const double *Xs = Ms + 64 * LD65;
            if (tx < s) {
                for (int j = 0; j < inner; ++j) {
                    const double a = Ms[tx + j * LD65];
#pragma unroll
                    for (int q = 0; q < NQ; ++q) acc[q] += a * Xs[j + cq[q]];
                }
            }
            __syncthreads();  // this buffer is refilled by the stage after next
        }
        if (tx < s) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int c = ty + 4 * q;
                if (c < kc) {
                    double &y = Yw[vi(yv, tx, c0 + c)];
                    y = (overwrite ? 0.0 : y) + T.alpha * acc[q];
                }
            }
        }
    }
}

// register-tiled SEGMUL for segments of <= 64 rows: every piece (dense, transposed dense or
// low-rank U[seg] W) streamed through L1 with no staging and no barriers
template <int NQ>
__device__ void segmul_tiled(const ExecArgs &A, const DTask &T, int k) {
    const DView &yv = T.v[0];
    const int s = yv.rows;
    const bool overwrite = T.flags & 1;
    const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
    double *Yw = vp(A, yv);
    for (int c0 = 0; c0 < k; c0 += 4 * NQ) {
        const int kc = min(4 * NQ, k - c0);
        double acc[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
        if (tx < s) {
            for (int p = T.pc_beg; p < T.pc_end; ++p) {
                const DPiece &pc = A.pieces[p];
                const int inner = pc.kind == 0 ? pc.mat.cols : vcols(A, pc.mat);
                tile_fma<NQ>(acc, strided(A, pc.mat), tx, 0, inner, strided(A, pc.x), nullptr, c0,
                             ty, kc);
            }
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int c = ty + 4 * q;
                if (c < kc) {
                    double &y = Yw[vi(yv, tx, c0 + c)];
                    y = (overwrite ? 0.0 : y) + T.alpha * acc[q];
                }
            }
        }
    }
}

__device__ void task_segmul(const ExecArgs &A, const DTask &T, double *sm) {
    const DView &yv = T.v[0];
    const int s = yv.rows;
    const int k = vcols(A, yv);
    double *Yg = vp(A, yv);
    const bool overwrite = T.flags & 1;
    if (s <= 64) {
        if (k <= 0) return;
        bool small_inner = true;
        for (int p = T.pc_beg; p < T.pc_end && small_inner; ++p) {
            const DPiece &pc = A.pieces[p];
            small_inner = pc.kind == 1 || pc.mat.cols <= 64;
        }
        if (small_inner) {
            if (k <= 8) segmul_staged<2>(A, T, k, sm);
            else if (k <= 16) segmul_staged<4>(A, T, k, sm);
            else if (k <= 32) segmul_staged<8>(A, T, k, sm);
            else segmul_staged<16>(A, T, k, sm);
        } else {
            if (k <= 8) segmul_tiled<2>(A, T, k);
            else if (k <= 16) segmul_tiled<4>(A, T, k);
            else if (k <= 32) segmul_tiled<8>(A, T, k);
            else segmul_tiled<16>(A, T, k);
        }
        return;
    }
    {
        bool fast = s <= 64 && !yv.trans;
        for (int p = T.pc_beg; p < T.pc_end && fast; ++p) {
            const DPiece &pc = A.pieces[p];
            fast = !pc.mat.trans && !pc.x.trans && (pc.kind == 1 || pc.mat.cols <= 128);
        }
        if (fast) {
            task_segmul_fast(A, T, sm);
            return;
        }
    }
    const int RP = s <= 64 ? 64 : (s <= 128 ? 128 : 256);
    const int G = NT / RP;            // thread groups over columns
    const int i = threadIdx.x % RP, g = threadIdx.x / RP;
    constexpr int NA = 16;
    const int CW = NA * G;            // columns per chunk
    for (int c0 = 0; c0 < k; c0 += CW) {
        double acc[NA];
#pragma unroll
        for (int q = 0; q < NA; ++q) acc[q] = 0.0;
        for (int p = T.pc_beg; p < T.pc_end; ++p) {
            const DPiece pc = A.pieces[p];
            const double *M = vp(A, pc.mat);
            const double *X = vp(A, pc.x);
            const int inner = pc.kind == 0 ? pc.mat.cols : vcols(A, pc.mat);
            if (i < s) {
                for (int j = 0; j < inner; ++j) {
                    const double a = M[vi(pc.mat, i, j)];
#pragma unroll
                    for (int q = 0; q < NA; ++q) {
                        int c = c0 + g + q * G;
                        if (c < k) acc[q] += a * X[vi(pc.x, j, c)];
                    }
                }
            }
        }
        if (i < s) {
#pragma unroll
            for (int q = 0; q < NA; ++q) {
                int c = c0 + g + q * G;
                if (c < k) {
                    double &y = Yg[vi(yv, i, c)];
                    y = (overwrite ? 0.0 : y) + T.alpha * acc[q];
                }
            }
        }
    }
    (void)sm;
}

// ---------------------------------------------------------------------------
// VTX: W (r x k, ld KC) = F^T X, F (n x r), X (n x k)
// ---------------------------------------------------------------------------
__device__ void task_vtx(const ExecArgs &A, const DTask &T, double *sm) {
    const DView &fv = T.v[0], &xv = T.v[1], &wv = T.v[2];
    const int n = fv.rows;
    const int r = vcols(A, fv);
    const int k = vcols(A, xv);
    const double *F = vp(A, fv);
    const double *X = vp(A, xv);
    double *W = vp(A, wv);
    if (r == 0 || k == 0) return;
    constexpr int CH = 64;
    constexpr int CL = CH + 1;       // odd stride: column walks hit distinct banks
    double *Fs = sm;                 // CH x r, ld CL
    double *Xs = sm + CL * KC_MAX;   // CH x k (k <= 128), ld CL
    constexpr int NP = 16;
    const int npair = r * k;
    double acc[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) acc[q] = 0.0;
    for (int j0 = 0; j0 < n; j0 += CH) {
        const int len = min(CH, n - j0);
        __syncthreads();
        for (int e = threadIdx.x; e < len * r; e += NT) {
            int j = e % len, c = e / len;
            Fs[j + c * CL] = F[vi(fv, j0 + j, c)];
        }
        for (int e = threadIdx.x; e < len * k; e += NT) {
            int j = e % len, c = e / len;
            Xs[j + c * CL] = X[vi(xv, j0 + j, c)];
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            int p = threadIdx.x + q * NT;
            if (p < npair) {
                int l = p % r, c = p / r;
                double s = 0.0;
                const double *fa = Fs + l * CL, *xa = Xs + c * CL;
                for (int j = 0; j < len; ++j) s += fa[j] * xa[j];
                acc[q] += s;
            }
        }
    }
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        int p = threadIdx.x + q * NT;
        if (p < npair) {
            int l = p % r, c = p / r;
            W[l + c * (i64)wv.ld] = acc[q];
        }
    }
}

// ---------------------------------------------------------------------------
// LRADD: C = C + alpha U2 V2^T recompressed at eps2 (_add_lr, hops.py:134-144)
// ---------------------------------------------------------------------------
__device__ void task_lradd(const ExecArgs &A, const DTask &T, int tid, double *sm) {
    const DView &cu = T.v[0], &cv = T.v[1], &u2 = T.v[2], &v2 = T.v[3];
    const int r2 = vcols(A, u2);
    if (r2 == 0) return;
    const int slot = cu.wslot;
    const int r1 = A.ranks[slot];
    const int K = r1 + r2;
    const int kcap = cu.cols;
    const i64 m = cu.rows, n = cv.rows;
    double *U = vp(A, cu);
    double *V = vp(A, cv);
    const double *U2 = vp(A, u2);
    const double *V2 = vp(A, v2);
    dev::RecompSmem &S = *reinterpret_cast<dev::RecompSmem *>(sm);
    if (K > kcap || K > KA_MAX) {
        // wider than the block's capacity or the recompression width: the update enters in
        // column chunks, recompressing after each (kept ranks <= KC_MAX leave room for the next
        // chunk when the capacity exceeds KC_MAX: the 2D operators' H-LU)
        const int cap = min(kcap, KA_MAX), rmax = min(kcap, KC_MAX);
        const Strided U2s = strided(A, u2), V2s = strided(A, v2);
        int rc = r1, done = 0;
        while (done < r2) {
            const int q = min(r2 - done, cap - rc);
            if (q <= 0) {
                if (threadIdx.x == 0) set_err(A, LH_ERANK, tid, -1);
                return;
            }
            for (i64 e = threadIdx.x; e < m * q; e += NT)
                U[e % m + (rc + e / m) * (i64)cu.ld] = T.alpha * U2s.p[(e % m) * U2s.si + (done + e / m) * U2s.sj];
            for (i64 e = threadIdx.x; e < n * q; e += NT)
                V[e % n + (rc + e / n) * (i64)cv.ld] = V2s.p[(e % n) * V2s.si + (done + e / n) * V2s.sj];
            __syncthreads();
            const int r = dev::recompress(U, cu.ld, m, V, cv.ld, n, rc + q, 1, T.alpha2, U, cu.ld, V, cv.ld, rmax, S);
            if (r > rmax) {
                if (threadIdx.x == 0) set_err(A, LH_ERANK, tid, -1);
                return;
            }
            rc = r;
            done += q;
            __syncthreads();
        }
        if (threadIdx.x == 0) A.ranks[slot] = rc;
        return;
    }
    constexpr int RS = (int)((sizeof(dev::RecompSmem) + 15) / 8) & ~1;
    constexpr i64 ROOM = SMEM_BYTES / 8 - RS;
    if ((m + n) * K <= ROOM) {
        // staged: [U1 alpha*U2] and [V1 V2] in shared memory (one cp.async round trip),
        // recompressed there, written back once
        double *Us = sm + RS, *Vs = Us + m * K;
        const Strided U1g{U, 1, cu.ld}, V1g{V, 1, cv.ld};
        stage_view(Us, (int)m, U1g, (int)m, r1, 0, nullptr);
        stage_view(Us + m * r1, (int)m, strided(A, u2), (int)m, r2, 0, nullptr);
        stage_view(Vs, (int)n, V1g, (int)n, r1, 0, nullptr);
        stage_view(Vs + n * r1, (int)n, strided(A, v2), (int)n, r2, 0, nullptr);
        cp_commit();
        cp_wait<0>();
        __syncthreads();
        for (i64 e = threadIdx.x; e < m * r2; e += NT) Us[m * r1 + e] *= T.alpha;
        __syncthreads();
        const int rmax = min(kcap, KC_MAX);
        int r = dev::recompress(Us, m, m, Vs, n, n, K, 1, T.alpha2, Us, m, Vs, n, rmax, S);
        if (r <= rmax) {
            for (i64 e = threadIdx.x; e < m * r; e += NT) U[e % m + (e / m) * (i64)cu.ld] = Us[e];
            for (i64 e = threadIdx.x; e < n * r; e += NT) V[e % n + (e / n) * (i64)cv.ld] = Vs[e];
        }
        if (threadIdx.x == 0) {
            if (r > rmax) set_err(A, LH_ERANK, tid, -1);
            else A.ranks[slot] = r;
        }
        return;
    }
    // copies with 8 independent loads in flight per thread (a load->store loop would pay one
    // memory round trip per element)
    auto copy_cols = [&](double *dst, i64 ldd, const DView &src, i64 rows, double scale) {
        const Strided S2 = strided(A, src);
        const i64 tot = rows * r2;
        for (i64 e0 = threadIdx.x; e0 < tot; e0 += 8 * NT) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const i64 e = e0 + (i64)q * NT;
                v[q] = e < tot ? S2.p[(e % rows) * S2.si + (e / rows) * S2.sj] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const i64 e = e0 + (i64)q * NT;
                if (e < tot) dst[e % rows + (r1 + e / rows) * ldd] = scale * v[q];
            }
        }
    };
    copy_cols(U, cu.ld, u2, m, T.alpha);
    copy_cols(V, cv.ld, v2, n, 1.0);
    __syncthreads();
    int r = dev::recompress(U, cu.ld, m, V, cv.ld, n, K, 1, T.alpha2, U, cu.ld, V, cv.ld,
                            min(kcap, KC_MAX), S);
    if (threadIdx.x == 0) {
        if (r > min(kcap, KC_MAX)) set_err(A, LH_ERANK, tid, -1);
        else A.ranks[slot] = r;
    }
}

// ---------------------------------------------------------------------------
// small dense kernels
// ---------------------------------------------------------------------------
__device__ void task_dgemm(const ExecArgs &A, const DTask &T) {
    const DView &cv = T.v[0], &av = T.v[1], &bv = T.v[2];
    const bool transB = T.flags & 1, overwrite = T.flags & 2;
    const int m = cv.rows, n = cv.cols;
    const int inner = vcols(A, av);
    double *C = vp(A, cv);
    const double *Am = vp(A, av);
    const double *Bm = vp(A, bv);
    for (int e = threadIdx.x; e < m * n; e += NT) {
        int i = e % m, j = e / m;
        double s = 0.0;
        for (int l = 0; l < inner; ++l)
            s += Am[vi(av, i, l)] * (transB ? Bm[vi(bv, j, l)] : Bm[vi(bv, l, j)]);
        double &c = C[vi(cv, i, j)];
        c = (overwrite ? 0.0 : c) + T.alpha * s;
    }
}

__device__ void task_dadd(const ExecArgs &A, const DTask &T) {
    const DView &cv = T.v[0], &dv = T.v[1];
    double *C = vp(A, cv);
    const double *D = vp(A, dv);
    for (int e = threadIdx.x; e < cv.rows * cv.cols; e += NT) {
        int i = e % cv.rows, j = e / cv.rows;
        C[vi(cv, i, j)] += T.alpha * D[vi(dv, i, j)];
    }
}

__device__ void task_densify(const ExecArgs &A, const DTask &T) {
    const DView &dv = T.v[0], &sv = T.v[1], &v2 = T.v[2];
    double *D = vp(A, dv);
    const double *S = vp(A, sv);
    if (T.flags & 1) {
        const int r = vcols(A, sv);
        const double *V = vp(A, v2);
        for (int e = threadIdx.x; e < dv.rows * dv.cols; e += NT) {
            int i = e % dv.rows, j = e / dv.rows;
            double s = 0.0;
            for (int l = 0; l < r; ++l) s += S[vi(sv, i, l)] * V[vi(v2, j, l)];
            D[vi(dv, i, j)] = s;
        }
    } else {
        for (int e = threadIdx.x; e < dv.rows * dv.cols; e += NT) {
            int i = e % dv.rows, j = e / dv.rows;
            D[vi(dv, i, j)] = S[vi(sv, i, j)];
        }
    }
}

__device__ __forceinline__ double hash_normal(uint32_t seed, uint64_t i) {
    // splitmix64 -> two uniforms -> Box-Muller
    uint64_t z = (uint64_t)seed * 0x9E3779B97F4A7C15ull + i * 0xBF58476D1CE4E5B9ull + 0x94D049BB133111EBull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    double u1 = ((z >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    uint64_t y = z * 0x2545F4914F6CDD1Dull + 0x9E3779B97F4A7C15ull;
    y ^= y >> 29;
    double u2 = ((y >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

__device__ void task_rand(const ExecArgs &A, const DTask &T) {
    const DView &dv = T.v[0];
    double *D = vp(A, dv);
    for (int e = threadIdx.x; e < dv.rows * dv.cols; e += NT) {
        int i = e % dv.rows, j = e / dv.rows;
        D[vi(dv, i, j)] = hash_normal((uint32_t)T.aux, (uint64_t)e);
    }
}

// T_CHECK: fail with the task's path if any |v0| exceeds alpha
__device__ void task_check(const ExecArgs &A, const DTask &T, int tid) {
    const DView &v = T.v[0];
    const double *G = vp(A, v);
    const i64 n = (i64)v.rows * v.cols;
    bool bad = false;
    for (i64 e = threadIdx.x; e < n; e += NT) bad |= fabs(G[vi(v, e % v.rows, e / v.rows)]) > T.alpha;
    if (__syncthreads_or(bad) && threadIdx.x == 0) set_err(A, LH_EINVAL, tid, T.path);
}

__device__ void task_orth(const ExecArgs &A, const DTask &T, double *sm) {
    const DView &dv = T.v[0];
    dev::RecompSmem &S = *reinterpret_cast<dev::RecompSmem *>(sm);
    constexpr int RS = (int)((sizeof(dev::RecompSmem) + 15) / 8) & ~1;
    const i64 m = dv.rows;
    const int k = dv.cols;
    double *G = vp(A, dv);
    if (!dv.trans && m * k <= SMEM_BYTES / 8 - RS) {
        double *Ys = sm + RS;
        stage_view(Ys, (int)m, strided(A, dv), (int)m, k, 0, nullptr);
        cp_commit();
        cp_wait<0>();
        __syncthreads();
        dev::cgs2(Ys, m, m, k, S.Ru, S.h, S.red);
        for (i64 e = threadIdx.x; e < m * k; e += NT) G[e % m + (e / m) * (i64)dv.ld] = Ys[e];
        return;
    }
    dev::cgs2(G, dv.ld, m, k, S.Ru, S.h, S.red);
}

__device__ void task_ident(const ExecArgs &A, const DTask &T) {
    const DView &dv = T.v[0];
    double *D = vp(A, dv);
    const bool zero = T.flags & 1;
    const int k = vcols(A, dv);
    for (int e = threadIdx.x; e < dv.rows * k; e += NT) {
        int i = e % dv.rows, j = e / dv.rows;
        D[vi(dv, i, j)] = (!zero && i == j) ? 1.0 : 0.0;
    }
}

// ---------------------------------------------------------------------------
// the persistent executor
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT, 1) exec_kernel(ExecArgs A) {
    extern __shared__ double4 smem_raw[];
    double *sm = reinterpret_cast<double *>(smem_raw);
    __shared__ int s_t;
    __shared__ int s_carry;  // successor this CTA made ready and keeps (work-first)
    __shared__ DTask s_task;
    if (threadIdx.x == 0) s_carry = -1;
    __syncthreads();
    while (true) {
        // pop the most urgent ready task: buckets by b-level class, highest first; a slot
        // below `tail` is reserved by a pusher and filled momentarily
        if (threadIdx.x == 0 && s_carry >= 0) {
            s_t = s_carry;
            s_task = A.tasks[s_carry];
            s_carry = -1;
        } else if (threadIdx.x == 0) {
            int t = -1;
            long long spins = 0;
            unsigned ns = 32;
            while (true) {
                int slot = -1;
                for (int b = NPRIO - 1; b >= 0 && slot < 0; --b) {
                    while (true) {
                        const int h = *(volatile const int32_t *)(A.heads + b);
                        const int tl = *(volatile const int32_t *)(A.tails + b);
                        if (h >= tl) break;
                        if (atomicCAS(A.heads + b, h, h + 1) == h) {
                            slot = A.qoff[b] + h;
                            break;
                        }
                    }
                }
                if (slot >= 0) {
                    // acquire: pairs with the pusher's release and invalidates this SM's L1
                    while ((t = ld_acquire(A.queue + slot)) < 0) __nanosleep(32);
                    break;
                }
                if (*(volatile const int32_t *)A.done_count >= A.ntasks) break;  // all done
                __nanosleep(ns);
                ns = ns < POLL_NS_MAX ? ns * 2 : POLL_NS_MAX;
                if (++spins > (1ll << 26)) {  // watchdog (tens of seconds): never hang
                    set_err(A, LH_EINTERNAL, -1, -2);
                    break;
                }
            }
            s_t = t;
            if (t >= 0) s_task = A.tasks[t];
        }
        __syncthreads();
        const int t = s_t;
        if (t < 0) return;
        const DTask &T = s_task;
        if (A.times && threadIdx.x == 0) A.times[2 * t] = gtimer();
        switch (T.type) {
            case T_GETRF: task_getrf(A, T, t, sm); break;
            case T_TRSM: task_trsm(A, T, t, sm); break;
            case T_SEGMUL: task_segmul(A, T, sm); break;
            case T_VTX: task_vtx(A, T, sm); break;
            case T_LRADD: task_lradd(A, T, t, sm); break;
            case T_DGEMM: task_dgemm(A, T); break;
            case T_DADD: task_dadd(A, T); break;
            case T_DENSIFY: task_densify(A, T); break;
            case T_IDENT: task_ident(A, T); break;
            case T_RAND: task_rand(A, T); break;
            case T_ORTH: task_orth(A, T, sm); break;
            case T_CHECK: task_check(A, T, t); break;
            default: break;
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            // release side: the barrier made the CTA's writes visible to warp 0; its
            // gpu-scope acq_rel fences publish them before the counter decrements
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            if (A.times && threadIdx.x == 0) A.times[2 * t + 1] = gtimer();
            const int sb = A.succ_beg[t], se = A.succ_beg[t + 1];
            auto push = [&](int s, int b) {
                const int pos = atomicAdd(A.tails + b, 1);
                st_release(A.queue + A.qoff[b] + pos, s);
            };
            // successors made ready by this completion: the most urgent one is kept and run
            // next by this CTA (no queue round trip on a dependency chain), the rest pushed
            int hold = -1, hold_b = -1;
            for (int q = sb + threadIdx.x; q < se; q += 32) {
                const int e = A.succ[q];
                const int s = e & SUCC_MASK, b = (int)((unsigned)e >> SUCC_SHIFT);
                if (atomicSub(A.remaining + s, 1) == 1) {
                    // last predecessor: acquire the other predecessors' releases
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    if (b > hold_b) {
                        if (hold >= 0) push(hold, hold_b);
                        hold = s;
                        hold_b = b;
                    } else {
                        push(s, b);
                    }
                }
            }
            const int key = hold >= 0 ? (hold_b << 5) | (31 - threadIdx.x) : -1;
            int best = key;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
            if (hold >= 0 && key != best) push(hold, hold_b);
            if (best >= 0 && key == best) s_carry = hold;
            __syncwarp();
            if (threadIdx.x == 0) atomicAdd(A.done_count, 1);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
Plan::~Plan() {
    cudaFree(d_tasks);
    cudaFree(d_deps);
    cudaFree(d_pieces);
    cudaFree(d_done);
    if (own_temp) cudaFree(d_temp);
    cudaFree(d_ranks);
    cudaFree(d_err);
    cudaFree(d_succ_beg);
    cudaFree(d_succ);
    cudaFree(d_rem_init);
    cudaFree(d_rem);
    cudaFree(d_queue_init);
    cudaFree(d_queue);
    cudaFree(d_qoff);
    cudaFree(d_ctr);
}

void Plan::upload(cudaStream_t s) {
    const int32_t n = (int32_t)tasks.size();
    // successor CSR, initial dependency counts, initial ready FIFO (tasks without deps)
    std::vector<int32_t> sb(n + 1, 0), sc(deps.size()), rem(n), q0(std::max(n, 1), -1);
    for (int32_t t = 0; t < n; ++t)
        for (int32_t k = 0; k < tasks[t].dep_cnt; ++k) ++sb[deps[tasks[t].dep_beg + k] + 1];
    for (int32_t t = 0; t < n; ++t) sb[t + 1] += sb[t];
    std::vector<int32_t> fill(sb.begin(), sb.end() - 1);
    LH_REQUIRE(n < (1 << 28), LH_EINTERNAL, "task count exceeds the successor encoding");
    std::vector<int32_t> cnt(NPRIO, 0), qoff(NPRIO, 0), pos(NPRIO, 0);
    for (int32_t t = 0; t < n; ++t) ++cnt[tasks[t].prio];
    for (int b = 1; b < NPRIO; ++b) qoff[b] = qoff[b - 1] + cnt[b - 1];
    for (int32_t t = 0; t < n; ++t) {
        rem[t] = tasks[t].dep_cnt;
        const int32_t code = t | (tasks[t].prio << 28);
        for (int32_t k = 0; k < tasks[t].dep_cnt; ++k) sc[fill[deps[tasks[t].dep_beg + k]]++] = code;
        if (rem[t] == 0) {
            const int b = tasks[t].prio;
            q0[qoff[b] + pos[b]++] = t;
        }
    }
    ctr_init.assign(2 * NPRIO + 2, 0);
    for (int b = 0; b < NPRIO; ++b) ctr_init[NPRIO + b] = pos[b];  // tails
    d_qoff = dupload(qoff, s);
    d_ctr = dalloc<int32_t>(2 * NPRIO + 2);
    d_succ_beg = dupload(sb, s);
    d_succ = dupload(sc, s);
    d_rem_init = dupload(rem, s);
    d_queue_init = dupload(q0, s);
    d_rem = dalloc<int32_t>(std::max(n, 1));
    d_queue = dalloc<int32_t>(std::max(n, 1));
    d_tasks = dupload(tasks, s);
    d_deps = dupload(deps, s);
    d_pieces = dupload(pieces, s);
    d_done = dalloc<int32_t>((i64)tasks.size() + 2);
    if (own_temp) d_temp = dalloc<double>(std::max<i64>(temp_len, 1));
    d_ranks = dalloc<int32_t>(std::max(nslots_total + 1, 1));
    d_err = dalloc<int32_t>(4);
    LH_CUDA(cudaStreamSynchronize(s));
}

static int exec_grid(Ctx &ctx) {
    static bool attr = false;
    if (!attr) {
        LH_CUDA(cudaFuncSetAttribute((const void *)exec_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
        attr = true;
    }
    int per_sm = 0;
    LH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, exec_kernel, NT, SMEM_BYTES));
    LH_REQUIRE(per_sm >= 1, LH_EINTERNAL, "executor kernel cannot be resident");
    return ctx.num_sms * per_sm;
}

static double g_last_mean_task_us = 0.0;

// Task-level profile (LEVYH_TASK_PROFILE=<file>): per-type busy time and the measured
// critical path (latest-finishing predecessor chain) with its per-type composition.
static void report_profile(const Plan &P, const std::vector<unsigned long long> &tm, const char *label) {
    const char *path = getenv("LEVYH_TASK_PROFILE");
    if (!path) return;
    FILE *f = fopen(path, "a");
    if (!f) return;
    const int n = (int)P.tasks.size();
    const char *names[] = {"?", "GETRF", "TRSM", "SEGMUL", "VTX", "LRADD", "DGEMM", "DADD",
                           "DENSIFY", "IDENT", "NOP", "RAND", "ORTH"};
    double busy[13] = {0}, cnt[13] = {0}, cp_busy[13] = {0}, cp_cnt[13] = {0};
    unsigned long long t0 = ~0ull, t1 = 0;
    int last = 0;
    for (int i = 0; i < n; ++i) {
        int ty = std::min(std::max(P.tasks[i].type, 0), 12);
        busy[ty] += (tm[2 * i + 1] - tm[2 * i]) * 1e-9;
        cnt[ty] += 1;
        t0 = std::min(t0, tm[2 * i]);
        if (tm[2 * i + 1] > t1) {
            t1 = tm[2 * i + 1];
            last = i;
        }
    }
    double wait = 0.0;
    int len = 0;
    for (int t = last; t >= 0;) {
        const DTask &T = P.tasks[t];
        int ty = std::min(std::max(T.type, 0), 12);
        cp_busy[ty] += (tm[2 * t + 1] - tm[2 * t]) * 1e-9;
        cp_cnt[ty] += 1;
        ++len;
        int best = -1;
        unsigned long long be = 0;
        for (int k = 0; k < T.dep_cnt; ++k) {
            int p = P.deps[T.dep_beg + k];
            if (best < 0 || tm[2 * p + 1] > be) {
                be = tm[2 * p + 1];
                best = p;
            }
        }
        if (best >= 0 && tm[2 * t] > be) wait += (tm[2 * t] - be) * 1e-9;
        t = best;
    }
    fprintf(f, "== %s: %d tasks, span %.4f s, critical path %d tasks, waits on path %.4f s\n", label, n,
            (t1 - t0) * 1e-9, len, wait);
    for (int ty = 1; ty <= 12; ++ty)
        if (cnt[ty] > 0)
            fprintf(f, "  %-8s count %9.0f busy %9.4f s mean %8.2f us | on path %7.0f tasks %8.4f s\n",
                    names[ty], cnt[ty], busy[ty], 1e6 * busy[ty] / cnt[ty], cp_cnt[ty], cp_busy[ty]);
    fclose(f);
}

// Run a plan; F / X / RHS bases.  Ranks of F (and X) are copied in and back out.
// run_plan_launch enqueues (stream-ordered, returns at once), run_plan_finish waits and
// raises the executor's errors.
struct PlanRun {
    ExecArgs A;
    bool prof = false;
    int err[4] = {0, 0, 0, 0};
    double *xbuf = nullptr;  // scratch of a propagator column part (Plan::x_len >= 0)
};

static void run_plan_launch(Ctx &ctx, Plan &P, HMat &F, HMat *X, double *rhs, int rhs_slot_val,
                            PlanRun &R) {
    cudaStream_t s = ctx.stream;
    LH_CUDA(cudaMemsetAsync(P.d_done, 0, sizeof(int32_t) * (P.tasks.size() + 2), s));
    LH_CUDA(cudaMemsetAsync(P.d_err, 0, sizeof(int32_t) * 4, s));
    if (!P.tasks.empty()) {
        LH_CUDA(cudaMemcpyAsync(P.d_rem, P.d_rem_init, sizeof(int32_t) * P.tasks.size(),
                                cudaMemcpyDeviceToDevice, s));
        LH_CUDA(cudaMemcpyAsync(P.d_queue, P.d_queue_init, sizeof(int32_t) * P.tasks.size(),
                                cudaMemcpyDeviceToDevice, s));
        LH_CUDA(cudaMemcpyAsync(P.d_ctr, P.ctr_init.data(), sizeof(int32_t) * P.ctr_init.size(),
                                cudaMemcpyHostToDevice, s));
    }
    if (F.nslots)
        LH_CUDA(cudaMemcpyAsync(P.d_ranks, F.d_ranks, sizeof(int32_t) * F.nslots,
                                cudaMemcpyDeviceToDevice, s));
    if (X && X->nslots)
        LH_CUDA(cudaMemcpyAsync(P.d_ranks + P.slot_off_x, X->d_ranks, sizeof(int32_t) * X->nslots,
                                cudaMemcpyDeviceToDevice, s));
    if (rhs_slot_val >= 0)
        LH_CUDA(cudaMemcpyAsync(P.d_ranks + P.rhs_slot, &rhs_slot_val, sizeof(int32_t),
                                cudaMemcpyHostToDevice, s));
    ExecArgs &A = R.A;
    A.tasks = P.d_tasks;
    A.ntasks = (int32_t)P.tasks.size();
    A.deps = P.d_deps;
    A.pieces = P.d_pieces;
    A.done = P.d_done;
    A.heads = P.d_ctr;
    A.tails = P.d_ctr + NPRIO;
    A.done_count = P.d_ctr + 2 * NPRIO;
    A.qoff = P.d_qoff;
    A.queue = P.d_queue;
    A.remaining = P.d_rem;
    A.succ_beg = P.d_succ_beg;
    A.succ = P.d_succ;
    A.err = P.d_err;
    A.base[B_F] = F.d_arena;
    A.base[B_TMP] = P.d_temp;
    A.base[B_RHS] = rhs;
    A.base[B_X] = X ? X->d_arena : nullptr;
    if (X && P.x_len >= 0) {
        // a propagator column part: its views address [x_base, x_base + x_len) of the Z layout,
        // held by the part's scratch buffer (X->d_arena is not allocated yet)
        LH_REQUIRE(R.xbuf != nullptr, LH_EINTERNAL, "propagator part without a scratch buffer");
        A.base[B_X] = R.xbuf - P.x_base;
    }
    A.base[B_INV] = F.d_inv;
    A.ranks = P.d_ranks;
    A.perm = F.d_perm;
    A.times = nullptr;
    R.prof = (getenv("LEVYH_TASK_PROFILE") != nullptr ||
              getenv("LEVYH_TASK_PROFILE_STATS") != nullptr) && A.ntasks > 0;
    if (R.prof) A.times = dalloc<unsigned long long>(2 * (i64)A.ntasks);
    if (A.ntasks > 0) {
        int grid = exec_grid(ctx);
        void *args[] = {&A};
        LH_CUDA(cudaLaunchCooperativeKernel((const void *)exec_kernel, grid, NT, args, SMEM_BYTES, s));
    }
    LH_CUDA(cudaMemcpyAsync(R.err, P.d_err, sizeof(R.err), cudaMemcpyDeviceToHost, s));
    if (F.nslots)
        LH_CUDA(cudaMemcpyAsync(F.d_ranks, P.d_ranks, sizeof(int32_t) * F.nslots,
                                cudaMemcpyDeviceToDevice, s));
    if (X && X->nslots)
        LH_CUDA(cudaMemcpyAsync(X->d_ranks, P.d_ranks + P.slot_off_x, sizeof(int32_t) * X->nslots,
                                cudaMemcpyDeviceToDevice, s));
}

static void run_plan_finish(Ctx &ctx, Plan &P, PlanRun &R, const char *label) {
    LH_CUDA(cudaStreamSynchronize(ctx.stream));
    ExecArgs &A = R.A;
    if (R.prof) {
        std::vector<unsigned long long> tm(2 * (size_t)A.ntasks);
        LH_CUDA(cudaMemcpy(tm.data(), A.times, sizeof(unsigned long long) * tm.size(),
                           cudaMemcpyDeviceToHost));
        cudaFree(A.times);
        double sum = 0.0;
        for (int i = 0; i < A.ntasks; ++i) sum += (tm[2 * i + 1] - tm[2 * i]) * 1e-3;
        g_last_mean_task_us = sum / A.ntasks;
        report_profile(P, tm, label);
    }
    const int *err = R.err;
    if (err[0] == LH_ESINGULAR) {
        std::string msg = err[2] >= 0 && err[2] < (int)P.paths.size() ? P.paths[err[2]]
                                                                      : "singular diagonal block";
        throw Error(LH_ESINGULAR, msg);
    }
    if (err[0] == LH_ERANK)
        throw Error(LH_ERANK, "low-rank capacity exceeded during H-arithmetic (increase kcap)");
    if (err[0] == LH_EINVAL && err[2] >= 0 && err[2] < (int)P.paths.size())
        throw Error(LH_EINVAL, P.paths[err[2]]);
    if (err[0] != 0) throw Error(err[0], "executor failure (task " + std::to_string(err[1]) + ")");
}

static void run_plan(Ctx &ctx, Plan &P, HMat &F, HMat *X, double *rhs, int rhs_slot_val,
                     const char *label = "plan", double *xbuf = nullptr) {
    PlanRun R;
    R.xbuf = xbuf;
    run_plan_launch(ctx, P, F, X, rhs, rhs_slot_val, R);
    run_plan_finish(ctx, P, R, label);
}

// ---------------------------------------------------------------------------
// background planning: plans depend only on the block structure, so the H-LU plan is
// built on a host thread as soon as a square H-matrix is assembled, and the two
// triangular-inverse plans and the propagator plan right after it (overlapping the GPU
// execution of the LU)
// ---------------------------------------------------------------------------
void triangle_layout(HMat &X, const HMat &F, bool lower, int kcap);
void block_layout(HMat &X, const HMat &F, int part, int kcap);

// column capacity of the propagator's low-rank blocks: rank + sketch width (14) before each
// recompression; the eps2 ranks of Z stay <= ~10 on these operators (LEVYH_PROP_KCAP overrides)
static int prop_kcap() {
    static const int v = getenv("LEVYH_PROP_KCAP") ? std::min(std::max(atoi(getenv("LEVYH_PROP_KCAP")), 16),
                                                              (int)KA_MAX)
                                                   : 32;
    return v;
}

// the propagator's capacity for a factor whose low-rank blocks were laid out wider than
// KC_MAX (series builds with high expansion ranks): the full recompression width
static int prop_kcap_for(const HMat &F) {
    int mx = 0;
    for (const Node &nd : F.nodes)
        if (nd.kind == K_LR && nd.vpar < 0) mx = std::max(mx, nd.kcap);
    return mx > KC_MAX ? KA_MAX : prop_kcap();
}

struct PlanJob {
    HMat shadow;   // structure-only copy the H-LU planner mutates (no device memory)
    HMat fshadow;  // the factor's structure as the H-LU leaves it (mark_lu_leaves), read-only
    std::shared_ptr<Plan> lu;
    i64 perm_len = 0;
    HMat X[2];
    std::shared_ptr<Plan> inv[2];
    HMat Z;
    std::shared_ptr<Plan> prop;
    std::vector<std::shared_ptr<Plan>> prop_parts;  // column parts run one by one (large N)
    bool prop_uploaded = false;  // device copies made by the planning thread (own stream)
    int device = -1;             // device of the thread that assembled the matrix
    PlanStream lu_stream;  // the H-LU plan in chunks, when hlu() arrives before planning ends
    std::string error, inv_error, prop_error;
    std::shared_ptr<std::atomic<bool>> cancel = std::make_shared<std::atomic<bool>>(false);
    std::future<void> f_lu, f_inv, f_prop;  // last members: joined first, after ~PlanJob raised cancel
    ~PlanJob() { cancel->store(true); }     // a matrix dropped while planning: stop at the next task
};

static void copy_structure(HMat &D, const HMat &S) {
    D.refined = S.refined;
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
    D.arena_len = S.arena_len;
}

static void patch_eps(Plan &P, double eps2) {
    for (DTask &t : P.tasks)
        if (t.type == T_LRADD) t.alpha2 = eps2;
}

// Plans depend only on the block structure, so they are built on host threads as soon as
// a square H-matrix is assembled: the H-LU plan, and concurrently the propagator plan
// (itself split over column blocks) against the factor's structure from mark_lu_leaves.
// The triangular-inverse plans are added when LEVYH_BG_INVERSE is set.
void start_background_plans(HMat &H) {
    if (H.nrows != H.ncols || H.factored || getenv("LEVYH_NO_BG_PLAN")) return;
    auto job = std::make_shared<PlanJob>();
    refine_dense_leaves(H);
    copy_structure(job->shadow, H);
    copy_structure(job->fshadow, H);
    job->shadow.plan_cancel = job->fshadow.plan_cancel = job->cancel;
    PlanJob *j = job.get();
    if (const char *e = getenv("LEVYH_STREAM_MIN_CHUNK")) j->lu_stream.min_chunk = std::max(1, atoi(e));
    try {
        i64 pl = 0, il = 0;
        mark_lu_leaves(j->fshadow, pl, il);
        j->fshadow.factored = true;
    } catch (const std::exception &e) {
        return;  // not LU-factorizable: hlu reports it
    }
    job->f_lu = std::async(std::launch::async, [j] {
        try {
            j->lu = plan_hlu(j->shadow, 1e-10, j->perm_len, &j->lu_stream);
        } catch (const std::exception &e) {
            j->error = e.what();
            std::lock_guard<std::mutex> lk(j->lu_stream.mu);  // release a waiting consumer
            j->lu_stream.done = true;
            j->lu_stream.cv.notify_all();
        }
    });
    cudaGetDevice(&j->device);
    if (!getenv("LEVYH_NO_BG_PROP"))
    job->f_prop = std::async(std::launch::async, [j] {
        try {
            block_layout(j->Z, j->fshadow, 2, prop_kcap_for(j->fshadow));
            j->prop = plan_propagator(j->fshadow, j->Z, 1e-10, 8, &j->prop_parts);
            if (!j->prop) return;  // parts: uploaded one at a time by prepare_propagator
            // upload on a stream of this thread once the H-LU planning (and with it the
            // streamed H-LU chunk uploads) is done: the copies overlap the H-LU's last chunks
            if (j->device >= 0 && !getenv("LEVYH_NO_BG_UPLOAD")) {
                j->f_lu.wait();
                // only when the plan is small against free device memory (the propagator may
                // never be requested: e.g. stepping by substitution at the largest sizes)
                LH_CUDA(cudaSetDevice(j->device));
                size_t fr = 0, tot = 0;
                LH_CUDA(cudaMemGetInfo(&fr, &tot));
                const Plan &pp = *j->prop;
                const double need = (double)pp.tasks.size() * (sizeof(DTask) + 24) +
                                    (double)pp.deps.size() * 8 + (double)pp.pieces.size() * sizeof(DPiece) +
                                    (double)pp.temp_len * 8;
                if (need > 0.25 * (double)fr) return;
                LH_CUDA(cudaSetDevice(j->device));
                cudaStream_t st;
                LH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
                j->prop->upload(st);
                LH_CUDA(cudaStreamSynchronize(st));
                LH_CUDA(cudaStreamDestroy(st));
                j->prop_uploaded = true;
            }
        } catch (const std::exception &e) {
            j->prop_error = e.what();
        }
    });
    if (getenv("LEVYH_BG_INVERSE")) {
        job->f_inv = std::async(std::launch::async, [j] {
            try {
                for (int mode = 0; mode < 2; ++mode)
                    triangle_layout(j->X[mode], j->fshadow, mode == 0, KA_MAX);
                auto f0 = std::async(std::launch::async,
                                     [j] { j->inv[0] = plan_inverse(j->fshadow, j->X[0], 0, 1e-10); });
                j->inv[1] = plan_inverse(j->fshadow, j->X[1], 1, 1e-10);
                f0.get();
            } catch (const std::exception &e) {
                j->inv_error = e.what();
            }
        });
    }
    H.bg_plan = job;
}

static void check_leaf_layout(const HMat &F, const PlanJob &job) {
    LH_REQUIRE(F.inv_len == job.fshadow.inv_len && job.perm_len == job.fshadow.perm_len,
               LH_EINTERNAL, "background plans disagree on the diagonal-leaf layout");
    for (size_t b = 0; b < F.nodes.size(); ++b) {
        const Node &x = F.nodes[b], &y = job.fshadow.nodes[b];
        LH_REQUIRE(x.kind == y.kind && x.poff == y.poff && x.ioff == y.ioff, LH_EINTERNAL,
                   "background plans disagree on the diagonal-leaf layout");
    }
}

// Run the H-LU as chunks of the plan still being built on the background thread, one chunk
// ahead: the next cut is requested when a chunk launches, uploaded on a second stream while
// it runs, and launched as soon as it finishes.  The chunks share one temp pool (grown by
// copy between chunks).
static void hlu_streamed(Ctx &ctx, HMat &F, double eps2, PlanJob &job) {
    PlanStream &st = job.lu_stream;
    double *temp = nullptr;
    i64 temp_cap = 0;
    int nchunks = 0;
    i64 ntasks = 0;
    cudaStream_t up;
    LH_CUDA(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    LH_CUDA(cudaEventCreate(&e0));
    LH_CUDA(cudaEventCreate(&e1));
    float exec_ms = 0.f;
    auto take = [&]() -> std::shared_ptr<Plan> {
        std::unique_lock<std::mutex> lk(st.mu);
        st.want.store(true);
        st.cv.wait(lk, [&] { return !st.chunks.empty() || st.done; });
        if (st.chunks.empty()) return nullptr;
        std::shared_ptr<Plan> C = st.chunks.front();
        st.chunks.pop_front();
        return C;
    };
    auto prepare = [&](Plan &C) {
        if (eps2 != 1e-10) patch_eps(C, eps2);
        C.upload(up);  // host CSR + copies on the second stream (synchronous on it)
    };
    auto grow_temp = [&](Plan &C) {
        if (C.temp_len > temp_cap) {
            double *nt = dalloc<double>(std::max<i64>(C.temp_len, 1));
            if (temp) {
                LH_CUDA(cudaMemcpyAsync(nt, temp, sizeof(double) * temp_cap, cudaMemcpyDeviceToDevice,
                                        ctx.stream));
                LH_CUDA(cudaStreamSynchronize(ctx.stream));
                cudaFree(temp);
            }
            temp = nt;
            temp_cap = C.temp_len;
        }
        C.d_temp = temp;
    };
    try {
        std::shared_ptr<Plan> cur = take();
        if (cur) {
            prepare(*cur);
            grow_temp(*cur);
        }
        PlanRun R;
        while (cur) {
            LH_CUDA(cudaEventRecord(e0, ctx.stream));
            run_plan_launch(ctx, *cur, F, nullptr, nullptr, -1, R);
            LH_CUDA(cudaEventRecord(e1, ctx.stream));
            auto tl = std::chrono::steady_clock::now();
            std::shared_ptr<Plan> nxt = take();  // cut while `cur` runs
            if (nxt) prepare(*nxt);
            run_plan_finish(ctx, *cur, R, "hlu");
            float ms = 0.f;
            LH_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            exec_ms += ms;
            if (getenv("LEVYH_PLAN_VERBOSE"))
                fprintf(stderr, "[levyh] hlu chunk %d: %zu tasks, exec %.3f s (host wall %.3f s)\n", nchunks,
                        cur->tasks.size(), ms / 1e3,
                        std::chrono::duration<double>(std::chrono::steady_clock::now() - tl).count());
            ++nchunks;
            ntasks += (i64)cur->tasks.size();
            cur.reset();  // frees the chunk's device arrays (not the shared temp pool)
            if (nxt) grow_temp(*nxt);
            cur = nxt;
        }
    } catch (...) {
        cudaFree(temp);
        cudaStreamDestroy(up);
        throw;
    }
    cudaFree(temp);
    cudaStreamDestroy(up);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    auto tw = std::chrono::steady_clock::now();
    job.f_lu.wait();
    LH_REQUIRE(job.error.empty(), LH_EINTERNAL, "H-LU planning failed: " + job.error);
    LH_REQUIRE(ntasks == (i64)job.lu->tasks.size(), LH_EINTERNAL, "streamed H-LU plan incomplete");
    if (getenv("LEVYH_PLAN_VERBOSE"))
        fprintf(stderr, "[levyh] hlu streamed: %d chunks, exec %.3f s, waited for the plan end %.3f s\n",
                nchunks, exec_ms / 1e3,
                std::chrono::duration<double>(std::chrono::steady_clock::now() - tw).count());
    F.lu_stats[3] = exec_ms / 1e3;
    F.lu_stats[4] = nchunks;
}

// lu_stats[6..7]: the plan's algorithmic flops and bytes at the factor's final ranks (temporaries,
// whose ranks are gone with the plan's rank array, at the mean stored rank)
static void record_plan_work(HMat &F, const Plan &P) {
    double mean = 0.0;
    for (int32_t r : F.h_ranks) mean += r;
    if (!F.h_ranks.empty()) mean /= (double)F.h_ranks.size();
    plan_work(P, F.h_ranks, mean, F.lu_stats[6], F.lu_stats[7]);
}

void hlu(Ctx &ctx, HMat &F, double eps2) {
    LH_REQUIRE(F.nrows == F.ncols, LH_EINVAL, "LU requires a square matrix");
    LH_REQUIRE(!F.factored, LH_EINVAL, "matrix is already factored");
    i64 perm_len = 0;
    std::shared_ptr<Plan> P;
    PlanJob *job = F.bg_plan ? static_cast<PlanJob *>(F.bg_plan.get()) : nullptr;
    if (job && job->f_lu.valid()) {
        bool streamed = false;
        {
            std::lock_guard<std::mutex> lk(job->lu_stream.mu);
            if (!job->lu_stream.done && !getenv("LEVYH_NO_STREAM_LU")) {
                job->lu_stream.engaged = true;
                streamed = true;
            }
        }
        if (streamed) {
            // the factor's storage layout is known up front (mark_lu_leaves)
            F.d_perm = dalloc<int32_t>(std::max<i64>(job->fshadow.perm_len, 1));
            F.perm_len = job->fshadow.perm_len;
            F.inv_len = job->fshadow.inv_len;
            F.d_inv = dalloc<double>(std::max<i64>(F.inv_len, 1));
            F.factored = true;
            F.mv_plan.reset();
            auto ts0 = std::chrono::steady_clock::now();
            hlu_streamed(ctx, F, eps2, *job);
            auto ts1 = std::chrono::steady_clock::now();
            F.nodes = job->shadow.nodes;
            check_leaf_layout(F, *job);
            F.sync_ranks(ctx.stream);
            if (getenv("LEVYH_PLAN_VERBOSE"))
                fprintf(stderr, "[levyh] hlu streamed: chunks %.3f s, finish %.3f s\n",
                        std::chrono::duration<double>(ts1 - ts0).count(),
                        std::chrono::duration<double>(std::chrono::steady_clock::now() - ts1).count());
            F.lu_stats[0] = (double)job->lu->tasks.size();
            F.lu_stats[1] = job->lu->build_seconds;
            F.lu_stats[2] = (double)job->lu->temp_len * 8.0;
            record_plan_work(F, *job->lu);
            job->lu.reset();
            return;
        }
        job->f_lu.wait();
        if (job->error.empty() && job->lu) {
            P = std::move(job->lu);
            F.nodes = job->shadow.nodes;  // diagonal leaves K_FDENSE with pivot/inverse offsets
            F.inv_len = job->shadow.inv_len;
            perm_len = job->perm_len;
            check_leaf_layout(F, *job);
            if (eps2 != 1e-10) patch_eps(*P, eps2);
        }
    }
    if (!P) P = plan_hlu(F, eps2, perm_len);  // marks diagonal leaves K_FDENSE
    F.d_perm = dalloc<int32_t>(std::max<i64>(perm_len, 1));
    F.perm_len = perm_len;
    F.d_inv = dalloc<double>(std::max<i64>(F.inv_len, 1));
    P->upload(ctx.stream);
    F.factored = true;
    F.mv_plan.reset();
    LH_CUDA(cudaStreamSynchronize(ctx.stream));
    auto t0 = std::chrono::steady_clock::now();
    run_plan(ctx, *P, F, nullptr, nullptr, -1, "hlu");
    F.lu_stats[3] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    F.lu_stats[4] = 1;
    F.sync_ranks(ctx.stream);
    F.lu_stats[0] = (double)P->tasks.size();
    F.lu_stats[1] = P->build_seconds;
    F.lu_stats[2] = (double)P->temp_len * 8.0;
    record_plan_work(F, *P);
}

struct SolvePlans {
    std::shared_ptr<Plan> sub;  // substitution DAG
    int cap = 0;
    std::shared_ptr<HMat> XL, XU;   // triangular inverses
    std::shared_ptr<MvPlan> mvL, mvU;
    std::shared_ptr<HMat> Z;        // propagator (A+)^{-1} = (L U)^{-1} on the full block tree
    std::shared_ptr<MvPlan> mvZ;
    std::shared_ptr<HMat> ZS;       // Z with shared leaf bases (zshared.cu), single-RHS path
    std::shared_ptr<MvPlan> mvZS;
    double zs_stats[3] = {0, 0, 0};
    double zs_probe = 0.0;  // relative probe error of the single-RHS form against Z
    const MvPlan &z1plan() const { return mvZS ? *mvZS : *mvZ; }
    HMat &z1mat() const { return mvZS ? *ZS : *Z; }
    int g_method = -1;
    int g_kernels = 0;  // kernel nodes in the cached step graph
    int32_t last_path[3] = {-1, 0, 0};  // lh_cn_last_path: shape, multi-RHS DMMA, pipelined host step
    std::shared_ptr<Plan> tri[3][2];  // dense-RHS triangular solves by (mode, unit)
    double *tmp = nullptr;          // scratch vector(s)
    i64 tmp_len = 0;
    cudaGraphExec_t graph = nullptr;  // cached CN step
    const double *g_u = nullptr, *g_y = nullptr;
    uint64_t g_hm = 0;  // HMat::id of the hminus the graph was captured with
    uint64_t g_gen = 0;  // and its storage generation (HMat::gen)
    // host-buffer CN step (cn_step_host): pipelined graph keyed by the host pointers
    cudaGraphExec_t hgraph = nullptr;
    const double *hg_in = nullptr;
    double *hg_out = nullptr;
    uint64_t hg_hm = 0;
    cudaStream_t side = nullptr;
    std::vector<cudaEvent_t> hev;
    double *hx = nullptr, *hy = nullptr;  // device x and y of the host step
    ~SolvePlans() {
        if (graph) cudaGraphExecDestroy(graph);
        if (hgraph) cudaGraphExecDestroy(hgraph);
        for (cudaEvent_t e : hev) cudaEventDestroy(e);
        if (side) cudaStreamDestroy(side);
        if (hx) cudaFree(hx);
        if (hy) cudaFree(hy);
        if (tmp) cudaFree(tmp);
    }
};

static SolvePlans &plans_of(HMat &F) {
    if (!F.solve_plan) F.solve_plan = std::make_shared<SolvePlans>();
    return *static_cast<SolvePlans *>(F.solve_plan.get());
}

static void solve_substitution(Ctx &ctx, HMat &F, double *b, i64 ldb, int nrhs) {
    LH_REQUIRE(ldb == F.nrows, LH_EINVAL, "solve expects a packed right-hand side (ldb == n)");
    SolvePlans &S = plans_of(F);
    const int CAP = 64;
    if (!S.sub) {
        S.sub = plan_solve(F, F.nrows, CAP);
        S.sub->upload(ctx.stream);
    }
    for (int c0 = 0; c0 < nrhs; c0 += CAP) {
        int kc = std::min(CAP, nrhs - c0);
        run_plan(ctx, *S.sub, F, nullptr, b + (i64)c0 * ldb, kc, "solve");
    }
}

// X: same block tree as F; part 0 / 1 keep the lower / upper triangle (leaves of the other
// triangle are K_ZERO), part 2 keeps every block.  Low-rank leaves get kcap columns.
void triangle_layout(HMat &X, const HMat &F, bool lower, int kcap) {
    block_layout(X, F, lower ? 0 : 1, kcap);
}

void block_layout(HMat &X, const HMat &F, int part, int kcap) {
    X.rt = F.rt;
    X.ct = F.ct;
    X.rt_hold = F.rt_hold;
    X.ct_hold = F.ct_hold;
    X.nrows = F.nrows;
    X.ncols = F.ncols;
    X.root = F.root;
    X.nodes = F.nodes;
    X.refined = F.refined;
    for (Node &nd : X.nodes)  // virtual children of refined leaves: plain dense storage here
        if (nd.vpar >= 0) {
            nd.kind = K_DENSE;
            nd.ioff = -1;
        }
    i64 off = 0;
    int32_t slots = 0;
    walk_leaves(X);
    for (int32_t b : X.leafblocks) {
        Node &nd = X.nodes[b];
        bool diag = (nd.r0 == nd.c0 && nd.m == nd.n);
        bool other = part == 0 ? (nd.c0 >= nd.r0 + nd.m)
                   : part == 1 ? (nd.r0 >= nd.c0 + nd.n)
                               : false;
        if (other && !diag) {
            nd.kind = K_ZERO;
            continue;
        }
        if (nd.kind == K_FDENSE || nd.kind == K_DENSE) {
            nd.kind = K_DENSE;
            nd.doff = off;
            off += nd.m * nd.n;
        } else if (nd.kind == K_LR) {
            nd.kcap = kcap;
            nd.rslot = slots++;
            nd.uoff = off;
            off += nd.m * kcap;
            nd.voff = off;
            off += nd.n * kcap;
        }
    }
    X.arena_len = off;
    X.nslots = slots;
}

void prepare_inverse(Ctx &ctx, HMat &F, double eps2) {
    LH_REQUIRE(F.factored, LH_EINVAL, "prepare_inverse needs an H-LU factorization");
    SolvePlans &S = plans_of(F);
    if (S.XL) return;
    int kcap = KA_MAX;  // room for rank + sketch width before recompression
    PlanJob *job = F.bg_plan ? static_cast<PlanJob *>(F.bg_plan.get()) : nullptr;
    bool use_bg = false;
    if (job && job->f_inv.valid()) {
        job->f_inv.wait();
        use_bg = job->inv_error.empty() && job->inv[0] && job->inv[1];
    }
    for (int mode = 0; mode < 2; ++mode) {
        auto X = std::make_shared<HMat>();
        std::shared_ptr<Plan> P;
        if (use_bg) {
            copy_structure(*X, job->X[mode]);
            X->nslots = job->X[mode].nslots;
            X->arena_len = job->X[mode].arena_len;
            P = std::move(job->inv[mode]);  // the job lets go: the plan dies after its run
            if (eps2 != 1e-10) patch_eps(*P, eps2);
        } else {
            triangle_layout(*X, F, mode == 0, kcap);
        }
        X->d_arena = dalloc<double>(std::max<i64>(X->arena_len, 1));
        X->d_ranks = dalloc<int32_t>(std::max(X->nslots, 1));
        LH_CUDA(cudaMemsetAsync(X->d_ranks, 0, sizeof(int32_t) * std::max(X->nslots, 1), ctx.stream));
        if (!P) P = plan_inverse(F, *X, mode, eps2);
        P->upload(ctx.stream);
        run_plan(ctx, *P, F, X.get(), nullptr, -1, mode == 0 ? "inverse L" : "inverse U");
        X->sync_ranks(ctx.stream);
        std::vector<int32_t> blocks;
        for (int32_t b : X->leafblocks)
            if (X->nodes[b].kind != K_ZERO) blocks.push_back(b);
        auto mv = build_mv_plan(*X, blocks, ctx.stream);
        if (mode == 0) {
            S.XL = X;
            S.mvL = mv;
        } else {
            S.XU = X;
            S.mvU = mv;
        }
    }
    if (!S.tmp) {
        S.tmp_len = F.nrows;
        S.tmp = dalloc<double>(S.tmp_len);
    }
}

i64 compress_near_field(Ctx &ctx, HMat &H, double eps);
i64 coarsen_hmat(Ctx &ctx, HMat &H, double eps);
bool build_shared_basis(Ctx &ctx, HMat &Z, double eps, HMat &ZS, std::shared_ptr<MvPlan> &plan,
                        double *stats);
bool build_h2(Ctx &ctx, HMat &Z, double eps, int split, HMat &ZS, std::shared_ptr<MvPlan> &plan,
              double *stats);
std::shared_ptr<Tree> refine_tree_leaves(const Tree &T, int maxleaf);

// relative 2-norm difference of two matvec plans of the same operator on a seeded probe vector
static double probe_rel_err(Ctx &ctx, const MvPlan &Pa, HMat &Ha, const MvPlan &Pb, HMat &Hb) {
    const i64 n = Ha.ncols;
    std::vector<double> x(n);
    uint64_t st = 0x9E3779B97F4A7C15ull;
    for (i64 i = 0; i < n; ++i) {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        x[i] = (double)(st >> 11) * 0x1.0p-53 - 0.5;
    }
    double *d = dalloc<double>(3 * n);
    LH_CUDA(cudaMemcpyAsync(d, x.data(), sizeof(double) * n, cudaMemcpyHostToDevice, ctx.stream));
    mv_run(Pa, Ha, d, d + n, 1.0, 0.0, ctx.stream, ctx.num_sms);
    mv_run(Pb, Hb, d, d + 2 * n, 1.0, 0.0, ctx.stream, ctx.num_sms);
    std::vector<double> ya(n), yb(n);
    LH_CUDA(cudaMemcpyAsync(ya.data(), d + n, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx.stream));
    LH_CUDA(cudaMemcpyAsync(yb.data(), d + 2 * n, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx.stream));
    LH_CUDA(cudaStreamSynchronize(ctx.stream));
    cudaFree(d);
    double num = 0.0, den = 0.0;
    for (i64 i = 0; i < n; ++i) {
        num += (ya[i] - yb[i]) * (ya[i] - yb[i]);
        den += ya[i] * ya[i];
    }
    return den > 0.0 ? std::sqrt(num / den) : std::sqrt(num);
}

// contiguous device copies dst[d + i] = src[s + i], i < len (jobs cut to <= 64K doubles so the
// CTAs share the work evenly)
struct CopyJob {
    i64 src, dst, len;
};
__global__ void copy_jobs_kernel(const CopyJob *jobs, int n, const double *src, double *dst) {
    for (int j = blockIdx.x; j < n; j += gridDim.x) {
        const CopyJob J = jobs[j];
        for (i64 i = threadIdx.x; i < J.len; i += blockDim.x) dst[J.dst + i] = src[J.src + i];
    }
}
static void run_copy_jobs(Ctx &ctx, const std::vector<CopyJob> &in, const double *src, double *dst) {
    std::vector<CopyJob> jobs;
    const i64 CH = 65536;
    for (const CopyJob &J : in)
        for (i64 o = 0; o < J.len; o += CH) jobs.push_back({J.src + o, J.dst + o, std::min(CH, J.len - o)});
    if (jobs.empty()) return;
    CopyJob *d = dupload(jobs, ctx.stream);
    copy_jobs_kernel<<<(int)std::min<size_t>(jobs.size(), (size_t)ctx.num_sms * 8), NT, 0, ctx.stream>>>(
        d, (int)jobs.size(), src, dst);
    LH_CUDA(cudaGetLastError());
    LH_CUDA(cudaStreamSynchronize(ctx.stream));
    cudaFree(d);
}

// Tight re-layout of the blocks of H whose storage lies in [lo, hi) of `src` (offsets in H's
// layout): dense leaves m x n, low-rank blocks at capacity max(rank, 1); the new storage starts at
// `base` of the returned buffer's eventual home and the node offsets are rewritten to it.
// Returns the packed buffer (len doubles, zero beyond the copied ranks).
static double *compact_range(Ctx &ctx, HMat &H, const double *src, i64 src_base, i64 lo, i64 hi, i64 base,
                             i64 &len, std::vector<std::pair<i64, i64>> *regions = nullptr) {
    std::vector<CopyJob> jobs;
    i64 off = 0;
    for (int32_t b : H.leafblocks) {
        Node &nd = H.nodes[b];
        if (nd.vpar >= 0) continue;
        if (nd.kind == K_DENSE || nd.kind == K_FDENSE) {
            if (nd.doff < lo || nd.doff >= hi) continue;
            if (regions) regions->push_back({nd.doff, base + off});
            jobs.push_back({nd.doff - src_base, off, nd.m * nd.n});
            nd.doff = base + off;
            off += nd.m * nd.n;
        } else if (nd.kind == K_LR) {
            if (nd.uoff < lo || nd.uoff >= hi) continue;
            const int r = H.h_ranks[nd.rslot], kc = std::max(r, 1);
            if (regions) {
                regions->push_back({nd.uoff, base + off});
                regions->push_back({nd.voff, base + off + nd.m * kc});
            }
            jobs.push_back({nd.uoff - src_base, off, nd.m * r});
            nd.uoff = base + off;
            off += nd.m * kc;
            jobs.push_back({nd.voff - src_base, off, nd.n * r});
            nd.voff = base + off;
            off += nd.n * kc;
            nd.kcap = kc;
        }
    }
    len = off;
    double *d = dalloc<double>(std::max<i64>(off, 1));
    LH_CUDA(cudaMemsetAsync(d, 0, sizeof(double) * (size_t)std::max<i64>(off, 1), ctx.stream));
    run_copy_jobs(ctx, jobs, src, d);
    return d;
}

// The H-LU factor's arena at capacity max(rank, 1) (it is only read from here on): every
// block moves, so the views of the plans still to run on it are re-pointed, and the plans that
// were cut against the old layout (substitution, triangular solves) are dropped (rebuilt lazily).
static void compact_factor(Ctx &ctx, HMat &F, std::vector<std::shared_ptr<Plan>> &plans) {
    F.sync_ranks(ctx.stream);
    std::vector<std::pair<i64, i64>> starts;  // (old start, new start) of every region
    const i64 old_len = F.arena_len;
    i64 len = 0;
    double *na = compact_range(ctx, F, F.d_arena, 0, 0, old_len, 0, len, &starts);
    std::sort(starts.begin(), starts.end());
    auto remap = [&](DView &v) {
        if (v.base != B_F) return;
        auto it = std::upper_bound(starts.begin(), starts.end(), std::make_pair(v.off, (i64)INT64_MAX));
        LH_REQUIRE(it != starts.begin(), LH_EINTERNAL, "factor view outside every block");
        --it;
        v.off = v.off - it->first + it->second;
    };
    for (auto &P : plans) {
        for (DTask &t : P->tasks)
            for (DView &v : t.v) remap(v);
        for (DPiece &pc : P->pieces) {
            remap(pc.mat);
            remap(pc.x);
        }
    }
    cudaFree(F.d_arena);
    F.d_arena = na;
    F.arena_len = len;
    F.mv_plan.reset();
    F.inv_plan.reset();
    SolvePlans &S = plans_of(F);
    S.sub.reset();
    for (auto &m : S.tri)
        for (auto &q : m) q.reset();
    if (F.bg_plan) {
        PlanJob *job = static_cast<PlanJob *>(F.bg_plan.get());
        if (job->f_inv.valid()) job->f_inv.wait();
        job->inv[0].reset();  // cut against the old layout
        job->inv[1].reset();
    }
    ++F.gen;
    if (getenv("LEVYH_PLAN_VERBOSE"))
        fprintf(stderr, "[levyh] factor compacted: %.2f GB -> %.2f GB\n", 8e-9 * (double)old_len, 8e-9 * (double)len);
}

void prepare_propagator(Ctx &ctx, HMat &F, double eps2) {
    LH_REQUIRE(F.factored, LH_EINVAL, "prepare_propagator needs an H-LU factorization");
    SolvePlans &S = plans_of(F);
    if (S.Z) return;
    PlanJob *job = F.bg_plan ? static_cast<PlanJob *>(F.bg_plan.get()) : nullptr;
    auto Z = std::make_shared<HMat>();
    std::shared_ptr<Plan> P;
    std::vector<std::shared_ptr<Plan>> parts;
    bool uploaded = false;
    if (job && job->f_prop.valid()) {
        job->f_prop.wait();
        if (job->prop_error.empty() && (job->prop || !job->prop_parts.empty())) {
            copy_structure(*Z, job->Z);
            Z->nslots = job->Z.nslots;
            Z->arena_len = job->Z.arena_len;
            P = std::move(job->prop);
            parts = std::move(job->prop_parts);
            uploaded = job->prop_uploaded && P;
            if (eps2 != 1e-10) {
                if (P) patch_eps(*P, eps2);
                for (auto &q : parts) patch_eps(*q, eps2);
                if (uploaded)  // refresh the device task array
                    LH_CUDA(cudaMemcpyAsync(P->d_tasks, P->tasks.data(), sizeof(DTask) * P->tasks.size(),
                                            cudaMemcpyHostToDevice, ctx.stream));
            }
        }
    }
    if (!P && parts.empty()) {
        block_layout(*Z, F, 2, prop_kcap_for(F));
        P = plan_propagator(F, *Z, eps2, 8, &parts);
    }
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
    const bool verbose = getenv("LEVYH_PLAN_VERBOSE") != nullptr;
    auto memlog = [&](const char *what) {
        if (!verbose) return;
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        fprintf(stderr, "[levyh] propagator memory %s: %.2f GB used of %.2f\n", what, (tot - fr) * 1e-9, tot * 1e-9);
    };
    auto ta = now();
    memlog("before Z");
    if (verbose)
        fprintf(stderr, "[levyh] propagator: Z arena %.2f GB, plan %.2f GB on the device (%zu part(s))\n",
                8e-9 * (double)Z->arena_len, 1e-9 * (P ? plan_device_bytes(*P) : plan_device_bytes(*parts[0])),
                P ? (size_t)1 : parts.size());
    if (P) Z->d_arena = dalloc<double>(std::max<i64>(Z->arena_len, 1));
    Z->d_ranks = dalloc<int32_t>(std::max(Z->nslots, 1));
    LH_CUDA(cudaMemsetAsync(Z->d_ranks, 0, sizeof(int32_t) * std::max(Z->nslots, 1), ctx.stream));
    double ntask = 0.0, build_s = 0.0, temp_b = 0.0;
    auto t0 = now();
    if (P) {
        if (!uploaded) P->upload(ctx.stream);
        t0 = now();
        run_plan(ctx, *P, F, Z.get(), nullptr, -1, "propagator");
        ntask = (double)P->tasks.size();
        build_s = P->build_seconds;
        temp_b = (double)P->temp_len * 8.0;
        P.reset();
    } else {
        // large N: the independent column parts Z[:, J] = (LU)^-1 I[:, J] one after another.
        // The factor is compacted first; each part's DAG is uploaded, runs into a scratch buffer
        // of the part's extent, and the part is then packed at capacity max(rank, 1) and its DAG
        // freed; the packed parts form Z's arena at the end.
        compact_factor(ctx, F, parts);
        memlog("factor compacted");
        i64 xmax = 0;
        for (auto &q : parts) xmax = std::max(xmax, q->x_len);
        double *scratch = dalloc<double>(std::max<i64>(xmax, 1));
        std::vector<std::pair<double *, i64>> packed;
        i64 zlen = 0;
        t0 = now();
        try {
            for (auto &q : parts) {
                q->upload(ctx.stream);
                memlog("part uploaded");
                run_plan(ctx, *q, F, Z.get(), nullptr, -1, "propagator", scratch);
                ntask += (double)q->tasks.size();
                build_s = std::max(build_s, q->build_seconds);
                temp_b = std::max(temp_b, (double)q->temp_len * 8.0);
                Z->sync_ranks(ctx.stream);
                i64 len = 0;
                double *buf = compact_range(ctx, *Z, scratch, q->x_base, q->x_base, q->x_base + q->x_len, zlen, len);
                packed.push_back({buf, len});
                zlen += len;
                q.reset();
            }
        } catch (...) {
            cudaFree(scratch);
            for (auto &pb : packed) cudaFree(pb.first);
            throw;
        }
        parts.clear();
        cudaFree(scratch);
        memlog("parts packed");
        Z->d_arena = dalloc<double>(std::max<i64>(zlen, 1));
        i64 o = 0;
        for (auto &pb : packed) {
            LH_CUDA(cudaMemcpyAsync(Z->d_arena + o, pb.first, sizeof(double) * pb.second, cudaMemcpyDeviceToDevice,
                                    ctx.stream));
            LH_CUDA(cudaStreamSynchronize(ctx.stream));
            cudaFree(pb.first);
            o += pb.second;
        }
        Z->arena_len = zlen;
    }
    Z->sync_ranks(ctx.stream);
    auto t1 = now();
    memlog("Z computed");
    Z->lu_stats[0] = ntask;
    Z->lu_stats[1] = build_s;
    Z->lu_stats[2] = temp_b;
    Z->lu_stats[3] = sec(t0, t1);
    auto t2 = now();
    // near-field compression of Z: its off-diagonal dense leaves are
    // numerically low-rank, which cuts the bytes every CN step streams
    if (!getenv("LEVYH_NO_NF_COMPRESS")) {
        double nf_eps = 1e-2 * std::min(eps2, 1e-10);
        if (const char *e = getenv("LEVYH_NF_EPS")) nf_eps = atof(e);
        Z->lu_stats[4] = (double)compress_near_field(ctx, *Z, nf_eps);
    }
    // coarsening: 2 x 2 low-rank siblings merged into one block where that saves bytes
    if (!getenv("LEVYH_NO_COARSEN")) {
        double c_eps = eps2;
        if (const char *e = getenv("LEVYH_COARSEN_EPS")) c_eps = atof(e);
        Z->lu_stats[5] = (double)coarsen_hmat(ctx, *Z, c_eps);
    }
    auto t3 = now();
    memlog("near-field compressed + coarsened");
    S.mvZ = build_mv_plan(*Z, Z->leafblocks, ctx.stream);
    memlog("matvec plan of Z");
    // nested (H2) bases for the single-RHS step (zshared.cu), checked against the H-form of Z
    // on a probe vector; else shared leaf bases
    if (!getenv("LEVYH_NO_H2")) {
        double sb_eps = 1e-2 * std::min(eps2, 1e-10);
        if (const char *e = getenv("LEVYH_SB_EPS")) sb_eps = atof(e);
        const int split = getenv("LEVYH_H2_SPLIT") ? atoi(getenv("LEVYH_H2_SPLIT")) : -1;  // -1: automatic
        auto zs = std::make_shared<HMat>();
        std::shared_ptr<MvPlan> pz;
        // leaves above 64 rows (cfg5's 128): the nested bases are built on copies of the cluster
        // trees with those leaves split at 64 rows (Z's blocks keep their clusters)
        bool big = false;
        for (const Tree *T : {Z->rt, Z->ct})
            for (int32_t lc : T->leaves) big = big || T->nodes[lc].size() > 64;
        const Tree *rt0 = Z->rt, *ct0 = Z->ct;
        auto rh0 = Z->rt_hold, ch0 = Z->ct_hold;
        if (big && !getenv("LEVYH_NO_H2_REFINE")) {
            auto r64 = refine_tree_leaves(*Z->rt, 64);
            auto c64 = Z->ct == Z->rt ? r64 : refine_tree_leaves(*Z->ct, 64);
            Z->rt = r64.get();
            Z->ct = c64.get();
            Z->rt_hold = r64;
            Z->ct_hold = c64;
        }
        bool built = false;
        try {
            built = build_h2(ctx, *Z, sb_eps, split, *zs, pz, S.zs_stats);
        } catch (...) {
            Z->rt = rt0;
            Z->ct = ct0;
            Z->rt_hold = rh0;
            Z->ct_hold = ch0;
            throw;
        }
        Z->rt = rt0;
        Z->ct = ct0;
        Z->rt_hold = rh0;
        Z->ct_hold = ch0;
        if (built) {
            const double err = probe_rel_err(ctx, *S.mvZ, *Z, *pz, *zs);
            if (getenv("LEVYH_PLAN_VERBOSE")) fprintf(stderr, "[levyh] H2 probe: relative error %.3e\n", err);
            if (err <= 1e-10) {
                S.ZS = zs;
                S.mvZS = pz;
                S.zs_probe = err;
            }
        }
    }
    memlog("H2 form built");
    if (!S.mvZS && !getenv("LEVYH_NO_SHARED_BASIS")) {
        double sb_eps = 1e-2 * std::min(eps2, 1e-10);
        if (const char *e = getenv("LEVYH_SB_EPS")) sb_eps = atof(e);
        auto zs = std::make_shared<HMat>();
        std::shared_ptr<MvPlan> pz;
        if (build_shared_basis(ctx, *Z, sb_eps, *zs, pz, S.zs_stats)) {
            // same acceptance rule as the H2 form: a form that misses the probe is not installed
            // and the step streams the H-form of Z itself
            const double err = probe_rel_err(ctx, *S.mvZ, *Z, *pz, *zs);
            if (getenv("LEVYH_PLAN_VERBOSE"))
                fprintf(stderr, "[levyh] shared-basis probe: relative error %.3e\n", err);
            if (err <= 1e-10) {
                S.ZS = zs;
                S.mvZS = pz;
                S.zs_probe = err;
            }
        }
    }
    if (getenv("LEVYH_PLAN_VERBOSE"))
        fprintf(stderr, "[levyh] propagator: alloc+upload %.3f s, exec %.3f s, free plan %.3f s, "
                        "near-field compression + coarsening %.3f s (%.0f leaves, %.0f merges), matvec plan "
                        "%.3f s\n", sec(ta, t0), sec(t0, t1), sec(t1, t2), sec(t2, t3), Z->lu_stats[4],
                Z->lu_stats[5], sec(t3, now()));
    S.Z = Z;
    if (!S.tmp) {
        S.tmp_len = F.nrows;
        S.tmp = dalloc<double>(S.tmp_len);
    }
}

int step_graph_kernels(HMat &F) { return plans_of(F).g_kernels; }

void cn_last_path(HMat &F, int32_t *out) {
    SolvePlans &S = plans_of(F);
    for (int k = 0; k < 3; ++k) out[k] = S.last_path[k];
    out[3] = S.g_kernels;
}

// Y = alpha Z X + beta W for row-major multi-RHS blocks: the nested-basis walk as batched DMMA
// products (h2mm.cu) when Z has its H2 form, else the DMMA matmat of Z's H-form
static bool z_h2mm(const SolvePlans &S) {
    return S.mvZS && S.mvZS->h2 && S.mvZS->h2->mm && !getenv("LEVYH_NO_H2MM");
}
void propagator_stats(HMat &F, double *out) {
    SolvePlans &S = plans_of(F);
    LH_REQUIRE(S.Z != nullptr, LH_EINVAL, "call prepare_propagator first");
    for (int k = 0; k < 6; ++k) out[k] = S.Z->lu_stats[k];
    out[6] = S.mvZS ? (S.mvZS->h2 ? 2.0 : 1.0) : 0.0;
    out[7] = S.zs_probe;
    out[8] = S.zs_stats[0];
    out[9] = S.zs_stats[1];
    // multi-RHS form of Z and its flops per right-hand side: the H2 walk (h2mm.cu) plus the
    // segment matmat of the dense leaves and row bases, or the H-form matmat (2 x stored scalars)
    auto stored2 = [](HMat &H) {
        H.sync_ranks(nullptr);
        double sc = 0.0;
        for (int32_t b : H.leafblocks) {
            const Node &nd = H.nodes[b];
            if (nd.kind == K_LR) sc += (double)H.h_ranks[nd.rslot] * (nd.m + nd.n);
            else if (nd.kind != K_ZERO && nd.kind != K_HIER) sc += (double)nd.m * nd.n;
        }
        return 2.0 * sc;
    };
    if (z_h2mm(S)) {
        out[10] = S.mvZS->h2->mm->flops_per_rhs + stored2(*S.ZS);
        out[11] = 2.0;
    } else {
        out[10] = stored2(*S.Z);
        out[11] = 1.0;
    }
}

static void z_matmat(Ctx &ctx, SolvePlans &S, const double *X, double *Y, i64 ldk, double alpha, double beta,
                     const double *W, const MmBufs &bz) {
    if (z_h2mm(S)) h2mm_run(*S.mvZS->h2->mm, *S.mvZS, X, Y, ldk, alpha, beta, W, ctx.stream);
    else mm_run(*S.mvZ, X, Y, ldk, alpha, beta, W, bz.T, bz.part, ctx.stream);
}

static void solve_propagator(Ctx &ctx, HMat &F, double *b, i64 ldb, int nrhs) {
    SolvePlans &S = plans_of(F);
    LH_REQUIRE(S.Z != nullptr, LH_EINVAL, "call prepare_propagator first");
    if (nrhs >= mm_min_rhs()) {  // B <- Z B as one DMMA matmat
        const i64 n = F.nrows, ldk = mm_pad(nrhs);
        double *Xr = ctx.mm[0].ensure(n * ldk), *Yr = ctx.mm[1].ensure(n * ldk);
        MmBufs bb = mm_bufs(ctx, *S.mvZ, ldk);
        mm_transpose(b, ldb, Xr, ldk, n, nrhs, true, ctx.stream);
        z_matmat(ctx, S, Xr, Yr, ldk, 1.0, 0.0, nullptr, bb);
        mm_transpose(Yr, ldk, b, ldb, n, nrhs, false, ctx.stream);
        LH_CUDA(cudaStreamSynchronize(ctx.stream));
        return;
    }
    for (int q = 0; q < nrhs; ++q) {
        double *bq = b + (i64)q * ldb;
        mv_run(S.z1plan(), S.z1mat(), bq, S.tmp, 1.0, 0.0, ctx.stream, ctx.num_sms);
        LH_CUDA(cudaMemcpyAsync(bq, S.tmp, sizeof(double) * F.nrows, cudaMemcpyDeviceToDevice,
                                ctx.stream));
    }
}

// The one-matvec CN step u <- 2 Z u - u equals Z (A- u) only for A- = 2I - A+.  That is decided
// from provenance, not measured: derive() sets cn_pair_of when it built hminus from this
// factor's A+ and verified every stored entry (build.cu: pair_check_kernel); checkpoints keep
// the tags.  Anything else (an independently assembled A-) runs u <- Z (A- u).
static bool cn_pair_ok(const HMat &Hm, const HMat &F) { return Hm.cn_pair_tag != 0 && Hm.cn_pair_tag == F.pair_tag; }

static void solve_inverse(Ctx &ctx, HMat &F, double *b, i64 ldb, int nrhs) {
    SolvePlans &S = plans_of(F);
    LH_REQUIRE(S.XL != nullptr, LH_EINVAL, "call prepare_inverse first");
    for (int q = 0; q < nrhs; ++q) {
        double *bq = b + (i64)q * ldb;
        mv_run(*S.mvL, *S.XL, bq, S.tmp, 1.0, 0.0, ctx.stream, ctx.num_sms);
        mv_run(*S.mvU, *S.XU, S.tmp, bq, 1.0, 0.0, ctx.stream, ctx.num_sms);
    }
}

// trisolve_lower / trisolve_upper_right with a dense right-hand side (hops.py:282-310):
// T X = B with one triangle of T (mode 0 lower, 1 upper, 2 upper transposed), in place
void trisolve_dense(Ctx &ctx, HMat &T, int mode, bool unit, double *b, i64 ldb, int nrhs) {
    LH_REQUIRE(T.nrows == T.ncols, LH_EINVAL, "triangular solve needs a square H-matrix");
    LH_REQUIRE(mode >= 0 && mode <= 2, LH_EINVAL, "mode must be 0 (L), 1 (U) or 2 (U^T)");
    LH_REQUIRE(ldb == T.nrows, LH_EINVAL, "solve expects a packed right-hand side (ldb == n)");
    if (nrhs <= 0) return;
    SolvePlans &S = plans_of(T);
    const int CAP = 64;
    auto &P = S.tri[mode][unit ? 1 : 0];
    if (!P) {
        P = plan_trisolve_dense(T, T.nrows, CAP, mode, unit, mode == 0 ? "L" : "U");
        P->upload(ctx.stream);
    }
    for (int c0 = 0; c0 < nrhs; c0 += CAP) {
        const int kc = std::min(CAP, nrhs - c0);
        run_plan(ctx, *P, T, nullptr, b + (i64)c0 * ldb, kc, "trisolve");
    }
}

// trisolve_lower / trisolve_upper_right with an H-matrix right-hand side (hops.py:282-310):
// X (already a deep copy of B) solved in place on the executor
void trisolve_block(Ctx &ctx, HMat &T, HMat &X, int mode, bool unit, double eps2) {
    LH_REQUIRE(T.nrows == T.ncols, LH_EINVAL, "triangular solve needs a square H-matrix");
    auto P = plan_trisolve_block(T, X, mode, unit, eps2);
    P->upload(ctx.stream);
    run_plan(ctx, *P, T, &X, nullptr, -1, mode == 0 ? "trisolve_lower (block)" : "trisolve_upper_right (block)");
    X.sync_ranks(ctx.stream);
    X.mv_plan.reset();
}

// lowrank_add_recompress (hops.py:147-156): (u, v) <- recompressed u1 v1^T + u2 v2^T with the
// Frobenius-tail rule at eps2, as one LRADD task on the executor.  Device, column-major
// factors (ld = m resp. n); outputs need r1 + r2 columns; the new rank is returned.
int lowrank_add_recompress(Ctx &ctx, i64 m, i64 n, const double *u1, const double *v1, int r1,
                           const double *u2, const double *v2, int r2, double eps2, double *uo,
                           double *vo) {
    LH_REQUIRE(m > 0 && n > 0 && r1 >= 0 && r2 >= 0, LH_EINVAL, "invalid low-rank shapes");
    LH_REQUIRE(r1 + r2 <= KA_MAX, LH_ERANK, "r1 + r2 exceeds the recompression width");
    if (r2 == 0) {  // the task recompresses the target plus a non-empty addend
        std::swap(u1, u2);
        std::swap(v1, v2);
        std::swap(r1, r2);
    }
    if (r2 == 0) return 0;
    const int kcap = r1 + r2;
    HMat W;
    const i64 uo_off = 0, vo_off = m * kcap, u2_off = vo_off + n * kcap, v2_off = u2_off + m * r2;
    W.arena_len = v2_off + n * r2;
    W.d_arena = dalloc<double>(W.arena_len);
    W.nslots = 1;
    W.d_ranks = dalloc<int32_t>(1);
    cudaStream_t s = ctx.stream;
    if (r1 > 0) {
        LH_CUDA(cudaMemcpyAsync(W.d_arena + uo_off, u1, sizeof(double) * m * r1, cudaMemcpyDeviceToDevice, s));
        LH_CUDA(cudaMemcpyAsync(W.d_arena + vo_off, v1, sizeof(double) * n * r1, cudaMemcpyDeviceToDevice, s));
    }
    LH_CUDA(cudaMemcpyAsync(W.d_arena + u2_off, u2, sizeof(double) * m * r2, cudaMemcpyDeviceToDevice, s));
    LH_CUDA(cudaMemcpyAsync(W.d_arena + v2_off, v2, sizeof(double) * n * r2, cudaMemcpyDeviceToDevice, s));
    LH_CUDA(cudaMemcpyAsync(W.d_ranks, &r1, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    Plan P;
    DTask t;
    std::memset(&t, 0, sizeof(t));
    for (auto &v : t.v) v.wslot = -1;
    t.type = T_LRADD;
    t.path = -1;
    t.alpha = 1.0;
    t.alpha2 = eps2;
    t.v[0] = DView{uo_off, (int32_t)m, kcap, (int32_t)m, 0, B_F, 0, 0};
    t.v[1] = DView{vo_off, (int32_t)n, kcap, (int32_t)n, 0, B_F, 0, 0};
    t.v[2] = DView{u2_off, (int32_t)m, r2, (int32_t)m, -1, B_F, 0, 0};
    t.v[3] = DView{v2_off, (int32_t)n, r2, (int32_t)n, -1, B_F, 0, 0};
    P.tasks.push_back(t);
    P.nslots_total = 1;
    P.slot_off_x = 1;
    P.slot_off_tmp = 1;
    P.upload(s);
    run_plan(ctx, P, W, nullptr, nullptr, -1, "lowrank_add_recompress");
    W.sync_ranks(s);
    const int r = W.h_ranks[0];
    if (r > 0) {
        LH_CUDA(cudaMemcpyAsync(uo, W.d_arena + uo_off, sizeof(double) * m * r, cudaMemcpyDeviceToDevice, s));
        LH_CUDA(cudaMemcpyAsync(vo, W.d_arena + vo_off, sizeof(double) * n * r, cudaMemcpyDeviceToDevice, s));
    }
    LH_CUDA(cudaStreamSynchronize(s));
    return r;
}

void solve(Ctx &ctx, HMat &F, double *b, i64 ldb, int nrhs, int method) {
    LH_REQUIRE(F.factored, LH_EINVAL, "solve needs an H-LU factorization");
    if (nrhs <= 0) return;
    if (method == 0) solve_substitution(ctx, F, b, ldb, nrhs);
    else if (method == 1) solve_inverse(ctx, F, b, ldb, nrhs);
    else if (method == 2) solve_propagator(ctx, F, b, ldb, nrhs);
    else throw Error(LH_EINVAL, "solve method must be 0 (substitution), 1 (inverse factors) or 2 (propagator)");
}

// ---------------------------------------------------------------------------
// micro-benchmark: chains of R identical tasks through the real executor
// kind 0: GETRF 64x64 (independent blocks, chained); 1: TRSM (inverse GEMM) with k
// columns; 2: SEGMUL with one dense 64x64 piece and k columns.  out[0] = executor
// wall time per task (us, includes hand-off), out[1] = mean task body (us).
// ---------------------------------------------------------------------------
__global__ void fill_random_kernel(double *p, i64 n, double diag_boost, int m) {
    for (i64 e = (i64)blockIdx.x * NT + threadIdx.x; e < n; e += (i64)gridDim.x * NT) {
        uint64_t z = e * 0x9E3779B97F4A7C15ull + 12345;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z ^= z >> 31;
        double v = ((z >> 11) * (1.0 / 9007199254740992.0)) - 0.5;
        i64 w = e % ((i64)m * m);
        if (w % m == w / m) v += diag_boost;
        p[e] = v;
    }
}

void task_bench(Ctx &ctx, int kind, int R, int k, bool chain, double *out) {
    const int m = 64;
    HMat F;  // synthetic storage owner
    F.arena_len = (i64)R * m * m + (i64)R * m * 64;
    F.d_arena = dalloc<double>(F.arena_len);
    F.d_perm = dalloc<int32_t>((i64)R * m);
    F.inv_len = (i64)R * m * m;
    F.d_inv = dalloc<double>(F.inv_len);
    fill_random_kernel<<<1024, NT, 0, ctx.stream>>>(F.d_arena, F.arena_len, 8.0, m);
    fill_random_kernel<<<1024, NT, 0, ctx.stream>>>(F.d_inv, F.inv_len, 1.0, m);
    LH_CUDA(cudaMemsetAsync(F.d_perm, 0, sizeof(int32_t) * R * m, ctx.stream));
    std::vector<int32_t> permh((size_t)R * m);
    for (int r = 0; r < R; ++r)
        for (int i = 0; i < m; ++i) permh[(size_t)r * m + i] = i;
    upload(F.d_perm, permh, ctx.stream);
    Plan P;
    for (int r = 0; r < R; ++r) {
        DTask t;
        std::memset(&t, 0, sizeof(t));
        for (auto &v : t.v) v.wslot = -1;
        t.path = -1;
        const i64 dense_off = (i64)r * m * m, rhs_off = (i64)R * m * m + (i64)r * m * 64;
        DView D{dense_off, m, m, m, -1, B_F, 0, 0};
        DView Bv{rhs_off, m, k, m, -1, B_F, 0, 0};
        DView Iv{(i64)r * m * m, m, m, m, -1, B_INV, 0, 0};
        if (kind == 0 || kind == 3) {
            t.type = T_GETRF;
            t.aux = r * m;
            t.v[0] = D;
            t.v[1] = Iv;
            t.flags = kind == 0 ? 1 : 0;  // kind 3: LU without the packed leaf inverse
        } else if (kind == 1) {
            t.type = T_TRSM;
            t.flags = 0 | 32 | 64;
            t.aux = r * m;
            t.v[0] = D;
            t.v[1] = Bv;
            t.v[2] = Iv;
        } else {
            t.type = T_SEGMUL;
            t.alpha = -1.0;
            t.v[0] = Bv;
            t.pc_beg = (int32_t)P.pieces.size();
            DPiece pc;
            std::memset(&pc, 0, sizeof(pc));
            pc.kind = 0;
            pc.mat = D;
            pc.x = DView{(i64)R * m * m + (i64)((r + 1) % R) * m * 64, m, k, m, -1, B_F, 0, 0};
            P.pieces.push_back(pc);
            t.pc_end = (int32_t)P.pieces.size();
        }
        t.dep_beg = (int32_t)P.deps.size();
        t.dep_cnt = (chain && r > 0) ? 1 : 0;
        if (t.dep_cnt) P.deps.push_back(r - 1);
        P.tasks.push_back(t);
    }
    P.nslots_total = 0;
    P.upload(ctx.stream);
    setenv("LEVYH_TASK_PROFILE_STATS", "1", 1);
    LH_CUDA(cudaStreamSynchronize(ctx.stream));
    auto t0 = std::chrono::steady_clock::now();
    run_plan(ctx, P, F, nullptr, nullptr, -1, "bench");
    double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    out[0] = 1e6 * wall / R;
    out[1] = g_last_mean_task_us;
}

// algorithmic bytes of the two matvec phases over `blocks` (fp64): phase 1 reads V,
// phase 2 reads the dense leaves and U, reads x once and writes y once.
static void mv_bytes(const HMat &H, const std::vector<int32_t> &blocks, double &b1, double &b2) {
    b1 = b2 = 0.0;
    for (int32_t b : blocks) {
        const Node &nd = H.nodes[b];
        if (nd.kind == K_LR) {
            double r = H.h_ranks[nd.rslot];
            b1 += 8.0 * r * nd.n;
            b2 += 8.0 * r * nd.m;
        } else if (nd.kind == K_DENSE || nd.kind == K_FDENSE) {
            b2 += 8.0 * nd.m * nd.n;
        }
    }
    b2 += 16.0 * H.nrows;
}

// Per-kernel CUDA-event timing of one CN step.  method 1: out[0..5] = mean ms of vtx(H-),
// seg(H-), vtx(XL), seg(XL), vtx(XU), seg(XU); out[6..11] their algorithmic bytes;
// out[12..14] stored scalars of H-, XL, XU.  method 2: out[0..1] / out[6..7] = vtx(Z), seg(Z)
// of the step u <- 2 Z u - u (rest 0); out[12] H-, out[13] Z.  out[15] stored scalars of F.
void step_profile(Ctx &ctx, HMat &Hm, HMat &F, double *u, int iters, int method, double *out) {
    SolvePlans &S = plans_of(F);
    if (method == 2) LH_REQUIRE(S.Z != nullptr, LH_EINVAL, "call prepare_propagator first");
    else LH_REQUIRE(S.XL != nullptr, LH_EINVAL, "call prepare_inverse first");
    double *y = (double *)ctx.ensure_scratch(sizeof(double) * (size_t)Hm.nrows);
    Hm.sync_ranks(ctx.stream);
    struct Mv {
        const MvPlan *P;
        HMat *H;
        double *x, *y;
        double alpha, beta;
        const double *z;
    };
    std::vector<Mv> mv;
    if (method == 2) {
        S.z1mat().sync_ranks(ctx.stream);
        mv.push_back({&S.z1plan(), &S.z1mat(), u, y, 2.0, -1.0, u});
    } else {
        S.XL->sync_ranks(ctx.stream);
        S.XU->sync_ranks(ctx.stream);
        mv.push_back({&get_mv_plan(Hm, ctx.stream), &Hm, u, y, 1.0, 0.0, nullptr});
        mv.push_back({S.mvL.get(), S.XL.get(), y, S.tmp, 1.0, 0.0, nullptr});
        mv.push_back({S.mvU.get(), S.XU.get(), S.tmp, u, 1.0, 0.0, nullptr});
    }
    if (method == 2 && S.z1plan().h2 && S.z1plan().h2->step2) {
        const MvPlan &Pz = S.z1plan();
        // two-kernel H2 step (h2step.cu): xpad / K1 / K2 timed separately; bytes are the ring
        // operands each kernel streams plus its vector writes (yd by K1, y by K2) and the
        // staging copy of x (read + write)
        // as cn_steps runs it: u copied into the staging buffer once, then K1 + K2 in place
        cudaEvent_t ev[4];
        for (auto &e : ev) LH_CUDA(cudaEventCreate(&e));
        double acc3[3] = {0, 0, 0};
        LH_CUDA(cudaEventRecord(ev[3], ctx.stream));
        h2s_load(*Pz.h2, u, ctx.stream);
        LH_CUDA(cudaEventRecord(ev[0], ctx.stream));
        LH_CUDA(cudaEventSynchronize(ev[0]));

        for (int it = 0; it < iters; ++it) {
            h2s_step_inplace(*Pz.h2, 2.0, -1.0, ctx.stream, ev);
            LH_CUDA(cudaEventSynchronize(ev[2]));
            for (int k = 0; k < 2; ++k) {
                float ms = 0.f;
                LH_CUDA(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
                acc3[k + 1] += ms;
            }
        }
        h2s_store(*Pz.h2, u, ctx.stream);
        LH_CUDA(cudaStreamSynchronize(ctx.stream));
        for (auto &e : ev) cudaEventDestroy(e);
        for (int k = 0; k < 16; ++k) out[k] = 0.0;
        const H2S &S2 = *Pz.h2->step2;
        for (int k = 0; k < 3; ++k) out[k] = acc3[k] / std::max(iters, 1);
        out[6] = 0.0;  // the staging copy runs once per cn_steps call, not per step
        out[7] = (double)S2.bytes1 + 8.0 * Hm.nrows;
        out[8] = (double)S2.bytes2 + 8.0 * Hm.nrows;
        out[11] = 1.0;  // layout flag: (staging copy: 0 per step), K1, K2
    } else {
    const int nk = 2 * (int)mv.size();
    cudaEvent_t ev[7];
    for (auto &e : ev) LH_CUDA(cudaEventCreate(&e));
    std::vector<double> acc(6, 0.0);
    for (int it = 0; it < iters; ++it) {
        for (size_t q = 0; q < mv.size(); ++q) {
            const Mv &m = mv[q];
            LH_CUDA(cudaEventRecord(ev[2 * q], ctx.stream));
            mv_vtx_launch(*m.P, *m.H, m.x, ctx.num_sms, ctx.stream);
            LH_CUDA(cudaEventRecord(ev[2 * q + 1], ctx.stream));
            mv_seg_launch(*m.P, *m.H, m.x, m.y, m.alpha, m.beta, ctx.stream, ctx.num_sms, m.z);
        }
        LH_CUDA(cudaEventRecord(ev[nk], ctx.stream));
        if (method == 2)
            LH_CUDA(cudaMemcpyAsync(u, y, sizeof(double) * Hm.nrows, cudaMemcpyDeviceToDevice,
                                    ctx.stream));
        LH_CUDA(cudaEventSynchronize(ev[nk]));
        for (int k = 0; k < nk; ++k) {
            float ms = 0.f;
            LH_CUDA(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
            acc[k] += ms;
        }
    }
    LH_CUDA(cudaStreamSynchronize(ctx.stream));
    for (auto &e : ev) cudaEventDestroy(e);
    for (int k = 0; k < 16; ++k) out[k] = 0.0;
    for (int k = 0; k < nk; ++k) out[k] = acc[k] / std::max(iters, 1);
    }
    auto nonzero = [](const HMat &H) {
        std::vector<int32_t> bl;
        for (int32_t b : H.leafblocks)
            if (H.nodes[b].kind != K_ZERO) bl.push_back(b);
        return bl;
    };
    auto stored = [](const HMat &H, const std::vector<int32_t> &blocks) {
        double s = 0.0;
        for (int32_t b : blocks) {
            const Node &nd = H.nodes[b];
            if (nd.kind == K_LR) s += (double)H.h_ranks[nd.rslot] * (nd.m + nd.n);
            else if (nd.kind != K_ZERO && nd.kind != K_HIER) s += (double)nd.m * nd.n;
        }
        return s;
    };
    for (size_t q = 0; q < mv.size() && out[11] == 0.0; ++q) {
        const auto bl = nonzero(*mv[q].H);
        mv_bytes(*mv[q].H, bl, out[6 + 2 * q], out[7 + 2 * q]);
        if (mv[q].z && mv[q].z != mv[q].y) out[7 + 2 * q] += 8.0 * mv[q].H->nrows;  // reads z
        if (mv[q].P->cpl) out[6 + 2 * q] += (double)mv[q].P->cpl->bytes;  // coupling (phase 1 side)
        if (mv[q].P->h2) out[6 + 2 * q] += (double)mv[q].P->h2->bytes;  // H2 walk (phase 1 side)
    }
    out[12] = stored(Hm, Hm.leafblocks);
    if (method == 2) {
        out[13] = stored(S.z1mat(), S.z1mat().leafblocks) + (S.mvZS ? S.zs_stats[1] : 0.0);
    } else {
        out[13] = stored(*S.XL, nonzero(*S.XL));
        out[14] = stored(*S.XU, nonzero(*S.XU));
    }
    F.sync_ranks(ctx.stream);
    out[15] = stored(F, F.leafblocks);
}

static int count_kernel_nodes(cudaGraph_t g) {
    size_t nn = 0;
    LH_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    LH_CUDA(cudaGraphGetNodes(g, nodes.data(), &nn));
    int k = 0;
    for (auto nd : nodes) {
        cudaGraphNodeType ty;
        LH_CUDA(cudaGraphNodeGetType(nd, &ty));
        k += ty == cudaGraphNodeTypeKernel;
    }
    return k;
}

void cn_steps(Ctx &ctx, HMat &Hm, HMat &F, double *u, i64 ldu, int nrhs, int nsteps, int method) {
    LH_REQUIRE(F.factored, LH_EINVAL, "cn_steps needs an H-LU factorization of A+");
    LH_REQUIRE(Hm.nrows == F.nrows, LH_EINVAL, "operator sizes differ");
    // A-'s matvec plan only when the step reads A- (not for u <- 2 Z u - u on the CN pair, so a
    // spilled A- stays on the host)
    const bool pair2 = method == 2 && cn_pair_ok(Hm, F);
    MvPlan *Pmp = pair2 ? nullptr : &get_mv_plan(Hm, ctx.stream);
    double *y = (double *)ctx.ensure_scratch(sizeof(double) * (size_t)Hm.nrows);
    if (method == 1 || method == 2) {
        SolvePlans &S = plans_of(F);
        if (method == 1) LH_REQUIRE(S.XL != nullptr, LH_EINVAL, "call prepare_inverse first");
        else LH_REQUIRE(S.Z != nullptr, LH_EINVAL, "call prepare_propagator first");
        // method 1: one step = 3 H-matvecs (A-, L^-1, U^-1); method 2: u <- 2 Z u - u, one
        // H-matvec of the propagator (Z A- u with two when hminus is not 2I - A+).  The step
        // is captured once as a CUDA graph, cached per (operator, vector, scratch, method).
        const int shape = method == 2 ? (cn_pair_ok(Hm, F) ? 2 : 3) : 1;
        S.last_path[0] = shape;
        S.last_path[1] = method == 2 && nrhs >= mm_min_rhs() ? (z_h2mm(S) ? 2 : 1) : 0;
        S.last_path[2] = 0;
        if (method == 2 && nrhs >= mm_min_rhs()) {
            // K right-hand sides: U row-major on the device for the whole run, each step one
            // (or two) DMMA matmats: U <- 2 Z U - U, or U <- Z (A- U)
            const i64 n = Hm.nrows, ldk = mm_pad(nrhs);
            double *Xr = ctx.mm[0].ensure(n * ldk), *Yr = ctx.mm[1].ensure(n * ldk);
            // the two plans share the context's grow-only scratch: size it for both before taking
            // pointers (a later, larger request would reallocate under the first plan's pointers)
            mm_bufs(ctx, *S.mvZ, ldk);
            MmBufs bm = shape == 3 ? mm_bufs(ctx, *Pmp, ldk) : MmBufs{};
            MmBufs bz = mm_bufs(ctx, *S.mvZ, ldk);
            mm_transpose(u, ldu, Xr, ldk, n, nrhs, true, ctx.stream);
            for (int k = 0; k < nsteps; ++k) {
                if (shape == 2) {
                    z_matmat(ctx, S, Xr, Yr, ldk, 2.0, -1.0, Xr, bz);
                } else {
                    mm_run(*Pmp, Xr, Yr, ldk, 1.0, 0.0, nullptr, bm.T, bm.part, ctx.stream);
                    std::swap(Xr, Yr);
                    z_matmat(ctx, S, Xr, Yr, ldk, 1.0, 0.0, nullptr, bz);
                }
                std::swap(Xr, Yr);
            }
            mm_transpose(Xr, ldk, u, ldu, n, nrhs, false, ctx.stream);
            LH_CUDA(cudaStreamSynchronize(ctx.stream));
            return;
        }
        const MvPlan &Pz1 = S.z1plan();
        const bool inplace = shape == 2 && Pz1.h2 && Pz1.h2->step2 && !getenv("LEVYH_NO_INPLACE_STEP");
        for (int q = 0; q < nrhs; ++q) {
            double *uq = u + (i64)q * ldu;
            if (inplace) {
                // two-kernel H2 step on the staging copy: u in once, K1 + K2 per step (captured
                // once), u out once
                const int key = 4;  // graph shape tag of the in-place step
                if (!(S.graph && S.g_hm == Hm.id && S.g_gen == Hm.gen && S.g_method == key)) {
                    if (S.graph) {
                        cudaGraphExecDestroy(S.graph);
                        S.graph = nullptr;
                    }
                    cudaGraph_t g;
                    LH_CUDA(cudaStreamBeginCapture(ctx.stream, cudaStreamCaptureModeThreadLocal));
                    try {
                        h2s_step_inplace(*Pz1.h2, 2.0, -1.0, ctx.stream);
                    } catch (...) {
                        cudaStreamEndCapture(ctx.stream, &g);
                        throw;
                    }
                    LH_CUDA(cudaStreamEndCapture(ctx.stream, &g));
                    S.g_kernels = count_kernel_nodes(g);
                    LH_CUDA(cudaGraphInstantiate(&S.graph, g, 0));
                    cudaGraphDestroy(g);
                    S.g_u = nullptr;
                    S.g_hm = Hm.id;
                    S.g_gen = Hm.gen;
                    S.g_y = nullptr;
                    S.g_method = key;
                }
                h2s_load(*Pz1.h2, uq, ctx.stream);
                for (int k = 0; k < nsteps; ++k) LH_CUDA(cudaGraphLaunch(S.graph, ctx.stream));
                h2s_store(*Pz1.h2, uq, ctx.stream);
                continue;
            }
            if (!(S.graph && S.g_u == uq && S.g_hm == Hm.id && S.g_gen == Hm.gen && S.g_y == y &&
                  S.g_method == shape)) {
                if (S.graph) {
                    cudaGraphExecDestroy(S.graph);
                    S.graph = nullptr;
                }
                cudaGraph_t g;
                LH_CUDA(cudaStreamBeginCapture(ctx.stream, cudaStreamCaptureModeThreadLocal));
                try {
                    if (shape == 1) {
                        mv_run(*Pmp, Hm, uq, y, 1.0, 0.0, ctx.stream, ctx.num_sms);
                        mv_run(*S.mvL, *S.XL, y, S.tmp, 1.0, 0.0, ctx.stream, ctx.num_sms);
                        mv_run(*S.mvU, *S.XU, S.tmp, uq, 1.0, 0.0, ctx.stream, ctx.num_sms);
                    } else if (shape == 2) {
                        mv_run(S.z1plan(), S.z1mat(), uq, y, 2.0, -1.0, ctx.stream, ctx.num_sms, uq);
                        LH_CUDA(cudaMemcpyAsync(uq, y, sizeof(double) * Hm.nrows,
                                                cudaMemcpyDeviceToDevice, ctx.stream));
                    } else {
                        mv_run(*Pmp, Hm, uq, y, 1.0, 0.0, ctx.stream, ctx.num_sms);
                        mv_run(S.z1plan(), S.z1mat(), y, uq, 1.0, 0.0, ctx.stream, ctx.num_sms);
                    }
                } catch (...) {
                    cudaStreamEndCapture(ctx.stream, &g);
                    throw;
                }
                LH_CUDA(cudaStreamEndCapture(ctx.stream, &g));
                S.g_kernels = count_kernel_nodes(g);
                LH_CUDA(cudaGraphInstantiate(&S.graph, g, 0));
                cudaGraphDestroy(g);
                S.g_u = uq;
                S.g_hm = Hm.id;
                S.g_gen = Hm.gen;
                S.g_y = y;
                S.g_method = shape;
            }
            for (int k = 0; k < nsteps; ++k) LH_CUDA(cudaGraphLaunch(S.graph, ctx.stream));
        }
        LH_CUDA(cudaStreamSynchronize(ctx.stream));
        return;
    }
    LH_REQUIRE(method == 0, LH_EINVAL, "cn_steps method must be 0, 1 or 2");
    {
        SolvePlans &S = plans_of(F);
        S.last_path[0] = 0;
        S.last_path[1] = S.last_path[2] = 0;
    }
    for (int q = 0; q < nrhs; ++q) {
        double *uq = u + (i64)q * ldu;
        for (int k = 0; k < nsteps; ++k) {
            mv_run(*Pmp, Hm, uq, y, 1.0, 0.0, ctx.stream, ctx.num_sms);
            LH_CUDA(cudaMemcpyAsync(uq, y, sizeof(double) * Hm.nrows, cudaMemcpyDeviceToDevice,
                                    ctx.stream));
            solve_substitution(ctx, F, uq, Hm.nrows, 1);
        }
    }
}

static bool is_pinned(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// One CN step with HOST buffers (the reference-facing call: levy.step_cn, levy.py:295-306,
// on numpy vectors).  Method 2 with the CN pair (u <- 2 Z u - u) runs as one captured graph
// in which u arrives and the new u leaves in pieces overlapped with the V^T u and segment
// kernels (mv_run_host); any other case copies in, steps on the device and copies out.
void cn_step_host(Ctx &ctx, HMat &Hm, HMat &F, const double *u_in, double *u_out, int method) {
    LH_REQUIRE(F.factored, LH_EINVAL, "cn_steps needs an H-LU factorization of A+");
    LH_REQUIRE(Hm.nrows == F.nrows, LH_EINVAL, "operator sizes differ");
    const i64 n = Hm.nrows;
    SolvePlans &S = plans_of(F);
    if (!S.hx) {
        S.hx = dalloc<double>(n);
        S.hy = dalloc<double>(n);
    }
    bool pipelined = method == 2 && S.Z && is_pinned(u_in) && is_pinned(u_out) &&
                     !getenv("LEVYH_NO_HOST_PIPE");
    if (pipelined) pipelined = cn_pair_ok(Hm, F) && S.z1plan().npiece > 0 && S.z1plan().nbatch > 0;
    if (!pipelined) {
        LH_CUDA(cudaMemcpyAsync(S.hx, u_in, sizeof(double) * n, cudaMemcpyHostToDevice, ctx.stream));
        cn_steps(ctx, Hm, F, S.hx, n, 1, 1, method);
        LH_CUDA(cudaMemcpyAsync(u_out, S.hx, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx.stream));
        LH_CUDA(cudaStreamSynchronize(ctx.stream));
        return;
    }
    const MvPlan &P = S.z1plan();
    if (!(S.hgraph && S.hg_in == u_in && S.hg_out == u_out && S.hg_hm == Hm.id)) {
        if (S.hgraph) {
            cudaGraphExecDestroy(S.hgraph);
            S.hgraph = nullptr;
        }
        if (!S.side) LH_CUDA(cudaStreamCreateWithFlags(&S.side, cudaStreamNonBlocking));
        while ((int)S.hev.size() < 2 * P.npiece + 2) {
            cudaEvent_t e;
            LH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            S.hev.push_back(e);
        }
        cudaGraph_t g;
        LH_CUDA(cudaStreamBeginCapture(ctx.stream, cudaStreamCaptureModeThreadLocal));
        try {
            if (P.h2 && P.h2->step2 && !getenv("LEVYH_HOST_PIECES"))  // two-kernel step: copy in, step, copy out
                h2s_launch_host(*P.h2, u_in, S.hy, u_out, 2.0, -1.0, ctx.stream);
            else
                mv_run_host(P, u_in, S.hx, S.hy, u_out, 2.0, -1.0, true, ctx.stream, S.side, S.hev.data(),
                            ctx.num_sms);
        } catch (...) {
            cudaStreamEndCapture(ctx.stream, &g);
            throw;
        }
        LH_CUDA(cudaStreamEndCapture(ctx.stream, &g));
        LH_CUDA(cudaGraphInstantiate(&S.hgraph, g, 0));
        cudaGraphDestroy(g);
        S.hg_in = u_in;
        S.hg_out = u_out;
        S.hg_hm = Hm.id;
    }
    LH_CUDA(cudaGraphLaunch(S.hgraph, ctx.stream));
    LH_CUDA(cudaStreamSynchronize(ctx.stream));
    S.last_path[0] = 2;
    S.last_path[1] = 0;
    S.last_path[2] = 1;
}

}  // namespace lh

namespace lh {
// Phase-timed recompression (debug): every CTA recompresses its own copy of U (m x K),
// V (n x K) staged in shared memory, `reps` times; out[p] = mean ns of phase p
// (0 stage, 1 QR(U), 2 QR(V), 3 C = Ru Rv^T, 4 Jacobi SVD, 5 truncation + apply; 6 rank).
__global__ void __launch_bounds__(NT, 1) recomp_bench_kernel(const double *U0, const double *V0, int m,
                                                             int n, int K, int reps,
                                                             unsigned long long *acc) {
    extern __shared__ double4 smem_raw[];
    double *sm = reinterpret_cast<double *>(smem_raw);
    dev::RecompSmem &S = *reinterpret_cast<dev::RecompSmem *>(sm);
    constexpr int RS = (int)((sizeof(dev::RecompSmem) + 15) / 8) & ~1;
    double *Us = sm + RS, *Vs = Us + (i64)m * K;
    unsigned long long t[7];
    unsigned long long tot[6] = {0, 0, 0, 0, 0, 0};
    int r = 0, sweeps = 0;
    for (int rep = 0; rep < reps; ++rep) {
        __syncthreads();
        t[0] = gtimer();
        for (int e = threadIdx.x; e < m * K; e += NT) Us[e] = U0[e];
        for (int e = threadIdx.x; e < n * K; e += NT) Vs[e] = V0[e];
        __syncthreads();
        t[1] = gtimer();
        dev::cgs2(Us, m, m, K, S.Ru, S.h, S.red);
        __syncthreads();
        t[2] = gtimer();
        dev::cgs2(Vs, n, n, K, S.Rv, S.h, S.red);
        __syncthreads();
        t[3] = gtimer();
        for (int e = threadIdx.x; e < K * K; e += NT) {
            int i = e % K, j = e / K;
            double s = 0.0;
            for (int l = 0; l < K; ++l) s += S.Ru[i + l * dev::KA_MAX] * S.Rv[j + l * dev::KA_MAX];
            S.Cc[i + j * dev::KA_MAX] = s;
        }
        __syncthreads();
        t[4] = gtimer();
        sweeps = dev::jacobi_svd(S.Cc, S.Rv, K, S.sigma, S.ord, S.red);
        __syncthreads();
        t[5] = gtimer();
        r = dev::truncation_rank(S.sigma, S.ord, K, 1, 1e-10);
        for (int e = threadIdx.x; e < K * r; e += NT) {
            int l = e % K, c = e / K;
            S.Ru[l + c * dev::KA_MAX] = S.Cc[l + S.ord[c] * dev::KA_MAX];
        }
        __syncthreads();
        for (int e = threadIdx.x; e < K * r; e += NT) {
            int l = e % K, c = e / K;
            S.Cc[l + c * dev::KA_MAX] = S.Rv[l + S.ord[c] * dev::KA_MAX];
        }
        __syncthreads();
        dev::apply_coeffs(Us, m, m, K, S.Ru, dev::KA_MAX, r, Us, m);
        dev::apply_coeffs(Vs, n, n, K, S.Cc, dev::KA_MAX, r, Vs, n);
        __syncthreads();
        t[6] = gtimer();
        for (int p = 0; p < 6; ++p) tot[p] += t[p + 1] - t[p];
    }
    if (threadIdx.x == 0) {
        for (int p = 0; p < 6; ++p) atomicAdd(acc + p, tot[p]);
        atomicAdd(acc + 6, (unsigned long long)r);
        atomicAdd(acc + 7, (unsigned long long)sweeps);
    }
}

void recomp_bench(Ctx &ctx, int m, int n, int K, int reps, const double *U_host, const double *V_host,
                  double *out) {
    LH_REQUIRE(K >= 1 && K <= KA_MAX && m >= 1 && n >= 1, LH_EINVAL, "recomp_bench: bad shape");
    constexpr int RS = (int)((sizeof(dev::RecompSmem) + 15) / 8) & ~1;
    const i64 smem = 8 * (RS + (i64)(m + n) * K);
    LH_REQUIRE(smem <= SMEM_BYTES, LH_EINVAL, "recomp_bench: operands exceed shared memory");
    double *U = dalloc<double>((i64)m * K), *V = dalloc<double>((i64)n * K);
    unsigned long long *acc = dalloc<unsigned long long>(8);
    LH_CUDA(cudaMemcpyAsync(U, U_host, sizeof(double) * m * K, cudaMemcpyHostToDevice, ctx.stream));
    LH_CUDA(cudaMemcpyAsync(V, V_host, sizeof(double) * n * K, cudaMemcpyHostToDevice, ctx.stream));
    LH_CUDA(cudaMemsetAsync(acc, 0, sizeof(unsigned long long) * 8, ctx.stream));
    LH_CUDA(cudaFuncSetAttribute((const void *)recomp_bench_kernel,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    recomp_bench_kernel<<<ctx.num_sms, NT, SMEM_BYTES, ctx.stream>>>(U, V, m, n, K, reps, acc);
    LH_CUDA(cudaGetLastError());
    unsigned long long h[8];
    LH_CUDA(cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
    LH_CUDA(cudaStreamSynchronize(ctx.stream));
    for (int p = 0; p < 6; ++p) out[p] = (double)h[p] / ((double)ctx.num_sms * reps);
    out[6] = (double)h[6] / ctx.num_sms;
    out[7] = (double)h[7] / ctx.num_sms;
    LH_CUDA(cudaFree(U));
    LH_CUDA(cudaFree(V));
    LH_CUDA(cudaFree(acc));
}
}  // namespace lh
