// Krylov consumers of the GPU H-matrix engine: preconditioned CG and right-preconditioned
// restarted GMRES (levyh.solvers, /root/reference/pkg/src/levyh/solvers.py:46-153).
//
// Vectors stay on the device for the whole run.  The operator and the (inverse)
// preconditioner are lh_operator descriptors: an H-matvec, an H-LU solve, a dense row-major
// matrix (solvers.py:39-43 _as_operator) or a host callback on device pointers.  Scalars that
// feed the next vector update (CG's alpha and beta, the modified Gram-Schmidt projections)
// stay in a small device array and are read by the kernels directly; the host reads back
// only what the reference's control flow branches on (p'Ap, the residual norm, the
// Hessenberg column for the Givens update) -- one D2H per iteration.
//
// Every reduction is deterministic: a grid of fixed size writes per-CTA partials, and the
// last CTA to finish (atomic ticket) sums them in index order.
#include <cmath>
#include <vector>

#include "core.h"
#include "dev.cuh"

namespace lh {
void matvec(Ctx &ctx, HMat &H, const double *x, i64 ldx, double *y, i64 ldy, int nrhs);
void solve(Ctx &ctx, HMat &F, double *b, i64 ldb, int nrhs, int method);

// lh_operator with the handle resolved (capi.cpp)
struct KOp {
    int kind = LH_OP_IDENTITY;
    HMat *h = nullptr;
    int method = 0;
    const double *a = nullptr;
    i64 lda = 0;
    lh_apply_fn fn = nullptr;
    void *user = nullptr;
};

namespace {

constexpr int KT = 256;     // threads per CTA of the vector kernels
constexpr int KGRID = 296;  // 2 CTAs per SM of the 148: one wave, fixed (determinism)

// device scalar slots
enum { S_RZ0 = 0, S_RZ1, S_PAP, S_RR, S_NSLOTS };
constexpr int S_HCOL = 8;  // GMRES Hessenberg column: [S_HCOL, S_HCOL + restart + 2)

struct RedBuf {
    double *partials;  // KGRID
    unsigned *ticket;  // 1
};

__device__ __forceinline__ double coef(const double *sc, int num, int den, double sign) {
    double a = num >= 0 ? sc[num] : 1.0;
    if (den >= 0) a /= sc[den];
    return sign * a;
}

// Finish a grid reduction: every CTA contributes `v`; the last CTA writes sum to *out.
__device__ __forceinline__ void grid_reduce(double v, RedBuf rb, double *out) {
    __shared__ double red[KT / 32];
    __shared__ bool last;
    double s = dev::block_sum(v, red);
    if (threadIdx.x == 0) {
        rb.partials[blockIdx.x] = s;
        __threadfence();
        unsigned t = atomicAdd(rb.ticket, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double p = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += KT) p += ((volatile double *)rb.partials)[i];
    // fixed-order combine: thread i holds partials i, i + KT, ... ; block_sum is a fixed tree
    double tot = dev::block_sum(p, red);
    if (threadIdx.x == 0) {
        *out = tot;
        *rb.ticket = 0u;
    }
}

// y <- y + c x with c = sign * sc[num] / sc[den] (num/den < 0: 1); then optionally
// out = y . z (z == nullptr: no reduction).  x == nullptr: y <- c y (scale).
__global__ void __launch_bounds__(KT) axpy_dot_kernel(const double *__restrict__ x, double *y,
                                                      i64 n, const double *sc, int num, int den,
                                                      double sign, const double *z, RedBuf rb,
                                                      double *out) {
    const double c = coef(sc, num, den, sign);
    double acc = 0.0;
    for (i64 i = (i64)blockIdx.x * KT + threadIdx.x; i < n; i += (i64)gridDim.x * KT) {
        double v = x ? fma(c, x[i], y[i]) : c * y[i];
        y[i] = v;
        if (z) acc = fma(v, z[i], acc);
    }
    if (z) grid_reduce(acc, rb, out);
}

// w <- a x + b y (a, b host immediates; w may alias x or y); optionally out = w . w
__global__ void __launch_bounds__(KT) axpby_kernel(double a, const double *x, double b,
                                                   const double *y, double *w, i64 n, int norm,
                                                   RedBuf rb, double *out) {
    double acc = 0.0;
    for (i64 i = (i64)blockIdx.x * KT + threadIdx.x; i < n; i += (i64)gridDim.x * KT) {
        double v = a * x[i] + (y ? b * y[i] : 0.0);
        w[i] = v;
        acc = fma(v, v, acc);
    }
    if (norm) grid_reduce(acc, rb, out);
}

// p <- z + (sc[num] / sc[den]) p
__global__ void __launch_bounds__(KT) xpby_kernel(const double *__restrict__ z, double *p, i64 n,
                                                  const double *sc, int num, int den) {
    const double c = coef(sc, num, den, 1.0);
    for (i64 i = (i64)blockIdx.x * KT + threadIdx.x; i < n; i += (i64)gridDim.x * KT)
        p[i] = fma(c, p[i], z[i]);
}

__global__ void __launch_bounds__(KT) dot_kernel(const double *__restrict__ x,
                                                 const double *__restrict__ y, i64 n, RedBuf rb,
                                                 double *out) {
    double acc = 0.0;
    for (i64 i = (i64)blockIdx.x * KT + threadIdx.x; i < n; i += (i64)gridDim.x * KT)
        acc = fma(x[i], y[i], acc);
    grid_reduce(acc, rb, out);
}

// Modified Gram-Schmidt step i of Arnoldi column j (solvers.py:125-127):
//   w <- w - H[i] V_i ;  H[i+1] = w . V_{i+1}  (or w . w after the last basis vector)
// One pass over w: the projection onto V_{i+1} is reduced while w is updated.
__global__ void __launch_bounds__(KT) mgs_kernel(double *w, const double *__restrict__ Vi,
                                                 const double *__restrict__ Vnext, i64 n,
                                                 const double *hi, RedBuf rb, double *hnext) {
    const double c = -*hi;
    double acc = 0.0;
    for (i64 i = (i64)blockIdx.x * KT + threadIdx.x; i < n; i += (i64)gridDim.x * KT) {
        double v = fma(c, Vi[i], w[i]);
        w[i] = v;
        acc = fma(v, Vnext ? Vnext[i] : v, acc);
    }
    grid_reduce(acc, rb, hnext);
}

// out = V[:, :k] y  (V column-major, ld = n; y on the device, k <= 64)
__global__ void __launch_bounds__(KT) gemv_basis_kernel(const double *__restrict__ V, i64 n, int k,
                                                        const double *__restrict__ y, double *out) {
    __shared__ double ys[64];
    if (threadIdx.x < k) ys[threadIdx.x] = y[threadIdx.x];
    __syncthreads();
    for (i64 i = (i64)blockIdx.x * KT + threadIdx.x; i < n; i += (i64)gridDim.x * KT) {
        double s = 0.0;
        for (int j = 0; j < k; ++j) s = fma(V[i + (i64)j * n], ys[j], s);
        out[i] = s;
    }
}

// Dense row-major matvec y = A x (one warp per row, two-wide loads)
__global__ void __launch_bounds__(KT) dense_gemv_kernel(const double *__restrict__ A, i64 lda,
                                                        i64 m, i64 n, const double *__restrict__ x,
                                                        double *__restrict__ y) {
    const int lane = threadIdx.x & 31;
    const i64 warps = (i64)gridDim.x * (KT / 32);
    for (i64 r = (i64)blockIdx.x * (KT / 32) + (threadIdx.x >> 5); r < m; r += warps) {
        const double *a = A + r * lda;
        double s = 0.0;
        for (i64 c = lane; c < n; c += 32) s = fma(a[c], x[c], s);
        s = dev::warp_sum(s);
        if (lane == 0) y[r] = s;
    }
}

// ---------------------------------------------------------------------------
struct Krylov {
    Ctx &ctx;
    cudaStream_t s;
    i64 n;
    double *sc = nullptr;
    RedBuf rb{};
    std::vector<double *> owned;

    Krylov(Ctx &c, i64 n_, int nslots) : ctx(c), s(c.stream), n(n_) {
        sc = alloc(nslots);
        rb.partials = alloc(KGRID);
        unsigned *t = nullptr;
        LH_CUDA(cudaMalloc(&t, sizeof(unsigned)));
        LH_CUDA(cudaMemsetAsync(t, 0, sizeof(unsigned), s));
        rb.ticket = t;
        LH_CUDA(cudaMemsetAsync(sc, 0, sizeof(double) * nslots, s));
    }
    ~Krylov() {
        cudaStreamSynchronize(s);
        for (double *p : owned) cudaFree(p);
        if (rb.ticket) cudaFree(rb.ticket);
    }
    double *alloc(i64 len) {
        double *p = dalloc<double>(len);
        owned.push_back(p);
        return p;
    }
    int grid() const { return (int)std::min<i64>(KGRID, std::max<i64>(1, (n + KT - 1) / KT)); }
    void launched() { LH_CUDA(cudaGetLastError()); }
    void dot(const double *x, const double *y, int slot) {
        dot_kernel<<<grid(), KT, 0, s>>>(x, y, n, rb, sc + slot);
        launched();
    }
    void axpy(const double *x, double *y, int num, int den, double sign, const double *z = nullptr,
              int slot = 0) {
        axpy_dot_kernel<<<grid(), KT, 0, s>>>(x, y, n, sc, num, den, sign, z, rb, sc + slot);
        launched();
    }
    void axpby(double a, const double *x, double b, const double *y, double *w, int norm_slot = -1) {
        axpby_kernel<<<grid(), KT, 0, s>>>(a, x, b, y, w, n, norm_slot >= 0, rb,
                                           sc + std::max(norm_slot, 0));
        launched();
    }
    void read(int slot, int cnt, double *host) {
        LH_CUDA(cudaMemcpyAsync(host, sc + slot, sizeof(double) * cnt, cudaMemcpyDeviceToHost, s));
        LH_CUDA(cudaStreamSynchronize(s));
    }
    void copy(double *dst, const double *src) {
        LH_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    }

    // y = op(x); x is not modified
    void apply(const KOp &op, const double *x, double *y) {
        switch (op.kind) {
        case LH_OP_IDENTITY: copy(y, x); break;
        case LH_OP_HMATVEC:
            matvec(ctx, *op.h, x, n, y, n, 1);
            break;
        case LH_OP_HSOLVE:
            copy(y, x);
            solve(ctx, *op.h, y, n, 1, op.method);
            break;
        case LH_OP_DENSE: {
            int g = (int)std::min<i64>(4 * 148, std::max<i64>(1, (n + 7) / 8));
            dense_gemv_kernel<<<g, KT, 0, s>>>(op.a, op.lda, n, n, x, y);
            launched();
            break;
        }
        case LH_OP_CALLBACK: {
            int rc = op.fn(op.user, x, y);
            LH_REQUIRE(rc == LH_OK, rc, "operator callback failed");
            break;
        }
        default: throw Error(LH_ETYPE, "unsupported operator kind");
        }
    }
};

void check_op(const KOp &op, i64 n, const char *what) {
    switch (op.kind) {
    case LH_OP_IDENTITY: return;
    case LH_OP_HMATVEC:
    case LH_OP_HSOLVE: {
        LH_REQUIRE(op.h != nullptr, LH_EINVAL, std::string(what) + ": null H-matrix");
        const HMat &H = *op.h;
        LH_REQUIRE(H.nrows == n && H.ncols == n, LH_EINVAL,
                   std::string(what) + ": operator size does not match the right-hand side");
        if (op.kind == LH_OP_HSOLVE)
            LH_REQUIRE(H.factored, LH_EINVAL, std::string(what) + ": solve needs an H-LU factorization");
        return;
    }
    case LH_OP_DENSE:
        LH_REQUIRE(op.a != nullptr && op.lda >= n, LH_EINVAL, std::string(what) + ": bad dense operand");
        return;
    case LH_OP_CALLBACK:
        LH_REQUIRE(op.fn != nullptr, LH_EINVAL, std::string(what) + ": null callback");
        return;
    default: throw Error(LH_ETYPE, std::string(what) + ": unsupported operator kind");
    }
}

}  // namespace

// solvers.py:46-88 pcg
void pcg(Ctx &ctx, const KOp &A, const KOp &M, const double *b, i64 n, double tol,
         int max_iter, double *x, double *res, int *iters, int *conv) {
    check_op(A, n, "pcg operator");
    check_op(M, n, "pcg preconditioner");
    *iters = 0;
    *conv = 0;
    Krylov K(ctx, n, S_NSLOTS);
    cudaStream_t s = ctx.stream;
    LH_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
    if (n == 0) {
        *conv = 1;
        return;
    }
    double *r = K.alloc(n), *z = K.alloc(n), *p = K.alloc(n), *Ap = K.alloc(n);
    K.copy(r, b);
    double hb[2];
    K.dot(b, b, S_RR);
    K.read(S_RR, 1, hb);
    const double normb = std::sqrt(hb[0]);
    if (normb == 0.0) {
        *conv = 1;
        return;
    }
    const bool precond = M.kind != LH_OP_IDENTITY;
    const double *zr = r;  // z = M(r); the identity preconditioner aliases r (solvers.py:56)
    if (precond) {
        K.apply(M, r, z);
        zr = z;
    }
    K.copy(p, zr);
    int rz = S_RZ0;  // ping-pong slot of r'z
    K.dot(r, zr, rz);
    for (int k = 0; k < max_iter; ++k) {
        K.apply(A, p, Ap);
        K.dot(p, Ap, S_PAP);
        K.axpy(p, x, rz, S_PAP, 1.0);                 // x += alpha p
        K.axpy(Ap, r, rz, S_PAP, -1.0, r, S_RR);      // r -= alpha Ap ; |r|^2
        double h[2];
        K.read(S_PAP, 2, h);  // S_PAP, S_RR adjacent
        if (!(h[0] > 0.0))
            throw Error(LH_ESINGULAR, "PCG breakdown: operator is not positive definite");
        const double rel = std::sqrt(h[1]) / normb;
        res[k] = rel;
        *iters = k + 1;
        if (rel <= tol) {
            *conv = 1;
            break;
        }
        if (precond) K.apply(M, r, z);
        const int rzn = rz ^ 1;
        K.dot(r, zr, rzn);
        xpby_kernel<<<K.grid(), KT, 0, s>>>(zr, p, n, K.sc, rzn, rz);  // p = z + (rz_new/rz) p
        K.launched();
        rz = rzn;
    }
    LH_CUDA(cudaStreamSynchronize(s));
}

// solvers.py:91-153 gmres_restarted (right preconditioning, Givens rotations)
void gmres(Ctx &ctx, const KOp &A, const KOp &M, const double *b, i64 n, double tol,
           int restart, int max_iter, double *x, double *res, int *iters, int *conv) {
    check_op(A, n, "gmres operator");
    check_op(M, n, "gmres preconditioner");
    LH_REQUIRE(restart >= 1 && restart <= 64, LH_EINVAL, "restart must be in [1, 64]");
    *iters = 0;
    *conv = 0;
    Krylov K(ctx, n, S_HCOL + restart + 2);
    cudaStream_t s = ctx.stream;
    LH_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
    if (n == 0) {
        *conv = 1;
        return;
    }
    double hb;
    K.dot(b, b, S_RR);
    K.read(S_RR, 1, &hb);
    const double normb = std::sqrt(hb);
    if (normb == 0.0) {
        *conv = 1;
        return;
    }
    const bool precond = M.kind != LH_OP_IDENTITY;
    double *V = K.alloc(n * (restart + 1));
    double *w = K.alloc(n), *t = K.alloc(n), *upd = K.alloc(n), *ydev = K.alloc(64);
    std::vector<double> H((restart + 1) * restart), cs(restart), sn(restart), g(restart + 1),
        col(restart + 2), y(restart);
    auto Hij = [&](int i, int j) -> double & { return H[(size_t)i * restart + j]; };
    int total = 0;
    bool last_ok = false;  // log.residuals[-1] <= tol
    while (total < max_iter && !*conv) {
        // r = b - A x ; beta = |r|
        K.apply(A, x, w);
        K.axpby(1.0, b, -1.0, w, w, S_RR);
        double b2;
        K.read(S_RR, 1, &b2);
        const double beta = std::sqrt(b2);
        if (beta / normb <= tol) {
            *conv = 1;
            break;
        }
        const int m = std::min(restart, max_iter - total);
        std::fill(H.begin(), H.end(), 0.0);
        std::fill(cs.begin(), cs.end(), 0.0);
        std::fill(sn.begin(), sn.end(), 0.0);
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = beta;
        K.axpby(1.0 / beta, w, 0.0, nullptr, V);  // V_0 = r / beta
        int j_done = 0;
        for (int j = 0; j < m; ++j) {
            double *Vj = V + (i64)j * n;
            if (precond) {
                K.apply(M, Vj, t);
                K.apply(A, t, w);
            } else {
                K.apply(A, Vj, w);
            }
            // modified Gram-Schmidt; slots S_HCOL + i hold H[i, j], S_HCOL + j + 1 holds |w|^2
            K.dot(w, V, S_HCOL);
            for (int i = 0; i <= j; ++i) {
                const double *Vnext = i < j ? V + (i64)(i + 1) * n : nullptr;
                mgs_kernel<<<K.grid(), KT, 0, s>>>(w, V + (i64)i * n, Vnext, n, K.sc + S_HCOL + i,
                                                   K.rb, K.sc + S_HCOL + i + 1);
                K.launched();
            }
            K.read(S_HCOL, j + 2, col.data());
            for (int i = 0; i <= j; ++i) Hij(i, j) = col[i];
            Hij(j + 1, j) = std::sqrt(col[j + 1]);
            if (Hij(j + 1, j) > 0)
                K.axpby(1.0 / Hij(j + 1, j), w, 0.0, nullptr, V + (i64)(j + 1) * n);
            for (int i = 0; i < j; ++i) {
                double tmp = cs[i] * Hij(i, j) + sn[i] * Hij(i + 1, j);
                Hij(i + 1, j) = -sn[i] * Hij(i, j) + cs[i] * Hij(i + 1, j);
                Hij(i, j) = tmp;
            }
            const double denom = std::hypot(Hij(j, j), Hij(j + 1, j));
            cs[j] = Hij(j, j) / denom;
            sn[j] = Hij(j + 1, j) / denom;
            Hij(j, j) = denom;
            Hij(j + 1, j) = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            j_done = j + 1;
            total += 1;
            const double rel = std::fabs(g[j + 1]) / normb;
            res[total - 1] = rel;
            *iters = total;
            last_ok = rel <= tol;
            if (last_ok) break;
        }
        // y = H[:j, :j]^{-1} g[:j]: H is upper triangular after the rotations (back substitution)
        for (int i = j_done - 1; i >= 0; --i) {
            double acc = g[i];
            for (int k = i + 1; k < j_done; ++k) acc -= Hij(i, k) * y[k];
            y[i] = acc / Hij(i, i);
        }
        if (j_done) {
            LH_CUDA(cudaMemcpyAsync(ydev, y.data(), sizeof(double) * j_done, cudaMemcpyHostToDevice, s));
            gemv_basis_kernel<<<K.grid(), KT, 0, s>>>(V, n, j_done, ydev, upd);
            K.launched();
            if (precond) {
                K.apply(M, upd, t);
                K.axpby(1.0, x, 1.0, t, x);
            } else {
                K.axpby(1.0, x, 1.0, upd, x);
            }
            LH_CUDA(cudaStreamSynchronize(s));  // ydev is reused by the next cycle
        }
        if (total > 0 && last_ok) *conv = 1;
    }
    LH_CUDA(cudaStreamSynchronize(s));
}

void dense_gemv(Ctx &ctx, const double *A, i64 lda, i64 m, i64 n, const double *x, double *y) {
    int g = (int)std::min<i64>(4 * 148, std::max<i64>(1, (m + 7) / 8));
    dense_gemv_kernel<<<g, KT, 0, ctx.stream>>>(A, lda, m, n, x, y);
    LH_CUDA(cudaGetLastError());
}

}  // namespace lh
