/*
 * levyh_b200.h -- C ABI of the B200-native Crank-Nicolson H-matrix hot path.
 *
 * Drop-in boundary for the reference package `levyh` (arxiv 1812.08324,
 * /root/reference/pkg/src/levyh).  Each entry point names the reference
 * function it replaces (file:line).  Plain pointers and sizes only: `*_dev`
 * arguments are CUDA device pointers (fp64 unless noted), `*_host` arguments
 * are host pointers.  Every call is ordered on the context's CUDA stream.
 *
 * Status codes map onto the reference's exception types:
 *   LH_EINVAL    -> ValueError            (hops.py:68-69, hmatrix.py:315-318, ...)
 *   LH_ESINGULAR -> numpy.linalg.LinAlgError, message carries the block path
 *                   ("zero pivot in dense diagonal leaf at root.11.22", hops.py:395-396)
 *   LH_ETYPE     -> TypeError             (hops.py:62, :401)
 * The message of the last failure is returned by lh_ctx_last_error().
 */
#ifndef LEVYH_B200_H
#define LEVYH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    LH_OK = 0,
    LH_EINVAL = 1,
    LH_ESINGULAR = 2,
    LH_ETYPE = 3,
    LH_ECUDA = 4,
    LH_ENOMEM = 5,
    LH_ERANK = 6,     /* rank capacity / ACA max-rank exceeded */
    LH_EINTERNAL = 7
};

typedef struct lh_ctx lh_ctx;
typedef struct lh_tree lh_tree;
typedef struct lh_hmat lh_hmat;

/* ---- context --------------------------------------------------------- */
int lh_ctx_create(int device, void *cuda_stream, lh_ctx **out);
void lh_ctx_destroy(lh_ctx *ctx);
const char *lh_ctx_last_error(const lh_ctx *ctx);
int lh_ctx_synchronize(lh_ctx *ctx);
/* the cudaStream_t every call of this context is ordered on (for caller-side events) */
void *lh_ctx_stream(const lh_ctx *ctx);
int lh_version(void);

/* ---- cluster tree: geometry.py:191-243 build_cluster_tree (bisection) -- */
int lh_tree_build(lh_ctx *ctx, const double *pts_host, int64_t n, int dim, int leaf_size,
                  lh_tree **out);
/* the same with the split rule of build_cluster_tree(strategy=...): 0 "bisection", 1 "kmeans2"
 * (geometry.py:157-188, deterministic 2-means; the 2D L-shape studies) */
int lh_tree_build_strategy(lh_ctx *ctx, const double *pts_host, int64_t n, int dim, int leaf_size,
                           int strategy, lh_tree **out);
void lh_tree_destroy(lh_tree *t);
int64_t lh_tree_num_nodes(const lh_tree *t);
/* lohi[2*i], lohi[2*i+1] = start, end; bbox[(2*i)*dim ...] lo then hi; kids[2*i..] (-1 = leaf) */
int lh_tree_nodes(const lh_tree *t, int64_t *lohi_host, double *bbox_host, int32_t *kids_host);
/* order[i_tree] = i_orig  (Permutation.inverse, geometry.py:239) */
int lh_tree_order(const lh_tree *t, int64_t *order_host);

/* Block partition only (host, no GPU): the decision order of hmatrix.py:319-337 with every
 * admissible block of min(m,n) > n_min reported as low-rank (kind 1, rank -1).  Call with
 * recs_host = NULL to get the counts; recs_host[5*b..] = row0,row1,col0,col1,kind. */
int lh_partition(const lh_tree *rt, const lh_tree *ct, int n_min, int n_block, double eta,
                 int64_t *recs_host, int64_t *nblocks, int64_t *nhier);

/* Host-only planning statistics of the H-LU / solve task DAGs for the partition of
 * (rt, ct) (no GPU): stats[0..7] = lu tasks, lu deps, lu temp doubles, lu plan seconds,
 * solve tasks, solve deps, solve critical-path tasks, lu critical-path tasks. */
int lh_plan_stats(const lh_tree *rt, const lh_tree *ct, int n_min, int n_block, double eta,
                  int kcap, double *stats_host);


/* ---- H-matrix construction: hmatrix.py:121-137 HConfig, :306-340 build_from_dense */
typedef struct {
    int32_t n_min;        /* HConfig.n_min                                   */
    int32_t n_block;      /* HConfig.n_block                                 */
    double eta;           /* HConfig.eta                                     */
    double eps1;          /* HConfig.eps1: keep sigma_k > eps1*sigma_1        */
    int32_t kcap;         /* low-rank column capacity (>= rank; slack for H-LU) */
    int32_t max_aca_rank; /* ACA iteration cap before recompression          */
    double aca_tol;       /* ACA stop: |u_k||v_k| <= aca_tol*|S_k|_F          */
} lh_hconfig;

/* Partition + ACA/QR/SVD compression of a Toeplitz operator A[i,j] = t[j - i + nrows - 1]
 * (t has nrows + ncols - 1 entries, device).  Matrix-free analogue of
 * build_from_dense(toeplitz(t), rt, ct, cfg) (hmatrix.py:306-340). */
int lh_hmat_build_toeplitz(lh_ctx *ctx, const lh_tree *rt, const lh_tree *ct, const double *t_dev,
                           const lh_hconfig *cfg, lh_hmat **out);
/* Sharded assembly: rank `rank` of `world` compresses its share of the
 * admissible blocks (longest-processing-time assignment by m + n, identical on every
 * rank).  The result is pending until every other rank's share has been unpacked:
 *   lh_hmat_shard_pack(buf = NULL) -> length; pack -> device buffer (doubles);
 *   exchange the buffers (e.g. NCCL all-gather); lh_hmat_shard_unpack for every source
 *   rank; lh_hmat_shard_finalize (dense conversions + local dense fill).
 * The finalized matrix equals the unsharded lh_hmat_build_toeplitz result bit for bit.
 * t_dev must stay valid until finalize. */
int lh_hmat_build_toeplitz_shard(lh_ctx *ctx, const lh_tree *rt, const lh_tree *ct,
                                 const double *t_dev, const lh_hconfig *cfg, int32_t rank,
                                 int32_t world, lh_hmat **out);
int lh_hmat_shard_pack(lh_ctx *ctx, lh_hmat *h, double *buf_dev, int64_t cap, int64_t *len);
int lh_hmat_shard_unpack(lh_ctx *ctx, lh_hmat *h, int32_t src_rank, const double *buf_dev,
                         int64_t len);
int lh_hmat_shard_finalize(lh_ctx *ctx, lh_hmat *h);
/* NCCL inside the library.  The context owns one communicator:
 * rank 0 calls lh_nccl_unique_id, the caller distributes the 128 bytes (any side channel, e.g.
 * torch.distributed.broadcast_object_list), every rank calls lh_nccl_init.  libnccl.so.2 is
 * opened at run time (the copy already loaded by the process first).  lh_nccl_ready: 1 once
 * initialised. */
int lh_nccl_unique_id(void *uid128_host);
int lh_nccl_init(lh_ctx *ctx, int32_t rank, int32_t world, const void *uid128_host);
int lh_nccl_ready(lh_ctx *ctx);
/* Sharded assembly over the context's communicator: the same result as lh_hmat_build_toeplitz
 * (bit for bit) with the ACA of the admissible blocks split across the ranks (longest-processing-
 * time assignment by m + n) and every rank's share cut into `stages` parts: stage s's factors
 * are all-gathered on a communication stream while stage s + 1 compresses.  stats_host (may be
 * NULL): compress seconds, host wait for the exchange, finalize seconds, bytes sent, received. */
int lh_hmat_build_toeplitz_nccl(lh_ctx *ctx, const lh_tree *rt, const lh_tree *ct, const double *t_dev,
                                const lh_hconfig *cfg, int32_t stages, double *stats_host, lh_hmat **out);
/* Broadcast of an H-matrix's device data (arena, ranks, leaf permutations and inverses) from
 * `root`; every rank holds the same structure and layout (e.g. an H-LU factor computed once and
 * shared by ranks that step disjoint right-hand-side columns). */
int lh_bcast_factors(lh_ctx *ctx, lh_hmat *h, int32_t root);
/* build_from_dense(A, rt, ct, cfg) with A on the device (tree order), element (i,j) at
 * A[i*lda + j] (row_major=1, numpy C order) or A[i + j*lda] (row_major=0). */
int lh_hmat_build_dense(lh_ctx *ctx, const lh_tree *rt, const lh_tree *ct, const double *A_dev,
                        int64_t lda, int row_major, const lh_hconfig *cfg, lh_hmat **out);
/* Same partition and ranks as `src`; low-rank blocks (lr_scale*U, V); dense blocks refilled
 * from the Toeplitz symbol t_dev.  Used for A- from A+ (hard part 4). kcap<=0: tight. */
int lh_hmat_derive_toeplitz(lh_ctx *ctx, const lh_hmat *src, const double *t_dev, double lr_scale,
                            int32_t kcap, lh_hmat **out);
int lh_hmat_clone(lh_ctx *ctx, const lh_hmat *src, int32_t kcap, lh_hmat **out);
void lh_hmat_destroy(lh_hmat *h);
/* Memory management (no reference counterpart: levyh keeps every operator in host RAM).
 * lh_hmat_spill moves an unfactored H-matrix's arena to host memory and frees its device
 * copy and matvec plan; every call that reads the arena (matvec, entry, exports, derive, hlu,
 * trisolve, save, steps that read A-) brings it back first.  Used for A- of the CN pair when
 * the step is u <- 2 Z u - u and never reads A- (levy.FracCNSystem.prepare(spill_minus=True),
 * cfg5 at N = 2^22).  lh_hmat_resident: 1 on the device, 0 spilled. */
int lh_hmat_spill(lh_ctx *ctx, lh_hmat *h);
int lh_hmat_resident(const lh_hmat *h);

/* ---- introspection: hmatrix.py:343-433 -------------------------------- */
int64_t lh_hmat_num_blocks(const lh_hmat *h);
/* recs[6*b ..] = row0,row1,col0,col1,kind(0 dense,1 lowrank,2 dense_lu),rank  (walk order) */
int lh_hmat_structure(lh_ctx *ctx, const lh_hmat *h, int64_t *recs_host);
/* stats[0..3] = dense_blocks, lowrank_blocks, stored_scalars, hier_nodes  (memory_report) */
int lh_hmat_memory(lh_ctx *ctx, const lh_hmat *h, int64_t *stats_host);
/* dense/dense_lu: a = m*n col-major (+ perm int64[m] into b for dense_lu as doubles);
 * lowrank: a = U (m*rank col-major), b = V (n*rank col-major). */
int lh_hmat_export_block(lh_ctx *ctx, const lh_hmat *h, int64_t block, double *a_host,
                         double *b_host);
/* hmatrix.py:416-433 h_entry: entry (i, j) in tree order, found by descending the block tree
 * on the host and reading only the containing leaf on the device (one value of a dense leaf,
 * one row of U and of V of a low-rank leaf).  LH_EINVAL outside the matrix, LH_ETYPE in an
 * LU-factored leaf. */
int lh_hmat_entry(lh_ctx *ctx, const lh_hmat *h, int64_t i, int64_t j, double *out_host);

/* Bulk export (host copies) for checkpointing and for timing the reference CPU path on
 * GPU-built factors.  sizes[0..2] = arena length (doubles), rank slots, permutation length.
 * recs[11*b ..] per leaf block (walk order): row0,row1,col0,col1,kind(1 dense,2 lowrank,
 * 3 dense_lu),dense_off,u_off,v_off,kcap,rank_slot,perm_off. */
int lh_hmat_layout(const lh_hmat *h, int64_t *recs_host, int64_t *sizes_host);
int lh_hmat_export_arena(lh_ctx *ctx, const lh_hmat *h, double *arena_host, int32_t *ranks_host,
                         int32_t *perm_host);

/* Checkpoints: one self-contained file with both cluster trees (and
 * their points), the block tree, the storage layout and the device arrays (arena, ranks,
 * leaf pivots, leaf inverses) of an H-matrix or an H-LU factor; eps2 is stored as metadata.
 * A loaded matrix is bit-identical to the saved one.  LH_EINVAL on a foreign, truncated or
 * corrupt file.  lh_hmat_load returns new tree handles (destroy with lh_tree_destroy). */
int lh_hmat_save(lh_ctx *ctx, const lh_hmat *h, double eps2, const char *path);
int lh_hmat_load(lh_ctx *ctx, const char *path, lh_tree **row_tree, lh_tree **col_tree,
                 lh_hmat **out, int32_t *factored, double *eps2);
/* The tree's input points (original order, n x dim row-major; NULL = query); returns dim. */
int lh_tree_points(const lh_tree *t, double *pts_host);

/* ---- H-arithmetic ------------------------------------------------------ */
/* hops.py:65-70 matvec / :73-85 mul_dense:  Y = H X, X is ncols x nrhs (col-major, ldx) */
int lh_hmat_matvec(lh_ctx *ctx, const lh_hmat *h, const double *x_dev, int64_t ldx, double *y_dev,
                   int64_t ldy, int32_t nrhs);
/* hops.py:411-421 hlu: in-place recursive H-LU with eps2 recompression.
 * On LH_ESINGULAR the message names the block path. */
int lh_hlu(lh_ctx *ctx, lh_hmat *h, double eps2);
/* hops.py:424-432 solve: forward (unit L, leaf pivots) + backward (U) substitution,
 * in place on B (n x nrhs, col-major, ldb). method 0 = substitution DAG, 1 = inverse factors,
 * 2 = propagator (one H-matvec of Z = (LU)^-1). */
int lh_solve(lh_ctx *ctx, lh_hmat *factor, double *b_dev, int64_t ldb, int32_t nrhs,
             int32_t method);
/* hops.py:282-310 trisolve_lower / trisolve_upper_right with a dense right-hand side:
 * T X = B in place on B (n x nrhs, col-major, ldb == n) using one triangle of T:
 * mode 0 lower (unit_diagonal = unit), 1 upper, 2 upper transposed (X U = B^T is solved as
 * U^T X^T = B^T by the caller).  LU-factored leaves use their LU (unit L with pivots);
 * a plain dense leaf with a zero diagonal entry fails with LH_ESINGULAR and the message
 * "singular triangular diagonal block at L.11..." (hops.py:179-182). */
int lh_trisolve_dense(lh_ctx *ctx, lh_hmat *t, int32_t mode, int32_t unit, double *b_dev,
                      int64_t ldb, int32_t nrhs);
/* hops.py:282-310 trisolve_lower / trisolve_upper_right with an H-matrix right-hand side B
 * (same cluster trees as T): *out = a new H-matrix X, a deep copy of B (low-rank capacity 32;
 * B is not modified) solved in place by the block recursion: mode 0 L X = B (unit_diagonal =
 * unit, _trisolve_block "L"), mode 2 X U = B (_trisolve_right_upper; unit must be 0).
 * Low-rank targets are recompressed at a Frobenius tail of eps2 relative (the reference passes
 * 0 and keeps rounding-noise singular values; 1e-14 keeps the ranks bounded).
 * A rank beyond the capacity fails with LH_ERANK. */
int lh_trisolve_block(lh_ctx *ctx, lh_hmat *t, const lh_hmat *b, int32_t mode, int32_t unit, double eps2,
                      lh_hmat **out);
/* hops.py:147-156 lowrank_add_recompress: (u_out, v_out) = recompressed u1 v1^T + u2 v2^T,
 * smallest rank r with ||tail||_F <= eps2 ||sum||_F (QR, QR, SVD).  Device, column-major,
 * ld = m (u) / n (v); outputs hold r1 + r2 <= 48 columns; *r_out = r. */
int lh_lowrank_add_recompress(lh_ctx *ctx, int64_t m, int64_t n, const double *u1, const double *v1,
                              int32_t r1, const double *u2, const double *v2, int32_t r2,
                              double eps2, double *u_out, double *v_out, int32_t *r_out);
/* Precompute the triangular-inverse factors used by method 1. */
int lh_prepare_inverse(lh_ctx *ctx, lh_hmat *factor, double eps2);
/* Precompute the propagator Z = (LU)^-1 as an H-matrix on the factor's block tree
 * (L- then U-solve of the identity, eps2 recompression), used by method 2. */
int lh_prepare_propagator(lh_ctx *ctx, lh_hmat *factor, double eps2);
/* out[0..9] = propagator task count, planning seconds, temp bytes, executor seconds,
 * off-diagonal dense leaves of Z stored low-rank after near-field compression, 2 x 2
 * low-rank sibling groups of Z merged by coarsening, the single-RHS form of Z (0 H-matrix,
 * 1 shared leaf bases, 2 nested H2 bases), the relative error of that form against the
 * H-matrix on a seeded probe vector, the mean leaf basis size, and the scalars of bases,
 * transfers and couplings outside the dense leaves and row bases; out[10] flops per right-hand
 * side of the multi-RHS product with Z and out[11] its form (2: the nested-basis walk as batched
 * DMMA products, 1: the DMMA matmat of the H-form) */
int lh_propagator_stats(lh_hmat *factor, double *out_host);
/* Kernel launches per CN step: kernel nodes of the step graph lh_cn_steps last captured
 * (methods 1 and 2), 0 before the first call. */
int32_t lh_step_graph_kernels(lh_hmat *factor);
/* Path the last lh_cn_steps / lh_cn_step_host call on this factor took: out[0] = step shape
 * (0 substitution, 1 triangular inverses, 2 u <- 2 Z u - u on the CN pair, 3 u <- Z (A- u)),
 * out[1] = 1 when the K right-hand sides ran as DMMA matmats (multi-RHS), out[2] = 1 when the
 * host step ran pipelined, out[3] = kernel nodes of the single-RHS step graph. */
int lh_cn_last_path(lh_hmat *factor, int32_t *out_host);
/* levy.py:309-330 run_cn loop: U <- solve(F, Hm U), nsteps times, in place.
 * method 2 with Hm = 2I - A+ (the CN pair: Hm derived from this factor's A+ by
 * lh_hmat_derive_toeplitz with lr_scale -1, every entry verified there) runs
 * U <- 2 Z U - U, one H-matvec per step; any other Hm runs U <- Z (Hm U).
 * nrhs >= 8 columns run as FP64 tensor-core (DMMA) matmats. */
int lh_cn_steps(lh_ctx *ctx, const lh_hmat *hminus, lh_hmat *factor, double *u_dev, int64_t ldu,
                int32_t nrhs, int32_t nsteps, int32_t method);

/* levy.py:295-306 step_cn on HOST vectors: u_out = one CN step of u_in (u_out may equal
 * u_in; both length n).  With pinned buffers and method 2 on the CN pair, u arrives and the
 * new u leaves in pieces overlapped with the step's kernels (one cached graph per buffer
 * pair); otherwise copy in, step, copy out.  Returns when u_out is written. */
int lh_cn_step_host(lh_ctx *ctx, const lh_hmat *hminus, lh_hmat *factor, const double *u_in_host,
                    double *u_out_host, int32_t method);

/* Measurement: CUDA-event timing of each kernel of one CN step, averaged over `iters`
 * steps applied to u_dev in place.  method 1: out[0..5] mean ms of vtx(H-), seg(H-),
 * vtx(L^-1), seg(L^-1), vtx(U^-1), seg(U^-1); out[6..11] their algorithmic bytes;
 * out[12..14] stored scalars of H-, L^-1, U^-1.  method 2: out[0..1], out[6..7] for
 * phase 1 of Z (V^T x, or the H2 walk when lh_propagator_stats reports form 2) and the
 * segment kernel (others 0); when Z runs the two-kernel H2 step, out[11] = 1 and out[1..2] /
 * out[7..8] are K1 (column walk + dense diagonal leaves) and K2 (couplings, row walk, row bases,
 * the new u written into the staging copy); out[0] = out[6] = 0 (the staging copy of u is made
 * once per lh_cn_steps call).  out[12] H-, out[13] Z in the form the step streams.  out[15]
 * stored scalars of the factor. */
int lh_step_profile(lh_ctx *ctx, const lh_hmat *hminus, lh_hmat *factor, double *u_dev,
                    int32_t iters, int32_t method, double *out_host);
/* out[0..6] = H-LU task count, planning seconds, temp bytes, executor seconds, number of
 * plan chunks executed (> 1 when the LU ran while its plan was still being built), and the
 * factorisation's algorithmic FP64 flops and operand bytes (task list evaluated at the factor's
 * final ranks; temporaries at the mean stored rank) */
int lh_hlu_stats(const lh_hmat *factor, double *out_host);

/* 2D Gaussian CN operator on an nx x (N / nx) tensor grid (levy.assemble_cn_2d, levy.py:275-292;
 * entries levy.py:178-206 _entries_a_2d): which 0 = A, 1 = A+, 2 = A-; row i / column j is grid
 * point order_host[i] / order_host[j] (a cluster tree's permutation), out_dev row-major N x N.
 * lam = the reference's window sum (host scalar).  The H-form is then build_from_dense
 * (lh_hmat_build_dense) of this matrix. */
int lh_cn2d_dense(lh_ctx *ctx, int64_t N, int32_t nx, double h, double eps_sq, double scale, double a,
                  double b, double c, double lam, double dt, int32_t which, const int64_t *order_host,
                  double *out_dev);

/* ---- Krylov consumers: levyh.solvers (solvers.py:39-153) ---------------- */
/* Operator for the Krylov solvers, y = op(x) on device vectors of length n, ordered on the
 * context's stream.  solvers.py:39-43 _as_operator accepts a callable or a dense matrix;
 * here: an H-matvec (hops.matvec), an H-LU solve (hops.solve with lh_solve's method), a
 * dense row-major matrix, or a host callback (returns an lh status code). */
typedef int (*lh_apply_fn)(void *user, const double *x_dev, double *y_dev);
enum { LH_OP_IDENTITY = 0, LH_OP_HMATVEC = 1, LH_OP_HSOLVE = 2, LH_OP_DENSE = 3, LH_OP_CALLBACK = 4 };
typedef struct {
    int32_t kind;         /* LH_OP_*                                           */
    lh_hmat *hmat;        /* HMATVEC: H; HSOLVE: the factored H-matrix (hlu)   */
    int32_t method;       /* HSOLVE: 0 substitution, 1 inverse, 2 propagator   */
    const double *a_dev;  /* DENSE: n x n row-major, leading dimension lda     */
    int64_t lda;
    lh_apply_fn fn;       /* CALLBACK                                          */
    void *user;
} lh_operator;

/* solvers.py:46-88 pcg: preconditioned conjugate gradient from x = 0; Minv NULL or
 * LH_OP_IDENTITY = no preconditioner.  residuals_host[k] = ||r_k|| / ||b|| for every
 * iteration (capacity max_iter); *iters, *converged as IterationLog.  p'Ap <= 0 fails with
 * LH_ESINGULAR "PCG breakdown: operator is not positive definite" (solvers.py:71-72). */
int lh_pcg(lh_ctx *ctx, const lh_operator *A, const lh_operator *Minv, const double *b_dev,
           int64_t n, double tol, int32_t max_iter, double *x_dev, double *residuals_host,
           int32_t *iters, int32_t *converged);
/* solvers.py:91-153 gmres_restarted: right-preconditioned restarted GMRES (modified
 * Gram-Schmidt Arnoldi, Givens rotations), restart <= 64; residuals as lh_pcg.
 * Stagnation returns LH_OK with *converged = 0. */
int lh_gmres_restarted(lh_ctx *ctx, const lh_operator *A, const lh_operator *Minv,
                       const double *b_dev, int64_t n, double tol, int32_t restart,
                       int32_t max_iter, double *x_dev, double *residuals_host, int32_t *iters,
                       int32_t *converged);
/* y = A x for a dense row-major m x n device matrix (the dense-operator path of the Krylov
 * solvers, solvers.py:42-43). */
int lh_dense_gemv(lh_ctx *ctx, const double *a_dev, int64_t lda, int64_t m, int64_t n,
                  const double *x_dev, double *y_dev);

/* ---- entry generation: fractional.py:285-405 + levy.py:169-206 -------- */
typedef struct {
    int32_t kind;   /* 0: power c|y|^(-1-2s); 1: CGMY; 2: tabulated nu(j*h), j=-M..M */
    double c, s;    /* power measure */
    double C, G, M, Y; /* CGMY */
    const double *table_dev; /* kind 2 */
} lh_measure;

typedef struct {
    double h;       /* grid spacing                       */
    int64_t N;      /* interior unknowns                   */
    int64_t M;      /* window offsets |j| <= M (L_W/h)     */
    double rho_r;   /* window radius                       */
    double tail;    /* tail mass beyond L_W                */
    double m2;      /* windowed second moment (host quad)  */
    double a, b, c; /* local coefficients (b = b_eff)      */
    double dt;      /* CN time step                        */
} lh_cn_params;

/* Smooth-measure series H-builder: build_from_expansion (hmatrix.py:243-291) with the
 * Gaussian family of gaussian_expansion_1d (hmatrix.py:171-186), as levy.CNSystem.hmatrix
 * calls it (levy.py:224-239).  Partition of hmatrix.py:319-337 (admissible blocks with
 * min(m,n) > n_min are low-rank, no dense fallback); low-rank factors around the row
 * cluster centre with n_terms = fixed_rank, or rank_bound_gaussian(...) + 1 per block when
 * delta > 0 (hmatrix.py:270-290); U carries `scale`.  Dense leaves: A[i,j] =
 * t_dev[n_rows - 1 + j - i] (entry_fn of a Toeplitz CN system) or, with t_dev NULL, the
 * kernel scale * exp(-eps_sq (x_i - y_j)^2).  Points are device arrays in tree order. */
int lh_hmat_build_gauss_series(lh_ctx *ctx, const lh_tree *rt, const lh_tree *ct, const double *t_dev,
                               const double *row_pts_dev, const double *col_pts_dev, double eps_sq,
                               double scale, int fixed_rank, double delta, const lh_hconfig *cfg,
                               lh_hmat **out);
/* The exact entries of a 2D Gaussian CN operator (levy._entries_a_2d / CNSystem.entries,
 * levy.py:178-206) as a dense-leaf source: the arguments of lh_cn2d_dense with the tree order on
 * the device. */
typedef struct {
    int32_t nx, which;            /* grid width; 0 = A, 1 = A+, 2 = A- */
    double h, eps_sq, scale;      /* grid spacing, Gaussian density scale * exp(-eps_sq |y|^2) */
    double a, b, c, lam, dt;
    const int64_t *order_dev;     /* order_dev[i] = grid index (iy nx + ix) of tree position i */
} lh_cn2d_entries;
/* build_from_expansion with gaussian_expansion_2d (hmatrix.py:189-216, :243-291) as
 * levy.CNSystem.hmatrix calls it for dim = 2 (levy.py:224-239): tensor-product factor families,
 * T terms per dimension (fixed_rank, or the Gaussian rank bound + 1 on the row cluster's diameter
 * when delta > 0), block rank T^2, U's first family carries `scale`.  Points: n x 2 row-major
 * device arrays in tree order.  Dense leaves from `entries` (exact operator entries) or, with
 * NULL, from the kernel scale * exp(-eps_sq |x_i - y_j|^2).  LH_ERANK when T^2 exceeds the
 * 32-column stored-rank limit (T > 5): such operators take lh_hmat_build_dense. */
int lh_hmat_build_gauss_series_2d(lh_ctx *ctx, const lh_tree *rt, const lh_tree *ct,
                                  const double *row_pts_dev, const double *col_pts_dev, double eps_sq,
                                  double scale, int fixed_rank, double delta, const lh_hconfig *cfg,
                                  const lh_cn2d_entries *entries, lh_hmat **out);
/* _expansion_terms (hmatrix.py:284-290): fixed_rank, or rank_bound_gaussian(sqrt(eps_sq),
 * diameter, delta) + 1 (hmatrix.py:270-281) when delta > 0; 1 for a zero diameter. */
int lh_gauss_series_terms(double eps_sq, double diameter, int fixed_rank, double delta);
/* Toeplitz symbols of levy.CNSystem for the Gaussian density scale*exp(-eps_sq y^2)
 * (levy.py:72-81, :169-176, :194-206, :249-263): A[i,j] = -nu((j-i)h) h, band -a/h^2 -+ b/2h,
 * diagonal 2a/h^2 - c + lam h with lam = sum_{j=1..n_off} nu(-jh) + nu(jh); A+- = I +- dt/2 A.
 * Lengths 2N-1 (device); lam_host (nullable) receives lam. */
int lh_gauss_cn_symbol(lh_ctx *ctx, int64_t N, double h, double eps_sq, double scale, int64_t n_off,
                       double a, double b, double c, double dt, double *tA_dev, double *tPlus_dev,
                       double *tMinus_dev, double *lam_host);

/* Writes the Toeplitz symbols tA, tPlus, tMinus (2N-1 each, device) of A and
 * A+- = I +- dt/2 A, and sums_host[0..2] = S0, Sg, Sd (GPU reduction). */
int lh_cn_symbol(lh_ctx *ctx, const lh_measure *nu, const lh_cn_params *p, double *tA_dev,
                 double *tPlus_dev, double *tMinus_dev, double *sums_host);

/* ---- matrix-free evaluators and variable-order assembly (fractional.py) ---- */
/* frac_apply_1d (fractional.py:338-361) / eval_i1 (:304-319): out[i], i = 0..2K, on the main grid
 * from the 2(M+K)+1 samples u_dev of the padded grid; conv = np.correlate(u, kern, 'valid') with
 * kern_j = nu(j h) w_j (_window_sums_1d, :285-301), then
 *   i1 = conv - u S0 - d1 Sg - d2 Sd,  out = i1 + far - u tail + d2 m2.
 * part 1 returns i1 alone (eval_i1 at K = 0).  far_dev (2K+1) may be NULL (zero far field).
 * sums_host (nullable) receives S0, Sg, Sd.  tail and m2 are host scalars as in lh_cn_symbol. */
int lh_frac_apply_1d(lh_ctx *ctx, const lh_measure *nu, double h, int64_t M, int64_t K, double rho_r,
                     double tail, double m2, const double *u_dev, const double *far_dev, int32_t part,
                     double *out_dev, double *sums_host);
/* frac_apply_2d (fractional.py:435-477) with the square window of _window_sums_2d (:413-432):
 * u_dev is the padded grid, row-major side x side with side = 2(M+K)+1, out_dev the main grid
 * (2K+1)^2.  The density is the 2D power density c r^(-2-2s) evaluated on the device, or, with
 * table_dev != NULL, nu.density2 tabulated by the caller on the (2M+1)^2 window offsets
 * (row-major, centre ignored).  sums_host (nullable): S0, Sgx, Sgy, Sdxx, Sdyy, Sdxy. */
int lh_frac_apply_2d(lh_ctx *ctx, double c, double s, const double *table_dev, double h, int64_t M,
                     int64_t K, double rho_r, double tail, double m2, const double *u_dev,
                     const double *far_dev, double *out_dev, double *sums_host);
/* assemble_variable_order (fractional.py:539-622): the dense variable-order stiffness matrix on
 * the L-shape, A_dev row-major m x m (device).  cells_host: m x 2 integer cell coordinates of
 * lshape_grid(n) (:504-520); s_host: the order s(x_i) per row, inside (0, 1) (LH_EINVAL
 * otherwise, :553-554).  Per row on the device: c_{2,s_i} (frac_kernel_constant), the kernel on
 * the (2 Mw + 1)^2 offsets, the six window sums, the graded second moment
 * (windowed_second_moment_radial_2d) and tail_mass_square_2d, the nine-point correction.
 * gl16_host / gl64_host: Gauss-Legendre nodes then weights (16 + 16, 64 + 64) as
 * numpy.polynomial.legendre.leggauss returns them.  rowinfo_host (nullable, 8 per row): S0, sgx,
 * sgy, sdxx, sdyy, sdxy, m2, tail. */
int lh_assemble_variable_order(lh_ctx *ctx, int32_t n, int64_t m, const int32_t *cells_host,
                               const double *s_host, double L_W, double rho_r, const double *gl16_host,
                               const double *gl64_host, double *A_dev, double *rowinfo_host);

#ifdef __cplusplus
}
#endif
#endif
