// H-matvec plan (see matvec.cu).
#pragma once

#include <memory>
#include <vector>

#include "core.h"

namespace lh {

// All operand offsets below index the plan's packed buffer (MvPlan::pbuf), which holds the
// operands in the order the kernels stream them: per segment its dense pieces then the U
// rows of its low-rank pieces, as COLUMNS of ld = even(rows) doubles (pad rows zero), then
// every V chunk.  A segment is therefore a sequence of columns, each with one coefficient:
// x[xc0 + j] for column j of a dense piece, t_b[c] for column c of a low-rank piece.
struct SegDesc {
    i64 y0;
    int32_t rows, ld;
    int32_t dbeg, dend;  // dense pieces (MvDense)
    int32_t lbeg, lend;  // low-rank pieces (MvLr)
    int32_t bbeg, bend;  // bulk-copy batches (SBatch)
    i64 poff;            // the segment's column stream: pbuf[poff + i + q * ld], q < ncol
    int32_t ncol, cmoff; // colmap[cmoff + q]: source row of column q's coefficient
};
struct MvDense {  // element (i, j) = pbuf[off + i + j * ld], multiplies x[xc0 + j]
    i64 off, xc0;
    int32_t ncols, pad;
};
struct MvLr {  // U rows at pbuf[off + i + c * ld], c < r; t_b = tvec[blk * KC_MAX + c]
    i64 off;
    int32_t r, blk;
};
struct VChunk {  // V rows at pbuf[voff + i + c * len], i < len, c < r, multiplies x[xc0 + i]
    i64 voff, xc0;
    int32_t len, r;  // r: rank | (first column << 16); a block of rank > 8 is split by columns
                     // into chunks of <= 8 (vc_rank / vc_col0)
    int32_t blk;   // the block's row of tvec (t_b = tvec[blk * KC_MAX + c])
    int32_t pidx;  // < 0: the chunk is the whole block (write t_b); else partial row index
};
__host__ __device__ inline int vc_rank(const VChunk &c) { return c.r & 0xffff; }
__host__ __device__ inline int vc_col0(const VChunk &c) { return c.r >> 16; }
struct VGroup {  // V chunks over the same x rows [xc0, xc0 + len): gchunks [cbeg, cend), m output rows
    i64 xc0;
    int32_t len, cbeg, cend, m;
    int32_t pad;
};
struct TJob {  // t_b = sum of the partials of chunks [cbeg, cend), written to tvec row blk
    int32_t blk, r, cbeg, cend;
};
// TMA segment kernel: a batch is K consecutive columns of one segment (K * ld <= one ring
// slot); the first kd of them belong to a dense piece (coefficients = an x slice), the rest to
// low-rank pieces (coefficients = tcol[tsrc .. tsrc + K - kd), gathered from tvec per step).
struct SBatch {
    i64 src;     // pbuf offset (doubles, even) of the batch's columns
    i64 tsrc;    // tcol offset (even) of the low-rank coefficients
    i64 xsrc;    // x element offset (even) of the x slice (kd > 0)
    int32_t K, kd, xadj, total;  // columns, dense columns, x[xc0] at slice[xadj], bytes in flight
};
struct PackJob {  // pbuf[dst + i + j * ld] = arena[src + i + j * src_ld], i < rows
    i64 src, src_ld, dst;
    int32_t rows, cols;
    int32_t ld, pad;
};

// Shared-leaf-basis coupling (zshared.cu): between phase 1 (x_hat_s = P_s^T x per column
// leaf, computed by the V^T x kernel) and phase 2 (the segments stream Q_t with coefficients
// y_hat_t), t_b = sum_s E_{s,b}^T x_hat_s per block and y_hat_t = sum_b C_{t,b} t_b per row leaf.
struct CplChunk {  // t_b partial: rows [0, nrow) of E data at ebuf[e0 + row * r + c], x_hat via xidx
    i64 e0;
    int32_t nrow, r, out, x0;  // out >= 0: partial row index; < 0: -(1 + block) direct
};
struct CplRow {    // y_hat_t[i] = sum_g cbuf[e0 + i + g * k] * tb[tidx[t0 + g]], g < ncol; -> tvec row blk
    i64 e0;
    int32_t ncol, k, blk, t0;
};
struct Coupling {
    int nchunk = 0, nrow = 0, ntj = 0, nb = 0;
    CplChunk *chunks = nullptr;
    int32_t *xidx = nullptr;  // tvec index of every E row (x_hat_s[l])
    CplRow *rows = nullptr;
    int32_t *tidx = nullptr;  // tb index of every C column (t_b[c])
    TJob *tjobs = nullptr;
    double *ebuf = nullptr, *cbuf = nullptr, *tb = nullptr, *part = nullptr;
    double *xg = nullptr, *tg = nullptr;  // x_hat / t_b gathered in coefficient order
    i64 nx = 0, nt = 0;
    i64 bytes = 0;  // algorithmic bytes of the coupling data per application
    ~Coupling();
};
void coupling_launch(const Coupling &C, const double *tvec_in, double *tvec_out, cudaStream_t s);

// Nested (H2) cluster bases for Z (zshared.cu: build_h2).  Every cluster tau of the column
// tree carries x_hat_tau = Pnest_tau^T x, computed bottom-up (leaf: P_s^T x_s; internal: Tc_tau^T
// [x_hat_c1; x_hat_c2]); every block b = (rho, sigma) is a k_rho x k_sigma coupling S_b; the row
// tree is walked top-down, y_hat_c = sum_{b: rho(b) = c} S_b x_hat_sigma(b) + Tr_p[c rows] y_hat_p,
// and y_hat of a row leaf is the coefficient of its basis Q_t in the segment kernel.
// Both walks are cut at subtrees of height <= split: one CTA per subtree, the column subtrees
// finish the top of the tree by last-arrival climbing, every row subtree walks its own path
// from the top.
struct H2Leaf {  // xh[xoff + j] = sum_i pb[poff + i + 64 j] x[x0 + i], i < rows, j < k
    i64 poff, x0;
    int32_t rows, k, xoff, pad;
};
struct H2Up {  // xh[xoff + j] = sum_i tu[toff + i k + j] [xh[xoff1 ..+k1]; xh[xoff2 ..+k2]]_i
    i64 toff;
    int32_t k, k1, k2, xoff, xoff1, xoff2, parent, pad;  // parent: H2Up index, -1 none
};
struct H2Down {  // y = sum_{e in [c0, c1)} S_e x_hat + td[toff + roff + i + j ldt] y_parent[j], j < kp
    i64 toff;
    int32_t ldt, roff, kp, k, yoff, yoffp, c0, c1, out, pad;  // yoffp < 0: parent = path end
};                     // (yoff: the node's y_hat / w slot; out: tcol offset of a row leaf's coefficients)
struct H2Cpl {  // w[i] += sum_j sb[soff + i + j kr] xh[xoff + j], j < kc
    i64 soff;
    int32_t kr, kc, xoff, pad;
};
struct H2CRec {  // a row cluster's couplings [c0, c1) with the first one inlined; w slot yoff
    i64 soff;
    int32_t kr, kc, xoff, yoff, c0, c1;
};
struct H2Sub {  // a subtree's transfer matrices [tbeg, tbeg + tlen) are staged in shared memory;
                // its x_hat / y_hat entries are [base, base + ...) locally
    i64 tbeg;
    int32_t tlen, base;
};
struct H2QLeaf {  // fused step: y[r0 + i] = alpha (yd[r0 + i] + sum_c Q[qoff + i + c rows] y_hat[c]) + beta z[r0 + i]
    i64 qoff, r0;     // Q_t in the ZS arena (column-major, ld = rows); first row
    int32_t rows, k;  // k = 0: a row leaf without a basis (dense part only)
    int32_t yloc, pad;  // y_hat_t at ys[yloc] of the subtree CTA (k > 0)
};
struct H2S;  // h2step.h: the two-kernel step
// multi-RHS H2 application (h2mm.cu): batched DMMA products, one launch per tree level
struct H2MMJob {  // C[crow .. +m] (=|+=) A (m x kk) B; A(i, j) = abase[aoff + i sa + j sb];
    i64 aoff;     // B rows: [b[r], b[r] + n[r]) concatenated, r < 4
    int32_t m, kk, sa, sb, crow, pad;
    int32_t b[4], n[4];
};
enum : int32_t { H2MM_X = 0, H2MM_XH = 1, H2MM_YH = 2 };               // B source / C target
enum : int32_t { H2MM_PB = 0, H2MM_TU = 1, H2MM_SB = 2, H2MM_TD = 3 };  // A base
struct H2MMLevel {
    int32_t beg, end, src, abase, dst, accum;
};
struct H2MM {
    H2MMJob *jobs = nullptr;
    int njobs = 0;
    std::vector<H2MMLevel> levels;
    i64 nxh = 0, nyrows = 0;  // rows of Xh and of Yh (whose first rows are the ZS plan's T rows)
    const double *pb = nullptr, *tu = nullptr, *td = nullptr, *sb = nullptr;
    double flops_per_rhs = 0.0;  // of the walk (the rows add the ZS plan's 2 x stored scalars)
    DevBuf xh, yh;
    ~H2MM();
};
struct H2MMInput {
    const std::vector<H2Leaf> *leaves = nullptr;
    const std::vector<H2Up> *ups = nullptr;
    std::vector<int> up_height;
    const std::vector<H2Down> *dns = nullptr;
    const std::vector<H2Cpl> *cpls = nullptr;
    std::vector<int> dn_depth;
    std::vector<int32_t> dn_row, dn_prow;  // Yh row of every node / of its parent (-1 none)
    i64 nxh = 0, nyrows = 0;
    const double *pb = nullptr, *tu = nullptr, *td = nullptr, *sb = nullptr;
};
std::shared_ptr<H2MM> build_h2mm(const H2MMInput &in, cudaStream_t st);
struct MvPlan;
// Y = alpha Z X + beta W (row-major, ldk a multiple of 64); zs: the ZS plan (dense + Q_t pieces)
void h2mm_run(H2MM &M, const MvPlan &zs, const double *X, double *Y, i64 ldk, double alpha, double beta,
              const double *W, cudaStream_t s);
struct H2 {
    int nsub_up = 0, nsub_dn = 0, maxh_up = 0, maxh_dn = 0, split = 0;
    std::shared_ptr<H2S> step2;  // two-kernel fused step (default when built)
    std::shared_ptr<H2MM> mm;    // multi-RHS walk (h2mm.cu)
    // fused single-RHS step: the dense diagonal leaves stream on a forked,
    // low-priority stream beside the walk into yd; the row walk applies Q_t y_hat_t itself
    H2QLeaf *qleaf = nullptr;    // per row subtree, [dn_qbeg[s], dn_qbeg[s+1])
    int32_t *dn_qbeg = nullptr;
    const double *zarena = nullptr;  // ZS arena (Q_t)
    double *yd = nullptr;            // dense-leaf part of y
    H2Leaf *leaves = nullptr;
    H2Up *ups = nullptr;
    H2Down *dns = nullptr;
    H2Cpl *cpls = nullptr;
    int32_t *up_lv = nullptr;    // nsub_up x (maxh_up + 1): ups ranges by height
    int32_t *cnt = nullptr;      // arrival counters per H2Up (zero between launches)
    H2Sub *up_sub = nullptr, *dn_sub = nullptr;
    int32_t *dn_path = nullptr;  // path node ids (H2Down) per row subtree, top-down
    int32_t *dn_pbeg = nullptr;  // nsub_dn + 1
    int32_t *dn_lv = nullptr;    // nsub_dn x (maxh_dn + 2): subtree nodes by depth, top-down
    double *pb = nullptr, *tu = nullptr, *td = nullptr, *sb = nullptr;
    double *xh = nullptr;
    double *wg = nullptr;          // couplings w of every row cluster (at its yoff)
    H2CRec *crec = nullptr;        // row clusters with couplings
    int32_t *up_chain = nullptr, *up_cbeg = nullptr;  // climb chain (H2Up ids) per column subtree
    int32_t *up_xcnt = nullptr, *dn_ycnt = nullptr;  // x_hat / y_hat slots per subtree
    int nleaf = 0, ncnode = 0;
    std::vector<i64> leaf_end;  // host: last row + 1 of every column leaf (leaves are in row order)
    int up_tmax = 0, up_xmax = 0, dn_tmax = 0, dn_ymax = 0;  // staged doubles per CTA
    int maxpath = 0;
    i64 bytes = 0;  // algorithmic bytes per application (P, transfers, couplings)
    ~H2();
};
// the walk writes the row-leaf coefficients straight into the segment kernel's tcol and the
// padded copy of x (xpad), so an H2 plan needs no tgather launch
// leaves = false: the column-leaf x_hat are already in place (h2_leaf_launch per x piece)
void h2_launch(const H2 &h, const double *x, double *tcol, double *xpad, i64 nx, cudaStream_t s, bool leaves = true);
// fused step: leaf / up / couple on s, then (after `dense_done`) the row walk finishing
// y = alpha (yd + Q y_hat) + beta z
void h2_launch_fused(const H2 &h, const double *x, double *y, double alpha, double beta, const double *z,
                     cudaStream_t s, cudaEvent_t dense_done);
void h2_leaf_launch(const H2 &h, int l0, int l1, const double *x, cudaStream_t s);
void treduce_launch(const TJob *jobs, int n, const double *part, double *out, cudaStream_t s);

struct MvPlan {
    int nseg = 0, nch = 0, nch16 = 0, ntj = 0, nbatch = 0, tma_grid = 0;
    std::shared_ptr<Coupling> cpl;     // set for shared-leaf-basis operators
    std::shared_ptr<H2> h2;            // set for nested-basis (H2) operators
    // split H2 plan: this plan holds the row-basis pieces; `dense` the dense leaves (lean
    // segment kernel, run on the forked stream beside the walk)
    std::shared_ptr<MvPlan> dense;
    // fused H2 step: the dense diagonal leaves alone (segment kernel in its smallest
    // configuration, written to h2->yd) beside the walk; the walk finishes y
    std::shared_ptr<MvPlan> fdense;
    int lean = 0;                      // segment kernel configuration: 0 full, 1 lean, 2 co-resident
    cudaStream_t fork = nullptr;
    cudaEvent_t fev[2] = {nullptr, nullptr};
    std::vector<int32_t> blk_of_node;  // tvec row of every low-rank node (-1 otherwise)
    double *pbuf = nullptr;  // packed operands
    i64 pbuf_len = 0;
    double *tvec = nullptr;  // t_b per low-rank block, KC_MAX per block
    double *tcol = nullptr;  // batch-ordered low-rank column coefficients (TMA kernel)
    int32_t *tmap = nullptr; // tcol[e] = tvec[tmap[e]] (-1: padding)
    i64 tcol_len = 0;
    double *xpad = nullptr;  // aligned, zero-padded copy of x (TMA kernel)
    i64 nx = 0;
    // multi-RHS (matmat.cu): coefficient row of every segment column, >= 0 a row of X
    // (dense piece), < 0 a row -(1 + blk * KC_MAX + c) of T = V^T X (low-rank piece)
    int32_t *colmap = nullptr;
    i64 ncolmap = 0;
    int nblk = 0, npart = 0;
    SegDesc *segs = nullptr;
    MvDense *dp = nullptr;
    MvLr *lp = nullptr;
    VChunk *chunks = nullptr;
    VChunk *chunks16 = nullptr;  // chunks of blocks with rank > 8
    VGroup *groups = nullptr;    // multi-RHS: chunks grouped by x rows (matmat.cu)
    VChunk *gchunks = nullptr;
    int ngroup = 0;
    TJob *tjobs = nullptr;
    double *part = nullptr;
    SBatch *batches = nullptr;
    int32_t *cta_seg = nullptr;  // TMA kernel: segments [cta_seg[c], cta_seg[c+1]) per CTA
    i64 n_dpieces = 0, n_lpieces = 0;
    // host-buffer pipelining (mv_run_host): x arrives and y leaves in npiece column / row
    // pieces; the V chunks are also stored piece by piece (a chunk belongs to the piece of
    // its last x row), the segments split at ycut with their own byte-balanced CTA ranges
    int npiece = 0;
    std::vector<i64> xcut, ycut;          // npiece + 1 each
    std::vector<int32_t> pch, pch16;      // chunk ranges per piece in chunks_pp / chunks16_pp
    VChunk *chunks_pp = nullptr, *chunks16_pp = nullptr;
    int32_t *cta_seg_pp = nullptr;        // npiece x (tma_grid + 1)
    ~MvPlan();
};

// tma_grid: CTAs of the segment kernel (byte-balanced contiguous segment ranges); 0 = one per SM
std::shared_ptr<MvPlan> build_mv_plan(HMat &H, const std::vector<int32_t> &blocks,
                                      cudaStream_t s, int tma_grid = 0);
void mv_run(const MvPlan &P, const HMat &H, const double *x, double *y, double alpha, double beta,
            cudaStream_t s, int num_sms, const double *z = nullptr);
MvPlan &get_mv_plan(HMat &H, cudaStream_t s);
void mv_vtx_launch(const MvPlan &P, const HMat &H, const double *x, int num_sms, cudaStream_t s);
void mv_seg_launch(const MvPlan &P, const HMat &H, const double *x, double *y, double alpha,
                   double beta, cudaStream_t s, int num_sms, const double *z = nullptr);
void matvec(Ctx &ctx, HMat &H, const double *x, i64 ldx, double *y, i64 ldy, int nrhs);
// y = alpha H x + beta z with x arriving from pinned host memory and y leaving to it, the
// transfers overlapped with the kernels piece by piece (copies on `side`, kernels on `s`;
// ev: >= 2 npiece + 2 events).  z = x_dev (z_is_x) or y_dev.  Capturable.
void mv_run_host(const MvPlan &P, const double *x_host, double *x_dev, double *y_dev,
                 double *y_host, double alpha, double beta, bool z_is_x, cudaStream_t s,
                 cudaStream_t side, cudaEvent_t *ev, int num_sms);

// multi-RHS (matmat.cu); row-major X, Y, Z with ldk = mm_pad(K)
i64 mm_pad(int k);
int mm_min_rhs();
void mm_transpose(const double *src, i64 lds, double *dst, i64 ldd, i64 n, int k, bool to_rowmajor,
                  cudaStream_t s);
void mm_run(const MvPlan &P, const double *X, double *Y, i64 ldk, double alpha, double beta,
            const double *Z, double *T, double *part, cudaStream_t s);
struct MmBufs {  // the context's multi-RHS scratch sized for plan P and K right-hand sides
    double *T, *part;
};
MmBufs mm_bufs(Ctx &ctx, const MvPlan &P, i64 ldk);
// the segment phase of mm_run alone, with T supplied by the caller (T row blk * KC_MAX + c)
void seg_mm_launch(const MvPlan &P, const double *X, const double *T, i64 ldk, double *Y, double alpha,
                   double beta, const double *Z, cudaStream_t s);

}  // namespace lh
