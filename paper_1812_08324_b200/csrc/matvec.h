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
void treduce_launch(const TJob *jobs, int n, const double *part, double *out, cudaStream_t s);

struct MvPlan {
    int nseg = 0, nch = 0, nch16 = 0, ntj = 0, nbatch = 0, tma_grid = 0;
    std::shared_ptr<Coupling> cpl;     // set for shared-leaf-basis operators
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

std::shared_ptr<MvPlan> build_mv_plan(HMat &H, const std::vector<int32_t> &blocks,
                                      cudaStream_t s);
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

}  // namespace lh
