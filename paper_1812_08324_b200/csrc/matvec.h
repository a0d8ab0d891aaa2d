// H-matvec plan (see matvec.cu).
#pragma once

#include <memory>
#include <vector>

#include "core.h"

namespace lh {

struct SegDesc {
    i64 y0;
    int32_t rows;
    int32_t dbeg, dend;
    int32_t lbeg, lend;
};
struct MvDense {  // element (i, j) of the piece = arena[off + i + j * ld], multiplies x[xc0 + j]
    i64 off, ld, xc0;
    int32_t ncols;
};
struct MvLr {  // U rows of the piece at arena[off + i + c * ld]; t_b from chunk partials [cbeg, cend)
    i64 off, ld;
    int32_t slot, cbeg, cend;
};
struct VChunk {  // V rows at arena[voff + i + c * ld], i < len, multiplies x[xc0 + i]
    i64 voff, ld, xc0;
    int32_t len, slot;
    i64 tout;      // >= 0: whole block in this chunk, write t_b at tvec[tout]
    int32_t pidx;  // else: partial row index
    int32_t pad;
};

struct TJob {  // t_b = sum of the partials of chunks [cbeg, cend) of the block in rank slot `slot`
    int32_t slot, cbeg, cend;
};

struct MvPlan {
    int nseg = 0, nch = 0, nch16 = 0, ntj = 0;
    VChunk *chunks16 = nullptr;  // chunks whose block rank exceeded 8 at plan time
    TJob *tjobs = nullptr;
    double *tvec = nullptr;  // KC_MAX per rank slot
    i64 n_dpieces = 0, n_lpieces = 0;
    SegDesc *segs = nullptr;
    MvDense *dp = nullptr;
    MvLr *lp = nullptr;
    VChunk *chunks = nullptr;
    double *part = nullptr;
    ~MvPlan();
};

std::shared_ptr<MvPlan> build_mv_plan(const HMat &H, const std::vector<int32_t> &blocks,
                                      cudaStream_t s);
void mv_run(const MvPlan &P, const HMat &H, const double *x, double *y, double alpha, double beta,
            cudaStream_t s, int num_sms, const double *z = nullptr);
MvPlan &get_mv_plan(HMat &H, cudaStream_t s);
void mv_vtx_launch(const MvPlan &P, const HMat &H, const double *x, int grid, cudaStream_t s);
void mv_seg_launch(const MvPlan &P, const HMat &H, const double *x, double *y, double alpha,
                   double beta, cudaStream_t s, int num_sms, const double *z = nullptr);
void matvec(Ctx &ctx, HMat &H, const double *x, i64 ldx, double *y, i64 ldy, int nrhs);

}  // namespace lh
