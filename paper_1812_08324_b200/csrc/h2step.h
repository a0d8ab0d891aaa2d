// Two-kernel single-RHS step of the nested-basis (H2) propagator (h2step.cu).
//
// Both kernels are persistent (one CTA per SM) and warp-specialised: one producer lane walks
// the CTA's list of work chunks and streams every chunk's operands into a shared-memory ring
// with cp.async.bulk (TMA engine, mbarrier completion), while eight consumer warps compute from
// shared memory.  Every operand of the walk is therefore in flight ahead of use, and each level
// of a cluster-tree walk costs one consumer barrier instead of one dependent global round trip.
//
//   K1 (up): per column subtree: x_hat of the leaves (P_s^T x from the staged bases and x),
//            the subtree's levels (T^T [x_hat_c1; x_hat_c2] from staged transfers), then the
//            top of the tree by last-arrival climbing (one dedicated warp), while the consumer
//            warps go on streaming the CTA's share of the dense diagonal leaves: yd = D x.
//   K2 (down): per row subtree: couplings w = S x_hat of its clusters and of the clusters on
//            its path (x_hat gathered once), the path chain and the levels (y_hat = w +
//            T_parent y_hat_parent from staged transfers), then the rows of its leaves:
//            y = alpha (yd + Q_t y_hat_t) + beta z.
// Reference semantics: hops.matvec (hops.py:50-70) of Z = (A+)^-1 in H2 form.
#pragma once

#include <vector>

#include "core.h"
#include "matvec.h"

namespace lh {

constexpr int H2S_ST = 4;                    // ring stages
constexpr int H2S_SLOTB = 40960 + 1024;      // bytes per ring slot (a 64 x 64 leaf + x slice)
constexpr int H2S_SLOTB2 = 32768;            // largest K2 ring slot when two CTAs share an SM (two stages each)
constexpr int H2S_CONS = 8;                  // consumer warps
constexpr int H2S_MAXP = 24;                 // path length (as H2_MAXP)
constexpr int H2S_XG = 512;                  // gathered x_hat entries per coupling chunk

enum : int32_t { C_LEAF = 0, C_ULVL = 1, C_DENSE = 2, C_CPL = 3, C_PATH = 4, C_DLVL = 5, C_Q = 6 };
enum : int32_t { F_NEWLVL = 1, F_END = 2, F_SEGFIRST = 4, F_SEGLAST = 8, F_BEGIN = 16 };

struct H2SChunk {           // 96 bytes (descriptor arrays are bulk-copied: sizes multiples of 16)
    int32_t type, flags;
    int32_t a, b;           // item range (dense: a = first row, b = rows)
    int32_t e0, e1, e2;     // dense: K, kd, xadj (x slice offset); F_BEGIN: w slots to clear
    int32_t ncopy;
    uint64_t src[4];        // absolute device addresses (16-byte aligned)
    int32_t bytes[4];       // multiples of 16
    int32_t dst[4];         // byte offsets in the slot (16-byte aligned)
};
struct H2SLeaf {  // x_hat = P^T x: P at slot[p] (ld 64, k columns), x rows at slot[xsl ..]
    int32_t p, xsl, rows, k, xs, pad;
    i64 xh;
};
struct H2SUp {  // x_hat = T^T [xs[xs1 ..+k1]; xs[xs2 ..+k2]], T row i at slot[t + i k]
    int32_t t, k, k1, k2, xs, xs1, xs2, pad;
    i64 xh, pad2;
};
struct H2SCplN {  // w[ws ..+kr] = sum_e S_e x_hat_e over couplings [c0, c1); rows ro .. ro+kr of the chunk
    int32_t ws, kr_ro, c0, c1;  // kr_ro = kr | ro << 8
};
struct H2SCplE {  // S (kr x kc, column-major) at slot[s]; x_hat at xh[xh ..+kc], gathered to slot[x0 + xo]
    int32_t s, kc, xo, xh;
};
struct H2SPath {  // chain step: y = w[ws] (+ T[t + roff + i + j ldt] y_prev[j], j < kp); out >= 0: ys slot
    int32_t ws, k, kp, ldt, roff, t, out, pad;
};
struct H2SDn {  // y[ys] = w[ws] + T[t + roff + i + j ldt] y[ysp + j], j < kp
    int32_t ys, ysp, ws, k, kp, ldt, roff, t;
};
struct H2SQ {  // rows of a row leaf: y = alpha (yd + Q y_hat) + beta z
    int32_t q, yd, zs, rows, k, ys;  // slot offsets (doubles) of Q, yd row 0, x/z row 0; ys: y_hat slot
    i64 r0;
};

struct H2S {
    int G = 0;                        // CTAs (one per SM)
    int G2 = 0, st2 = H2S_ST, slot2 = H2S_SLOTB;  // K2: CTAs, ring stages and slot bytes (one CTA per row
                                                  // subtree, two per SM on two-stage rings, when that fits)
    int smem1 = 0, smem2 = 0;         // dynamic shared memory of K1 / K2 (bytes)
    int xsmax = 0, wsmax = 0, ysmax = 0;
    H2SChunk *c1 = nullptr, *c2 = nullptr;
    int32_t *cb1 = nullptr, *cb2 = nullptr;  // chunk ranges per CTA
    // per-CTA ranges of the item arrays (the CTA preloads its descriptors into shared memory)
    int32_t *lb1 = nullptr, *ub1 = nullptr;
    int32_t *nb2 = nullptr, *eb2 = nullptr, *pb2 = nullptr, *db2 = nullptr, *qb2 = nullptr;
    int desc1 = 0, desc2 = 0;  // descriptor bytes per CTA (max)
    int32_t *sb1 = nullptr, *sl1 = nullptr;  // K1: column subtrees per CTA (climber)
    H2SLeaf *leaf = nullptr;
    H2SUp *up = nullptr;
    H2SCplN *cn = nullptr;
    H2SCplE *ce = nullptr;
    H2SPath *path = nullptr;
    H2SDn *dn = nullptr;
    H2SQ *q = nullptr;
    double *xpad = nullptr;  // 16-byte aligned copy of x (TMA source)
    double *yd = nullptr;    // dense-leaf part of y
    double *sb2 = nullptr, *td2 = nullptr;  // K2 operands reordered per row subtree
    i64 n = 0;
    i64 bytes1 = 0, bytes2 = 0;  // bytes streamed through the rings per application
    ~H2S();
};

// host-side description of the built H2 form (zshared.cu: build_h2) the step plan is cut from
struct H2SInput {
    i64 n = 0;
    const std::vector<H2Leaf> *leaves = nullptr;
    std::vector<int32_t> up_leaf_beg;            // column subtree s: leaves [beg[s], beg[s+1])
    const std::vector<H2Up> *ups = nullptr;
    const std::vector<int32_t> *up_lv = nullptr;  // nsub_up x (maxh_up + 1)
    const std::vector<H2Sub> *up_sub = nullptr;
    const std::vector<int32_t> *up_xcnt = nullptr;
    int maxh_up = 0, nsub_up = 0;
    const std::vector<H2Down> *dns = nullptr;
    const std::vector<int32_t> *dn_lv = nullptr;  // nsub_dn x (maxh_dn + 2)
    const std::vector<H2Sub> *dn_sub = nullptr;
    const std::vector<int32_t> *dn_ycnt = nullptr;
    const std::vector<int32_t> *dn_path = nullptr, *dn_pbeg = nullptr;
    const std::vector<H2Cpl> *cpls = nullptr;
    std::vector<std::pair<i64, i64>> dn_rows;  // row range of every row subtree root
    int maxh_dn = 0, nsub_dn = 0;
    struct RLeaf {
        i64 r0, rows, k, qoff, sub, yloc;
    };
    std::vector<RLeaf> rleaf;  // every row leaf in row order; qoff into the ZS arena (k > 0)
    const double *pb = nullptr, *tu = nullptr, *td = nullptr, *sb = nullptr, *zarena = nullptr;
    // the dense diagonal leaves as a segment plan (host copies of its segments and batches)
    std::vector<SegDesc> segs;
    std::vector<SBatch> batches;
    const double *pbuf = nullptr;
};
// cuts the two chunk lists; false (nothing installed) when a piece does not fit a ring slot
bool build_h2s(const H2SInput &in, H2 &h, int num_sms, cudaStream_t st);
// y = alpha Z x + beta z (z = x when z_is_x) with the two kernels, on stream s
void h2s_launch(const H2 &h, const double *x, double *y, double alpha, double beta, const double *z,
                cudaStream_t s);
// the same with events around the three launches (ev[0] xpad ev[1] K1 ev[2] K2 ev[3]); profiling
void h2s_launch_timed(const H2 &h, const double *x, double *y, double alpha, double beta, const double *z,
                      cudaStream_t s, cudaEvent_t *ev);
// CN stepping in place on the staging copy: h2s_load copies x in once, every h2s_step_inplace is
// x <- alpha Z x + beta x with the two kernels only (K2 writes the new x into the staging copy),
// h2s_store copies the state out.  ev (optional): events before K1, between, after K2.
void h2s_load(const H2 &h, const double *x, cudaStream_t s);
void h2s_step_inplace(const H2 &h, double alpha, double beta, cudaStream_t s, cudaEvent_t *ev = nullptr);
void h2s_store(const H2 &h, double *y, cudaStream_t s);
// the same with x arriving from (pinned) host memory straight into the aligned staging copy and
// y leaving to host memory; z = x (beta != 0).  Capturable.
void h2s_launch_host(const H2 &h, const double *x_host, double *y_dev, double *y_host, double alpha, double beta,
                     cudaStream_t s);

}  // namespace lh
