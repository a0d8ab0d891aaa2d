// Static task DAG for H-arithmetic (H-LU, triangular solves, triangular inverses).
//
// The host replays the reference recursion (hops.py:211-421) symbolically and
// records primitive tasks with their operand views; data dependencies come from
// row-interval tracking of every operand; ranks stay on the device, so the
// schedule is independent of the numerical values and can be cached per
// block structure.  csrc/lu.cu executes the DAG in one persistent kernel.
#pragma once

#include <sys/mman.h>

#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "core.h"

namespace lh {

// Allocator for the planner's large arrays (tens of millions of tasks): 2 MB-aligned blocks
// advised for transparent huge pages (far fewer first-touch faults when several planner
// threads fill them), and default-initialising construct (resize does not zero-fill).
template <class T>
struct HugeAlloc {
    using value_type = T;
    HugeAlloc() = default;
    template <class U>
    HugeAlloc(const HugeAlloc<U> &) {}
    T *allocate(size_t n) {
        const size_t bytes = n * sizeof(T), huge = (size_t)1 << 21;
        if (bytes >= huge) {
            const size_t sz = (bytes + huge - 1) / huge * huge;
            void *p = std::aligned_alloc(huge, sz);
            if (!p) throw std::bad_alloc();
            madvise(p, sz, MADV_HUGEPAGE);
            return static_cast<T *>(p);
        }
        void *p = std::malloc(bytes ? bytes : 1);
        if (!p) throw std::bad_alloc();
        return static_cast<T *>(p);
    }
    void deallocate(T *p, size_t) { std::free(p); }
    template <class U>
    void construct(U *p) {
        ::new (static_cast<void *>(p)) U;
    }
    template <class U, class... Args>
    void construct(U *p, Args &&...args) {
        ::new (static_cast<void *>(p)) U(std::forward<Args>(args)...);
    }
    template <class U>
    bool operator==(const HugeAlloc<U> &) const { return true; }
    template <class U>
    bool operator!=(const HugeAlloc<U> &) const { return false; }
};
template <class T>
using hvec = std::vector<T, HugeAlloc<T>>;

enum Base : int8_t { B_F = 0, B_TMP = 1, B_RHS = 2, B_X = 3, B_INV = 4 };
constexpr int NBASE = 5;
constexpr int LEAF_INV_MAX = 64;  // diagonal leaves up to this size also store packed inverses

struct DView {     // element (i, j) = base[off + (trans ? j + i*ld : i + j*ld)]
    i64 off;
    int32_t rows, cols, ld;
    int32_t wslot;  // >= 0: the number of COLUMNS is ranks[wslot] at run time (cols = capacity)
    int8_t base, trans;
    int16_t pad;
};

enum TaskType : int32_t {
    T_GETRF = 1,   // v0 dense leaf (m x m), aux = perm offset
    T_TRSM = 2,    // v0 triangle (factored leaf), v1 rhs (in place); flags: mode|unit<<4|perm<<5
    T_SEGMUL = 3,  // v0 = Y segment; pieces; alpha; flags&1: overwrite (beta = 0)
    T_VTX = 4,     // v2 = W (r x k) <- v0^T (n x r) v1 (n x k); W rank slot = r
    T_LRADD = 5,   // LR target U = v0, V = v1 ; += alpha * v2 v3^T ; recompress (eps in alpha2)
    T_DGEMM = 6,   // v0 (m x n) = beta*v0 + alpha * v1 * op(v2); flags&1: transB, flags&2: overwrite
    T_DADD = 7,    // v0 += alpha * v1
    T_DENSIFY = 8, // v0 (m x n) <- v1 v2^T (low rank) or copy v1 (dense, v2 unused)
    T_IDENT = 9,   // v0 <- identity (or zero if flags&1)
    T_NOP = 10,    // dependency barrier (temp-buffer reuse)
    T_RAND = 11,   // v0 <- N(0,1) samples, seed aux
    T_ORTH = 12,   // v0 (m x p) <- Q of its CGS2 QR, in place
    T_CHECK = 13,  // fail (path) if any |v0| > 1: a refined leaf's L21 needs cross-half pivoting
};

struct DTask {
    int32_t type, flags, path, aux;
    double alpha, alpha2;
    DView v[4];
    int32_t dep_beg, dep_cnt;
    int32_t pc_beg, pc_end;
    int32_t prio, pad;  // ready-queue bucket (b-level class; higher = more urgent)
};
constexpr int NPRIO = 8;

struct DPiece {     // SEGMUL piece: Y += alpha * mat * (X rows or W)
    int32_t kind;   // 0 dense: mat (seg x n) times X[xrow : xrow+n, :]; 1 low-rank: mat (seg x r) times w
    int32_t pad;
    DView mat;
    DView x;        // dense: X rows slice; low-rank: W (r x k)
};

struct Plan {
    hvec<DTask> tasks;
    hvec<int32_t> deps;
    hvec<DPiece> pieces;
    std::vector<std::string> paths;
    i64 temp_len = 0;
    int32_t nslots_total = 0;  // rank slots: F, X, temps
    int32_t slot_off_x = 0, slot_off_tmp = 0;
    int32_t rhs_slot = -1;       // slot holding the run-time RHS width (solve plans)
    bool own_temp = true;        // false: d_temp is lent by the caller (streamed chunks)
    // propagator column part run on its own: its B_X views address [x_base, x_base + x_len) of
    // the Z layout, which lives in a scratch buffer of x_len doubles while the part runs
    i64 x_base = 0, x_len = -1;
    // device copies
    DTask *d_tasks = nullptr;
    int32_t *d_deps = nullptr;
    DPiece *d_pieces = nullptr;
    int32_t *d_done = nullptr;  // one flag per task + counters
    int32_t *d_succ_beg = nullptr, *d_succ = nullptr;  // successor CSR
    int32_t *d_rem_init = nullptr, *d_rem = nullptr;   // dependency counters
    int32_t *d_queue_init = nullptr, *d_queue = nullptr;  // ready FIFO
    int32_t *d_qoff = nullptr, *d_ctr = nullptr;  // bucket offsets; heads, tails, done count
    std::vector<int32_t> ctr_init;
    double *d_temp = nullptr;
    int32_t *d_ranks = nullptr;
    int32_t *d_err = nullptr;
    double build_seconds = 0.0;
    ~Plan();
    void upload(cudaStream_t s);
};

// Algorithmic FP64 work of a plan: flops and operand bytes (each operand read or written once
// per task) summed over its tasks, with the run-time column counts taken from `ranks` (the
// factor's final ranks, indexed by rank slot) and `rank_other` for slots outside it (temporaries).
void plan_work(const Plan &P, const std::vector<int32_t> &ranks, double rank_other, double &flops, double &bytes);

}  // namespace lh
