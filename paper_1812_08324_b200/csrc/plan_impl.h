// Planner internals (host only).
#pragma once

#include <atomic>
#include <condition_variable>
#include <deque>
#include <initializer_list>
#include <mutex>
#include <map>
#include <memory>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "plan.h"

namespace lh {

typedef uint64_t u64;
constexpr int K_ZERO = 4;   // structurally zero block (triangular-inverse storage)
constexpr int KC = 32;      // rows of a W = F^T X temp (>= any rank)

struct PView {
    DView d;
    u64 obj;
    i64 r0;       // first row of this view inside its object
    bool whole;   // transposed: dependency on the whole object
    int32_t tmp = -1;
    int32_t vnode = -1;            // refined dense leaf: accesses also cover its virtual children
    const HMat *vh = nullptr;
    PView rows_(i64 a, i64 cnt) const;
    PView cols_(i64 a, i64 cnt) const;
    PView T() const;
};

// Per-object row-interval state for dependency tracking: the object's rows are covered by
// contiguous segments, each with its last writer and the readers since that write (up to
// four inline).  Objects are indexed densely (F / X block storage, the right-hand side,
// temporaries).
struct DepTracker {
    struct Seg {
        i64 a, b;
        int32_t writer;
        int32_t nr;
        int32_t rd[4];
        std::vector<int32_t> *more;  // readers beyond four (rare)
    };
    std::vector<std::vector<Seg>> objs;
    void access(int32_t task, u64 obj, i64 a, i64 b, bool write, std::vector<int32_t> &out);
    ~DepTracker();
};

struct Mref {
    HMat *H;
    int base;
    int32_t slot_off;
};

struct LeafRef {
    int32_t b;
    i64 r, c;
};

// A plan handed over in program-order chunks while the planner is still running: each
// chunk only depends on itself and on earlier chunks, which have run by the time it starts.
// Chunks are cut on demand (the consumer sets `want` when it is idle).
struct PlanStream {
    std::mutex mu;
    std::condition_variable cv;
    std::deque<std::shared_ptr<Plan>> chunks;
    bool engaged = false;  // a consumer is taking chunks (set under mu)
    bool done = false;     // planning finished (set under mu)
    std::atomic<bool> want{false};
    size_t min_chunk = 50000;
};

struct Planner {
    HMat &F;
    HMat *X;
    std::shared_ptr<Plan> P;
    DepTracker deps;
    double eps2 = 1e-10;
    i64 nF = 0, nX = 0;
    i64 perm_len = 0;
    i64 inv_len = 0;
    int32_t next_slot = 0;
    int32_t next_temp = 0;
    struct TempRec {
        i64 off;
        int cls;
        int32_t barrier;
        std::vector<int32_t> users;
    };
    struct FreeBlock {
        i64 off;
        std::vector<int32_t> users;
    };
    std::unordered_map<int32_t, TempRec> temps;
    std::map<int, std::deque<FreeBlock>> freelist;

    Planner(HMat &F, HMat *X);
    u64 key(int base, i64 id, int which) const;
    PView dense_view(const Mref &M, int32_t b) const;
    PView u_view(const Mref &M, int32_t b) const;
    PView v_view(const Mref &M, int32_t b) const;
    PView temp(i64 rows, i64 cols, int32_t wslot);
    void release(const PView &v);
    int32_t new_slot();
    int32_t emit(DTask t, std::initializer_list<std::pair<const PView *, bool>> acc,
                 const std::vector<std::pair<PView, bool>> *more = nullptr);
    int32_t add_path(const std::string &s);
    void leaves_of(const Mref &M, int32_t b, i64 r, i64 c, std::vector<LeafRef> &out) const;
    void segments_of(const Tree &T, int32_t cl, std::vector<std::pair<i64, i64>> &out) const;
    void segmul(const PView &Y, const Mref &M, int32_t a, const PView &X, bool trans, double alpha,
                bool overwrite);
    void solve_dense(const Mref &T, int32_t t, const PView &B, int mode, bool unit,
                     const std::string &path);
    void trisolve_left(const Mref &T, int32_t t, const Mref &Bm, int32_t b, int mode, bool unit,
                       const std::string &path);
    void trisolve_right_upper(const Mref &T, int32_t t, const Mref &Bm, int32_t b,
                              const std::string &path);
    void sub_lowrank(const Mref &Cm, int32_t c, const PView &U, const PView &V);
    void sub_dense(const Mref &Cm, int32_t c, const PView &D);
    void lr_sketch_update(const Mref &Cm, int32_t c, const Mref *Am, int32_t a, const Mref *Bm,
                          int32_t b, const PView *D);
    int32_t rand_seed = 1;
    // column filter on the target (B_X) matrix: only its blocks with columns in [flo, fhi)
    // are planned (independent column blocks of a left solve, planned on separate threads)
    bool filt = false;
    i64 flo = 0, fhi = 0;
    int colpart(const Mref &M, int32_t b) const;  // 0 outside, 1 inside, 2 straddles
    PView densify(const Mref &M, int32_t b);
    void schur(const Mref &Cm, int32_t c, const Mref &Am, int32_t a, const Mref &Bm, int32_t b);
    void lu_block(int32_t b, const std::string &path);
    void finalize();
    PlanStream *stream = nullptr;
    size_t cut_task = 0, cut_piece = 0;
    std::vector<int32_t> dbuf;  // emit's dependency scratch
    void cut_chunk();
};
void assign_priorities(Plan &P);

// a node the planner recurses into: a real hierarchical block or a refined dense leaf
inline bool hier(const Node &n) {
    return n.kind == K_HIER || ((n.kind == K_DENSE || n.kind == K_FDENSE) && n.kid[0] >= 0);
}
inline bool dense_leaf(const Node &n) { return n.kind == K_DENSE && n.kid[0] < 0; }
void refine_dense_leaves(HMat &H);
void dense_loc(const HMat &H, int32_t b, i64 &off, i64 &ld);

std::shared_ptr<Plan> plan_hlu(HMat &F, double eps2, i64 &perm_len_out,
                               PlanStream *stream = nullptr);
std::shared_ptr<Plan> plan_solve(HMat &F, i64 n, int nrhs_cap);
std::shared_ptr<Plan> plan_inverse(HMat &F, HMat &X, int mode, double eps2);
std::shared_ptr<Plan> plan_trisolve_dense(HMat &T, i64 n, int nrhs_cap, int mode, bool unit,
                                          const std::string &root);
std::shared_ptr<Plan> plan_trisolve_block(HMat &T, HMat &X, int mode, bool unit, double eps2);
// keep_parts: when the merged DAG's device footprint (plan_device_bytes) would exceed
// LEVYH_PROP_MERGE_GB (default 8 GB), the independent column parts are returned there instead
// of merged (and the result is null): they then run one after another, each uploaded, executed
// and freed (N = 2^22, where the merged DAG does not fit next to the factor and Z)
std::shared_ptr<Plan> plan_propagator(HMat &F, HMat &Z, double eps2, int max_parts = 8,
                                      std::vector<std::shared_ptr<Plan>> *keep_parts = nullptr);
double plan_device_bytes(const Plan &P);
std::shared_ptr<Plan> merge_plans(const std::vector<std::shared_ptr<Plan>> &parts);
void mark_lu_leaves(HMat &F, i64 &perm_len, i64 &inv_len);
int64_t critical_path(const Plan &P);

}  // namespace lh
