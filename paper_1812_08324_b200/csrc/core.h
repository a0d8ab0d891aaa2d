// Internal structures of the B200 H-matrix engine (host side).
// Public ABI: include/levyh_b200.h.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/levyh_b200.h"

namespace lh {

typedef int64_t i64;

// Error carrying an lh status code; converted to a return code at the C-ABI.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define LH_CUDA(call)                                                                        \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            throw ::lh::Error(LH_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define LH_REQUIRE(cond, code, msg)                   \
    do {                                              \
        if (!(cond)) throw ::lh::Error((code), (msg)); \
    } while (0)

// ---------------------------------------------------------------------------
// cluster tree (geometry.py:66-243)
// ---------------------------------------------------------------------------
struct Cluster {
    i64 lo, hi;          // tree-order range [lo, hi)
    double blo[2], bhi[2];
    int32_t kid[2];      // -1: leaf
    int32_t depth;
    i64 size() const { return hi - lo; }
    bool leaf() const { return kid[0] < 0; }
};

struct Tree {
    int dim = 1;
    i64 n = 0;
    int leaf_size = 64;
    std::vector<Cluster> nodes;  // nodes[0] is the root
    std::vector<i64> order;      // order[i_tree] = i_orig
    std::vector<int32_t> leaves; // leaf cluster ids in tree order
    std::vector<double> pts;     // the input points, original order, n x dim row-major
};

Tree *build_tree(const double *pts, i64 n, int dim, int leaf_size, int strategy = 0);  // 1: kmeans2
bool admissible(const Cluster &a, const Cluster &b, int dim, double eta);
double diameter(const Cluster &a, int dim);

// ---------------------------------------------------------------------------
// block tree (hmatrix.py:51-118)
// ---------------------------------------------------------------------------
enum Kind : int32_t { K_HIER = 0, K_DENSE = 1, K_LR = 2, K_FDENSE = 3 };

struct Node {
    int32_t kind;
    int32_t rcl, ccl;     // row / column cluster ids
    i64 r0, c0, m, n;     // absolute tree-order position and shape
    int32_t kid[4];       // HIER: 11, 12, 21, 22
    i64 rs, cs;           // HIER: row_split, col_split
    i64 doff;             // DENSE/FDENSE: arena offset, column-major, ld = m
    i64 uoff, voff;       // LR: U (m x kcap), V (n x kcap), column-major
    int32_t kcap;         // LR: column capacity
    int32_t rslot;        // LR: index into the rank array
    i64 poff;             // FDENSE: offset of the int32 net row permutation
    i64 ioff = -1;        // FDENSE: offset of the packed leaf inverse (L^-1 strict lower, U^-1 upper)
    int32_t depth;        // block-tree depth
    // H-arithmetic refinement of a dense leaf larger than 64 x 64 (plan.cpp: refine_dense_leaves):
    // the leaf keeps its kind for everything else, kid[] then name 2 x 2 virtual children whose
    // storage is a sub-block of the leaf's (doff relative to the virtual parent vpar)
    int32_t vpar = -1;
};

struct Ctx;

uint64_t next_hmat_id();

struct HMat {
    // process-unique identity: caches keyed on it never confuse a freed operator with a new one
    // allocated at the same address
    const uint64_t id = next_hmat_id();
    // CN pair provenance.  derive() gives the unfactored A+ a persistent random tag and copies it
    // into the A- it builds when it verified entry by entry that A- equals 2I - A+ (dense leaves
    // within 8 ulp of 2 on the diagonal, exact negatives elsewhere; low-rank blocks (-U, V)).
    // Both tags survive the in-place H-LU and checkpoints; 0 = none.
    mutable uint64_t pair_tag = 0;
    uint64_t cn_pair_tag = 0;
    const Tree *rt = nullptr, *ct = nullptr;
    std::shared_ptr<const Tree> rt_hold, ct_hold;  // keep trees alive
    i64 nrows = 0, ncols = 0;
    int32_t root = 0;
    std::vector<Node> nodes;
    std::vector<int32_t> leafblocks;  // non-HIER nodes in walk order (11,12,21,22)
    double *d_arena = nullptr;
    i64 arena_len = 0;
    int32_t *d_ranks = nullptr;
    std::vector<int32_t> h_ranks;     // host mirror (valid after sync_ranks)
    int32_t nslots = 0;
    int32_t *d_perm = nullptr;        // FDENSE permutations
    i64 perm_len = 0;
    double *d_inv = nullptr;          // FDENSE packed leaf inverses
    i64 inv_len = 0;
    // host spill (lh_hmat_spill): the arena lives in host memory and d_arena is null until
    // ensure_resident() brings it back; gen counts the moves (caches holding arena pointers key on it)
    double *h_spill = nullptr;
    uint64_t gen = 0;
    bool factored = false;
    bool refined = false;             // dense leaves > 64 split for the H-arithmetic planner
    double lu_stats[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // tasks, plan s, temp bytes, exec s, chunks / NF leaves, merges,
                                                    // [6] algorithmic flops, [7] algorithmic bytes (plan_work)
    // lazily built plans (opaque; see matvec.cu / plan.cpp)
    std::shared_ptr<void> mv_plan;
    std::shared_ptr<void> solve_plan;
    std::shared_ptr<void> inv_plan;
    std::shared_ptr<void> bg_plan;  // background H-LU + inverse planning (lu.cu: PlanJob)
    // set on the planners' structure copies: raised when the matrix is destroyed while its plans
    // are still being built (Planner::emit stops at the next task)
    std::shared_ptr<std::atomic<bool>> plan_cancel;
    std::shared_ptr<void> shard;    // pending sharded assembly (build.cu: ShardState)
    ~HMat();
    void sync_ranks(cudaStream_t s);
};

// Moves H's arena to pinned host memory and frees the device copy and H's matvec plan
// (derived operators that a step never reads: A- of the CN pair under the propagator).
void spill_arena(HMat &H, cudaStream_t s);
// Brings a spilled arena back (no-op when resident); every path that reads H's arena calls it.
void ensure_resident(HMat &H, cudaStream_t s);
struct Ctx;
void bcast_hmat(Ctx &ctx, HMat &H, int root);

// Partition exactly as build_from_dense decides it (hmatrix.py:319-337), with every
// admissible block with min(m,n) > n_min marked K_LR (compression decides later).
void partition(HMat &H, const Tree &rt, const Tree &ct, int n_min, int n_block, double eta);
void walk_leaves(HMat &H);

struct DevBuf {  // grow-only device buffer
    double *p = nullptr;
    i64 cap = 0;
    double *ensure(i64 n);
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf();
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool owns_stream = false;
    std::string last_error;
    int num_sms = 148;
    // reusable device scratch
    void *scratch = nullptr;
    size_t scratch_bytes = 0;
    void *ensure_scratch(size_t bytes);
    DevBuf mm[4];  // multi-RHS: X, Y (row-major), T = V^T X, chunk partials
    std::shared_ptr<void> nccl;  // communicator (nccl.cpp: lh_nccl_init)
    ~Ctx();
};

// NCCL (nccl.cpp): communicator owned by the context
void nccl_unique_id(void *out128);
void nccl_init(Ctx &ctx, int rank, int world, const void *uid128);
bool nccl_ready(Ctx &ctx);
int nccl_rank(Ctx &ctx);
int nccl_world(Ctx &ctx);
cudaStream_t nccl_stream(Ctx &ctx);
void nccl_allgather_f64(Ctx &ctx, const double *send, double *recv, size_t count, cudaStream_t s);
void nccl_allgather_i64(Ctx &ctx, const int64_t *send, int64_t *recv, size_t count, cudaStream_t s);
void nccl_bcast_bytes(Ctx &ctx, void *buf, size_t bytes, int root, cudaStream_t s);

// device memory helpers
template <class T>
T *dalloc(i64 count) {
    void *p = nullptr;
    if (count <= 0) count = 1;
    cudaError_t e = cudaMalloc(&p, sizeof(T) * (size_t)count);
    if (e != cudaSuccess)
        throw Error(LH_ENOMEM, std::string("cudaMalloc(") + std::to_string(sizeof(T) * count) +
                                   " bytes): " + cudaGetErrorString(e));
    return (T *)p;
}
template <class T, class A>
void upload(T *dst, const std::vector<T, A> &src, cudaStream_t s) {
    if (!src.empty())
        LH_CUDA(cudaMemcpyAsync(dst, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice, s));
}
template <class T, class A>
T *dupload(const std::vector<T, A> &src, cudaStream_t s) {
    T *p = dalloc<T>((i64)src.size());
    upload(p, src, s);
    return p;
}

}  // namespace lh
