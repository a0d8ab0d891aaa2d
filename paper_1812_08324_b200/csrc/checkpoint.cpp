// H-matrix / H-LU factor checkpoints (factor export and import for
// checkpointing the H-LU across runs).  One self-contained little-endian file:
//
//   "LHB200H1" | u32 version | u32 flags (1 factored, 2 refined, 4 one tree for rows+cols)
//   i64 nrows, ncols | i32 root, nslots | i64 arena_len, perm_len, inv_len | f64 eps2
//   tree(rows) [tree(cols)]  : i32 dim, leaf_size | i64 n | i64 nnodes | Cluster[] |
//                              i64 order[n] | i64 nleaves | i32 leaves[] | f64 pts[n*dim]
//   i64 nnodes | Node[] | i64 nleafblocks | i32 leafblocks[]
//   f64 arena[arena_len] | i32 ranks[nslots] | i32 perm[perm_len] | f64 inv[inv_len]
//   "LHB200END"
//
// Device arrays stream through a pinned double buffer (64 MB halves) so a 6 GB factor is
// written at disk speed without a host copy of the whole arena.  Loading rebuilds the exact
// HMat (block tree, layout, ranks, pivots, leaf inverses): matvec / solve / stepping on a
// loaded factor are bit-identical to the saved one.
#include <cstring>
#include <type_traits>

#include "core.h"

namespace lh {

static_assert(std::is_trivially_copyable<Cluster>::value, "Cluster must be POD");
static_assert(std::is_trivially_copyable<Node>::value, "Node must be POD");

namespace {

const char MAGIC[8] = {'L', 'H', 'B', '2', '0', '0', 'H', '1'};
const char TAIL[9] = {'L', 'H', 'B', '2', '0', '0', 'E', 'N', 'D'};
constexpr uint32_t VERSION = 1;
constexpr size_t STAGE = 64ull << 20;

struct File {
    FILE *f = nullptr;
    std::string path;
    File(const char *p, const char *mode) : path(p) {
        f = fopen(p, mode);
        LH_REQUIRE(f != nullptr, LH_EINVAL, std::string("cannot open checkpoint ") + p);
    }
    ~File() {
        if (f) fclose(f);
    }
    void put(const void *p, size_t n) {
        if (n && fwrite(p, 1, n, f) != n)
            throw Error(LH_EINVAL, "write failed: " + path);
    }
    void get(void *p, size_t n) {
        if (n && fread(p, 1, n, f) != n)
            throw Error(LH_EINVAL, "truncated or corrupt checkpoint: " + path);
    }
    template <class T>
    void put(const T &v) { put(&v, sizeof(T)); }
    template <class T>
    T get() {
        T v;
        get(&v, sizeof(T));
        return v;
    }
    template <class T>
    void put_vec(const std::vector<T> &v) {
        put<i64>((i64)v.size());
        put(v.data(), sizeof(T) * v.size());
    }
    template <class T>
    void get_vec(std::vector<T> &v, i64 limit) {
        i64 n = get<i64>();
        LH_REQUIRE(n >= 0 && n <= limit, LH_EINVAL, "corrupt checkpoint (array length): " + path);
        v.resize(n);
        get(v.data(), sizeof(T) * n);
    }
};

struct Pinned {
    char *p = nullptr;
    Pinned() { LH_CUDA(cudaMallocHost(&p, 2 * STAGE)); }
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
};

// device -> file, double-buffered: the copy of chunk k+1 overlaps the write of chunk k
void dev_to_file(File &F, const void *d, size_t bytes, cudaStream_t s, Pinned &pin) {
    const char *src = (const char *)d;
    cudaEvent_t ev[2];
    LH_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    LH_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    size_t nchunks = (bytes + STAGE - 1) / STAGE;
    auto issue = [&](size_t k) {
        size_t off = k * STAGE, len = std::min(STAGE, bytes - off);
        LH_CUDA(cudaMemcpyAsync(pin.p + (k & 1) * STAGE, src + off, len, cudaMemcpyDeviceToHost, s));
        LH_CUDA(cudaEventRecord(ev[k & 1], s));
    };
    try {
        if (nchunks) issue(0);
        for (size_t k = 0; k < nchunks; ++k) {
            LH_CUDA(cudaEventSynchronize(ev[k & 1]));
            if (k + 1 < nchunks) issue(k + 1);
            size_t off = k * STAGE, len = std::min(STAGE, bytes - off);
            F.put(pin.p + (k & 1) * STAGE, len);
        }
    } catch (...) {
        cudaStreamSynchronize(s);
        cudaEventDestroy(ev[0]);
        cudaEventDestroy(ev[1]);
        throw;
    }
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
}

// file -> device, double-buffered: the read of chunk k+1 overlaps the upload of chunk k
void file_to_dev(File &F, void *d, size_t bytes, cudaStream_t s, Pinned &pin) {
    char *dst = (char *)d;
    cudaEvent_t ev[2];
    LH_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    LH_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    bool used[2] = {false, false};
    size_t nchunks = (bytes + STAGE - 1) / STAGE;
    try {
        for (size_t k = 0; k < nchunks; ++k) {
            size_t off = k * STAGE, len = std::min(STAGE, bytes - off);
            if (used[k & 1]) LH_CUDA(cudaEventSynchronize(ev[k & 1]));  // buffer free again
            F.get(pin.p + (k & 1) * STAGE, len);
            LH_CUDA(cudaMemcpyAsync(dst + off, pin.p + (k & 1) * STAGE, len, cudaMemcpyHostToDevice, s));
            LH_CUDA(cudaEventRecord(ev[k & 1], s));
            used[k & 1] = true;
        }
        LH_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
        cudaStreamSynchronize(s);
        cudaEventDestroy(ev[0]);
        cudaEventDestroy(ev[1]);
        throw;
    }
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
}

void put_tree(File &F, const Tree &T) {
    F.put<int32_t>(T.dim);
    F.put<int32_t>(T.leaf_size);
    F.put<i64>(T.n);
    F.put_vec(T.nodes);
    F.put(T.order.data(), sizeof(i64) * T.order.size());
    F.put_vec(T.leaves);
    LH_REQUIRE((i64)T.pts.size() == T.n * T.dim, LH_EINTERNAL, "cluster tree without its points");
    F.put(T.pts.data(), sizeof(double) * T.pts.size());
}

std::shared_ptr<Tree> get_tree(File &F) {
    auto T = std::make_shared<Tree>();
    T->dim = F.get<int32_t>();
    T->leaf_size = F.get<int32_t>();
    T->n = F.get<i64>();
    LH_REQUIRE((T->dim == 1 || T->dim == 2) && T->n > 0 && T->n < (1ll << 40), LH_EINVAL,
               "corrupt checkpoint (cluster tree): " + F.path);
    F.get_vec(T->nodes, 4 * T->n);
    T->order.resize(T->n);
    F.get(T->order.data(), sizeof(i64) * T->n);
    F.get_vec(T->leaves, T->n);
    T->pts.resize(T->n * T->dim);
    F.get(T->pts.data(), sizeof(double) * T->pts.size());
    return T;
}

}  // namespace

void save_hmat(Ctx &ctx, HMat &H, double eps2, const char *path) {
    LH_REQUIRE(!H.shard, LH_EINVAL, "sharded assembly not finalized");
    LH_CUDA(cudaStreamSynchronize(ctx.stream));
    File F(path, "wb");
    F.put(MAGIC, 8);
    F.put<uint32_t>(VERSION);
    const bool one_tree = H.rt == H.ct;
    F.put<uint32_t>((H.factored ? 1u : 0u) | (H.refined ? 2u : 0u) | (one_tree ? 4u : 0u));
    F.put<i64>(H.nrows);
    F.put<i64>(H.ncols);
    F.put<int32_t>(H.root);
    F.put<int32_t>(H.nslots);
    F.put<i64>(H.arena_len);
    F.put<i64>(H.perm_len);
    F.put<i64>(H.inv_len);
    F.put<double>(eps2);
    put_tree(F, *H.rt);
    if (!one_tree) put_tree(F, *H.ct);
    F.put_vec(H.nodes);
    F.put_vec(H.leafblocks);
    Pinned pin;
    dev_to_file(F, H.d_arena, sizeof(double) * H.arena_len, ctx.stream, pin);
    if (H.nslots > 0) dev_to_file(F, H.d_ranks, sizeof(int32_t) * H.nslots, ctx.stream, pin);
    if (H.perm_len > 0) dev_to_file(F, H.d_perm, sizeof(int32_t) * H.perm_len, ctx.stream, pin);
    if (H.inv_len > 0) dev_to_file(F, H.d_inv, sizeof(double) * H.inv_len, ctx.stream, pin);
    F.put(TAIL, 9);
    LH_REQUIRE(fflush(F.f) == 0, LH_EINVAL, std::string("write failed: ") + path);
}

void load_hmat(Ctx &ctx, const char *path, HMat &H, std::shared_ptr<Tree> &rt,
               std::shared_ptr<Tree> &ct, double &eps2) {
    File F(path, "rb");
    char magic[8];
    F.get(magic, 8);
    LH_REQUIRE(memcmp(magic, MAGIC, 8) == 0, LH_EINVAL,
               std::string("not a levyh_b200 H-matrix checkpoint: ") + path);
    uint32_t ver = F.get<uint32_t>();
    LH_REQUIRE(ver == VERSION, LH_EINVAL, "unsupported checkpoint version " + std::to_string(ver));
    uint32_t flags = F.get<uint32_t>();
    H.nrows = F.get<i64>();
    H.ncols = F.get<i64>();
    H.root = F.get<int32_t>();
    H.nslots = F.get<int32_t>();
    H.arena_len = F.get<i64>();
    H.perm_len = F.get<i64>();
    H.inv_len = F.get<i64>();
    eps2 = F.get<double>();
    LH_REQUIRE(H.nrows > 0 && H.ncols > 0 && H.nslots >= 0 && H.arena_len >= 0 && H.perm_len >= 0 &&
                   H.inv_len >= 0,
               LH_EINVAL, std::string("corrupt checkpoint header: ") + path);
    rt = get_tree(F);
    ct = (flags & 4u) ? rt : get_tree(F);
    LH_REQUIRE(rt->n == H.nrows && ct->n == H.ncols, LH_EINVAL,
               std::string("corrupt checkpoint (tree sizes): ") + path);
    H.rt = rt.get();
    H.ct = ct.get();
    H.rt_hold = rt;
    H.ct_hold = ct;
    F.get_vec(H.nodes, 64 * (H.nrows + H.ncols) + 64);
    F.get_vec(H.leafblocks, (i64)H.nodes.size());
    LH_REQUIRE(H.root >= 0 && H.root < (int32_t)H.nodes.size(), LH_EINVAL,
               std::string("corrupt checkpoint (root): ") + path);
    H.factored = flags & 1u;
    H.refined = flags & 2u;
    Pinned pin;
    H.d_arena = dalloc<double>(std::max<i64>(H.arena_len, 1));
    file_to_dev(F, H.d_arena, sizeof(double) * H.arena_len, ctx.stream, pin);
    H.d_ranks = dalloc<int32_t>(std::max<int32_t>(H.nslots, 1));
    if (H.nslots > 0) file_to_dev(F, H.d_ranks, sizeof(int32_t) * H.nslots, ctx.stream, pin);
    if (H.perm_len > 0 || H.factored) {
        H.d_perm = dalloc<int32_t>(std::max<i64>(H.perm_len, 1));
        if (H.perm_len > 0) file_to_dev(F, H.d_perm, sizeof(int32_t) * H.perm_len, ctx.stream, pin);
    }
    if (H.inv_len > 0) {
        H.d_inv = dalloc<double>(H.inv_len);
        file_to_dev(F, H.d_inv, sizeof(double) * H.inv_len, ctx.stream, pin);
    }
    char tail[9];
    F.get(tail, 9);
    LH_REQUIRE(memcmp(tail, TAIL, 9) == 0, LH_EINVAL, std::string("corrupt checkpoint (trailer): ") + path);
    H.sync_ranks(ctx.stream);
}

}  // namespace lh
