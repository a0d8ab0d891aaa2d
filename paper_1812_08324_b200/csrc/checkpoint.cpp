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
constexpr uint32_t VERSION = 2;  // 2: CN-pair tags in the header
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

void check_tree(const Tree &T, const std::string &path) {
    const i64 nn = (i64)T.nodes.size();
    auto bad = [&](const char *what) {
        throw Error(LH_EINVAL, std::string("corrupt checkpoint (cluster tree ") + what + "): " + path);
    };
    if (nn < 1) bad("empty");
    for (const Cluster &c : T.nodes) {
        if (!(c.lo >= 0 && c.lo <= c.hi && c.hi <= T.n)) bad("range");
        for (int k = 0; k < 2; ++k)
            if (c.kid[k] < -1 || c.kid[k] >= nn) bad("child");
    }
    for (i64 v : T.order)
        if (v < 0 || v >= T.n) bad("order");
    for (int32_t l : T.leaves)
        if (l < 0 || l >= nn) bad("leaf");
}

// Every offset and index a later kernel dereferences must lie inside the arrays the file
// brought: a truncated or edited file is rejected here instead of faulting on the device.
void check_nodes(const HMat &H, const Tree &rt, const Tree &ct, const std::string &path) {
    const i64 nb = (i64)H.nodes.size();
    auto bad = [&](i64 b, const char *what) {
        throw Error(LH_EINVAL, std::string("corrupt checkpoint (block ") + std::to_string(b) + ": " + what +
                                   "): " + path);
    };
    auto in = [](i64 off, i64 len, i64 cap) { return off >= 0 && len >= 0 && off <= cap && len <= cap - off; };
    for (i64 b = 0; b < nb; ++b) {
        const Node &nd = H.nodes[b];
        if (nd.kind < K_HIER || nd.kind > 4) bad(b, "kind");
        const i64 cmin = nd.vpar >= 0 ? -1 : 0;  // virtual children split inside a leaf cluster: -1
        if (nd.rcl < cmin || nd.rcl >= (i64)rt.nodes.size() || nd.ccl < cmin || nd.ccl >= (i64)ct.nodes.size())
            bad(b, "cluster");
        if (!in(nd.r0, nd.m, H.nrows) || !in(nd.c0, nd.n, H.ncols)) bad(b, "position");
        if (nd.vpar < -1 || nd.vpar >= nb) bad(b, "parent");
        if (nd.kind == K_HIER || nd.vpar >= 0 || (nd.kind == K_DENSE || nd.kind == K_FDENSE))
            for (int k = 0; k < 4; ++k)
                if (nd.kid[k] < -1 || nd.kid[k] >= nb) bad(b, "child");
        if (nd.kind == K_DENSE || nd.kind == K_FDENSE) {
            // virtual children of a refined leaf (vpar >= 0) hold offsets relative to their parent
            i64 off = 0, ld = nd.m;
            int32_t q = (int32_t)b;
            for (int hops = 0; q >= 0 && hops < 64; ++hops) {
                off += H.nodes[q].doff;
                ld = H.nodes[q].m;
                if (H.nodes[q].vpar < 0) break;
                q = H.nodes[q].vpar;
            }
            if (q < 0 || H.nodes[q].vpar >= 0) bad(b, "refinement chain");
            if (nd.m > 0 && nd.n > 0 && !in(off, (nd.n - 1) * ld + nd.m, H.arena_len)) bad(b, "dense storage");
        }
        if (nd.kind == K_FDENSE) {
            if (!in(nd.poff, nd.m, H.perm_len)) bad(b, "pivots");
            if (nd.ioff != -1 && !in(nd.ioff, nd.m * nd.m, H.inv_len)) bad(b, "leaf inverse");
        }
        if (nd.kind == K_LR) {
            if (nd.kcap < 0 || nd.kcap > 64) bad(b, "capacity");
            if (nd.rslot < 0 || nd.rslot >= H.nslots) bad(b, "rank slot");
            if (!in(nd.uoff, nd.m * nd.kcap, H.arena_len) || !in(nd.voff, nd.n * nd.kcap, H.arena_len))
                bad(b, "low-rank storage");
        }
    }
    for (int32_t b : H.leafblocks)
        if (b < 0 || b >= nb || H.nodes[b].kind == K_HIER) bad(b, "leaf list");
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
    F.put<uint64_t>(H.pair_tag);
    F.put<uint64_t>(H.cn_pair_tag);
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
    H.pair_tag = F.get<uint64_t>();
    H.cn_pair_tag = F.get<uint64_t>();
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
    check_tree(*rt, path);
    if (ct != rt) check_tree(*ct, path);
    check_nodes(H, *rt, *ct, path);
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
    for (const Node &nd : H.nodes)
        LH_REQUIRE(nd.kind != K_LR || (H.h_ranks[nd.rslot] >= 0 && H.h_ranks[nd.rslot] <= nd.kcap), LH_EINVAL,
                   std::string("corrupt checkpoint (rank exceeds capacity): ") + path);
    if (H.perm_len > 0) {
        std::vector<int32_t> perm(H.perm_len);
        LH_CUDA(cudaMemcpy(perm.data(), H.d_perm, sizeof(int32_t) * H.perm_len, cudaMemcpyDeviceToHost));
        for (const Node &nd : H.nodes)
            if (nd.kind == K_FDENSE)
                for (i64 i = 0; i < nd.m; ++i)
                    LH_REQUIRE(perm[nd.poff + i] >= 0 && perm[nd.poff + i] < std::max<i64>(nd.m, 128), LH_EINVAL,
                               std::string("corrupt checkpoint (pivot out of range): ") + path);
    }
}

}  // namespace lh
