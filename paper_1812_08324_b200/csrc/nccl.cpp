// NCCL inside the C ABI: a communicator owned by the context, created
// from a unique id the caller distributes (lh_nccl_unique_id / lh_nccl_init), and the two
// collectives the hot path needs: the all-gather of the sharded ACA factors (build.cu:
// build_toeplitz_nccl) and a broadcast of an H-matrix's device data (lh_bcast_factors).
// libnccl is opened at run time (the copy the process already loaded, e.g. torch's, first),
// so the library itself does not link against NCCL.
#include <dlfcn.h>

#include <cstring>

#include "core.h"

namespace lh {

namespace {

typedef int (*GetUniqueIdFn)(void *);
struct Uid128 {  // ncclUniqueId, passed by value
    char b[128];
};
typedef int (*CommInitRankFn2)(void **, int, Uid128, int);
typedef int (*CommDestroyFn)(void *);
typedef int (*AllGatherFn)(const void *, void *, size_t, int, void *, cudaStream_t);
typedef int (*BroadcastFn)(const void *, void *, size_t, int, int, void *, cudaStream_t);
typedef const char *(*ErrStrFn)(int);

struct NcclLib {
    void *h = nullptr;
    GetUniqueIdFn get_uid = nullptr;
    CommInitRankFn2 init_rank = nullptr;
    CommDestroyFn destroy = nullptr;
    AllGatherFn allgather = nullptr;
    BroadcastFn bcast = nullptr;
    ErrStrFn errstr = nullptr;
};

NcclLib &nccl_lib() {
    static NcclLib L;
    static bool tried = false;
    if (!tried) {
        tried = true;
        const char *names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char *n : names) {
            L.h = dlopen(n, RTLD_NOW | RTLD_NOLOAD);  // the copy already in the process (torch)
            if (L.h) break;
        }
        for (const char *n : names) {
            if (L.h) break;
            L.h = dlopen(n, RTLD_NOW | RTLD_LOCAL);
        }
        if (L.h) {
            L.get_uid = (GetUniqueIdFn)dlsym(L.h, "ncclGetUniqueId");
            L.init_rank = (CommInitRankFn2)dlsym(L.h, "ncclCommInitRank");
            L.destroy = (CommDestroyFn)dlsym(L.h, "ncclCommDestroy");
            L.allgather = (AllGatherFn)dlsym(L.h, "ncclAllGather");
            L.bcast = (BroadcastFn)dlsym(L.h, "ncclBroadcast");
            L.errstr = (ErrStrFn)dlsym(L.h, "ncclGetErrorString");
        }
    }
    LH_REQUIRE(L.h && L.get_uid && L.init_rank && L.destroy && L.allgather && L.bcast, LH_EINVAL,
               "NCCL (libnccl.so.2) is not available in this process");
    return L;
}

void nccl_check(int rc, const char *what) {
    if (rc != 0) {
        NcclLib &L = nccl_lib();
        throw Error(LH_ECUDA, std::string(what) + ": " + (L.errstr ? L.errstr(rc) : std::to_string(rc)));
    }
}

constexpr int NCCL_UINT8 = 1, NCCL_INT64 = 4, NCCL_FLOAT64 = 8;

}  // namespace

struct NcclState {
    void *comm = nullptr;
    int rank = 0, world = 1;
    cudaStream_t cs = nullptr;  // the communication stream (overlaps the context's stream)
    ~NcclState() {
        if (comm) nccl_lib().destroy(comm);
        if (cs) cudaStreamDestroy(cs);
    }
};

static NcclState &nccl_of(Ctx &ctx) {
    LH_REQUIRE(ctx.nccl != nullptr, LH_EINVAL, "call lh_nccl_init on this context first");
    return *static_cast<NcclState *>(ctx.nccl.get());
}

void nccl_unique_id(void *out128) { nccl_check(nccl_lib().get_uid(out128), "ncclGetUniqueId"); }

void nccl_init(Ctx &ctx, int rank, int world, const void *uid128) {
    LH_REQUIRE(world >= 1 && rank >= 0 && rank < world, LH_EINVAL, "invalid NCCL rank/world");
    NcclLib &L = nccl_lib();
    auto st = std::make_shared<NcclState>();
    st->rank = rank;
    st->world = world;
    Uid128 u;
    std::memcpy(u.b, uid128, 128);
    LH_CUDA(cudaSetDevice(ctx.device));
    nccl_check(L.init_rank(&st->comm, world, u, rank), "ncclCommInitRank");
    LH_CUDA(cudaStreamCreateWithFlags(&st->cs, cudaStreamNonBlocking));
    ctx.nccl = st;
}

bool nccl_ready(Ctx &ctx) { return ctx.nccl != nullptr; }
int nccl_rank(Ctx &ctx) { return nccl_of(ctx).rank; }
int nccl_world(Ctx &ctx) { return nccl_of(ctx).world; }
cudaStream_t nccl_stream(Ctx &ctx) { return nccl_of(ctx).cs; }

void nccl_allgather_f64(Ctx &ctx, const double *send, double *recv, size_t count, cudaStream_t s) {
    NcclState &st = nccl_of(ctx);
    nccl_check(nccl_lib().allgather(send, recv, count, NCCL_FLOAT64, st.comm, s), "ncclAllGather");
}
void nccl_allgather_i64(Ctx &ctx, const int64_t *send, int64_t *recv, size_t count, cudaStream_t s) {
    NcclState &st = nccl_of(ctx);
    nccl_check(nccl_lib().allgather(send, recv, count, NCCL_INT64, st.comm, s), "ncclAllGather");
}
void nccl_bcast_bytes(Ctx &ctx, void *buf, size_t bytes, int root, cudaStream_t s) {
    NcclState &st = nccl_of(ctx);
    LH_REQUIRE(root >= 0 && root < st.world, LH_EINVAL, "invalid broadcast root");
    if (bytes == 0) return;
    nccl_check(nccl_lib().bcast(buf, buf, bytes, NCCL_UINT8, root, st.comm, s), "ncclBroadcast");
}

// every device array of H from `root` (all ranks hold the same structure and layout, e.g. a
// factor computed once and shared by ranks that step disjoint right-hand-side columns)
void bcast_hmat(Ctx &ctx, HMat &H, int root) {
    ensure_resident(H, ctx.stream);
    cudaStream_t s = ctx.stream;
    nccl_bcast_bytes(ctx, H.d_arena, sizeof(double) * (size_t)H.arena_len, root, s);
    nccl_bcast_bytes(ctx, H.d_ranks, sizeof(int32_t) * (size_t)std::max(H.nslots, 0), root, s);
    if (H.d_perm) nccl_bcast_bytes(ctx, H.d_perm, sizeof(int32_t) * (size_t)H.perm_len, root, s);
    if (H.d_inv) nccl_bcast_bytes(ctx, H.d_inv, sizeof(double) * (size_t)H.inv_len, root, s);
    LH_CUDA(cudaStreamSynchronize(s));
    H.sync_ranks(s);
}

}  // namespace lh
