// Host replay of the reference H-arithmetic recursion into a static task DAG.
//
// Mirrors, case by case:
//   hops.py:392-408 _lu_block          -> Planner::lu_block
//   hops.py:232-258 _trisolve_block    -> Planner::trisolve_left
//   hops.py:261-279 _trisolve_right_upper -> Planner::trisolve_right_upper
//   hops.py:211-229 _solve_dense_rhs   -> Planner::solve_dense
//   hops.py:348-369 _schur             -> Planner::schur
//   hops.py:318-345 _sub_lowrank/_sub_dense -> Planner::sub_lowrank / sub_dense
//   hops.py:73-100  mul_dense/tmul_dense -> Planner::segmul (per-row-segment tasks)
// Ranks are never read on the host: every width that depends on a rank is a
// run-time rank slot, so one plan serves every matrix with this block structure.
#include "plan_impl.h"

#include <algorithm>
#include <chrono>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <future>

namespace lh {

// ---------------------------------------------------------------------------
// views
// ---------------------------------------------------------------------------
PView PView::rows_(i64 a, i64 cnt) const {
    PView r = *this;
    if (!d.trans) {
        r.d.off += a;
        r.r0 += a;
    } else {
        r.d.off += a * d.ld;
    }
    r.d.rows = (int32_t)cnt;
    return r;
}
PView PView::cols_(i64 a, i64 cnt) const {
    PView r = *this;
    if (!d.trans) r.d.off += a * d.ld;
    else r.d.off += a;
    r.d.cols = (int32_t)cnt;
    return r;
}
PView PView::T() const {
    PView r = *this;
    std::swap(r.d.rows, r.d.cols);
    r.d.trans = !d.trans;
    r.whole = true;
    return r;
}

// ---------------------------------------------------------------------------
// dependency tracking: per object, disjoint row intervals with last writer + readers
// ---------------------------------------------------------------------------
static void add_reader(DepTracker::Seg &s, int32_t task) {
    if (s.nr > 0) {  // the same task touching twice in a row
        const int32_t last = s.nr <= 4 ? s.rd[s.nr - 1] : s.more->back();
        if (last == task) return;
    }
    if (s.nr < 4) s.rd[s.nr] = task;
    else {
        if (!s.more) s.more = new std::vector<int32_t>();
        s.more->push_back(task);
    }
    ++s.nr;
}

void DepTracker::access(int32_t task, u64 obj, i64 a, i64 b, bool write, std::vector<int32_t> &out) {
    if (obj >= objs.size()) objs.resize(std::max<size_t>(obj + 1, objs.size() + objs.size() / 2 + 16));
    std::vector<Seg> &v = objs[obj];
    if (v.empty()) v.push_back(Seg{0, INT64_MAX, -1, 0, {0, 0, 0, 0}, nullptr});
    // first segment containing row a (segments are sorted and cover [0, inf))
    size_t i = std::upper_bound(v.begin(), v.end(), a, [](i64 x, const Seg &s) { return x < s.a; }) -
               v.begin() - 1;
    auto split = [&](size_t k, i64 at) {  // split segment k at row `at` (a < at < b)
        Seg t = v[k];
        if (t.more) t.more = new std::vector<int32_t>(*t.more);
        v[k].b = at;
        t.a = at;
        v.insert(v.begin() + k + 1, t);
    };
    if (v[i].a < a) {
        split(i, a);
        ++i;
    }
    const size_t first = i;
    for (; i < v.size() && v[i].a < b; ++i) {
        if (v[i].b > b) split(i, b);
        Seg &s = v[i];
        if (s.writer >= 0 && s.writer != task) out.push_back(s.writer);
        if (write) {
            for (int k = 0; k < std::min(s.nr, 4); ++k)
                if (s.rd[k] != task) out.push_back(s.rd[k]);
            if (s.more) {
                for (int32_t r : *s.more)
                    if (r != task) out.push_back(r);
                delete s.more;
                s.more = nullptr;
            }
            s.writer = task;
            s.nr = 0;
        } else {
            add_reader(s, task);
        }
    }
    if (write && i - first > 1) {  // the written rows now share one state: merge them
        v[first].b = v[i - 1].b;
        v.erase(v.begin() + first + 1, v.begin() + i);
    }
}

DepTracker::~DepTracker() {
    for (auto &v : objs)
        for (auto &s : v) delete s.more;
}

// ---------------------------------------------------------------------------
// Planner
// ---------------------------------------------------------------------------
Planner::Planner(HMat &F, HMat *X) : F(F), X(X) {
    P = std::make_shared<Plan>();
    P->slot_off_x = F.nslots;
    P->slot_off_tmp = F.nslots + (X ? X->nslots : 0);
    next_slot = P->slot_off_tmp;
    nF = (i64)F.nodes.size();
    nX = X ? (i64)X->nodes.size() : 0;
    deps.objs.reserve((size_t)(3 * (nF + nX) + 1024));
    // measured on the 1D operators: ~29 (H-LU) to ~38 (propagator) tasks per block-tree node
    // and ~6 dependencies per task; reserving (virtual memory, touched only as used) avoids
    // regrowth copies of the multi-100-MB arrays
    const size_t est = (size_t)(nF + nX) * 40;
    P->tasks.reserve(est);
    P->deps.reserve(est * 7);
    P->pieces.reserve(est * 2);
}

// dense object ids: block storage of F (U, V, dense) and X, then the right-hand side, then
// the temporaries in creation order
u64 Planner::key(int base, i64 id, int which) const {
    if (base == B_F) return (u64)(3 * id + which);
    if (base == B_X) return (u64)(3 * nF + 3 * id + which);
    if (base == B_RHS) return (u64)(3 * (nF + nX));
    return (u64)(3 * (nF + nX) + 1 + id);  // B_TMP
}

// storage of a dense leaf or of a virtual child of a refined leaf: absolute offset, ld
void dense_loc(const HMat &H, int32_t b, i64 &off, i64 &ld) {
    off = 0;
    int32_t q = b;
    while (H.nodes[q].vpar >= 0) {
        off += H.nodes[q].doff;
        q = H.nodes[q].vpar;
    }
    off += H.nodes[q].doff;
    ld = H.nodes[q].m;
}

// Dense leaves larger than 64 x 64 are split 2 x 2 for the H-arithmetic planner (recursively):
// along the cluster tree where the leaf's cluster has children, else at row / column 64.
// The split leaf keeps its kind for the structure, the matvec and the exports; only the
// planner recurses into it, so every task runs on the 64-row fast paths.  (Leaf pivoting then
// acts per 64-row half: identical to partial pivoting over the whole leaf whenever that picks
// no cross-half pivot, which a T_CHECK task verifies after the leaf's L21 solve.)
void refine_dense_leaves(HMat &H) {
    if (H.refined) return;
    H.refined = true;
    if (getenv("LEVYH_NO_LEAF_SPLIT")) return;
    std::vector<int32_t> todo;
    for (int32_t b : H.leafblocks) {
        const Node &nd = H.nodes[b];
        if ((nd.kind == K_DENSE || nd.kind == K_FDENSE) && nd.kid[0] < 0 && nd.m > 64 && nd.n > 64)
            todo.push_back(b);
    }
    auto split = [](const Tree *T, int32_t cl, i64 size, int32_t &k0, int32_t &k1) -> i64 {
        if (T && cl >= 0 && !T->nodes[cl].leaf()) {
            k0 = T->nodes[cl].kid[0];
            k1 = T->nodes[cl].kid[1];
            return T->nodes[k0].size();
        }
        k0 = k1 = -1;
        return std::min<i64>(64, size / 2 > 0 ? 64 : size);
    };
    while (!todo.empty()) {
        const int32_t b = todo.back();
        todo.pop_back();
        const Node p = H.nodes[b];
        i64 poff, pld;
        dense_loc(H, b, poff, pld);
        (void)poff;
        int32_t r0c, r1c, c0c, c1c;
        const i64 rs = split(H.rt, p.rcl, p.m, r0c, r1c), cs = split(H.ct, p.ccl, p.n, c0c, c1c);
        if (rs <= 0 || rs >= p.m || cs <= 0 || cs >= p.n) continue;
        int32_t kids[4];
        for (int q = 0; q < 4; ++q) {
            Node c;
            std::memset(&c, 0, sizeof(c));
            const bool lo = q >> 1, rt = q & 1;
            c.kind = K_DENSE;
            c.rcl = lo ? r1c : r0c;
            c.ccl = rt ? c1c : c0c;
            c.r0 = p.r0 + (lo ? rs : 0);
            c.c0 = p.c0 + (rt ? cs : 0);
            c.m = lo ? p.m - rs : rs;
            c.n = rt ? p.n - cs : cs;
            for (auto &k : c.kid) k = -1;
            c.doff = (lo ? rs : 0) + (rt ? cs : 0) * pld;
            c.uoff = c.voff = -1;
            c.rslot = -1;
            c.ioff = -1;
            c.depth = p.depth + 1;
            c.vpar = b;
            kids[q] = (int32_t)H.nodes.size();
            H.nodes.push_back(c);
            if (c.m > 64 && c.n > 64) todo.push_back(kids[q]);
        }
        Node &pp = H.nodes[b];
        for (int q = 0; q < 4; ++q) pp.kid[q] = kids[q];
        pp.rs = rs;
        pp.cs = cs;
    }
}

PView Planner::dense_view(const Mref &M, int32_t b) const {
    const Node &nd = M.H->nodes[b];
    i64 off, ld;
    dense_loc(*M.H, b, off, ld);
    PView v{};
    v.d = DView{off, (int32_t)nd.m, (int32_t)nd.n, (int32_t)ld, -1, (int8_t)M.base, 0, 0};
    v.obj = key(M.base, b, 0);
    v.r0 = 0;
    v.whole = false;
    if (nd.kind != K_HIER && nd.kid[0] >= 0) {
        v.vnode = b;
        v.vh = M.H;
    }
    return v;
}
PView Planner::u_view(const Mref &M, int32_t b) const {
    const Node &nd = M.H->nodes[b];
    PView v{};
    v.d = DView{nd.uoff, (int32_t)nd.m, nd.kcap, (int32_t)nd.m, M.slot_off + nd.rslot,
                (int8_t)M.base, 0, 0};
    v.obj = key(M.base, b, 1);
    return v;
}
PView Planner::v_view(const Mref &M, int32_t b) const {
    const Node &nd = M.H->nodes[b];
    PView v{};
    v.d = DView{nd.voff, (int32_t)nd.n, nd.kcap, (int32_t)nd.n, M.slot_off + nd.rslot,
                (int8_t)M.base, 0, 0};
    v.obj = key(M.base, b, 2);
    return v;
}

// temporaries: size-class pools with delayed FIFO reuse; reuse adds WAR edges
// on every task that touched the previous occupant.
PView Planner::temp(i64 rows, i64 cols, int32_t wslot) {
    i64 need = std::max<i64>(rows * cols, 1);
    int cls = 0;
    while (((i64)1 << cls) < need) ++cls;
    auto &fl = freelist[cls];
    i64 off;
    std::vector<int32_t> prev;
    // reuse distance: a freed block is reused once this many blocks of its class were freed
    // after it (keeps independent work from serialising on WAR edges); large classes keep about
    // LEVYH_TEMP_WINDOW doubles (default 2^26 = 512 MB) in flight instead of 512 blocks
    static const i64 window = getenv("LEVYH_TEMP_WINDOW") ? atoll(getenv("LEVYH_TEMP_WINDOW")) : ((i64)1 << 26);
    const size_t MIN_AGE = (size_t)std::max<i64>(4, std::min<i64>(512, window >> cls));
    if (fl.size() > MIN_AGE) {
        off = fl.front().off;
        prev = std::move(fl.front().users);
        fl.pop_front();
    } else {
        off = P->temp_len;
        P->temp_len += (i64)1 << cls;
    }
    int32_t id = next_temp++;
    TempRec tr;
    tr.off = off;
    tr.cls = cls;
    tr.barrier = -1;
    if (!prev.empty()) {
        // every task touching the new occupant waits for every user of the old one
        DTask nop;
        std::memset(&nop, 0, sizeof(nop));
        nop.type = T_NOP;
        nop.path = -1;
        for (auto &vv : nop.v) vv.wslot = -1;
        std::sort(prev.begin(), prev.end());
        prev.erase(std::unique(prev.begin(), prev.end()), prev.end());
        nop.dep_beg = (int32_t)P->deps.size();
        nop.dep_cnt = (int32_t)prev.size();
        P->deps.insert(P->deps.end(), prev.begin(), prev.end());
        tr.barrier = (int32_t)P->tasks.size();
        P->tasks.push_back(nop);
    }
    temps[id] = std::move(tr);
    PView v{};
    v.d = DView{off, (int32_t)rows, (int32_t)cols, (int32_t)rows, wslot, B_TMP, 0, 0};
    v.obj = key(B_TMP, id, 0);
    v.tmp = id;
    return v;
}

void Planner::release(const PView &v) {
    auto it = temps.find(v.tmp);
    if (it == temps.end()) return;
    FreeBlock fb{it->second.off, std::move(it->second.users)};
    freelist[it->second.cls].push_back(std::move(fb));
    temps.erase(it);
}

int32_t Planner::new_slot() { return next_slot++; }

int32_t Planner::emit(DTask t, std::initializer_list<std::pair<const PView *, bool>> acc,
                      const std::vector<std::pair<PView, bool>> *more) {
    if (F.plan_cancel && F.plan_cancel->load(std::memory_order_relaxed))
        throw Error(LH_EINTERNAL, "planning cancelled: the matrix was destroyed");
    int32_t id = (int32_t)P->tasks.size();
    std::vector<int32_t> &d = dbuf;
    d.clear();
    auto touch = [&](const PView &v, bool w) {
        i64 a = v.whole ? 0 : v.r0;
        i64 b = v.whole ? INT64_MAX : v.r0 + v.d.rows;
        deps.access(id, v.obj, a, b, w, d);
        if (v.vnode >= 0) {  // the refined leaf's storage is also its virtual children's
            std::vector<int32_t> st{v.vnode};
            while (!st.empty()) {
                const Node &q = v.vh->nodes[st.back()];
                st.pop_back();
                for (int k = 0; k < 4; ++k)
                    if (q.kid[k] >= 0) {
                        deps.access(id, key(v.d.base, q.kid[k], 0), 0, INT64_MAX, w, d);
                        st.push_back(q.kid[k]);
                    }
            }
        }
        if (v.tmp >= 0) {
            auto it = temps.find(v.tmp);
            if (it != temps.end()) {
                if (it->second.barrier >= 0) d.push_back(it->second.barrier);
                it->second.users.push_back(id);
            }
        }
    };
    for (auto &p : acc) touch(*p.first, p.second);
    if (more)
        for (auto &p : *more) touch(p.first, p.second);
    std::sort(d.begin(), d.end());
    d.erase(std::unique(d.begin(), d.end()), d.end());
    t.dep_beg = (int32_t)P->deps.size();
    t.dep_cnt = (int32_t)d.size();
    P->deps.insert(P->deps.end(), d.begin(), d.end());
    P->tasks.push_back(t);
    if (stream && stream->want.load(std::memory_order_relaxed) &&
        P->tasks.size() - cut_task >= stream->min_chunk)
        cut_chunk();
    return id;
}

// tasks [cut_task, end) as a self-contained plan: dependencies on earlier chunks are dropped
// (those chunks have run), indices are rebased; temp offsets stay global (shared pool)
void Planner::cut_chunk() {
    auto C = std::make_shared<Plan>();
    const int32_t t0 = (int32_t)cut_task, p0 = (int32_t)cut_piece;
    const int32_t n = (int32_t)P->tasks.size();
    C->tasks.reserve(n - t0);
    for (int32_t i = t0; i < n; ++i) {
        DTask t = P->tasks[i];
        const int32_t *dp = P->deps.data() + t.dep_beg;
        const int32_t beg = (int32_t)C->deps.size();
        for (int32_t k = 0; k < t.dep_cnt; ++k)
            if (dp[k] >= t0) C->deps.push_back(dp[k] - t0);
        t.dep_beg = beg;
        t.dep_cnt = (int32_t)C->deps.size() - beg;
        t.pc_beg -= p0;
        t.pc_end -= p0;
        C->tasks.push_back(t);
    }
    C->pieces.assign(P->pieces.begin() + p0, P->pieces.end());
    C->paths = P->paths;
    C->temp_len = P->temp_len;
    C->nslots_total = next_slot;
    C->slot_off_x = P->slot_off_x;
    C->slot_off_tmp = P->slot_off_tmp;
    C->own_temp = false;
    assign_priorities(*C);
    cut_task = P->tasks.size();
    cut_piece = P->pieces.size();
    std::lock_guard<std::mutex> lk(stream->mu);
    stream->chunks.push_back(C);
    stream->want.store(false);
    stream->cv.notify_all();
}

static DTask mk(int32_t type) {
    DTask t;
    std::memset(&t, 0, sizeof(t));
    t.type = type;
    t.path = -1;
    for (auto &v : t.v) v.wslot = -1;
    return t;
}

// leaf blocks of a subtree with offsets relative to the subtree root
void Planner::leaves_of(const Mref &M, int32_t b, i64 r, i64 c, std::vector<LeafRef> &out) const {
    const Node &nd = M.H->nodes[b];
    if (hier(nd)) {
        leaves_of(M, nd.kid[0], r, c, out);
        leaves_of(M, nd.kid[1], r, c + nd.cs, out);
        leaves_of(M, nd.kid[2], r + nd.rs, c, out);
        leaves_of(M, nd.kid[3], r + nd.rs, c + nd.cs, out);
    } else {
        out.push_back({b, r, c});
    }
}

// row segments (leaf clusters) of a cluster subtree, relative to its start
void Planner::segments_of(const Tree &T, int32_t cl, std::vector<std::pair<i64, i64>> &out) const {
    const Cluster &c = T.nodes[cl];
    auto leaf_rows = [&](i64 lo, i64 size) {  // leaf clusters > 64 rows: 64-row segments
        if (!F.refined || getenv("LEVYH_NO_LEAF_SPLIT")) {
            out.push_back({lo, size});
            return;
        }
        for (i64 a = 0; a < size; a += 64) out.push_back({lo + a, std::min<i64>(64, size - a)});
    };
    if (c.leaf()) {
        leaf_rows(0, c.size());
        return;
    }
    std::vector<int32_t> st{cl};
    while (!st.empty()) {
        int32_t k = st.back();
        st.pop_back();
        const Cluster &q = T.nodes[k];
        if (q.leaf()) leaf_rows(q.lo - c.lo, q.size());
        else {
            st.push_back(q.kid[1]);
            st.push_back(q.kid[0]);
        }
    }
}

// Y (rows of op(A)) = beta*Y + alpha * op(A) * X    (mul_dense / tmul_dense, hops.py:73-100)
// A is a block subtree of M; X has rows = columns of op(A).
void Planner::segmul(const PView &Y, const Mref &M, int32_t a, const PView &X, bool trans,
                     double alpha, bool overwrite) {
    const Node &A = M.H->nodes[a];
    if (A.kind == K_ZERO) {
        if (overwrite) {
            DTask t = mk(T_IDENT);
            t.flags = 1;
            t.v[0] = Y.d;
            emit(t, {{&Y, true}});
        }
        return;
    }
    std::vector<LeafRef> lv;
    leaves_of(M, a, 0, 0, lv);
    // phase 1: W_b = F^T X for every low-rank leaf (F = V, or U when transposed)
    struct LRW {
        PView w;
        bool used;
    };
    std::vector<PView> W(lv.size());
    std::vector<bool> hasW(lv.size(), false);
    for (size_t q = 0; q < lv.size(); ++q) {
        const Node &nd = M.H->nodes[lv[q].b];
        if (nd.kind != K_LR) continue;
        PView F = trans ? u_view(M, lv[q].b) : v_view(M, lv[q].b);
        i64 xr = trans ? lv[q].r : lv[q].c;
        i64 n = trans ? nd.m : nd.n;
        PView Xs = X.rows_(xr, n);
        // W is (rank of F) x (columns of X); both widths are read at run time from
        // the operands, so W itself carries no rank slot.
        PView w = temp(KC, std::max<i64>(X.d.cols, 1), -1);
        w.d.ld = KC;
        DTask t = mk(T_VTX);
        t.v[0] = F.d;
        t.v[1] = Xs.d;
        t.v[2] = w.d;
        emit(t, {{&F, false}, {&Xs, false}, {&w, true}});
        W[q] = w;
        hasW[q] = true;
    }
    // phase 2: one task per output row segment; leaves bucketed by the segments they cover
    std::vector<std::pair<i64, i64>> segs;
    const int32_t scl = trans ? A.ccl : A.rcl;
    if (scl >= 0) segments_of(trans ? *M.H->ct : *M.H->rt, scl, segs);
    else segs.push_back({0, trans ? A.n : A.m});  // virtual child of a refined leaf (<= 64)
    std::vector<i64> starts(segs.size());
    for (size_t k = 0; k < segs.size(); ++k) starts[k] = segs[k].first;
    std::vector<std::vector<int32_t>> bucket(segs.size());
    for (size_t q = 0; q < lv.size(); ++q) {
        const Node &nd = M.H->nodes[lv[q].b];
        if (nd.kind == K_ZERO) continue;
        const i64 o0 = trans ? lv[q].c : lv[q].r, on = trans ? nd.n : nd.m;
        size_t k = std::upper_bound(starts.begin(), starts.end(), o0) - starts.begin() - 1;
        for (; k < segs.size() && segs[k].first < o0 + on; ++k) bucket[k].push_back((int32_t)q);
    }
    for (size_t sk = 0; sk < segs.size(); ++sk) {
        const auto &sg = segs[sk];
        i64 s0 = sg.first, s1 = sg.first + sg.second;
        PView Ys = Y.rows_(s0, s1 - s0);
        DTask t = mk(T_SEGMUL);
        t.alpha = alpha;
        t.flags = overwrite ? 1 : 0;
        t.v[0] = Ys.d;
        t.pc_beg = (int32_t)P->pieces.size();
        std::vector<std::pair<PView, bool>> more;
        more.reserve(2 * bucket[sk].size() + 1);
        for (int32_t q : bucket[sk]) {
            const Node &nd = M.H->nodes[lv[q].b];
            i64 o0 = trans ? lv[q].c : lv[q].r;   // output-row range of this leaf
            i64 on = trans ? nd.n : nd.m;
            i64 a0 = std::max(o0, s0), a1 = std::min(o0 + on, s1);
            LH_REQUIRE(a0 == s0 && a1 == s1, LH_EINTERNAL, "leaf block not aligned with segments");
            DPiece pc;
            std::memset(&pc, 0, sizeof(pc));
            if (nd.kind == K_LR) {
                PView F = trans ? v_view(M, lv[q].b) : u_view(M, lv[q].b);
                PView Fs = F.rows_(a0 - o0, a1 - a0);
                pc.kind = 1;
                pc.mat = Fs.d;
                pc.x = W[q].d;
                more.push_back({Fs, false});
                more.push_back({W[q], false});
            } else {
                PView D = dense_view(M, lv[q].b);
                PView Ds = trans ? D.T().rows_(a0 - o0, a1 - a0) : D.rows_(a0 - o0, a1 - a0);
                i64 xr = trans ? lv[q].r : lv[q].c;
                i64 n = trans ? nd.m : nd.n;
                PView Xs = X.rows_(xr, n);
                pc.kind = 0;
                pc.mat = Ds.d;
                pc.x = Xs.d;
                more.push_back({Ds, false});
                more.push_back({Xs, false});
            }
            P->pieces.push_back(pc);
        }
        t.pc_end = (int32_t)P->pieces.size();
        more.push_back({Ys, true});
        emit(t, {}, &more);
    }
    for (size_t q = 0; q < lv.size(); ++q)
        if (hasW[q]) release(W[q]);
}

// T X = B for a dense right-hand side view B (hops.py:211-229); mode 0 L, 1 U, 2 Ut
void Planner::solve_dense(const Mref &T, int32_t t, const PView &B, int mode, bool unit,
                          const std::string &path) {
    const Node &nd = T.H->nodes[t];
    if (!hier(nd)) {
        LH_REQUIRE(nd.kind == K_FDENSE || nd.kind == K_DENSE, LH_ETYPE,
                   "triangular solve needs a dense diagonal leaf at " + path);
        PView Tv = dense_view(T, t);
        DTask k = mk(T_TRSM);
        k.v[0] = Tv.d;
        k.v[1] = B.d;
        if (nd.kind == K_FDENSE) {
            // _leaf_solve on a FactoredDense leaf: unit L with the leaf pivots, non-unit U
            k.flags = mode | (mode == 0 ? 16 : 0) | 32;
            k.aux = (int32_t)nd.poff;
            if (nd.ioff >= 0) {  // apply the packed leaf inverse written by the leaf's GETRF
                k.flags |= 64;
                k.v[2] = DView{nd.ioff, (int32_t)nd.m, (int32_t)nd.m, (int32_t)nd.m, -1, B_INV, 0, 0};
            }
        } else {
            // plain dense triangle (trisolve_lower / trisolve_upper_right on an unfactored
            // H-matrix): zero diagonal raises with the block path (hops.py:179-182)
            k.flags = mode | (unit ? 16 : 0) | 128;
            k.path = add_path("singular triangular diagonal block at " + path);
        }
        emit(k, {{&Tv, false}, {&B, true}});
        return;
    }
    i64 s = nd.rs;
    PView B1 = B.rows_(0, s), B2 = B.rows_(s, nd.m - s);
    const bool virt = nd.kind != K_HIER;  // refined leaf: its halves report the leaf's path
    const std::string p11 = virt ? path : path + ".11", p22 = virt ? path : path + ".22";
    if (mode == 0) {
        solve_dense(T, nd.kid[0], B1, mode, unit, p11);
        segmul(B2, T, nd.kid[2], B1, false, -1.0, false);
        solve_dense(T, nd.kid[3], B2, mode, unit, p22);
    } else if (mode == 1) {
        solve_dense(T, nd.kid[3], B2, mode, unit, p22);
        segmul(B1, T, nd.kid[1], B2, false, -1.0, false);
        solve_dense(T, nd.kid[0], B1, mode, unit, p11);
    } else {
        solve_dense(T, nd.kid[0], B1, mode, unit, p11);
        segmul(B2, T, nd.kid[1], B1, true, -1.0, false);
        solve_dense(T, nd.kid[3], B2, mode, unit, p22);
    }
}

// hops.py:232-258: T X = B in place on block b of matrix Bm (mode 0 L, 1 U)
int Planner::colpart(const Mref &M, int32_t b) const {
    if (!filt || M.base != B_X) return 1;
    const Node &nd = M.H->nodes[b];
    const i64 a = nd.c0, e = nd.c0 + nd.n;
    if (e <= flo || a >= fhi) return 0;
    return (a >= flo && e <= fhi) ? 1 : 2;
}

void Planner::trisolve_left(const Mref &T, int32_t t, const Mref &Bm, int32_t b, int mode,
                            bool unit, const std::string &path) {
    const Node &B = Bm.H->nodes[b];
    if (B.kind == K_ZERO) return;
    const int cp = colpart(Bm, b);
    if (cp == 0) return;
    if (cp == 2 && !hier(B)) throw Error(LH_EINTERNAL, "column split straddles a leaf");
    if (B.kind == K_LR) {
        solve_dense(T, t, u_view(Bm, b), mode, unit, path);
        return;
    }
    const Node &Tn = T.H->nodes[t];
    if (dense_leaf(B) || !hier(Tn)) {
        LH_REQUIRE(B.kind == K_DENSE, LH_ETYPE,
                   "hierarchical right-hand side against a leaf triangle at " + path);
        solve_dense(T, t, dense_view(Bm, b), mode, unit, path);
        return;
    }
    LH_REQUIRE(hier(B), LH_ETYPE, "hierarchical right-hand side against a leaf triangle at " + path);
    const int32_t c00 = Tn.kid[0], c01 = Tn.kid[1], c10 = Tn.kid[2], c11 = Tn.kid[3];
    const int32_t b00 = B.kid[0], b01 = B.kid[1], b10 = B.kid[2], b11 = B.kid[3];
    const bool virt = Tn.kind != K_HIER;
    const std::string p11 = virt ? path : path + ".11", p22 = virt ? path : path + ".22";
    if (mode == 0) {
        trisolve_left(T, c00, Bm, b00, mode, unit, p11);
        trisolve_left(T, c00, Bm, b01, mode, unit, p11);
        schur(Bm, b10, T, c10, Bm, b00);
        schur(Bm, b11, T, c10, Bm, b01);
        trisolve_left(T, c11, Bm, b10, mode, unit, p22);
        trisolve_left(T, c11, Bm, b11, mode, unit, p22);
    } else {
        trisolve_left(T, c11, Bm, b10, mode, unit, p22);
        trisolve_left(T, c11, Bm, b11, mode, unit, p22);
        schur(Bm, b00, T, c01, Bm, b10);
        schur(Bm, b01, T, c01, Bm, b11);
        trisolve_left(T, c00, Bm, b00, mode, unit, p11);
        trisolve_left(T, c00, Bm, b01, mode, unit, p11);
    }
}

// hops.py:261-279: X U = B in place on block b
void Planner::trisolve_right_upper(const Mref &T, int32_t t, const Mref &Bm, int32_t b,
                                   const std::string &path) {
    const Node &B = Bm.H->nodes[b];
    if (B.kind == K_ZERO) return;
    if (B.kind == K_LR) {
        solve_dense(T, t, v_view(Bm, b), 2, true, path);
        return;
    }
    const Node &Tn = T.H->nodes[t];
    if (dense_leaf(B) || !hier(Tn)) {
        LH_REQUIRE(B.kind == K_DENSE, LH_ETYPE,
                   "hierarchical right-hand side against a leaf triangle at " + path);
        solve_dense(T, t, dense_view(Bm, b).T(), 2, true, path);
        return;
    }
    LH_REQUIRE(hier(B), LH_ETYPE, "hierarchical right-hand side against a leaf triangle at " + path);
    const int32_t c00 = Tn.kid[0], c01 = Tn.kid[1], c11 = Tn.kid[3];
    const int32_t b00 = B.kid[0], b01 = B.kid[1], b10 = B.kid[2], b11 = B.kid[3];
    const bool virt = Tn.kind != K_HIER;
    const std::string p11 = virt ? path : path + ".11", p22 = virt ? path : path + ".22";
    trisolve_right_upper(T, c00, Bm, b00, p11);
    trisolve_right_upper(T, c00, Bm, b10, p11);
    schur(Bm, b01, Bm, b00, T, c01);
    schur(Bm, b11, Bm, b10, T, c01);
    trisolve_right_upper(T, c11, Bm, b01, p22);
    trisolve_right_upper(T, c11, Bm, b11, p22);
}

// hops.py:318-331: C -= U V^T
void Planner::sub_lowrank(const Mref &Cm, int32_t c, const PView &U, const PView &V) {
    const Node &C = Cm.H->nodes[c];
    if (C.kind == K_ZERO) throw Error(LH_EINTERNAL, "update into a structurally zero block");
    if (dense_leaf(C)) {
        PView Cv = dense_view(Cm, c);
        DTask t = mk(T_DGEMM);
        t.alpha = -1.0;
        t.flags = 1;  // C += alpha * U * V^T
        t.v[0] = Cv.d;
        t.v[1] = U.d;
        t.v[2] = V.d;
        emit(t, {{&U, false}, {&V, false}, {&Cv, true}});
    } else if (C.kind == K_LR) {
        PView Cu = u_view(Cm, c), Cv = v_view(Cm, c);
        DTask t = mk(T_LRADD);
        t.alpha = -1.0;
        t.alpha2 = eps2;
        t.v[0] = Cu.d;
        t.v[1] = Cv.d;
        t.v[2] = U.d;
        t.v[3] = V.d;
        Cu.whole = Cv.whole = true;
        emit(t, {{&U, false}, {&V, false}, {&Cu, true}, {&Cv, true}});
    } else {
        i64 rs = C.rs, cs = C.cs;
        sub_lowrank(Cm, C.kid[0], U.rows_(0, rs), V.rows_(0, cs));
        sub_lowrank(Cm, C.kid[1], U.rows_(0, rs), V.rows_(cs, C.n - cs));
        sub_lowrank(Cm, C.kid[2], U.rows_(rs, C.m - rs), V.rows_(0, cs));
        sub_lowrank(Cm, C.kid[3], U.rows_(rs, C.m - rs), V.rows_(cs, C.n - cs));
    }
}

// hops.py:334-345: C -= D
void Planner::sub_dense(const Mref &Cm, int32_t c, const PView &D) {
    const Node &C = Cm.H->nodes[c];
    if (dense_leaf(C)) {
        PView Cv = dense_view(Cm, c);
        DTask t = mk(T_DADD);
        t.alpha = -1.0;
        t.v[0] = Cv.d;
        t.v[1] = D.d;
        emit(t, {{&D, false}, {&Cv, true}});
    } else if (C.kind == K_LR) {
        lr_sketch_update(Cm, c, nullptr, -1, nullptr, -1, &D);
    } else if (C.kind == K_ZERO) {
        throw Error(LH_EINTERNAL, "update into a structurally zero block");
    } else {
        i64 rs = C.rs, cs = C.cs;
        sub_dense(Cm, C.kid[0], D.rows_(0, rs).cols_(0, cs));
        sub_dense(Cm, C.kid[1], D.rows_(0, rs).cols_(cs, C.n - cs));
        sub_dense(Cm, C.kid[2], D.rows_(rs, C.m - rs).cols_(0, cs));
        sub_dense(Cm, C.kid[3], D.rows_(rs, C.m - rs).cols_(cs, C.n - cs));
    }
}

// C (low-rank) -= M with M = A B (implicit, both block subtrees) or M = D (explicit dense).
// The reference converts such updates through a dense SVD (_sub_dense -> _svd_lowrank,
// hops.py:334-345, :159-163), which would materialise whole admissible blocks.  Here M
// is sketched: Y = M Omega (p Gaussian columns), Q = orth(Y), Z = M^T Q, and C -= Q Z^T
// goes through the same eps2 Frobenius recompression (_add_lr).
constexpr int P_SKETCH = 14;  // products of admissible blocks have eps-ranks <= ~8 here
void Planner::lr_sketch_update(const Mref &Cm, int32_t c, const Mref *Am, int32_t a,
                               const Mref *Bm, int32_t b, const PView *D) {
    const Node &C = Cm.H->nodes[c];
    const int p = P_SKETCH;
    PView Om = temp(C.n, p, -1);
    {
        DTask t = mk(T_RAND);
        t.aux = rand_seed++;
        t.v[0] = Om.d;
        emit(t, {{&Om, true}});
    }
    PView Y = temp(C.m, p, -1);
    if (D) {
        DTask t = mk(T_DGEMM);
        t.alpha = 1.0;
        t.flags = 2;
        t.v[0] = Y.d;
        t.v[1] = D->d;
        t.v[2] = Om.d;
        emit(t, {{D, false}, {&Om, false}, {&Y, true}});
    } else {
        const Node &B = Bm->H->nodes[b];
        PView T1 = temp(B.m, p, -1);
        segmul(T1, *Bm, b, Om, false, 1.0, true);
        segmul(Y, *Am, a, T1, false, 1.0, true);
        release(T1);
    }
    release(Om);
    {
        DTask t = mk(T_ORTH);
        t.v[0] = Y.d;
        emit(t, {{&Y, true}});
    }
    PView Z = temp(C.n, p, -1);
    if (D) {
        DTask t = mk(T_DGEMM);
        t.alpha = 1.0;
        t.flags = 2;
        t.v[0] = Z.d;
        t.v[1] = D->T().d;
        t.v[2] = Y.d;
        PView Dt = D->T();
        emit(t, {{&Dt, false}, {&Y, false}, {&Z, true}});
    } else {
        const Node &A = Am->H->nodes[a];
        PView T2 = temp(A.n, p, -1);
        segmul(T2, *Am, a, Y, true, 1.0, true);
        segmul(Z, *Bm, b, T2, true, 1.0, true);
        release(T2);
    }
    sub_lowrank(Cm, c, Y, Z);
    release(Y);
    release(Z);
}

// dense temp copy of a block subtree (hmatrix.py:402-413 to_dense)
PView Planner::densify(const Mref &M, int32_t b) {
    const Node &nd = M.H->nodes[b];
    PView D = temp(nd.m, nd.n, -1);
    std::vector<LeafRef> lv;
    leaves_of(M, b, 0, 0, lv);
    for (auto &l : lv) {
        const Node &q = M.H->nodes[l.b];
        PView Ds = D.rows_(l.r, q.m).cols_(l.c, q.n);
        DTask t = mk(T_DENSIFY);
        if (q.kind == K_ZERO) {
            t.type = T_IDENT;
            t.flags = 1;
            t.v[0] = Ds.d;
            emit(t, {{&Ds, true}});
        } else if (q.kind == K_LR) {
            PView U = u_view(M, l.b), V = v_view(M, l.b);
            t.v[0] = Ds.d;
            t.v[1] = U.d;
            t.v[2] = V.d;
            t.flags = 1;
            emit(t, {{&U, false}, {&V, false}, {&Ds, true}});
        } else {
            PView S = dense_view(M, l.b);
            t.v[0] = Ds.d;
            t.v[1] = S.d;
            emit(t, {{&S, false}, {&Ds, true}});
        }
    }
    return D;
}

static bool is_zero(const Node &n) { return n.kind == K_ZERO; }

// hops.py:348-369: C -= A B
void Planner::schur(const Mref &Cm, int32_t c, const Mref &Am, int32_t a, const Mref &Bm, int32_t b) {
    const Node &A = Am.H->nodes[a];
    const Node &B = Bm.H->nodes[b];
    const Node &C = Cm.H->nodes[c];
    if (is_zero(A) || is_zero(B)) return;  // structurally zero operand: no update
    const int cp = colpart(Cm, c);
    if (cp == 0) return;
    if (cp == 2) {  // only the block recursion may cross a column split
        if (!(hier(C) && hier(A) && hier(B) && A.cs == B.rs && C.rs == A.rs && C.cs == B.cs))
            throw Error(LH_EINTERNAL, "column split straddles a product update");
    }
    if (A.kind == K_LR) {
        PView Av = v_view(Am, a);
        PView W = temp(B.n, Av.d.cols, Av.d.wslot);  // tmul_dense(B, A.v): B^T A.v
        segmul(W, Bm, b, Av, true, 1.0, true);
        sub_lowrank(Cm, c, u_view(Am, a), W);
        release(W);
    } else if (B.kind == K_LR) {
        PView Bu = u_view(Bm, b);
        PView W = temp(A.m, Bu.d.cols, Bu.d.wslot);  // mul_dense(A, B.u)
        segmul(W, Am, a, Bu, false, 1.0, true);
        sub_lowrank(Cm, c, W, v_view(Bm, b));
        release(W);
    } else if (C.kind == K_LR) {
        // dense product into an admissible target: sketched instead of a dense SVD
        lr_sketch_update(Cm, c, &Am, a, &Bm, b, nullptr);
    } else if (dense_leaf(A) && dense_leaf(B)) {
        PView Ad = dense_view(Am, a), Bd = dense_view(Bm, b);
        if (dense_leaf(C)) {
            PView Cv = dense_view(Cm, c);
            DTask t = mk(T_DGEMM);
            t.alpha = -1.0;
            t.v[0] = Cv.d;
            t.v[1] = Ad.d;
            t.v[2] = Bd.d;
            emit(t, {{&Ad, false}, {&Bd, false}, {&Cv, true}});
        } else {
            PView D = temp(A.m, B.n, -1);
            DTask t = mk(T_DGEMM);
            t.alpha = 1.0;
            t.flags = 2;
            t.v[0] = D.d;
            t.v[1] = Ad.d;
            t.v[2] = Bd.d;
            emit(t, {{&Ad, false}, {&Bd, false}, {&D, true}});
            sub_dense(Cm, c, D);
            release(D);
        }
    } else if (dense_leaf(A)) {
        // tmul_dense(B, A.d^T)^T
        PView Ad = dense_view(Am, a);
        PView D = temp(B.n, A.m, -1);
        segmul(D, Bm, b, Ad.T(), true, 1.0, true);
        sub_dense(Cm, c, D.T());
        release(D);
    } else if (dense_leaf(B)) {
        PView Bd = dense_view(Bm, b);
        PView D = temp(A.m, B.n, -1);
        segmul(D, Am, a, Bd, false, 1.0, true);
        sub_dense(Cm, c, D);
        release(D);
    } else if (hier(C) && hier(A) && hier(B)) {
        if (A.cs != B.rs || C.rs != A.rs || C.cs != B.cs) {
            PView Bd = densify(Bm, b);
            PView D = temp(A.m, B.n, -1);
            segmul(D, Am, a, Bd, false, 1.0, true);
            sub_dense(Cm, c, D);
            release(D);
            release(Bd);
            return;
        }
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j)
                for (int k = 0; k < 2; ++k)
                    schur(Cm, C.kid[2 * i + j], Am, A.kid[2 * i + k], Bm, B.kid[2 * k + j]);
    } else {
        PView Bd = densify(Bm, b);
        PView D = temp(A.m, B.n, -1);
        segmul(D, Am, a, Bd, false, 1.0, true);
        sub_dense(Cm, c, D);
        release(D);
        release(Bd);
    }
}

// hops.py:392-408
void Planner::lu_block(int32_t b, const std::string &path) {
    Node &nd = F.nodes[b];
    Mref Fm{&F, B_F, 0};
    if (dense_leaf(nd)) {
        LH_REQUIRE(nd.m == nd.n, LH_EINTERNAL, "non-square diagonal leaf");
        PView D = dense_view(Fm, b);
        DTask t = mk(T_GETRF);
        t.aux = (int32_t)perm_len;
        nd.poff = perm_len;
        perm_len += nd.m;
        t.v[0] = D.d;
        if (nd.m <= LEAF_INV_MAX) {  // also write the packed leaf inverse (L^-1 | U^-1)
            nd.ioff = inv_len;
            inv_len += nd.m * nd.m;
            t.v[1] = DView{nd.ioff, (int32_t)nd.m, (int32_t)nd.m, (int32_t)nd.m, -1, B_INV, 0, 0};
            t.flags = 1;
        }
        t.path = add_path("zero pivot in dense diagonal leaf at " + path);
        emit(t, {{&D, true}});
        nd.kind = K_FDENSE;
        return;
    }
    LH_REQUIRE(hier(nd), LH_ETYPE,
               std::string("cannot LU-factorize diagonal block of type ") +
                   (nd.kind == K_LR ? "LowRank" : "Dense") + " at " + path);
    const bool virt = nd.kind != K_HIER;  // refined dense leaf: blocked LU of its halves
    const int32_t k0 = nd.kid[0], k1 = nd.kid[1], k2 = nd.kid[2], k3 = nd.kid[3];
    lu_block(k0, virt ? path : path + ".11");
    trisolve_left(Fm, k0, Fm, k1, 0, true, virt ? path : path + ".12");
    trisolve_right_upper(Fm, k0, Fm, k2, virt ? path : path + ".21");
    if (virt) {
        // partial pivoting over the whole leaf would have picked a pivot from the lower half
        // iff some |L21| > 1: fail loudly rather than return a differently pivoted factor
        PView L21 = dense_view(Fm, k2);
        DTask t = mk(T_CHECK);
        t.alpha = 1.0 + 1e-12;
        t.v[0] = L21.d;
        t.path = add_path("leaf LU needs pivoting across its 64-row halves at " + path +
                          " (set LEVYH_NO_LEAF_SPLIT=1)");
        emit(t, {{&L21, false}});
    }
    schur(Fm, k3, Fm, k2, Fm, k1);
    lu_block(k3, virt ? path : path + ".22");
    if (virt) {  // the leaf itself now holds its LU (factored for every other consumer)
        Node &me = F.nodes[b];
        me.kind = K_FDENSE;
        me.poff = F.nodes[k0].poff;
        me.ioff = -1;
    }
}

int32_t Planner::add_path(const std::string &s) {
    P->paths.push_back(s);
    return (int32_t)P->paths.size() - 1;
}

// b-level priority classes (critical-path friendly); tasks stay in program order
// (topological) and the ready-queue executor takes them in readiness order
void assign_priorities(Plan &P) {
    auto &T = P.tasks;
    const int32_t n = (int32_t)T.size();
    // estimated microseconds per task incl. ~3 us hand-off (measured on B200, r01)
    auto cost = [&](const DTask &t) -> double {
        switch (t.type) {
            case T_GETRF: return 90.0;
            case T_TRSM: return 9.0;
            case T_SEGMUL: return 6.0 + 1.5 * (t.pc_end - t.pc_beg);
            case T_VTX: return 8.0 + t.v[0].rows / 500.0;
            case T_LRADD: return 120.0 + (t.v[0].rows + t.v[1].rows) / 100.0;
            case T_ORTH: return 60.0 + t.v[0].rows / 200.0;
            case T_DGEMM: return 23.0;
            case T_RAND: return 20.0;
            case T_NOP: return 0.5;
            default: return 8.0;
        }
    };
    // b-level (cost of the longest path from the task to the end) -> NPRIO buckets; the
    // backward pass touches only dense float arrays (not the 184-byte task records)
    std::vector<float> c(n), bl(n);
    std::vector<int32_t> db(n), dc(n);
    for (int32_t i = 0; i < n; ++i) {
        c[i] = bl[i] = (float)cost(T[i]);
        db[i] = T[i].dep_beg;
        dc[i] = T[i].dep_cnt;
    }
    const int32_t *deps = P.deps.data();
    for (int32_t i = n - 1; i >= 0; --i) {
        const int32_t *dp = deps + db[i];
        const float bi = bl[i];
        for (int32_t k = 0; k < dc[i]; ++k) {
            const int32_t p = dp[k];
            bl[p] = std::max(bl[p], c[p] + bi);
        }
    }
    float mx = 1e-30f;
    for (int32_t i = 0; i < n; ++i) mx = std::max(mx, bl[i]);
    for (int32_t i = 0; i < n; ++i) T[i].prio = std::min(NPRIO - 1, (int)(NPRIO * bl[i] / mx));
}

void Planner::finalize() {
    P->nslots_total = next_slot;
    if (getenv("LEVYH_TEMP_HIST")) {  // planner diagnostics: pooled temp blocks per size class
        for (auto &kv : freelist)
            fprintf(stderr, "[levyh] temp class 2^%d: %zu blocks pooled, %.3f GB\n", kv.first, kv.second.size(),
                    8e-9 * (double)kv.second.size() * (double)((i64)1 << kv.first));
    }
    bool engaged = false;
    if (stream) {
        std::lock_guard<std::mutex> lk(stream->mu);
        engaged = stream->engaged;
    }
    if (!engaged) assign_priorities(*P);  // streamed chunks carry their own priorities
    if (stream) {  // hand the tail to an engaged consumer, then signal completion
        bool engaged;
        {
            std::lock_guard<std::mutex> lk(stream->mu);
            engaged = stream->engaged;
        }
        if (engaged && P->tasks.size() > cut_task) cut_chunk();
        std::lock_guard<std::mutex> lk(stream->mu);
        stream->done = true;
        stream->cv.notify_all();
    }
}

// longest dependency chain (in tasks, NOPs excluded); tasks are topologically ordered
void plan_work(const Plan &P, const std::vector<int32_t> &ranks, double rank_other, double &flops, double &bytes) {
    auto cols = [&](const DView &v) -> double {
        if (v.wslot < 0) return (double)v.cols;
        const double r = v.wslot < (int32_t)ranks.size() ? (double)ranks[v.wslot] : rank_other;
        return std::min(r, (double)v.cols);
    };
    auto size = [&](const DView &v) { return (double)v.rows * cols(v); };
    double fl = 0.0, by = 0.0;
    for (const DTask &t : P.tasks) {
        const DView *v = t.v;
        switch (t.type) {
        case T_GETRF: {  // LU with partial pivoting of an m x m leaf (+ its packed inverse when stored)
            const double m = v[0].rows;
            fl += 2.0 / 3.0 * m * m * m;
            by += 2.0 * m * m;
            break;
        }
        case T_TRSM: {
            const double m = v[0].rows, k = cols(v[1]);
            fl += m * m * k;
            by += 0.5 * m * m + 2.0 * (double)v[1].rows * k;
            break;
        }
        case T_SEGMUL: {
            const double k = cols(v[0]);
            by += 2.0 * size(v[0]);
            for (int32_t q = t.pc_beg; q < t.pc_end; ++q) {
                const DPiece &pc = P.pieces[q];
                const double inner = pc.kind == 0 ? (double)pc.mat.cols : cols(pc.mat);
                fl += 2.0 * (double)pc.mat.rows * inner * k;
                by += (double)pc.mat.rows * inner + inner * k;
            }
            break;
        }
        case T_VTX: {  // W (r x k) = v0^T (n x r) v1 (n x k)
            const double n = v[0].rows, r = cols(v[0]), k = cols(v[1]);
            fl += 2.0 * n * r * k;
            by += n * r + n * k + r * k;
            break;
        }
        case T_LRADD: {  // CGS2 QR of [U U2] and [V V2], K x K core, Jacobi SVD, apply
            const double m = v[0].rows, n = v[1].rows, r2 = cols(v[2]);
            const double r1 = std::min(cols(v[0]), std::max(0.0, (double)v[0].cols - r2));
            const double K = r1 + r2;
            fl += 4.0 * (m + n) * K * K + 14.0 * K * K * K + 2.0 * (m + n) * K * std::min(K, r1 + 1.0);
            by += 2.0 * (m + n) * K + (m + n) * r2;
            break;
        }
        case T_DGEMM: {
            const double m = v[0].rows, n = cols(v[0]);
            const double k = (t.flags & 1) ? cols(v[2]) : (double)v[2].rows;
            fl += 2.0 * m * n * std::min(k, cols(v[1]));
            by += 2.0 * m * n + size(v[1]) + size(v[2]);
            break;
        }
        case T_DADD:
            fl += size(v[0]);
            by += 3.0 * size(v[0]);
            break;
        case T_DENSIFY: {
            const double r = v[2].rows > 0 ? cols(v[1]) : 0.0;
            fl += 2.0 * size(v[0]) * r;
            by += size(v[0]) + (r > 0 ? ((double)v[1].rows + v[2].rows) * r : size(v[1]));
            break;
        }
        case T_IDENT:
        case T_RAND:
            by += size(v[0]);
            break;
        case T_ORTH: {
            const double m = v[0].rows, p = cols(v[0]);
            fl += 4.0 * m * p * p;
            by += 2.0 * m * p;
            break;
        }
        case T_CHECK:
            by += size(v[0]);
            break;
        default:
            break;
        }
    }
    flops = fl;
    bytes = 8.0 * by;
}

int64_t critical_path(const Plan &P) {
    std::vector<int64_t> d(P.tasks.size(), 0);
    int64_t best = 0;
    for (size_t i = 0; i < P.tasks.size(); ++i) {
        int64_t l = 0;
        const DTask &t = P.tasks[i];
        for (int32_t k = 0; k < t.dep_cnt; ++k) l = std::max(l, d[P.deps[t.dep_beg + k]]);
        d[i] = l + (t.type == T_NOP ? 0 : 1);
        best = std::max(best, d[i]);
    }
    return best;
}

// ---------------------------------------------------------------------------
// entry points
// ---------------------------------------------------------------------------
std::shared_ptr<Plan> plan_hlu(HMat &F, double eps2, i64 &perm_len_out, PlanStream *stream) {
    auto t0 = std::chrono::steady_clock::now();
    refine_dense_leaves(F);
    Planner pl(F, nullptr);
    pl.eps2 = eps2;
    pl.stream = stream;
    pl.lu_block(F.root, "root");
    pl.finalize();
    perm_len_out = pl.perm_len;
    F.inv_len = pl.inv_len;
    pl.P->build_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return pl.P;
}

// forward (unit L with leaf pivots) + backward (U) substitution on a dense RHS (hops.py:424-432)
std::shared_ptr<Plan> plan_solve(HMat &F, i64 n, int nrhs_cap) {
    auto t0 = std::chrono::steady_clock::now();
    refine_dense_leaves(F);
    Planner pl(F, nullptr);
    Mref Fm{&F, B_F, 0};
    PView B{};
    pl.P->rhs_slot = pl.new_slot();
    B.d = DView{0, (int32_t)n, nrhs_cap, (int32_t)n, pl.P->rhs_slot, B_RHS, 0, 0};
    B.obj = pl.key(B_RHS, 0, 0);
    pl.solve_dense(Fm, F.root, B, 0, true, "root");
    pl.solve_dense(Fm, F.root, B, 1, false, "root");
    pl.finalize();
    pl.P->build_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return pl.P;
}

// T X = B for a dense right-hand side, one triangle of T (hops.py:282-310 trisolve_lower /
// trisolve_upper_right on dense B): mode 0 lower, 1 upper, 2 upper transposed
std::shared_ptr<Plan> plan_trisolve_dense(HMat &T, i64 n, int nrhs_cap, int mode, bool unit,
                                          const std::string &root) {
    auto t0 = std::chrono::steady_clock::now();
    refine_dense_leaves(T);
    Planner pl(T, nullptr);
    Mref Tm{&T, B_F, 0};
    PView B{};
    pl.P->rhs_slot = pl.new_slot();
    B.d = DView{0, (int32_t)n, nrhs_cap, (int32_t)n, pl.P->rhs_slot, B_RHS, 0, 0};
    B.obj = pl.key(B_RHS, 0, 0);
    pl.solve_dense(Tm, T.root, B, mode, unit, root);
    pl.finalize();
    pl.P->build_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return pl.P;
}

// hops.py:282-310 with an H-matrix right-hand side: X (a deep copy of B, same block tree as T's
// columns) <- T^{-1} X in place by the block recursion (_trisolve_block for mode 0 / 1,
// _trisolve_right_upper for mode 2: X U = B), low-rank targets recompressed at eps2
std::shared_ptr<Plan> plan_trisolve_block(HMat &T, HMat &X, int mode, bool unit, double eps2) {
    auto t0 = std::chrono::steady_clock::now();
    refine_dense_leaves(T);
    Planner pl(T, &X);
    pl.eps2 = eps2;
    Mref Tm{&T, B_F, 0};
    Mref Xm{&X, B_X, T.nslots};
    if (mode == 2) pl.trisolve_right_upper(Tm, T.root, Xm, X.root, "U");
    else pl.trisolve_left(Tm, T.root, Xm, X.root, mode, unit, mode == 0 ? "L" : "U");
    pl.finalize();
    pl.P->build_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return pl.P;
}

// X <- T^{-1} X with X initialised to the identity (lower: mode 0 unit L with pivots; upper: mode 1)
std::shared_ptr<Plan> plan_inverse(HMat &F, HMat &X, int mode, double eps2) {
    auto t0 = std::chrono::steady_clock::now();
    Planner pl(F, &X);
    pl.eps2 = eps2;
    Mref Fm{&F, B_F, 0};
    Mref Xm{&X, B_X, F.nslots};
    // identity initialisation of every stored leaf
    for (int32_t b : X.leafblocks) {
        const Node &nd = X.nodes[b];
        if (nd.kind == K_DENSE) {
            PView D = pl.dense_view(Xm, b);
            DTask t = mk(T_IDENT);
            t.flags = (nd.r0 == nd.c0 && nd.m == nd.n) ? 0 : 1;
            t.v[0] = D.d;
            pl.emit(t, {{&D, true}});
        }
    }
    pl.trisolve_left(Fm, F.root, Xm, X.root, mode, mode == 0, "root");
    pl.finalize();
    pl.P->build_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return pl.P;
}

// Z <- (L U)^{-1} on the full block structure of F: Z = I, then Z <- L^{-1} Z (unit L with
// leaf pivots) while the strict upper triangle of Z is still structurally zero, then
// Z <- U^{-1} Z on every block.  Same task vocabulary as plan_inverse; the CN step
// (A+)^{-1} A- = 2 (A+)^{-1} - I then costs one H-matvec of Z.
// With filt, only the columns [lo, hi) of Z are planned: column blocks of a left solve are
// independent, so they are planned on separate threads and merged into one DAG.
static std::shared_ptr<Plan> plan_propagator_part(HMat &F, HMat &Z, double eps2, bool filt,
                                                  i64 lo, i64 hi, int32_t seed0) {
    Planner pl(F, &Z);
    pl.eps2 = eps2;
    pl.filt = filt;
    pl.flo = lo;
    pl.fhi = hi;
    pl.rand_seed = seed0;
    Mref Fm{&F, B_F, 0};
    Mref Zm{&Z, B_X, F.nslots};
    auto in_range = [&](const Node &nd) { return !filt || (nd.c0 >= lo && nd.c0 + nd.n <= hi); };
    std::vector<std::pair<int32_t, int32_t>> upper;  // (block, stored kind) of strict-upper leaves
    for (int32_t b : Z.leafblocks) {
        Node &nd = Z.nodes[b];
        const bool diag = (nd.r0 == nd.c0 && nd.m == nd.n);
        if (!diag && nd.c0 >= nd.r0 + nd.m) {
            upper.push_back({b, nd.kind});
            nd.kind = K_ZERO;
            continue;
        }
        if (nd.kind == K_DENSE && in_range(nd)) {
            PView D = pl.dense_view(Zm, b);
            DTask t = mk(T_IDENT);
            t.flags = diag ? 0 : 1;
            t.v[0] = D.d;
            pl.emit(t, {{&D, true}});
        }
    }
    pl.trisolve_left(Fm, F.root, Zm, Z.root, 0, true, "root");
    for (auto &u : upper) {  // the upper triangle becomes live storage: zero dense, rank 0
        Node &nd = Z.nodes[u.first];
        nd.kind = u.second;
        if (nd.kind == K_DENSE && in_range(nd)) {
            PView D = pl.dense_view(Zm, u.first);
            DTask t = mk(T_IDENT);
            t.flags = 1;
            t.v[0] = D.d;
            pl.emit(t, {{&D, true}});
        }
    }
    pl.trisolve_left(Fm, F.root, Zm, Z.root, 1, false, "root");
    pl.finalize();
    return pl.P;
}

static void structure_copy(HMat &D, const HMat &S) {
    D.refined = S.refined;
    D.rt = S.rt;
    D.ct = S.ct;
    D.rt_hold = S.rt_hold;
    D.ct_hold = S.ct_hold;
    D.nrows = S.nrows;
    D.ncols = S.ncols;
    D.root = S.root;
    D.nodes = S.nodes;
    D.leafblocks = S.leafblocks;
    D.nslots = S.nslots;
    D.arena_len = S.arena_len;
}

// concatenation of independent DAGs: task, dependency, piece and path indices and the
// temp-pool offsets of each part are shifted past the previous parts (parts copied in
// parallel, each into its own slice)
std::shared_ptr<Plan> merge_plans(const std::vector<std::shared_ptr<Plan>> &parts) {
    auto M = std::make_shared<Plan>();
    const size_t np = parts.size();
    std::vector<size_t> t0(np + 1, 0), d0(np + 1, 0), p0(np + 1, 0), s0(np + 1, 0);
    std::vector<i64> toff(np + 1, 0);
    for (size_t k = 0; k < np; ++k) {
        t0[k + 1] = t0[k] + parts[k]->tasks.size();
        d0[k + 1] = d0[k] + parts[k]->deps.size();
        p0[k + 1] = p0[k] + parts[k]->pieces.size();
        s0[k + 1] = s0[k] + parts[k]->paths.size();
        toff[k + 1] = toff[k] + parts[k]->temp_len;
        M->nslots_total = std::max(M->nslots_total, parts[k]->nslots_total);
    }
    M->tasks.resize(t0[np]);
    M->deps.resize(d0[np]);
    M->pieces.resize(p0[np]);
    M->slot_off_x = parts[0]->slot_off_x;
    M->slot_off_tmp = parts[0]->slot_off_tmp;
    M->temp_len = toff[np];
    std::vector<std::future<void>> fut;
    for (size_t k = 0; k < np; ++k)
        fut.push_back(std::async(std::launch::async, [&, k] {
            const Plan &p = *parts[k];
            const i64 to = toff[k];
            auto fix = [&](DView &v) {
                if (v.base == B_TMP) v.off += to;
            };
            DTask *T = M->tasks.data() + t0[k];
            for (size_t i = 0; i < p.tasks.size(); ++i) {
                DTask t = p.tasks[i];
                t.dep_beg += (int32_t)d0[k];
                t.pc_beg += (int32_t)p0[k];
                t.pc_end += (int32_t)p0[k];
                if (t.path >= 0) t.path += (int32_t)s0[k];
                for (auto &v : t.v) fix(v);
                T[i] = t;
            }
            int32_t *D = M->deps.data() + d0[k];
            for (size_t i = 0; i < p.deps.size(); ++i) D[i] = p.deps[i] + (int32_t)t0[k];
            DPiece *Pc = M->pieces.data() + p0[k];
            for (size_t i = 0; i < p.pieces.size(); ++i) {
                DPiece pc = p.pieces[i];
                fix(pc.mat);
                fix(pc.x);
                Pc[i] = pc;
            }
        }));
    for (auto &p : parts) M->paths.insert(M->paths.end(), p->paths.begin(), p->paths.end());
    for (auto &f : fut) f.get();
    return M;
}

// column ranges of the column clusters `depth` levels below the root (fewer when a leaf
// cluster is reached first)
static std::vector<std::pair<i64, i64>> column_blocks(const Tree &T, int depth) {
    std::vector<int32_t> cur{0};
    for (int d = 0; d < depth; ++d) {
        std::vector<int32_t> nxt;
        for (int32_t c : cur) {
            if (T.nodes[c].leaf()) return {};
            nxt.push_back(T.nodes[c].kid[0]);
            nxt.push_back(T.nodes[c].kid[1]);
        }
        cur.swap(nxt);
    }
    std::vector<std::pair<i64, i64>> out;
    for (int32_t c : cur) out.push_back({T.nodes[c].lo, T.nodes[c].lo + T.nodes[c].size()});
    return out;
}

double plan_device_bytes(const Plan &P) {
    return (double)P.tasks.size() * (sizeof(DTask) + 24) + (double)P.deps.size() * 8 +
           (double)P.pieces.size() * sizeof(DPiece) + (double)P.temp_len * 8;
}

std::shared_ptr<Plan> plan_propagator(HMat &F, HMat &Z, double eps2, int max_parts,
                                      std::vector<std::shared_ptr<Plan>> *keep_parts) {
    auto t0 = std::chrono::steady_clock::now();
    std::shared_ptr<Plan> P;
    if (const char *e = getenv("LEVYH_PROP_PARTS")) max_parts = atoi(e);
    int depth = 0, parts = 1;
    while ((2 << depth) <= max_parts) ++depth;
    // a split `depth` levels down is clean iff no leaf block sits above that depth: then
    // every leaf, and every product update of a leaf, lies inside one column block
    std::vector<std::pair<int32_t, int>> st{{Z.root, 0}};
    while (!st.empty() && depth > 0) {
        auto [b, d] = st.back();
        st.pop_back();
        const Node &nd = Z.nodes[b];
        if (nd.kind != K_HIER) {
            depth = std::min(depth, d);
            continue;
        }
        if (d + 1 >= depth) continue;
        for (int q = 0; q < 4; ++q) st.push_back({nd.kid[q], d + 1});
    }
    auto cols = depth > 0 ? column_blocks(*Z.ct, depth) : std::vector<std::pair<i64, i64>>{};
    // large operators: the column parts run one after another, each into a scratch buffer of its
    // own extent (prepare_propagator compacts each part as it finishes), so Z is laid out with
    // every part's blocks contiguous
    const double parts_gb = getenv("LEVYH_PROP_PARTS_GB") ? atof(getenv("LEVYH_PROP_PARTS_GB")) : 40.0;
    const bool parts_mode = keep_parts && cols.size() >= 2 && 8e-9 * (double)Z.arena_len > parts_gb;
    std::vector<i64> part_off;
    if (parts_mode) {
        part_off.assign(cols.size() + 1, 0);
        i64 off = 0;
        for (size_t k = 0; k < cols.size(); ++k) {
            part_off[k] = off;
            for (int32_t b : Z.leafblocks) {
                Node &nd = Z.nodes[b];
                if (nd.c0 < cols[k].first || nd.c0 >= cols[k].second) continue;
                LH_REQUIRE(nd.c0 + nd.n <= cols[k].second, LH_EINTERNAL, "propagator part split crosses a leaf");
                if (nd.kind == K_DENSE) {
                    nd.doff = off;
                    off += nd.m * nd.n;
                } else if (nd.kind == K_LR) {
                    nd.uoff = off;
                    off += nd.m * nd.kcap;
                    nd.voff = off;
                    off += nd.n * nd.kcap;
                }
            }
        }
        part_off[cols.size()] = off;
        LH_REQUIRE(off == Z.arena_len, LH_EINTERNAL, "propagator part layout lost blocks");
    }
    if (cols.size() >= 2) {
        std::vector<HMat> Zs(cols.size());
        std::vector<std::future<std::shared_ptr<Plan>>> fut;
        for (size_t k = 0; k < cols.size(); ++k) {
            structure_copy(Zs[k], Z);
            fut.push_back(std::async(std::launch::async, [&, k] {
                auto ts = std::chrono::steady_clock::now();
                auto r = plan_propagator_part(F, Zs[k], eps2, true, cols[k].first, cols[k].second,
                                              1 + (int32_t)k * (1 << 24));
                if (getenv("LEVYH_PLAN_VERBOSE"))
                    fprintf(stderr, "[levyh]   part %zu: %zu tasks %.3f s\n", k, r->tasks.size(),
                            std::chrono::duration<double>(std::chrono::steady_clock::now() - ts).count());
                return r;
            }));
        }
        std::vector<std::shared_ptr<Plan>> parts_v;
        bool ok = true;
        for (auto &f : fut) {
            try {
                parts_v.push_back(f.get());
            } catch (const std::exception &) {
                ok = false;  // defensive: the split check above should make this unreachable
            }
        }
        if (ok && parts_mode) {
            size_t nt = 0;
            double dev_bytes = 0.0;
            for (size_t k = 0; k < parts_v.size(); ++k) {
                auto &q = parts_v[k];
                nt += q->tasks.size();
                dev_bytes = std::max(dev_bytes, plan_device_bytes(*q));
                q->build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                q->x_base = part_off[k];
                q->x_len = part_off[k + 1] - part_off[k];
            }
            if (getenv("LEVYH_PLAN_VERBOSE"))
                fprintf(stderr, "[levyh] propagator plan: %zu tasks in %zu column parts run one by one (largest "
                                "part %.1f GB on the device, Z arena %.1f GB), %.3f s\n",
                        nt, parts_v.size(), dev_bytes * 1e-9, 8e-9 * (double)Z.arena_len, parts_v[0]->build_seconds);
            *keep_parts = std::move(parts_v);
            return nullptr;
        }
        if (ok) {
            auto tm = std::chrono::steady_clock::now();
            P = merge_plans(parts_v);
            parts = (int)parts_v.size();
            if (getenv("LEVYH_PLAN_VERBOSE"))
                fprintf(stderr, "[levyh]   merge %.3f s\n",
                        std::chrono::duration<double>(std::chrono::steady_clock::now() - tm).count());
        }
    }
    if (!P) P = plan_propagator_part(F, Z, eps2, false, 0, 0, 1);
    P->build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (getenv("LEVYH_PLAN_VERBOSE"))
        fprintf(stderr, "[levyh] propagator plan: %zu tasks, %d column parts, %.3f s\n",
                P->tasks.size(), parts, P->build_seconds);
    return P;
}

// the diagonal-leaf bookkeeping lu_block does while planning (pivot and packed-inverse
// offsets in recursion order, kind K_FDENSE), without planning: lets every plan that
// reads the factor start before the H-LU plan exists
static void mark_rec(HMat &F, int32_t b, i64 &perm_len, i64 &inv_len) {
    Node &nd = F.nodes[b];
    if (dense_leaf(nd)) {
        nd.poff = perm_len;
        perm_len += nd.m;
        if (nd.m <= LEAF_INV_MAX) {
            nd.ioff = inv_len;
            inv_len += nd.m * nd.m;
        }
        nd.kind = K_FDENSE;
        return;
    }
    LH_REQUIRE(hier(nd), LH_ETYPE, "cannot LU-factorize a low-rank diagonal block");
    mark_rec(F, nd.kid[0], perm_len, inv_len);
    mark_rec(F, nd.kid[3], perm_len, inv_len);
    if (nd.kind != K_HIER) {  // refined leaf (see lu_block)
        nd.kind = K_FDENSE;
        nd.poff = F.nodes[nd.kid[0]].poff;
        nd.ioff = -1;
    }
}

void mark_lu_leaves(HMat &F, i64 &perm_len, i64 &inv_len) {
    refine_dense_leaves(F);
    perm_len = inv_len = 0;
    mark_rec(F, F.root, perm_len, inv_len);
    F.inv_len = inv_len;
    F.perm_len = perm_len;
}

}  // namespace lh
