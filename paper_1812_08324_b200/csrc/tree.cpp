// Cluster tree and block partition (host).  Bit-exact restatement of
// geometry.py:142-263 (median bisection, bbox admissibility) and of the
// decision order of hmatrix.py:306-340 (build_from_dense).
#include <algorithm>
#include <cmath>
#include <numeric>

#include "core.h"

namespace lh {

double diameter(const Cluster &a, int dim) {
    // geometry.py:89-91  float(np.linalg.norm(bbox_hi - bbox_lo))
    double s = 0.0;
    for (int d = 0; d < dim; ++d) {
        double v = a.bhi[d] - a.blo[d];
        s += v * v;
    }
    return std::sqrt(s);
}

bool admissible(const Cluster &a, const Cluster &b, int dim, double eta) {
    // geometry.py:246-263
    double s = 0.0;
    for (int d = 0; d < dim; ++d) {
        double g = std::max(a.blo[d] - b.bhi[d], b.blo[d] - a.bhi[d]);
        g = std::max(g, 0.0);
        s += g * g;
    }
    double dist = std::sqrt(s);
    if (dist <= 0.0) return false;
    return std::min(diameter(a, dim), diameter(b, dim)) <= eta * dist;
}

namespace {

struct TreeBuilder {
    const double *pts;
    int dim, leaf_size;
    Tree *T;
    std::vector<i64> tmp;
    std::vector<double> key;
    int strategy = 0;  // 0 bisection, 1 kmeans2

    // _split_kmeans2 (geometry.py:157-188): deterministic 2-means, centroids seeded with the
    // extremes of the projection onto the bbox diagonal (first index on ties), assignment ties
    // to centroid 0, at most 50 iterations, even index split when a cluster empties or every
    // point coincides.  Same floating-point operations as numpy: squared distances summed x
    // then y, centroids as sequential sums over the members in index order / count.
    // Returns the cluster-0 (left) mask over idx[b, e).
    std::vector<char> kmeans2(const std::vector<i64> &idx, i64 b, i64 e, const Cluster &c) const {
        const i64 n = e - b;
        std::vector<char> left(n, 0);
        double diag[2] = {0, 0};
        bool any = false;
        for (int d = 0; d < dim; ++d) {
            diag[d] = c.bhi[d] - c.blo[d];
            any = any || diag[d] > 0;
        }
        auto even = [&]() {
            std::fill(left.begin(), left.end(), 0);
            for (i64 k = 0; k < n / 2; ++k) left[k] = 1;
            return left;
        };
        if (!any) return even();
        auto P = [&](i64 k, int d) { return pts[idx[b + k] * dim + d]; };
        i64 amin = 0, amax = 0;
        double pmin = 0, pmax = 0;
        for (i64 k = 0; k < n; ++k) {
            double pr = 0.0;
            for (int d = 0; d < dim; ++d) pr += P(k, d) * diag[d];
            if (k == 0 || pr < pmin) pmin = pr, amin = k;
            if (k == 0 || pr > pmax) pmax = pr, amax = k;
        }
        double cen[2][2];
        for (int d = 0; d < dim; ++d) {
            cen[0][d] = P(amin, d);
            cen[1][d] = P(amax, d);
        }
        std::vector<char> assign(n, 0), na(n, 0);
        bool have = false;
        for (int it = 0; it < 50; ++it) {
            for (i64 k = 0; k < n; ++k) {
                double d0 = 0.0, d1 = 0.0;
                for (int d = 0; d < dim; ++d) {
                    const double a0 = P(k, d) - cen[0][d], a1 = P(k, d) - cen[1][d];
                    d0 = d0 + a0 * a0;
                    d1 = d1 + a1 * a1;
                }
                na[k] = d1 < d0;
            }
            if (have && na == assign) break;
            assign = na;
            have = true;
            i64 n1 = 0;
            for (char v : assign) n1 += v;
            if (n1 == 0 || n1 == n) return even();
            double s[2][2] = {{0, 0}, {0, 0}};
            for (i64 k = 0; k < n; ++k)
                for (int d = 0; d < dim; ++d) s[assign[k]][d] = s[assign[k]][d] + P(k, d);
            for (int d = 0; d < dim; ++d) {
                cen[0][d] = s[0][d] / (double)(n - n1);
                cen[1][d] = s[1][d] / (double)n1;
            }
        }
        for (i64 k = 0; k < n; ++k) left[k] = !assign[k];
        return left;
    }

    int32_t build(std::vector<i64> &idx, i64 b, i64 e, i64 start, int depth) {
        // geometry.py:225-236; idx[b:e] are original point ids of this node
        Cluster c;
        c.lo = start;
        c.hi = start + (e - b);
        c.depth = depth;
        c.kid[0] = c.kid[1] = -1;
        for (int d = 0; d < 2; ++d) c.blo[d] = c.bhi[d] = 0.0;
        for (int d = 0; d < dim; ++d) {
            double lo = pts[idx[b] * dim + d], hi = lo;
            for (i64 k = b + 1; k < e; ++k) {
                double v = pts[idx[k] * dim + d];
                lo = std::min(lo, v);  // numpy min/max ignore order for finite data
                hi = std::max(hi, v);
            }
            c.blo[d] = lo;
            c.bhi[d] = hi;
        }
        int32_t id = (int32_t)T->nodes.size();
        T->nodes.push_back(c);
        i64 n = e - b;
        if (n <= leaf_size) {
            for (i64 k = b; k < e; ++k) T->order[start + (k - b)] = idx[k];
            T->leaves.push_back(id);
            return id;
        }
        if (strategy == 1) {
            const std::vector<char> left = kmeans2(idx, b, e, c);
            std::vector<i64> L, R;
            for (i64 k = 0; k < n; ++k) (left[k] ? L : R).push_back(idx[b + k]);
            const i64 nl = (i64)L.size();
            std::copy(L.begin(), L.end(), idx.begin() + b);
            std::copy(R.begin(), R.end(), idx.begin() + b + nl);
            int32_t k0 = build(idx, b, b + nl, start, depth + 1);
            int32_t k1 = build(idx, b + nl, e, start + nl, depth + 1);
            T->nodes[id].kid[0] = k0;
            T->nodes[id].kid[1] = k1;
            return id;
        }
        // _split_bisection (geometry.py:146-154): widest axis (first on ties),
        // stable argsort, first n//2 of the sorted order go left; the left child keeps
        // the original relative order of its members (idx[mask]).
        int axis = 0;
        double best = c.bhi[0] - c.blo[0];
        for (int d = 1; d < dim; ++d) {
            double w = c.bhi[d] - c.blo[d];
            if (w > best) { best = w; axis = d; }
        }
        bool sorted = true;
        for (i64 k = b + 1; k < e && sorted; ++k)
            sorted = pts[idx[k - 1] * dim + axis] <= pts[idx[k] * dim + axis];
        i64 half = n / 2;
        if (!sorted) {
            std::vector<i64> ord(n);
            std::iota(ord.begin(), ord.end(), (i64)0);
            std::stable_sort(ord.begin(), ord.end(), [&](i64 p, i64 q) {
                return pts[idx[b + p] * dim + axis] < pts[idx[b + q] * dim + axis];
            });
            std::vector<char> left(n, 0);
            for (i64 k = 0; k < half; ++k) left[ord[k]] = 1;
            std::vector<i64> L, R;
            L.reserve(half);
            R.reserve(n - half);
            for (i64 k = 0; k < n; ++k) (left[k] ? L : R).push_back(idx[b + k]);
            std::copy(L.begin(), L.end(), idx.begin() + b);
            std::copy(R.begin(), R.end(), idx.begin() + b + half);
        }
        int32_t k0 = build(idx, b, b + half, start, depth + 1);
        int32_t k1 = build(idx, b + half, e, start + half, depth + 1);
        T->nodes[id].kid[0] = k0;
        T->nodes[id].kid[1] = k1;
        return id;
    }
};

}  // namespace

Tree *build_tree(const double *pts, i64 n, int dim, int leaf_size, int strategy) {
    LH_REQUIRE(n > 0, LH_EINVAL, "point set must be nonempty");
    LH_REQUIRE(dim == 1 || dim == 2, LH_EINVAL, "only 1D and 2D point sets are supported");
    LH_REQUIRE(leaf_size >= 1, LH_EINVAL, "leaf_size must be >= 1");
    for (i64 k = 0; k < n * dim; ++k)
        LH_REQUIRE(std::isfinite(pts[k]), LH_EINVAL, "points must have finite coordinates");
    Tree *T = new Tree();
    T->dim = dim;
    T->n = n;
    T->leaf_size = leaf_size;
    T->pts.assign(pts, pts + n * dim);
    T->order.assign(n, 0);
    std::vector<i64> idx(n);
    std::iota(idx.begin(), idx.end(), (i64)0);
    LH_REQUIRE(strategy == 0 || strategy == 1, LH_EINVAL, "unknown strategy");
    TreeBuilder tb{pts, dim, leaf_size, T, {}, {}, strategy};
    tb.build(idx, 0, n, 0, 0);
    return T;
}

// ---------------------------------------------------------------------------
// partition (hmatrix.py:319-337)
// ---------------------------------------------------------------------------
namespace {
struct Partitioner {
    HMat &H;
    const Tree &rt, &ct;
    int n_min;
    double eta;
    i64 nmax;
    int32_t rec(int32_t r, int32_t c, int depth) {
        const Cluster &R = rt.nodes[r];
        const Cluster &C = ct.nodes[c];
        i64 m = R.size(), n = C.size();
        Node nd{};
        nd.rcl = r;
        nd.ccl = c;
        nd.r0 = R.lo;
        nd.c0 = C.lo;
        nd.m = m;
        nd.n = n;
        nd.depth = depth;
        nd.kid[0] = nd.kid[1] = nd.kid[2] = nd.kid[3] = -1;
        nd.rslot = -1;
        nd.doff = nd.uoff = nd.voff = nd.poff = -1;
        bool can_split = !R.leaf() && !C.leaf();
        bool hier = false;
        if ((m > nmax || n > nmax) && can_split) {
            hier = true;  // forced subdivision
        } else if (admissible(R, C, rt.dim, eta) && std::min(m, n) > n_min) {
            nd.kind = K_LR;
        } else if (std::min(m, n) <= n_min || !can_split) {
            nd.kind = K_DENSE;
        } else {
            hier = true;
        }
        int32_t id = (int32_t)H.nodes.size();
        H.nodes.push_back(nd);
        if (hier) {
            int32_t a = rec(R.kid[0], C.kid[0], depth + 1);
            int32_t b = rec(R.kid[0], C.kid[1], depth + 1);
            int32_t cc = rec(R.kid[1], C.kid[0], depth + 1);
            int32_t d = rec(R.kid[1], C.kid[1], depth + 1);
            Node &me = H.nodes[id];
            me.kind = K_HIER;
            me.kid[0] = a;
            me.kid[1] = b;
            me.kid[2] = cc;
            me.kid[3] = d;
            me.rs = rt.nodes[R.kid[0]].size();
            me.cs = ct.nodes[C.kid[0]].size();
        }
        return id;
    }
};
}  // namespace

void walk_leaves(HMat &H) {
    H.leafblocks.clear();
    std::vector<int32_t> st{H.root};
    while (!st.empty()) {
        int32_t b = st.back();
        st.pop_back();
        const Node &nd = H.nodes[b];
        if (nd.kind == K_HIER) {
            for (int k = 3; k >= 0; --k) st.push_back(nd.kid[k]);
        } else {
            H.leafblocks.push_back(b);
        }
    }
}

void partition(HMat &H, const Tree &rt, const Tree &ct, int n_min, int n_block, double eta) {
    LH_REQUIRE(n_block >= 2, LH_EINVAL, "n_block must be >= 2");
    H.rt = &rt;
    H.ct = &ct;
    H.nrows = rt.n;
    H.ncols = ct.n;
    H.nodes.clear();
    i64 mx = std::max(rt.n, ct.n);
    i64 nmax = (mx + n_block - 1) / n_block;  // math.ceil(max/n_block)
    Partitioner p{H, rt, ct, n_min, eta, nmax};
    H.root = p.rec(0, 0, 0);
    walk_leaves(H);
}

}  // namespace lh
