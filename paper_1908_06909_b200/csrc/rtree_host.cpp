// rtree_host.cpp -- the paper's R*-tree over the hull faces (NEXT-3).
//
// "an R*-tree is precomputed for the boundary elements in a pre-processing
// step ... We have chosen 10 as maximum number elements and 4 as minimum"
// (§2.5).  Built here by R*-tree insertion (Beckmann et
// al. 1990): ChooseSubtree by least overlap enlargement above the leaves and
// least volume enlargement higher up, forced reinsertion of the 30 % entries
// farthest from a node's centre on its level's first overflow per inserted
// face, and the margin / overlap split.  Flattened for the GPU's depth-first
// search (kernels.cu entry_rtree_kernel): node = [count, leaf, child[10],
// lo[10][3], hi[10][3]] as 72 int32 words; leaf children index bvh_faces.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "internal.h"

namespace tetproj {

namespace {

constexpr int kMaxFan = 10, kMinFan = 4, kReinsert = 3;   // 30 % of M + 1

struct Box {
    float lo[3], hi[3];
};

struct RStar {
    struct Node {
        int level;                 // 0 = leaf (children are faces)
        std::vector<int> ch;
        std::vector<Box> bx;
    };
    std::vector<Node> nodes;
    int root = 0;
    double pad = 0;                // flat boxes (faces in a coordinate plane) get volume
    std::vector<char> reinserted;  // per level, for the face being inserted
    struct Pending {
        int entry;
        Box b;
        int level;
    };
    std::vector<Pending> pending;

    static Box join(const Box& a, const Box& b) {
        Box r;
        for (int i = 0; i < 3; ++i) {
            r.lo[i] = std::min(a.lo[i], b.lo[i]);
            r.hi[i] = std::max(a.hi[i], b.hi[i]);
        }
        return r;
    }
    double vol(const Box& b) const {
        double v = 1;
        for (int i = 0; i < 3; ++i) v *= (double)b.hi[i] - b.lo[i] + pad;
        return v;
    }
    static double margin(const Box& b) {
        double m = 0;
        for (int i = 0; i < 3; ++i) m += (double)b.hi[i] - b.lo[i];
        return m;
    }
    double overlap(const Box& a, const Box& b) const {
        double v = 1;
        for (int i = 0; i < 3; ++i) {
            const double lo = std::max(a.lo[i], b.lo[i]), hi = std::min(a.hi[i], b.hi[i]);
            if (hi < lo) return 0;
            v *= hi - lo + pad;
        }
        return v;
    }
    Box cover(int nid) const {
        const Node& n = nodes[nid];
        Box r = n.bx[0];
        for (size_t i = 1; i < n.bx.size(); ++i) r = join(r, n.bx[i]);
        return r;
    }

    int choose(int nid, const Box& b) const {
        const Node& n = nodes[nid];
        const int c = (int)n.ch.size();
        int best = 0;
        double b1 = INFINITY, b2 = INFINITY, b3 = INFINITY;
        for (int i = 0; i < c; ++i) {
            const Box e = join(n.bx[i], b);
            const double enl = vol(e) - vol(n.bx[i]);
            double ov = 0;
            if (n.level == 1)   // children are leaves: least overlap enlargement
                for (int j = 0; j < c; ++j)
                    if (j != i) ov += overlap(e, n.bx[j]) - overlap(n.bx[i], n.bx[j]);
            const double a = vol(n.bx[i]);
            if (ov < b1 || (ov == b1 && (enl < b2 || (enl == b2 && a < b3)))) {
                b1 = ov;
                b2 = enl;
                b3 = a;
                best = i;
            }
        }
        return best;
    }

    int split(int nid) {
        Node& n = nodes[nid];
        const int E = (int)n.ch.size();
        std::vector<int> idx(E);
        auto sorted = [&](int axis, bool by_hi) {
            std::vector<int> o(E);
            for (int i = 0; i < E; ++i) o[i] = i;
            std::stable_sort(o.begin(), o.end(), [&](int a, int b) {
                const float va = by_hi ? n.bx[a].hi[axis] : n.bx[a].lo[axis];
                const float vb = by_hi ? n.bx[b].hi[axis] : n.bx[b].lo[axis];
                return va < vb;
            });
            return o;
        };
        auto group_box = [&](const std::vector<int>& o, int from, int to) {
            Box r = n.bx[o[from]];
            for (int i = from + 1; i < to; ++i) r = join(r, n.bx[o[i]]);
            return r;
        };
        // ChooseSplitAxis: least sum of margins over all distributions
        int axis = 0;
        double best_s = INFINITY;
        for (int a = 0; a < 3; ++a) {
            double s = 0;
            for (int h = 0; h < 2; ++h) {
                const std::vector<int> o = sorted(a, h == 1);
                for (int k = kMinFan; k <= E - kMinFan; ++k)
                    s += margin(group_box(o, 0, k)) + margin(group_box(o, k, E));
            }
            if (s < best_s) { best_s = s; axis = a; }
        }
        // ChooseSplitIndex: least overlap, then least volume
        std::vector<int> best_o;
        int best_k = kMinFan;
        double bo = INFINITY, bv = INFINITY;
        for (int h = 0; h < 2; ++h) {
            const std::vector<int> o = sorted(axis, h == 1);
            for (int k = kMinFan; k <= E - kMinFan; ++k) {
                const Box g1 = group_box(o, 0, k), g2 = group_box(o, k, E);
                const double ov = overlap(g1, g2), v = vol(g1) + vol(g2);
                if (ov < bo || (ov == bo && v < bv)) {
                    bo = ov;
                    bv = v;
                    best_o = o;
                    best_k = k;
                }
            }
        }
        Node sib;
        sib.level = n.level;
        std::vector<int> ch1;
        std::vector<Box> bx1;
        for (int i = 0; i < E; ++i) {
            const int s = best_o[i];
            if (i < best_k) { ch1.push_back(n.ch[s]); bx1.push_back(n.bx[s]); }
            else { sib.ch.push_back(n.ch[s]); sib.bx.push_back(n.bx[s]); }
        }
        n.ch.swap(ch1);
        n.bx.swap(bx1);
        nodes.push_back(sib);   // invalidates n
        return (int)nodes.size() - 1;
    }

    void reinsert(int nid) {
        const Box c = cover(nid);
        double cc[3];
        for (int i = 0; i < 3; ++i) cc[i] = 0.5 * ((double)c.lo[i] + c.hi[i]);
        Node& n = nodes[nid];
        const int E = (int)n.ch.size();
        std::vector<std::pair<double, int>> d(E);
        for (int i = 0; i < E; ++i) {
            double s = 0;
            for (int a = 0; a < 3; ++a) {
                const double x = 0.5 * ((double)n.bx[i].lo[a] + n.bx[i].hi[a]) - cc[a];
                s += x * x;
            }
            d[i] = {s, i};
        }
        std::sort(d.begin(), d.end());   // ascending: the last kReinsert are the farthest
        std::vector<int> ch;
        std::vector<Box> bx;
        for (int i = 0; i < E - kReinsert; ++i) {
            ch.push_back(n.ch[d[i].second]);
            bx.push_back(n.bx[d[i].second]);
        }
        for (int i = E - kReinsert; i < E; ++i)   // close reinsert: nearest of them first
            pending.push_back({n.ch[d[i].second], n.bx[d[i].second], n.level});
        n.ch.swap(ch);
        n.bx.swap(bx);
    }

    // insert below nid; returns a new sibling of nid after a split, else -1
    int insert_at(int nid, int entry, const Box& b, int level) {
        if (nodes[nid].level == level) {
            nodes[nid].ch.push_back(entry);
            nodes[nid].bx.push_back(b);
        } else {
            const int i = choose(nid, b);
            const int child = nodes[nid].ch[i];
            const int sib = insert_at(child, entry, b, level);
            nodes[nid].bx[i] = cover(child);
            if (sib >= 0) {
                const Box sb = cover(sib);
                nodes[nid].ch.push_back(sib);
                nodes[nid].bx.push_back(sb);
            }
        }
        if ((int)nodes[nid].ch.size() <= kMaxFan) return -1;
        const int L = nodes[nid].level;
        if (nid != root && !reinserted[L]) {   // OverflowTreatment
            reinserted[L] = 1;
            reinsert(nid);
            return -1;
        }
        return split(nid);
    }

    void insert_one(int entry, const Box& b, int level) {
        const int sib = insert_at(root, entry, b, level);
        if (sib >= 0) {
            Node r;
            r.level = nodes[root].level + 1;
            const Box b0 = cover(root), b1 = cover(sib);
            r.ch = {root, sib};
            r.bx = {b0, b1};
            nodes.push_back(r);
            root = (int)nodes.size() - 1;
            reinserted.resize(nodes[root].level + 1, 0);
        }
    }

    void insert(int face, const Box& b) {
        std::fill(reinserted.begin(), reinserted.end(), 0);
        insert_one(face, b, 0);
        while (!pending.empty()) {   // same data rectangle: flags stay set
            const Pending p = pending.front();
            pending.erase(pending.begin());
            insert_one(p.entry, p.b, p.level);
        }
    }
};

}  // namespace

void build_hull_rtree(HostMesh& M) {
    const int64_t B = (int64_t)M.bvh_faces.size() / 4;
    M.rtree_nodes.clear();
    if (B == 0) return;
    // face boxes from the BVH's face records (same face order, float rounded outward)
    std::vector<Box> fb(B);
    double span = 0;
    for (int64_t h = 0; h < B; ++h) {
        for (int i = 0; i < 3; ++i) {
            float lo = INFINITY, hi = -INFINITY;
            for (int j = 0; j < 3; ++j) {
                const float x = (float)M.vtx[4 * (size_t)M.bvh_faces[4 * h + j] + i];
                lo = std::min(lo, x);
                hi = std::max(hi, x);
            }
            fb[h].lo[i] = std::nextafter(lo, -INFINITY);
            fb[h].hi[i] = std::nextafter(hi, INFINITY);
            span = std::max(span, (double)std::fabs(lo) + std::fabs(hi));
        }
    }
    RStar t;
    t.pad = 1e-3 * span;
    t.nodes.push_back(RStar::Node{0, {}, {}});
    t.root = 0;
    t.reinserted.assign(1, 0);
    for (int64_t h = 0; h < B; ++h) t.insert((int)h, fb[h]);
    // flatten depth-first (root = node 0)
    std::vector<int> order, flat(t.nodes.size(), -1);
    std::vector<int> st = {t.root};
    while (!st.empty()) {
        const int n = st.back();
        st.pop_back();
        flat[n] = (int)order.size();
        order.push_back(n);
        if (t.nodes[n].level > 0)
            for (int i = (int)t.nodes[n].ch.size() - 1; i >= 0; --i) st.push_back(t.nodes[n].ch[i]);
    }
    M.rtree_nodes.assign(order.size() * 72, 0);
    for (size_t f = 0; f < order.size(); ++f) {
        const RStar::Node& n = t.nodes[order[f]];
        int32_t* w = &M.rtree_nodes[72 * f];
        w[0] = (int32_t)n.ch.size();
        w[1] = n.level == 0 ? 1 : 0;
        float* lo = reinterpret_cast<float*>(w + 12);
        float* hi = reinterpret_cast<float*>(w + 42);
        for (size_t i = 0; i < n.ch.size(); ++i) {
            w[2 + i] = n.level == 0 ? n.ch[i] : flat[n.ch[i]];
            for (int a = 0; a < 3; ++a) {
                lo[3 * i + a] = n.bx[i].lo[a];
                hi[3 * i + a] = n.bx[i].hi[a];
            }
        }
    }
}

}  // namespace tetproj
