// mesh_host.cpp -- host-side mesh preparation for libtetproj:
// grid snap, exact validation, orientation fix, convexity, Morton reorder and
// packing into the device layout.  Not timed ("precomputed ...
// in a pre-processing step").
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <climits>
#include <cstring>
#include <numeric>
#include <unordered_map>

#include "internal.h"

namespace tetproj {
namespace {

typedef __int128 i128;

// Face k of a positively oriented tet lists the nodes opposite node k with its
// normal (b-a)x(c-a) pointing out of the tet.
const int kFace[4][3] = {{1, 2, 3}, {0, 3, 2}, {0, 1, 3}, {0, 2, 1}};

int grid_exponent(double r) {
    int k;
    double m = std::frexp(64.0 * r, &k);
    return ((m == 0.5) ? k - 1 : k) - 30;  // ceil(log2(64 r)) - 30
}

bool snap(double x, double C, double g, long long& out) {
    double q = std::nearbyint((x - C) / g);
    if (!(std::fabs(q) <= 2147483647.0)) return false;
    out = (long long)q;
    return true;
}

// sign of det[b-a, c-a, d-a]: float filter, exact int128 when unsure.
int orient_filtered(const int32_t* a, const int32_t* b, const int32_t* c, const int32_t* d) {
    double e1[3], e2[3], e3[3];
    for (int i = 0; i < 3; ++i) {
        e1[i] = (double)b[i] - a[i];
        e2[i] = (double)c[i] - a[i];
        e3[i] = (double)d[i] - a[i];
    }
    // e1 x e2 is exact in double (|e| < 2^26 -> products < 2^52)
    double n0 = e1[1] * e2[2] - e1[2] * e2[1];
    double n1 = e1[2] * e2[0] - e1[0] * e2[2];
    double n2 = e1[0] * e2[1] - e1[1] * e2[0];
    double v = n0 * e3[0] + n1 * e3[1] + n2 * e3[2];
    double bound = 1e-14 * (std::fabs(n0 * e3[0]) + std::fabs(n1 * e3[1]) + std::fabs(n2 * e3[2]));
    if (v > bound) return 1;
    if (v < -bound) return -1;
    i128 E1[3], E2[3], E3[3];
    for (int i = 0; i < 3; ++i) {
        E1[i] = (i128)b[i] - a[i];
        E2[i] = (i128)c[i] - a[i];
        E3[i] = (i128)d[i] - a[i];
    }
    i128 N0 = E1[1] * E2[2] - E1[2] * E2[1];
    i128 N1 = E1[2] * E2[0] - E1[0] * E2[2];
    i128 N2 = E1[0] * E2[1] - E1[1] * E2[0];
    i128 w = N0 * E3[0] + N1 * E3[1] + N2 * E3[2];
    return (w > 0) - (w < 0);
}

uint64_t spread21(uint64_t x) {
    x &= 0x1fffff;
    x = (x | x << 32) & 0x1f00000000ffffULL;
    x = (x | x << 16) & 0x1f0000ff0000ffULL;
    x = (x | x << 8) & 0x100f00f00f00f00fULL;
    x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
    x = (x | x << 2) & 0x1249249249249249ULL;
    return x;
}

// Hilbert index of a point with 21-bit coordinates (Skilling's transpose
// algorithm, 3 dimensions): consecutive indices are face-adjacent cells, a
// tighter locality than the Morton order's jumps (TETPROJ_SFC=hilbert).
uint64_t hilbert21(uint32_t x0, uint32_t x1, uint32_t x2) {
    uint32_t X[3] = {x0 & 0x1fffff, x1 & 0x1fffff, x2 & 0x1fffff};
    const uint32_t M = 1u << 20;
    for (uint32_t Q = M; Q > 1; Q >>= 1) {   // inverse undo of excess work
        const uint32_t P = Q - 1;
        for (int i = 0; i < 3; ++i) {
            if (X[i] & Q) {
                X[0] ^= P;
            } else {
                const uint32_t t = (X[0] ^ X[i]) & P;
                X[0] ^= t;
                X[i] ^= t;
            }
        }
    }
    X[1] ^= X[0];                             // Gray encode
    X[2] ^= X[1];
    uint32_t t = 0;
    for (uint32_t Q = M; Q > 1; Q >>= 1)
        if (X[2] & Q) t ^= Q - 1;
    for (int i = 0; i < 3; ++i) X[i] ^= t;
    // interleave the transposed bits, X[0] most significant per level
    return (spread21(X[0]) << 2) | (spread21(X[1]) << 1) | spread21(X[2]);
}

// BVH over the hull faces for the per-ray entry finder (TET_ENTRY_BVH):
// faces sorted by the Morton code of their centroid, complete binary tree by
// median split, <= 4 faces per leaf, float boxes rounded outward (the boxes
// only prune; the entering decision is exact at the leaves).
void build_hull_bvh(HostMesh& M, const std::vector<int32_t>& P, const std::vector<int32_t>& T,
                    const std::vector<std::pair<int32_t, int>>& hull,
                    const std::vector<int32_t>& vnew) {
    const int64_t B = (int64_t)hull.size();
    struct Face { float lo[3], hi[3]; uint64_t key; int32_t v[3]; };
    std::vector<Face> f(B);
    long long mn[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX}, mx[3] = {LLONG_MIN, LLONG_MIN, LLONG_MIN};
    for (int64_t h = 0; h < B; ++h) {
        const int t = hull[h].first, k = hull[h].second;
        for (int j = 0; j < 3; ++j) f[h].v[j] = T[4 * (int64_t)t + kFace[k][j]];
        for (int i = 0; i < 3; ++i) {
            long long lo = LLONG_MAX, hi = LLONG_MIN;
            for (int j = 0; j < 3; ++j) {
                lo = std::min(lo, (long long)P[3 * f[h].v[j] + i]);
                hi = std::max(hi, (long long)P[3 * f[h].v[j] + i]);
            }
            f[h].lo[i] = std::nextafter((float)lo, -INFINITY);
            f[h].hi[i] = std::nextafter((float)hi, INFINITY);
            mn[i] = std::min(mn[i], lo);
            mx[i] = std::max(mx[i], hi);
        }
    }
    long long span = 1;
    for (int i = 0; i < 3; ++i) span = std::max(span, mx[i] - mn[i] + 1);
    int shift = 0;
    while ((span >> shift) >= (1 << 20)) ++shift;
    for (int64_t h = 0; h < B; ++h) {
        uint64_t key = 0;
        for (int i = 0; i < 3; ++i) {
            long long c = 0;
            for (int j = 0; j < 3; ++j) c += P[3 * f[h].v[j] + i];
            key |= spread21((uint64_t)(((c / 3) - mn[i]) >> shift)) << i;
        }
        f[h].key = key;
    }
    std::sort(f.begin(), f.end(), [](const Face& a, const Face& b) { return a.key < b.key; });
    // faces in BVH order: (tet, k) internal + vertex ids
    M.bvh_faces.resize((size_t)B * 4);
    for (int64_t h = 0; h < B; ++h)
        for (int j = 0; j < 3; ++j) M.bvh_faces[4 * h + j] = vnew[f[h].v[j]];
    // entry code per face: find (t,k) again by matching the face record order
    {
        std::unordered_map<uint64_t, int32_t> code;   // sorted-vertex-triple hash -> code
        code.reserve(B * 2);
        auto key3 = [](int32_t a, int32_t b, int32_t c) {
            int32_t x[3] = {a, b, c};
            std::sort(x, x + 3);
            return ((uint64_t)(uint32_t)x[0] * 0x9E3779B97F4A7C15ULL) ^ ((uint64_t)(uint32_t)x[1] << 21) ^
                   ((uint64_t)(uint32_t)x[2] * 0xC2B2AE3D27D4EB4FULL);
        };
        for (int64_t h = 0; h < B; ++h) {
            const int t = hull[h].first, k = hull[h].second;
            const int32_t a = T[4 * (int64_t)t + kFace[k][0]], b = T[4 * (int64_t)t + kFace[k][1]],
                          c = T[4 * (int64_t)t + kFace[k][2]];
            code[key3(a, b, c)] = M.hull[2 * h] * 4 + M.hull[2 * h + 1];
        }
        for (int64_t h = 0; h < B; ++h)
            M.bvh_faces[4 * h + 3] = code[key3(f[h].v[0], f[h].v[1], f[h].v[2])];
    }
    // nodes: implicit recursion on [lo, hi) ranges, stored depth-first
    M.bvh_nodes.clear();
    struct Rec { int64_t lo, hi, node; };
    std::vector<Rec> stack;
    auto push_node = [&]() {
        M.bvh_nodes.resize(M.bvh_nodes.size() + 8);
        return (int64_t)(M.bvh_nodes.size() / 8 - 1);
    };
    const int64_t root = push_node();
    stack.push_back({0, B, root});
    while (!stack.empty()) {
        Rec r = stack.back();
        stack.pop_back();
        float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int64_t h = r.lo; h < r.hi; ++h)
            for (int i = 0; i < 3; ++i) {
                lo[i] = std::min(lo[i], f[h].lo[i]);
                hi[i] = std::max(hi[i], f[h].hi[i]);
            }
        float* nd = reinterpret_cast<float*>(&M.bvh_nodes[8 * r.node]);
        for (int i = 0; i < 3; ++i) { nd[i] = lo[i]; nd[3 + i] = hi[i]; }
        if (r.hi - r.lo <= 4) {   // leaf: -(first+1), count
            M.bvh_nodes[8 * r.node + 6] = -(int32_t)(r.lo + 1);
            M.bvh_nodes[8 * r.node + 7] = (int32_t)(r.hi - r.lo);
        } else {
            const int64_t mid = (r.lo + r.hi) / 2;
            const int64_t L = push_node(), R = push_node();
            M.bvh_nodes[8 * r.node + 6] = (int32_t)L;
            M.bvh_nodes[8 * r.node + 7] = (int32_t)R;
            stack.push_back({mid, r.hi, R});
            stack.push_back({r.lo, mid, L});
        }
    }
}

}  // namespace

tet_status prepare_mesh(const double* verts, int64_t nv, const int32_t* tets,
                        const int32_t* nbrs, int64_t nt, const int32_t* bfaces,
                        int64_t nb, uint32_t flags, HostMesh& M, std::string& err) {
    if (!verts || !tets || !nbrs || (nb > 0 && !bfaces) || nv < 4 || nt < 1 || nb < 4 ||
        nt > (int64_t)(1 << 29) || nv > 0x7fffffff) {
        err = "tet_mesh_create: bad arguments";
        return TET_E_ARG;
    }
    // ---- grid snap (Numeric contract) ----
    double lo[3], hi[3];
    for (int i = 0; i < 3; ++i) lo[i] = hi[i] = verts[i];
    for (int64_t v = 0; v < nv; ++v)
        for (int i = 0; i < 3; ++i) {
            double x = verts[3 * v + i];
            if (!std::isfinite(x)) { err = "non-finite vertex coordinate"; return TET_E_ARG; }
            lo[i] = std::min(lo[i], x);
            hi[i] = std::max(hi[i], x);
        }
    double c[3], r = 0;
    for (int i = 0; i < 3; ++i) c[i] = 0.5 * (lo[i] + hi[i]);
    for (int64_t v = 0; v < nv; ++v)
        for (int i = 0; i < 3; ++i) r = std::max(r, std::fabs(verts[3 * v + i] - c[i]));
    if (!(r > 0)) { err = "degenerate vertex set"; return TET_E_ARG; }
    M.e = grid_exponent(r);
    M.g = std::ldexp(1.0, M.e);
    for (int i = 0; i < 3; ++i) M.C[i] = std::nearbyint(c[i] / M.g) * M.g;
    std::vector<int32_t> P((size_t)nv * 3);
    for (int64_t v = 0; v < nv; ++v)
        for (int i = 0; i < 3; ++i) {
            long long q;
            if (!snap(verts[3 * v + i], M.C[i], M.g, q)) { err = "vertex outside grid"; return TET_E_ARG; }
            P[3 * v + i] = (int32_t)q;
        }
    // ---- tets: indices, distinct nodes, exact orientation ----
    std::vector<int32_t> T(tets, tets + 4 * nt), N(nbrs, nbrs + 4 * nt);
    std::vector<char> swapped(nt, 0);
    for (int64_t t = 0; t < nt; ++t) {
        int32_t* q = &T[4 * t];
        for (int k = 0; k < 4; ++k) {
            if (q[k] < 0 || q[k] >= nv) { err = "node index out of range in tet " + std::to_string(t); return TET_E_MESH; }
            if (N[4 * t + k] < -1 || N[4 * t + k] >= nt) { err = "neighbour index out of range"; return TET_E_MESH; }
        }
        for (int i = 0; i < 4; ++i)
            for (int j = i + 1; j < 4; ++j)
                if (q[i] == q[j]) { err = "repeated node in tet " + std::to_string(t); return TET_E_MESH; }
        int s = orient_filtered(&P[3 * q[0]], &P[3 * q[1]], &P[3 * q[2]], &P[3 * q[3]]);
        if (s == 0) { err = "flat tet " + std::to_string(t); return TET_E_MESH; }
        if (s < 0) {
            if (!(flags & TET_F_FIX_ORIENTATION)) { err = "negatively oriented tet " + std::to_string(t); return TET_E_MESH; }
            std::swap(q[0], q[1]);
            std::swap(N[4 * t], N[4 * t + 1]);
            swapped[t] = 1;
        }
    }
    // ---- reciprocity + face tags k' ----
    std::vector<int8_t> kback((size_t)nt * 4, -1);
    auto face_key = [&](int64_t t, int k, int32_t out[3]) {
        for (int i = 0, j = 0; i < 4; ++i)
            if (i != k) out[j++] = T[4 * t + i];
        std::sort(out, out + 3);
    };
    for (int64_t t = 0; t < nt; ++t)
        for (int k = 0; k < 4; ++k) {
            int32_t n = N[4 * t + k];
            if (n < 0) continue;
            int32_t f1[3], f2[3];
            face_key(t, k, f1);
            int found = -1;
            for (int k2 = 0; k2 < 4; ++k2) {
                if (N[4 * (int64_t)n + k2] != t) continue;
                face_key(n, k2, f2);
                if (f1[0] == f2[0] && f1[1] == f2[1] && f1[2] == f2[2]) found = k2;
            }
            if (found < 0) { err = "non-reciprocal neighbours at tet " + std::to_string(t); return TET_E_MESH; }
            kback[4 * t + k] = (int8_t)found;
        }
    // ---- hull list == {nbr == -1} (caller indexing) ----
    std::vector<int64_t> have, given;
    std::vector<std::pair<int32_t, int>> hull;
    for (int64_t t = 0; t < nt; ++t)
        for (int k = 0; k < 4; ++k)
            if (N[4 * t + k] < 0) {
                hull.push_back({(int32_t)t, k});
                int kc = swapped[t] ? (k == 0 ? 1 : k == 1 ? 0 : k) : k;
                have.push_back(t * 4 + kc);
            }
    for (int64_t b = 0; b < nb; ++b) {
        int32_t t = bfaces[2 * b], k = bfaces[2 * b + 1];
        if (t < 0 || t >= nt || k < 0 || k > 3) { err = "boundary face out of range"; return TET_E_MESH; }
        given.push_back((int64_t)t * 4 + k);
    }
    std::sort(have.begin(), have.end());
    std::sort(given.begin(), given.end());
    if (have != given) { err = "boundary list does not match nbrs == -1"; return TET_E_MESH; }
    // ---- hull: closed 2-manifold, locally and globally convex ----
    const int64_t B = (int64_t)hull.size();
    std::unordered_map<uint64_t, int64_t> edge;  // directed edge -> hull face
    edge.reserve(B * 4);
    auto fv = [&](int64_t h, int j) { return T[4 * (int64_t)hull[h].first + kFace[hull[h].second][j]]; };
    for (int64_t h = 0; h < B; ++h)
        for (int j = 0; j < 3; ++j) {
            uint64_t key = ((uint64_t)(uint32_t)fv(h, j) << 32) | (uint32_t)fv(h, (j + 1) % 3);
            if (!edge.emplace(key, h).second) { err = "non-manifold hull"; return TET_E_MESH; }
        }
    for (int64_t h = 0; h < B; ++h)
        for (int j = 0; j < 3; ++j) {
            int32_t a = fv(h, j), b = fv(h, (j + 1) % 3);
            auto it = edge.find(((uint64_t)(uint32_t)b << 32) | (uint32_t)a);
            if (it == edge.end()) { err = "open hull"; return TET_E_MESH; }
            int64_t h2 = it->second;
            int32_t d = -1;
            for (int jj = 0; jj < 3; ++jj) {
                int32_t x = fv(h2, jj);
                if (x != a && x != b) d = x;
            }
            if (orient_filtered(&P[3 * fv(h, 0)], &P[3 * fv(h, 1)], &P[3 * fv(h, 2)], &P[3 * d]) > 0) {
                err = "hull is not convex (reflex hull edge)";
                return TET_E_NONCONVEX;
            }
        }
    {   // global: every hull vertex on the inner side of every hull plane
        std::vector<int32_t> hv;
        for (int64_t h = 0; h < B; ++h)
            for (int j = 0; j < 3; ++j) hv.push_back(fv(h, j));
        std::sort(hv.begin(), hv.end());
        hv.erase(std::unique(hv.begin(), hv.end()), hv.end());
        for (int64_t h = 0; h < B; ++h) {
            const int32_t *a = &P[3 * fv(h, 0)], *b = &P[3 * fv(h, 1)], *cc = &P[3 * fv(h, 2)];
            double e1[3], e2[3];
            for (int i = 0; i < 3; ++i) { e1[i] = (double)b[i] - a[i]; e2[i] = (double)cc[i] - a[i]; }
            double n0 = e1[1] * e2[2] - e1[2] * e2[1], n1 = e1[2] * e2[0] - e1[0] * e2[2],
                   n2 = e1[0] * e2[1] - e1[1] * e2[0];
            for (int32_t v : hv) {
                const int32_t* d = &P[3 * v];
                double x = n0 * ((double)d[0] - a[0]) + n1 * ((double)d[1] - a[1]) + n2 * ((double)d[2] - a[2]);
                double bound = 1e-14 * (std::fabs(n0 * ((double)d[0] - a[0])) + std::fabs(n1 * ((double)d[1] - a[1])) +
                                        std::fabs(n2 * ((double)d[2] - a[2])));
                if (x < -bound) continue;
                if (orient_filtered(a, b, cc, d) > 0) { err = "hull is not convex"; return TET_E_NONCONVEX; }
            }
        }
    }
    // ---- Morton (SFC) reorder of tets by centroid ----
    std::vector<int32_t> order(nt);
    std::iota(order.begin(), order.end(), 0);
    M.reordered = !(flags & TET_F_NO_REORDER);
    if (M.reordered) {
        long long mn[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX}, mx[3] = {LLONG_MIN, LLONG_MIN, LLONG_MIN};
        std::vector<long long> cen((size_t)nt * 3);
        for (int64_t t = 0; t < nt; ++t)
            for (int i = 0; i < 3; ++i) {
                long long s = 0;
                for (int k = 0; k < 4; ++k) s += P[3 * T[4 * t + k] + i];
                cen[3 * t + i] = s;
                mn[i] = std::min(mn[i], s);
                mx[i] = std::max(mx[i], s);
            }
        long long span = 1;
        for (int i = 0; i < 3; ++i) span = std::max(span, mx[i] - mn[i] + 1);
        int shift = 0;
        while ((span >> shift) >= (1 << 21)) ++shift;
        // Morton order by default; TETPROJ_SFC=hilbert measured the same
        // (c3 1.636e11 vs 1.639e11, c5 1.679e11 vs 1.675e11, profiles/README.md)
        const char* sfc = std::getenv("TETPROJ_SFC");
        const bool hilbert = sfc && std::string(sfc) == "hilbert";
        std::vector<uint64_t> key(nt);
        for (int64_t t = 0; t < nt; ++t) {
            uint64_t k = 0;
            if (hilbert)
                k = hilbert21((uint32_t)((cen[3 * t] - mn[0]) >> shift),
                              (uint32_t)((cen[3 * t + 1] - mn[1]) >> shift),
                              (uint32_t)((cen[3 * t + 2] - mn[2]) >> shift));
            else
                for (int i = 0; i < 3; ++i) k |= spread21((uint64_t)((cen[3 * t + i] - mn[i]) >> shift)) << i;
            key[t] = k;
        }
        std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return key[a] < key[b]; });
    }
    std::vector<int32_t> inv(nt);
    for (int64_t i = 0; i < nt; ++i) inv[order[i]] = (int32_t)i;
    // vertices renumbered by first use in the new tet order
    std::vector<int32_t> vnew(nv, -1);
    int32_t nvu = 0;
    for (int64_t i = 0; i < nt; ++i)
        for (int k = 0; k < 4; ++k) {
            int32_t v = T[4 * (int64_t)order[i] + k];
            if (vnew[v] < 0) vnew[v] = nvu++;
        }
    M.nv = nvu;
    M.nt = nt;
    M.nb = B;
    M.vtx.assign((size_t)nvu * 4, 0);
    double rmax2 = 0;
    long long bmn[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX}, bmx[3] = {LLONG_MIN, LLONG_MIN, LLONG_MIN};
    for (int64_t v = 0; v < nv; ++v) {
        if (vnew[v] < 0) continue;
        double s = 0;
        for (int i = 0; i < 3; ++i) {
            M.vtx[4 * (size_t)vnew[v] + i] = P[3 * v + i];
            s += (double)P[3 * v + i] * P[3 * v + i];
            bmn[i] = std::min(bmn[i], (long long)P[3 * v + i]);
            bmx[i] = std::max(bmx[i], (long long)P[3 * v + i]);
        }
        rmax2 = std::max(rmax2, s);
    }
    M.rmax = std::sqrt(rmax2) * (1 + 1e-12) + 1;
    double br2 = 0;
    for (int i = 0; i < 3; ++i) M.bs_c[i] = 0.5 * ((double)bmn[i] + (double)bmx[i]);
    for (int64_t v = 0; v < nv; ++v) {
        if (vnew[v] < 0) continue;
        double s = 0;
        for (int i = 0; i < 3; ++i) s += (P[3 * v + i] - M.bs_c[i]) * (P[3 * v + i] - M.bs_c[i]);
        br2 = std::max(br2, s);
    }
    M.bs_r = std::sqrt(br2) * (1 + 1e-12) + 1;
    // Face tags: face k of tet t (opposite node k) -> two int32
    // words, stored at position r = rank of node k's vertex id among the
    // tet's four (new) vertex ids:
    //   lo = n     (neighbour across the face, internal index); -1 on the hull
    //   hi = apex  (vertex id of n's node opposite the shared face); -1 on the hull
    // The walker holds all four vertex ids of t (three face slots + apex), so
    // it finds the exit face's position by ranking the dropped vertex among
    // them -- no node list or local-index bookkeeping in the loop -- and the
    // tag gives the next tet and its apex (gathered one step ahead).
    M.rec.assign((size_t)nt * 8, 0);
    M.tnode.assign((size_t)nt * 4, 0);
    M.perm.assign(nt, 0);
    for (int64_t i = 0; i < nt; ++i) {
        int64_t t = order[i];
        M.perm[i] = (int32_t)t;
        int32_t ids[4];
        for (int k = 0; k < 4; ++k) ids[k] = M.tnode[4 * i + k] = vnew[T[4 * t + k]];
        for (int k = 0; k < 4; ++k) {
            int r = 0;
            for (int j = 0; j < 4; ++j) r += ids[j] < ids[k];
            int32_t n = N[4 * t + k];
            if (n < 0) {
                M.rec[8 * i + 2 * r] = -1;
                M.rec[8 * i + 2 * r + 1] = -1;
                continue;
            }
            const int kp = kback[4 * t + k];
            M.rec[8 * i + 2 * r] = inv[n];
            M.rec[8 * i + 2 * r + 1] = vnew[T[4 * (int64_t)n + kp]];
        }
    }
    // 16-B face tags carrying the next apex's COORDINATES (DESIGN.md §5,
    // "FT16 walk"): tag r of tet i (same rank order as rec) packs
    //   w3 = n (26 bits; 2^26 - 1 on the hull) | apex id bits 0..5 << 26
    //   w0 = X << 6 | apex id bits 6..11,  w1 = Y << 6 | bits 12..17,
    //   w2 = Z << 6 | bits 18..23
    // (X, Y, Z = the apex's grid coordinates, |.| <= 2^24 + 1 < 2^25 by the
    // numeric contract), so the walker learns the next tet, its apex id AND
    // the apex position from one 16-B load -- no vertex gather in the loop.
    // Meshes with >= 2^26 - 1 tets or >= 2^24 vertices keep the rec walk.
    M.ft16 = nt < (1 << 26) - 1 && nvu < (1 << 24);
    if (M.ft16) {
        M.tag16.assign((size_t)nt * 16, 0);
        for (int64_t i = 0; i < nt; ++i) {
            const int64_t t = order[i];
            int32_t ids[4];
            for (int k = 0; k < 4; ++k) ids[k] = vnew[T[4 * t + k]];
            for (int k = 0; k < 4; ++k) {
                int r = 0;
                for (int j = 0; j < 4; ++j) r += ids[j] < ids[k];
                const int32_t n = N[4 * t + k];
                uint32_t n26 = 0x3FFFFFFu, apex = 0;
                int32_t X[3] = {0, 0, 0};
                if (n >= 0) {
                    const int32_t va = T[4 * (int64_t)n + kback[4 * t + k]];
                    n26 = (uint32_t)inv[n];
                    apex = (uint32_t)vnew[va];
                    for (int c = 0; c < 3; ++c) X[c] = P[3 * (int64_t)va + c];
                }
                uint32_t* w = reinterpret_cast<uint32_t*>(&M.tag16[16 * i + 4 * r]);
                w[0] = ((uint32_t)X[0] << 6) | ((apex >> 6) & 63u);
                w[1] = ((uint32_t)X[1] << 6) | ((apex >> 12) & 63u);
                w[2] = ((uint32_t)X[2] << 6) | ((apex >> 18) & 63u);
                w[3] = n26 | ((apex & 63u) << 26);
            }
        }
    }
    M.hull.resize((size_t)B * 2);
    for (int64_t h = 0; h < B; ++h) {
        M.hull[2 * h] = inv[hull[h].first];
        M.hull[2 * h + 1] = hull[h].second;
    }
    build_hull_bvh(M, P, T, hull, vnew);
    build_hull_rtree(M);
    return TET_OK;
}

tet_status prepare_geometry(const HostMesh& M, const tet_geometry* g,
                            std::vector<AngleGeom>& ang, std::vector<AngleAux>& aux,
                            std::string& err) {
    if (!g || !g->vecs || g->n_angles < 1 || g->n_v < 1 || g->n_u < 1 ||
        (g->beam != TET_BEAM_CONE && g->beam != TET_BEAM_PARALLEL)) {
        err = "bad geometry arguments";
        return TET_E_ARG;
    }
    ang.resize(g->n_angles);
    aux.resize(g->n_angles);
    const double lim = 2147483647.0;
    for (int a = 0; a < g->n_angles; ++a) {
        const double* q = g->vecs + 12 * (size_t)a;
        for (int i = 0; i < 12; ++i)
            if (!std::isfinite(q[i])) { err = "non-finite geometry"; return TET_E_ARG; }
        AngleGeom& G = ang[a];
        double mx = std::max(std::fabs(q[0]), std::max(std::fabs(q[1]), std::fabs(q[2])));
        for (int i = 0; i < 3; ++i) {
            bool ok = true;
            if (g->beam == TET_BEAM_CONE) ok &= snap(q[i], M.C[i], M.g, G.o[i]);
            else {
                if (!(mx > 0)) { err = "zero ray direction"; return TET_E_GEOMETRY; }
                G.o[i] = (long long)std::nearbyint((q[i] / mx) * 1048576.0);
            }
            ok &= snap(q[3 + i], M.C[i], M.g, G.p00[i]);
            ok &= snap(q[6 + i], 0.0, M.g, G.du[i]);
            ok &= snap(q[9 + i], 0.0, M.g, G.dv[i]);
            if (!ok) { err = "geometry outside the grid span"; return TET_E_GEOMETRY; }
        }
        // all ray points within +-(2^31-1): extremes are at the detector corners
        for (int cu = 0; cu < 2; ++cu)
            for (int cv = 0; cv < 2; ++cv)
                for (int i = 0; i < 3; ++i) {
                    double p = (double)G.p00[i] + (double)cu * (g->n_u - 1) * G.du[i] +
                               (double)cv * (g->n_v - 1) * G.dv[i];
                    double o = g->beam == TET_BEAM_CONE ? (double)G.o[i] : p - (double)G.o[i];
                    if (std::fabs(p) > lim || std::fabs(o) > lim) { err = "ray points outside the grid span"; return TET_E_GEOMETRY; }
                }
        AngleAux& X = aux[a];
        double U[3], V[3];
        for (int i = 0; i < 3; ++i) {
            X.S[i] = (double)G.o[i];
            X.P00[i] = (double)G.p00[i];
            U[i] = (double)G.du[i];
            V[i] = (double)G.dv[i];
        }
        X.N[0] = U[1] * V[2] - U[2] * V[1];
        X.N[1] = U[2] * V[0] - U[0] * V[2];
        X.N[2] = U[0] * V[1] - U[1] * V[0];
        double nn = std::sqrt(X.N[0] * X.N[0] + X.N[1] * X.N[1] + X.N[2] * X.N[2]);
        if (!(nn > 0)) { err = "detector steps are parallel or zero"; return TET_E_GEOMETRY; }
        double VxN[3] = {V[1] * X.N[2] - V[2] * X.N[1], V[2] * X.N[0] - V[0] * X.N[2], V[0] * X.N[1] - V[1] * X.N[0]};
        double NxU[3] = {X.N[1] * U[2] - X.N[2] * U[1], X.N[2] * U[0] - X.N[0] * U[2], X.N[0] * U[1] - X.N[1] * U[0]};
        double su = U[0] * VxN[0] + U[1] * VxN[1] + U[2] * VxN[2];
        double sv = V[0] * NxU[0] + V[1] * NxU[1] + V[2] * NxU[2];
        for (int i = 0; i < 3; ++i) { X.Us[i] = VxN[i] / su; X.Vs[i] = NxU[i] / sv; }
        if (g->beam == TET_BEAM_CONE) {
            // mesh strictly between the source plane and the detector plane
            double n[3] = {X.N[0] / nn, X.N[1] / nn, X.N[2] / nn};
            double dS = 0, dc = 0;
            for (int i = 0; i < 3; ++i) {
                dS += n[i] * (X.S[i] - X.P00[i]);
                dc += n[i] * (M.bs_c[i] - X.P00[i]);
            }
            double r = M.bs_r * (1 + 1e-9) + 2;
            bool ok = (dS > 0) ? (dc > r && dS - dc > r) : (dc < -r && dc - dS > r);
            if (!ok) { err = "cone geometry: mesh not strictly between source and detector"; return TET_E_GEOMETRY; }
        } else {
            double dn = X.S[0] * X.N[0] + X.S[1] * X.N[1] + X.S[2] * X.N[2];
            (void)dn;
        }
    }
    return TET_OK;
}

}  // namespace tetproj
