// Test harness (CPU): build a mesh's host-side structures with the product's
// host code (prepare_mesh -> BVH faces + R*-tree) and check the R*-tree's
// invariants: every hull face in exactly one leaf, non-root fan-out in
// [4, 10], every child box inside its parent's box and every
// face's vertices inside its leaf box.  Input: a raw mesh file written by
// tests/test_rtree_host.py.  Prints "nodes faces depth bad".
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "../../paper_1908_06909_b200/csrc/internal.h"

using namespace tetproj;

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    FILE* f = fopen(argv[1], "rb");
    if (!f) return 2;
    long long nv = 0, nt = 0, nb = 0;
    if (fread(&nv, 8, 1, f) != 1 || fread(&nt, 8, 1, f) != 1 || fread(&nb, 8, 1, f) != 1) return 2;
    std::vector<double> v(nv * 3);
    std::vector<int> t(nt * 4), n(nt * 4), b(nb * 2);
    if (fread(v.data(), 8, v.size(), f) != v.size() || fread(t.data(), 4, t.size(), f) != t.size() ||
        fread(n.data(), 4, n.size(), f) != n.size() || fread(b.data(), 4, b.size(), f) != b.size())
        return 2;
    fclose(f);
    HostMesh M;
    std::string err;
    if (prepare_mesh(v.data(), nv, t.data(), n.data(), nt, b.data(), nb, 1, M, err) != TET_OK) {
        printf("prepare_mesh failed: %s\n", err.c_str());
        return 1;
    }
    const size_t faces = M.bvh_faces.size() / 4;
    std::vector<int> seen(faces, 0);
    int bad = 0, depth_max = 0;
    std::function<void(int, int, const float*, const float*)> rec =
        [&](int nd, int depth, const float* plo, const float* phi) {
            const int* w = &M.rtree_nodes[72 * (size_t)nd];
            const int cnt = w[0], leaf = w[1];
            if (nd != 0 && (cnt < 4 || cnt > 10)) ++bad;
            if (cnt < 1 || cnt > 10) { ++bad; return; }
            depth_max = std::max(depth_max, depth);
            const float* lo = reinterpret_cast<const float*>(w + 12);
            const float* hi = reinterpret_cast<const float*>(w + 42);
            for (int c = 0; c < cnt; ++c) {
                if (plo)
                    for (int i = 0; i < 3; ++i)
                        if (lo[3 * c + i] < plo[i] || hi[3 * c + i] > phi[i]) ++bad;
                if (leaf) {
                    const int fc = w[2 + c];
                    if (fc < 0 || (size_t)fc >= faces) { ++bad; continue; }
                    seen[fc]++;
                    for (int j = 0; j < 3; ++j)
                        for (int i = 0; i < 3; ++i) {
                            const float x = (float)M.vtx[4 * (size_t)M.bvh_faces[4 * fc + j] + i];
                            if (x < lo[3 * c + i] || x > hi[3 * c + i]) ++bad;
                        }
                } else {
                    rec(w[2 + c], depth + 1, lo + 3 * c, hi + 3 * c);
                }
            }
        };
    rec(0, 0, nullptr, nullptr);
    for (int x : seen) bad += x != 1;
    printf("%zu %zu %d %d\n", M.rtree_nodes.size() / 72, faces, depth_max, bad);
    return 0;
}
