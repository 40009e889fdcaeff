// internal.h -- types shared by the host preparation, the kernels and the C ABI
// of libtetproj (product path; independent of oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/tetproj.h"

namespace tetproj {

// Per-angle scan geometry on the integer grid.
struct AngleGeom {
    long long o[3];    // cone: source S; parallel: direction d (ray o = p - d)
    long long p00[3];  // centre of pixel (v=0,u=0)
    long long du[3];   // u step
    long long dv[3];   // v step
};

// Per-angle doubles used only to bound the detector footprint of hull faces
// (never for a crossing decision).
struct AngleAux {
    double S[3];      // cone source / parallel direction (grid units)
    double P00[3];
    double N[3];      // U x V
    double Us[3];     // dual vector: u = (Q - P00) . Us
    double Vs[3];     // dual vector: v = (Q - P00) . Vs
};

// Host-side prepared mesh (internal SFC order).
struct HostMesh {
    int64_t nv = 0, nt = 0, nb = 0;
    int e = 0;                 // grid exponent, g = 2^e
    double g = 0, C[3] = {0, 0, 0};
    std::vector<int32_t> vtx;  // [V][4] grid coords (x,y,z,0), internal vertex order
    std::vector<int32_t> rec;  // [T][8] four face tags (lo, hi) -- see mesh_host.cpp
    std::vector<int32_t> tag16;// [T][16] four 16-B tags with apex coordinates (FT16 walk)
    bool ft16 = false;         // the mesh fits the FT16 tag encoding
    std::vector<int32_t> tnode;// [T][4] vertex ids (ray initialisation, entry finder)
    std::vector<int32_t> hull; // [B][2] (t, k) internal order
    std::vector<int32_t> perm; // [T] internal -> caller tet index
    std::vector<int32_t> bvh_nodes;  // [N][8] float lo[3], hi[3] | left, right (leaf: -(first+1), count)
    std::vector<int32_t> bvh_faces;  // [B][4] vertex ids (outward order) | entry code tet<<2|k
    std::vector<int32_t> rtree_nodes;  // [N][72] R*-tree over bvh_faces (rtree_host.cpp)
    double rmax = 0;           // max |X|_2 over vertices (grid units)
    double bs_c[3] = {0, 0, 0}, bs_r = 0;  // bounding sphere (grid units)
    bool reordered = false;
};

// Prepare (validate, orient, snap, reorder, pack).  Returns TET_OK or an
// error with text in `err`.
tet_status prepare_mesh(const double* verts, int64_t nv, const int32_t* tets,
                        const int32_t* nbrs, int64_t nt, const int32_t* bfaces,
                        int64_t nb, uint32_t flags, HostMesh& out, std::string& err);

// The paper's R*-tree over the hull faces (fan-out 4..10), from bvh_faces.
void build_hull_rtree(HostMesh& M);

// Snap a geometry to the mesh grid and validate it.
tet_status prepare_geometry(const HostMesh& m, const tet_geometry* g,
                            std::vector<AngleGeom>& ang, std::vector<AngleAux>& aux,
                            std::string& err);

// ------------------------------------------------------------- device ----
struct DevMesh {
    const int4* rec = nullptr;   // [2T] face tags
    const int4* tag16 = nullptr; // [4T] FT16 face tags (nullptr: rec walk)
    const int4* tnode = nullptr; // [T] node ids
    const int4* vtx = nullptr;   // [V]
    const int2* hull = nullptr;  // [B]
    const int* perm = nullptr;   // [T]
    const int4* bvh_nodes = nullptr;  // [2N] hull-face BVH (TET_ENTRY_BVH)
    const int4* bvh_faces = nullptr;  // [B]
    const int* rtree = nullptr;  // [N][72] R*-tree nodes (TET_ENTRY_RTREE)
    int64_t nv = 0, nt = 0, nb = 0;
    double g = 0, rmax = 0;
    double C[3] = {0, 0, 0};     // grid origin (world units)
    size_t l2_window_bytes = 0;  // L2 persistence window over rec (0 = off)
    double l2_hit_ratio = 0;
};

struct MtOptions {
    double eps0 = 1e-9, eps_growth = 10.0;
    int max_escalations = 12;
};

enum StatSlot {
    ST_RAYS = 0, ST_HIT, ST_CROSS, ST_LOST, ST_STUCK, ST_EXACT, ST_CONFLICT, ST_MAXC, ST_ESC,
    ST_COUNT
};

// Block-uniform half of the walker's shear frame, one per angle (kernels.cu
// make_frame_uni): cone -> q = source S (grid units); parallel -> q = (sx, sy,
// axis variant) of the angle's direction, scale = |d|/|d_k| g.  tau bounds the
// sign-filter error of every ray of the angle.  Passed by value as a
// __grid_constant__ kernel parameter (kUniMaxAngles angles per launch).
constexpr int kUniMaxAngles = 256;
struct UniFrame {
    double q[3];
    double tau;
    double scale;
};
struct UniFrames {
    UniFrame f[kUniMaxAngles];
};

struct LaunchChunk {
    const AngleGeom* ang;   // device, chunk-local angles
    const AngleGeom* host_ang;   // host copy of the same angles (uniform frames)
    const AngleAux* aux;    // device
    int beam, n_angles, nv, nu;
    int exact_heavy = 0;     // walk shape for exact-heavy scans (kernels.cu TraceShape)
};

// kernel launchers (kernels.cu)
size_t entry_scratch_bytes(const DevMesh& m, int n_angles);
cudaError_t launch_entry(const DevMesh& m, const LaunchChunk& c, int* entry, void* scratch,
                         unsigned long long* stats, cudaStream_t s);
cudaError_t launch_entry_bvh(const DevMesh& m, const LaunchChunk& c, int* entry,
                             unsigned long long* stats, cudaStream_t s);
cudaError_t launch_entry_rtree(const DevMesh& m, const LaunchChunk& c, int* entry,
                               unsigned long long* stats, cudaStream_t s);
cudaError_t launch_forward(const DevMesh& m, const LaunchChunk& c, const int* entry,
                           const float* mu_int, float* proj, unsigned long long* stats,
                           cudaStream_t s);
cudaError_t launch_backward(const DevMesh& m, const LaunchChunk& c, const int* entry,
                            const float* y, double* acc, unsigned long long* stats,
                            cudaStream_t s);
cudaError_t launch_mt(const DevMesh& m, const LaunchChunk& c, bool back, bool single,
                      const MtOptions& o, const int* entry, const float* mu_int, float* proj,
                      const float* y, double* acc, unsigned long long* stats, cudaStream_t s);
cudaError_t launch_gather_mu(const DevMesh& m, const float* mu, float* mu_int,
                             cudaStream_t s);
cudaError_t launch_scatter_x(const DevMesh& m, const double* acc, float* x, int accumulate,
                             cudaStream_t s);
cudaError_t launch_scatter_acc(const DevMesh& m, const double* acc, double* out,
                               cudaStream_t s);

}  // namespace tetproj
