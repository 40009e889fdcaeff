/*
 * include/tetproj.h -- C ABI of the B200-native tetrahedral-mesh X-ray
 * projector / backprojector (hot path of arXiv:1908.06909).
 *
 * The operator (§2.1, lines 22-33):
 *     A_ji = length of (ray j) ∩ (tet i)              "each entry represents the
 *                                                       length of the line-element
 *                                                       intersection"
 *     tet_project     : proj_j = sum_i A_ji mu_i       Eq. 2
 *     tet_backproject : x_i    = sum_j A_ji y_j        Eq. 3, the
 *                                                       exact adjoint of tet_project
 * computed matrix-free ("calculating the elements of A on the fly",
 * PAPER.md:34) by walking each ray from tet to tet through shared faces
 * (Alg. 2) on the graph mesh of §2.2.
 * Face crossings are decided by EXACT signs of det[a-o, b-o, p-o] on an
 * integer grid with a symbolic perturbation (readings R2-R5), so
 * no ray is lost or double-counted at edges and vertices.
 *
 * Conventions
 *  - Every call returns tet_status (TET_OK = 0) and never throws or aborts;
 *    tet_last_error() gives a thread-local description of the last failure.
 *  - Arrays are in the CALLER's tet / ray order.  Rays are ordered
 *    [angle][v][u] (row v, column u), ray id = (a*n_v + v)*n_u + u.
 *  - Data pointers (mu, proj, x) may be DEVICE pointers (on the mesh's device)
 *    or HOST pointers (pinned or pageable); the library detects which.  With
 *    device pointers the call is asynchronous on `cuda_stream` (unless `st`
 *    is non-NULL); with host pointers the call copies through device scratch
 *    and returns after the results are in host memory.
 *  - `cuda_stream` is a cudaStream_t (NULL = legacy default stream).
 */
#ifndef TETPROJ_H
#define TETPROJ_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tet_mesh* tet_mesh_t;   /* opaque; immutable after create; safe for
                                          concurrent project/backproject calls on
                                          different streams                        */
typedef enum {
    TET_OK = 0,
    TET_E_ARG = 1,        /* null / negative / non-finite argument              */
    TET_E_MESH = 2,       /* bad index, repeated node, flat or (without
                             TET_F_FIX_ORIENTATION) negative tet, non-reciprocal
                             neighbours, hull list != {nbr == -1}, open or
                             non-manifold hull                                   */
    TET_E_NONCONVEX = 3,  /* hull not convex ("the volumetric mesh must be
                             convex")                             */
    TET_E_GEOMETRY = 4,   /* ray points outside the grid span, zero step, or a
                             cone source / detector that is not strictly outside
                             the mesh on opposite sides                         */
    TET_E_CUDA = 5,       /* CUDA runtime error (text in tet_last_error)         */
    TET_E_NOMEM = 6,
    TET_E_RAYS = 7        /* TET_F_STRICT and lost|stuck|entry_conflicts > 0     */
} tet_status;

enum { TET_BEAM_CONE = 0, TET_BEAM_PARALLEL = 1 };

enum {
    TET_F_FIX_ORIENTATION = 1, /* swap nodes 0,1 (and nbrs 0,1) of negative tets  */
    TET_F_NO_REORDER = 2,      /* keep caller tet order inside (no SFC reorder)   */
    TET_F_STRICT = 4           /* lost/stuck rays make calls fail with TET_E_RAYS */
};

/* Scan geometry: explicit per-angle vectors (the paper fixes no convention and
 * cites TIGRE).  vecs is HOST memory [n_angles][12] doubles:
 *   cone     : source xyz        | pixel(v=0,u=0) centre xyz | u-step xyz | v-step xyz
 *   parallel : ray direction xyz | pixel(v=0,u=0) centre xyz | u-step xyz | v-step xyz
 * Pixel (v,u) centre = P00 + u*Ustep + v*Vstep.  All points and steps are
 * snapped to the mesh's integer grid; the
 * operator integrates the whole line through (source, pixel) -- for cone
 * beams the call checks the mesh lies strictly between source and detector,
 * so line ∩ mesh == segment ∩ mesh.                                            */
typedef struct {
    int32_t beam, n_angles, n_v, n_u;
    const double* vecs;
} tet_geometry;

typedef struct {
    uint64_t rays;              /* rays traced (all pixels x angles)             */
    uint64_t rays_hit;          /* rays that entered the mesh                    */
    uint64_t crossings;         /* tets visited (incl. zero-length crossings)    */
    uint64_t lost;              /* inconsistent exit pattern (must be 0)         */
    uint64_t stuck;             /* walk exceeded n_tets steps (must be 0)        */
    uint64_t exact_fallbacks;   /* signs decided by the int128 exact path        */
    uint64_t entry_conflicts;   /* pixels claimed by >1 hull face (must be 0)    */
    uint32_t max_crossings_per_ray;
    uint32_t _pad;
    uint64_t escalations;       /* paper-faithful modes: epsilon escalations      */
} tet_stats;

/* Traversal mode (tet_project_ex / tet_backproject_ex).
 *   TET_TRAVERSE_EXACT  : exact Plücker signs + SoS (default; R2-R5)
 *   TET_TRAVERSE_MT_F64 : the paper's Alg. 1 (Möller-Trumbore with safety
 *                         parameter eps) inside Alg. 2 (eps
 *                         escalation x eps_growth until two faces are hit,
 *                         swap check on zero-length steps)
 *                         in double precision on world coordinates
 *   TET_TRAVERSE_MT_F32 : the same in single precision (the failure mode of
 *                         fig:singledouble)
 * The MT modes exist to reproduce the paper's robustness study: rays whose
 * escalation exceeds max_escalations are counted as `lost` and contribute what
 * was summed so far; walks longer than n_tets steps are `stuck`.             */
enum { TET_TRAVERSE_EXACT = 0, TET_TRAVERSE_MT_F64 = 1, TET_TRAVERSE_MT_F32 = 2 };
/* Entry finder (the "index of a tetrahedron on the mesh boundary" each ray
 * starts from):
 *   TET_ENTRY_RASTER : per (hull face, angle) exact rasterisation of the face's
 *                      detector footprint (default)
 *   TET_ENTRY_BVH    : per-ray search of a binary BVH over the hull faces
 *   TET_ENTRY_RTREE  : per-ray depth-first search of the paper's R*-tree over
 *                      the hull faces (fan-out 4..10)
 * All take the same exact entering decision, so results are identical.      */
enum { TET_ENTRY_RASTER = 0, TET_ENTRY_BVH = 1, TET_ENTRY_RTREE = 2 };
typedef struct {
    int32_t traversal;         /* TET_TRAVERSE_*                                 */
    int32_t max_escalations;   /* MT modes: 12 (SPEC.md:314 reading)            */
    double eps0;               /* MT modes: 1e-9 ("eps <- 10^-9")  */
    double eps_growth;         /* MT modes: 10 ("eps <- eps*10")   */
    int32_t entry;             /* TET_ENTRY_*                                    */
    int32_t _reserved;
} tet_options;

/* Create a mesh on CUDA device `device` (§2.2 graph + boundary list).
 *   verts  [n_verts][3] double   world coordinates (host)
 *   tets   [n_tets][4]  int32    vertex indices (host)
 *   nbrs   [n_tets][4]  int32    nbrs[t][k] = tet across the face opposite
 *                                tets[t][k], -1 on the hull (host)
 *   bfaces [n_bfaces][2] int32   (t, k) with nbrs[t][k] == -1 (host)
 * Host arrays are read during the call and not retained.  Validation (exact
 * orientation, reciprocity, hull == {nbr == -1}, closed manifold hull, exact
 * convexity) happens here, before the device is touched: a mesh error is
 * reported (TET_E_MESH / TET_E_NONCONVEX) even when `device` does not exist;
 * a valid mesh on a missing device gives TET_E_CUDA.  On success *out owns
 * all device memory of the mesh until tet_mesh_destroy.                    */
tet_status tet_mesh_create(const double* verts, int64_t n_verts,
                           const int32_t* tets, const int32_t* nbrs, int64_t n_tets,
                           const int32_t* bfaces, int64_t n_bfaces,
                           int device, uint32_t flags, tet_mesh_t* out);
tet_status tet_mesh_destroy(tet_mesh_t m);

/* Forward projection, Eq. 2:
 *   mu   [n_tets] float, caller tet order (device or host)
 *   proj [n_angles][n_v][n_u] float (device or host), overwritten
 * st (host, nullable): if non-NULL the call synchronises cuda_stream and fills
 * it.  Performance note (results are unaffected): a call with st whose exact
 * fallbacks exceed 5 % of its crossings switches the mesh's later calls
 * (both directions) to a walk compiled for exact-heavy scans, and a later
 * call with st below that rate switches back.                               */
tet_status tet_project(tet_mesh_t m, const tet_geometry* g, const float* mu, float* proj,
                       void* cuda_stream, tet_stats* st);

/* Backprojection, Eq. 3, exact adjoint of tet_project:
 *   proj [n_angles][n_v][n_u] float (device or host)
 *   x    [n_tets] float, caller order: x = A^T proj  (accumulate = 0)
 *                                      x += A^T proj (accumulate != 0)
 * Sums are accumulated in double on the device and rounded once.             */
tet_status tet_backproject(tet_mesh_t m, const tet_geometry* g, const float* proj, float* x,
                           int accumulate, void* cuda_stream, tet_stats* st);

/* Backprojection into a caller-provided double accumulator (device pointer,
 * caller order) without rounding: acc += A^T proj.  For callers that reduce
 * partial sums in double (paper_1908_06909_b200.dist.dist_backproject with
 * precision="f64"); the default multi-GPU path all-reduces the f32 result of
 * tet_backproject (each rank's sum rounded once: <= W * 2^-24 relative for W
 * ranks, R15).                                                     */
tet_status tet_backproject_f64(tet_mesh_t m, const tet_geometry* g, const float* proj,
                               double* acc, void* cuda_stream, tet_stats* st);

/* tet_project / tet_backproject with traversal options (NULL = exact). */
tet_status tet_project_ex(tet_mesh_t m, const tet_geometry* g, const float* mu, float* proj,
                          const tet_options* opt, void* cuda_stream, tet_stats* st);
tet_status tet_backproject_ex(tet_mesh_t m, const tet_geometry* g, const float* proj, float* x,
                              int accumulate, const tet_options* opt, void* cuda_stream,
                              tet_stats* st);

/* Plans: a scan bound to a mesh.  PAPER.md Alg. 2 (lines 120-144) starts each
 * ray by "Read initial intersection element": the entry tet of every ray is
 * an input of the walk, and for a fixed scan it is the same for every
 * projection and backprojection.  tet_plan_create validates and snaps the
 * geometry once and runs the entry finder (opt->entry) for all rays into a
 * device entry map (4 B per ray, from the mesh's memory pool); the plan's
 * project / backproject calls walk from that map and skip the entry stage.
 * Results are identical to tet_project / tet_backproject with the same
 * geometry and options (the same kernels on the same entry map; backprojection
 * sums are rounded from double, so only the atomics' order differs).
 *   g, opt  host; copied (the caller's arrays are not retained); opt NULL =
 *           exact traversal, raster entry finder
 *   stream  creation is stream-ordered on cuda_stream: the plan may be used on
 *           that stream at once, on another one after synchronising with it
 *   *out    owned by the caller until tet_plan_destroy; the mesh must outlive
 *           it.  Plans are immutable: concurrent calls on different streams
 *           are safe.
 * Errors: TET_E_ARG (null / unknown option), TET_E_GEOMETRY (as tet_project),
 * TET_E_NOMEM / TET_E_CUDA (device); on error *out = NULL.                   */
typedef struct tet_plan* tet_plan_t;
tet_status tet_plan_create(tet_mesh_t m, const tet_geometry* g, const tet_options* opt,
                           void* cuda_stream, tet_plan_t* out);
/* Releases the plan's device memory stream-ordered on cuda_stream (which must
 * be ordered after every use of the plan, as for cudaFreeAsync) into the
 * mesh's memory pool, where later calls and plans reuse it; the pool returns
 * it to the device at tet_mesh_destroy.  NULL is a no-op. */
tet_status tet_plan_destroy(tet_plan_t p, void* cuda_stream);
/* tet_project / tet_backproject / tet_backproject_f64 on the plan's scan and
 * options; same array contracts, stats include the entry finder's counters
 * (exact_fallbacks, entry_conflicts) from tet_plan_create. */
tet_status tet_plan_project(tet_plan_t p, const float* mu, float* proj, void* cuda_stream,
                            tet_stats* st);
tet_status tet_plan_backproject(tet_plan_t p, const float* proj, float* x, int accumulate,
                                void* cuda_stream, tet_stats* st);
tet_status tet_plan_backproject_f64(tet_plan_t p, const float* proj, double* acc,
                                    void* cuda_stream, tet_stats* st);

/* Introspection (for tests / bench).  info[0..7] = n_verts, n_tets, n_bfaces,
 * device, grid exponent e (g = 2^e), bytes of device mesh data, L2 persisting
 * window bytes, reordered (0/1).                                              */
tet_status tet_mesh_info(tet_mesh_t m, int64_t info[8]);

/* Which walk and entry structures the mesh carries:
 *   feat[0] = walk of exact traversals: 1 = FT16 (16-B face tags with apex
 *             coordinates; exact-heavy scans still take the record walk),
 *             0 = 32-B record walk (mesh beyond the FT16 encoding, or
 *             TETPROJ_WALKER=rec at create)
 *   feat[1] = bytes of FT16 tags on the device (0 without)
 *   feat[2] = R*-tree nodes over the hull faces (TET_ENTRY_RTREE)
 *   feat[3] = binary BVH nodes over the hull faces (TET_ENTRY_BVH)          */
tet_status tet_mesh_features(tet_mesh_t m, int64_t feat[4]);

/* Kernel timing for benchmarks / profiling.  When enabled, every call records
 * CUDA events around each of its kernel launches on the call's stream (no
 * synchronisation is added).  tet_kernel_times() -- only after that stream
 * has been synchronised -- returns per kernel class [0 entry finder,
 * 1 forward walk, 2 backward walk, 3 permutes] the milliseconds during which
 * at least one launch of the class was running (the union of the launch
 * intervals: a call's angle chunks alternate between two streams and their
 * launches may overlap) and the launch counts, and resets them.             */
enum { TET_K_ENTRY = 0, TET_K_FORWARD = 1, TET_K_BACKWARD = 2, TET_K_PERMUTE = 3, TET_K_COUNT = 4 };
tet_status tet_set_kernel_timing(tet_mesh_t m, int enable);
tet_status tet_kernel_times(tet_mesh_t m, double ms[4], int64_t launches[4]);

/* Last error text of the calling thread (never NULL). */
const char* tet_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* TETPROJ_H */
