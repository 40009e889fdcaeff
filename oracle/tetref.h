/*
 * oracle/tetref.h -- CPU double-precision ORACLE of the tetrahedral-mesh CT
 * projector / backprojector of arXiv:1908.06909 (Eq. 1-3, Alg. 2).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * product path (paper_1908_06909_b200/, include/tetproj.h).
 *
 * All arrays are host memory in the caller's tet / ray order.  Values are
 * double.  Every function returns 0 on success, a positive code otherwise
 * (text in tetref_last_error()).
 */
#ifndef TETREF_H
#define TETREF_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tetref_mesh tetref_mesh;

typedef struct {
    int32_t beam;          /* 0 = cone, 1 = parallel                        */
    int32_t n_angles, n_v, n_u;
    const double* vecs;    /* [n_angles][12]     */
} tetref_geometry;

typedef struct {
    int64_t rays, rays_hit, crossings, lost, stuck, max_crossings;
} tetref_stats;

int  tetref_mesh_create(const double* verts, int64_t n_verts, const int32_t* tets,
                        const int32_t* nbrs, int64_t n_tets, const int32_t* bfaces,
                        int64_t n_bfaces, uint32_t flags /* 1 = fix orientation */,
                        tetref_mesh** out);
void tetref_mesh_destroy(tetref_mesh* m);
const char* tetref_last_error(void);
double tetref_grid_spacing(const tetref_mesh* m);

/* forward: out[i] = sum_t a(ray_ids[i], t) mu[t]   (Eq. 2)
 * ray id = (angle * n_v + v) * n_u + u;  ray_ids == NULL means all rays.  */
int tetref_project(const tetref_mesh* m, const tetref_geometry* g, const double* mu,
                   int64_t n_rays, const int64_t* ray_ids, double* out, int nthreads,
                   tetref_stats* st);
/* backward: x[t] += sum_i a(ray_ids[i], t) y[i]   (Eq. 3) */
int tetref_backproject(const tetref_mesh* m, const tetref_geometry* g, const double* y,
                       int64_t n_rays, const int64_t* ray_ids, double* x, int nthreads,
                       tetref_stats* st);
/* the walk of one ray: tets visited in order and their chords (world units) */
int tetref_ray_path(const tetref_mesh* m, const tetref_geometry* g, int64_t ray_id,
                    int64_t cap, int32_t* tets, double* chords, int64_t* n_out);
/* exact symbolically-perturbed side(ray(o,p), edge(a,b)) on grid integers */
int tetref_side(const int64_t o[3], const int64_t p[3], const int64_t a[3],
                const int64_t b[3]);
/* grid coordinates of the snapped ray (o, p) of a ray id */
int tetref_ray_points(const tetref_mesh* m, const tetref_geometry* g, int64_t ray_id,
                      int64_t o[3], int64_t p[3]);
/* snapped vertex grid coordinates [n_verts][3] */
int tetref_vertex_grid(const tetref_mesh* m, int64_t* out);

/* ---- NEXT-1: the paper's own traversal (Alg. 1 + Alg. 2) --
 * eps-guarded Möller-Trumbore with eps escalation, in double (single = 0) or
 * float (single = 1) on world coordinates; first element = the exact
 * entering hull tet.  Rays whose escalation exceeds max_escalations are
 * `lost` (they keep what they summed), walks longer than
 * 10 ceil(T^(1/3)) + 100 elements are `stuck` (tetref_mt.inc).          */
typedef struct {
    int32_t single;            /* 0 = double, 1 = float arithmetic            */
    int32_t max_escalations;   /* 12 (SPEC.md:314 reading)                    */
    double eps0;               /* 1e-9 ("eps <- 10^-9")        */
    double eps_growth;         /* 10   ("eps <- eps * 10")     */
    int32_t no_swap_check;     /* 1: skip Alg. 2's swap check (pins what it does) */
    int32_t _pad;
} tetref_mt_options;

typedef struct {
    int64_t rays, rays_hit, crossings, lost, stuck, max_crossings, escalations;
} tetref_mt_stats;

int tetref_mt_project(const tetref_mesh* m, const tetref_geometry* g, const double* mu,
                      int64_t n_rays, const int64_t* ray_ids, double* out,
                      const tetref_mt_options* opt, int nthreads, tetref_mt_stats* st);
int tetref_mt_backproject(const tetref_mesh* m, const tetref_geometry* g, const double* y,
                          int64_t n_rays, const int64_t* ray_ids, double* x,
                          const tetref_mt_options* opt, int nthreads, tetref_mt_stats* st);
/* Alg. 1 alone on one triangle (ray r1 -> r2), in double or float */
int tetref_mt_hit_f64(const double r1[3], const double r2[3], const double p1[3],
                      const double p2[3], const double p3[3], double eps, double* t);
int tetref_mt_hit_f32(const double r1[3], const double r2[3], const double p1[3],
                      const double p2[3], const double p3[3], double eps, double* t);

#ifdef __cplusplus
}
#endif
#endif
