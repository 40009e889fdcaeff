/*
 * oracle/tetref.c -- plain, slow, obviously-correct CPU ORACLE of the
 * tetrahedral-mesh X-ray projector / backprojector of arXiv:1908.06909.
 *
 * TEST INFRASTRUCTURE ONLY (see tetref.h).  Independent of the CUDA path:
 * no shared code, headers, tables or constants.
 *
 * What it computes (§2.1, Eq. 1-3, lines 22-33):
 *     a_ij = length of (ray j) ∩ (tet i)
 *     proj_j = sum_i a_ij mu_i                         (Eq. 2)
 *     x_i    = sum_j a_ij y_j                          (Eq. 3, PAPER.md:31-33;
 *                                  printed "b_i" read as b_j, R1)
 * How (Alg. 2, in its order):
 *     1. find the first boundary element of the ray   (§2.5)
 *        -- here by scanning EVERY hull face (no tree; brute force is the
 *        obviously-correct version of "the index of a tetrahedron on the mesh
 *        boundary");
 *     2. in the current element compute the two intersected faces and their
 *        parameters t1, t2 ("four triangle-ray intersections");
 *     3. sum += l*(t2-t1)*x, l = |R2-R1|;
 *     4. move to the neighbour across the t2 face, stop at -1.
 * Readings where the paper is silent:
 *     R2  the ray-triangle test is the EXACT sign of det[a-o, b-o, p-o] on the
 *         integer grid (replacing the epsilon-guarded Moller-Trumbore of Alg. 1,
 *         whose purpose -- "two intersections" always found, PAPER.md:75 -- is
 *         met exactly), with zeros resolved by Simulation of Simplicity: the
 *         line is perturbed to o + (d, d^2, d^4), p + (d, d^2, d^4) +
 *         (d^8, d^16, d^32) and the sign is that of the first non-zero term
 *         of  [det, -(ExD)x, -(ExD)y, -(ExD)z, (AxB)x, -Ez, Ey, (AxB)y, -Ex]
 *         (A=a-o, B=b-o, D=p-o, E=b-a)  -- this replaces the epsilon loop and
 *         the "check if they need to be swapped" step;
 *     R3  a face (a,b,c) is crossed iff side(a,b) = side(b,c) = side(c,a);
 *         with (a,b,c) ordered so its normal points out of the tet, -1 means
 *         entering and +1 leaving;
 *     R4  t of a crossed face = n.(a-o) / n.(p-o), n = (b-a)x(c-a), in double
 *         from exact integer dot products; chord = max(0, t2 - t1)*|p-o|*g;
 *     R5  numeric contract: vertices and ray points snapped to a power-of-two
 *         integer grid, A integrates line ∩ hull.
 */
#include "tetref.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef __int128 i128;

struct tetref_mesh {
    int64_t nv, nt, nb;
    int64_t (*v)[3];     /* snapped grid coordinates */
    int32_t (*tet)[4];   /* positively oriented */
    int32_t (*nbr)[4];
    int32_t (*hull)[2];  /* (t, k): nbr[t][k] == -1 */
    double g;            /* grid spacing (world units) */
    double C[3];         /* grid origin (world units) */
};

static _Thread_local char g_err[512];
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
const char* tetref_last_error(void) { return g_err; }

/* face k of a positively oriented tet (n0,n1,n2,n3), listed so that the normal
 * (b-a)x(c-a) points OUT of the tet: the face opposite node k. */
static const int FACE[4][3] = {{1, 2, 3}, {0, 3, 2}, {0, 1, 3}, {0, 2, 1}};

/* ---------------------------------------------------------------- exact -- */
static int sgn128(i128 x) { return (x > 0) - (x < 0); }

/* det[A, B, D] = D . (A x B) for integer 3-vectors (magnitudes < 2^34). */
static i128 det3(const i128 A[3], const i128 B[3], const i128 D[3]) {
    i128 cx = A[1] * B[2] - A[2] * B[1];
    i128 cy = A[2] * B[0] - A[0] * B[2];
    i128 cz = A[0] * B[1] - A[1] * B[0];
    return D[0] * cx + D[1] * cy + D[2] * cz;
}

/* Reading R2: sign of det[a-o, b-o, p-o] under the SoS perturbation. */
int tetref_side(const int64_t o[3], const int64_t p[3], const int64_t a[3],
                const int64_t b[3]) {
    i128 A[3], B[3], D[3], E[3];
    for (int i = 0; i < 3; ++i) {
        A[i] = (i128)a[i] - o[i];
        B[i] = (i128)b[i] - o[i];
        D[i] = (i128)p[i] - o[i];
        E[i] = (i128)b[i] - a[i];
    }
    i128 AxB[3] = {A[1] * B[2] - A[2] * B[1], A[2] * B[0] - A[0] * B[2],
                   A[0] * B[1] - A[1] * B[0]};
    i128 ExD[3] = {E[1] * D[2] - E[2] * D[1], E[2] * D[0] - E[0] * D[2],
                   E[0] * D[1] - E[1] * D[0]};
    i128 terms[9] = {det3(A, B, D), -ExD[0], -ExD[1], -ExD[2], AxB[0],
                     -E[2],         E[1],    AxB[1],  -E[0]};
    for (int i = 0; i < 9; ++i)
        if (terms[i] != 0) return sgn128(terms[i]);
    return 0; /* only when a == b (never for a valid mesh) */
}

/* orient3d(a,b,c,d) = det[b-a, c-a, d-a] */
static int orient(const int64_t a[3], const int64_t b[3], const int64_t c[3],
                  const int64_t d[3]) {
    i128 A[3], B[3], D[3];
    for (int i = 0; i < 3; ++i) {
        A[i] = (i128)b[i] - a[i];
        B[i] = (i128)c[i] - a[i];
        D[i] = (i128)d[i] - a[i];
    }
    /* det[A,B,D] with rows A,B,D = D.(AxB) */
    return sgn128(det3(A, B, D));
}

/* ----------------------------------------------------------------- grid -- */
static int grid_exponent(double r) {
    int k;
    double m = frexp(64.0 * r, &k);
    int c = (m == 0.5) ? k - 1 : k; /* ceil(log2(64 r)) */
    return c - 30;
}

static int snap_scalar(double x, double C, double g, int64_t* out) {
    double q = nearbyint((x - C) / g);
    if (!(fabs(q) <= 2147483647.0)) return 1;
    *out = (int64_t)q;
    return 0;
}

/* ------------------------------------------------------------------ mesh -- */
void tetref_mesh_destroy(tetref_mesh* m) {
    if (!m) return;
    free(m->v);
    free(m->tet);
    free(m->nbr);
    free(m->hull);
    free(m);
}

double tetref_grid_spacing(const tetref_mesh* m) { return m->g; }

int tetref_vertex_grid(const tetref_mesh* m, int64_t* out) {
    memcpy(out, m->v, sizeof(int64_t) * 3 * m->nv);
    return 0;
}

static int cmp_i64x3(const void* x, const void* y) {
    const int64_t* a = (const int64_t*)x;
    const int64_t* b = (const int64_t*)y;
    for (int i = 0; i < 3; ++i)
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
}

int tetref_mesh_create(const double* verts, int64_t nv, const int32_t* tets,
                       const int32_t* nbrs, int64_t nt, const int32_t* bfaces,
                       int64_t nb, uint32_t flags, tetref_mesh** out) {
    if (!verts || !tets || !nbrs || !out || nv < 4 || nt < 1 || nb < 4 || (nb && !bfaces))
        return fail(1, "bad arguments");
    *out = NULL;
    /* --- snap (Numeric contract) --- */
    double lo[3], hi[3];
    for (int i = 0; i < 3; ++i) lo[i] = hi[i] = verts[i];
    for (int64_t v = 0; v < nv; ++v)
        for (int i = 0; i < 3; ++i) {
            double x = verts[3 * v + i];
            if (!isfinite(x)) return fail(1, "non-finite vertex");
            if (x < lo[i]) lo[i] = x;
            if (x > hi[i]) hi[i] = x;
        }
    double c[3], r = 0.0;
    for (int i = 0; i < 3; ++i) c[i] = 0.5 * (lo[i] + hi[i]);
    for (int64_t v = 0; v < nv; ++v)
        for (int i = 0; i < 3; ++i) {
            double d = fabs(verts[3 * v + i] - c[i]);
            if (d > r) r = d;
        }
    if (!(r > 0.0)) return fail(1, "degenerate vertex set");
    tetref_mesh* m = (tetref_mesh*)calloc(1, sizeof *m);
    m->nv = nv;
    m->nt = nt;
    m->g = ldexp(1.0, grid_exponent(r));
    for (int i = 0; i < 3; ++i) m->C[i] = nearbyint(c[i] / m->g) * m->g;
    m->v = malloc(sizeof(*m->v) * nv);
    m->tet = malloc(sizeof(*m->tet) * nt);
    m->nbr = malloc(sizeof(*m->nbr) * nt);
    for (int64_t v = 0; v < nv; ++v)
        for (int i = 0; i < 3; ++i)
            if (snap_scalar(verts[3 * v + i], m->C[i], m->g, &m->v[v][i])) {
                tetref_mesh_destroy(m);
                return fail(1, "vertex outside grid span");
            }
    /* --- tets: indices, distinctness, exact orientation --- */
    int* swapped = calloc(nt, sizeof(int));
    int rc = 0;
    for (int64_t t = 0; t < nt && !rc; ++t) {
        for (int k = 0; k < 4; ++k) {
            m->tet[t][k] = tets[4 * t + k];
            m->nbr[t][k] = nbrs[4 * t + k];
            if (m->tet[t][k] < 0 || m->tet[t][k] >= nv) rc = fail(2, "node index out of range");
            if (m->nbr[t][k] < -1 || m->nbr[t][k] >= nt) rc = fail(2, "neighbour out of range");
        }
        if (rc) break;
        for (int i = 0; i < 4; ++i)
            for (int j = i + 1; j < 4; ++j)
                if (m->tet[t][i] == m->tet[t][j]) rc = fail(2, "repeated node");
        if (rc) break;
        int s = orient(m->v[m->tet[t][0]], m->v[m->tet[t][1]], m->v[m->tet[t][2]],
                       m->v[m->tet[t][3]]);
        if (s == 0) rc = fail(2, "flat tet");
        else if (s < 0) {
            if (!(flags & 1)) rc = fail(2, "negatively oriented tet");
            else { /* swap nodes 0,1 and the neighbours across their faces */
                int32_t x = m->tet[t][0]; m->tet[t][0] = m->tet[t][1]; m->tet[t][1] = x;
                x = m->nbr[t][0]; m->nbr[t][0] = m->nbr[t][1]; m->nbr[t][1] = x;
                swapped[t] = 1;
            }
        }
    }
    /* --- neighbour reciprocity: same face, listed back --- */
    for (int64_t t = 0; t < nt && !rc; ++t)
        for (int k = 0; k < 4 && !rc; ++k) {
            int32_t n = m->nbr[t][k];
            if (n < 0) continue;
            int found = 0;
            for (int k2 = 0; k2 < 4; ++k2) {
                if (m->nbr[n][k2] != t) continue;
                int64_t f1[3], f2[3];
                for (int i = 0, j = 0; i < 4; ++i) if (i != k) f1[j++] = m->tet[t][i];
                for (int i = 0, j = 0; i < 4; ++i) if (i != k2) f2[j++] = m->tet[n][i];
                /* sort both triples */
                for (int a = 0; a < 3; ++a) for (int b = a + 1; b < 3; ++b) {
                    if (f1[b] < f1[a]) { int64_t x = f1[a]; f1[a] = f1[b]; f1[b] = x; }
                    if (f2[b] < f2[a]) { int64_t x = f2[a]; f2[a] = f2[b]; f2[b] = x; }
                }
                if (f1[0] == f2[0] && f1[1] == f2[1] && f1[2] == f2[2]) found = 1;
            }
            if (!found) rc = fail(2, "non-reciprocal neighbours");
        }
    /* --- hull list == {(t,k): nbr == -1} (as sets, caller indexing) --- */
    int64_t nh = 0;
    for (int64_t t = 0; t < nt; ++t)
        for (int k = 0; k < 4; ++k) nh += (m->nbr[t][k] < 0);
    if (!rc && nh != nb) rc = fail(2, "boundary list does not match nbrs == -1");
    m->nb = nh;
    m->hull = malloc(sizeof(*m->hull) * (nh ? nh : 1));
    if (!rc) {
        int64_t (*given)[3] = malloc(sizeof(*given) * nb);
        int64_t (*have)[3] = malloc(sizeof(*have) * nb);
        int64_t h = 0;
        for (int64_t t = 0; t < nt; ++t)
            for (int k = 0; k < 4; ++k)
                if (m->nbr[t][k] < 0) {
                    m->hull[h][0] = (int32_t)t;
                    m->hull[h][1] = k;
                    /* caller's local index of this face */
                    int kc = swapped[t] ? (k == 0 ? 1 : k == 1 ? 0 : k) : k;
                    have[h][0] = t; have[h][1] = kc; have[h][2] = 0; ++h;
                }
        for (int64_t b = 0; b < nb; ++b) {
            given[b][0] = bfaces[2 * b]; given[b][1] = bfaces[2 * b + 1]; given[b][2] = 0;
        }
        qsort(given, nb, sizeof *given, cmp_i64x3);
        qsort(have, nb, sizeof *have, cmp_i64x3);
        if (memcmp(given, have, sizeof(*given) * nb)) rc = fail(2, "boundary list does not match nbrs == -1");
        free(given);
        free(have);
    }
    /* --- closed hull: every directed hull edge (a,b) matched by (b,a) --- */
    if (!rc) {
        int64_t ne = 3 * nh;
        int64_t (*e)[3] = malloc(sizeof(*e) * ne);
        for (int64_t h = 0; h < nh; ++h) {
            int t = m->hull[h][0], k = m->hull[h][1];
            for (int j = 0; j < 3; ++j) {
                e[3 * h + j][0] = m->tet[t][FACE[k][j]];
                e[3 * h + j][1] = m->tet[t][FACE[k][(j + 1) % 3]];
                e[3 * h + j][2] = 0;
            }
        }
        qsort(e, ne, sizeof *e, cmp_i64x3);
        for (int64_t i = 0; i < ne && !rc; ++i) {
            if (i + 1 < ne && e[i][0] == e[i + 1][0] && e[i][1] == e[i + 1][1])
                rc = fail(2, "non-manifold hull (repeated directed edge)");
            int64_t key[3] = {e[i][1], e[i][0], 0};
            if (!rc && !bsearch(key, e, ne, sizeof *e, cmp_i64x3))
                rc = fail(2, "open hull (unmatched edge)");
        }
        free(e);
    }
    /* --- convexity: no vertex strictly outside any hull face plane
     *     (the only constraint of the method) --- */
    if (!rc) {
        char* used = calloc(nv, 1);
        for (int64_t t = 0; t < nt; ++t)
            for (int k = 0; k < 4; ++k) used[m->tet[t][k]] = 1;
        for (int64_t h = 0; h < nh && !rc; ++h) {
            int t = m->hull[h][0], k = m->hull[h][1];
            const int64_t* a = m->v[m->tet[t][FACE[k][0]]];
            const int64_t* b = m->v[m->tet[t][FACE[k][1]]];
            const int64_t* cc = m->v[m->tet[t][FACE[k][2]]];
            for (int64_t v = 0; v < nv; ++v)
                if (used[v] && orient(a, b, cc, m->v[v]) > 0) {
                    rc = fail(3, "mesh is not convex");
                    break;
                }
        }
        free(used);
    }
    free(swapped);
    if (rc) {
        tetref_mesh_destroy(m);
        return rc;
    }
    *out = m;
    return 0;
}

/* ------------------------------------------------------------- geometry -- */
typedef struct {
    int64_t S[3];   /* cone: source; parallel: direction */
    int64_t P00[3], U[3], V[3];
} snapped_angle;

static int snap_angle(const tetref_mesh* m, const tetref_geometry* g, int a,
                      snapped_angle* s) {
    const double* q = g->vecs + 12 * (int64_t)a;
    for (int i = 0; i < 3; ++i) {
        if (g->beam == 0) {
            if (snap_scalar(q[i], m->C[i], m->g, &s->S[i])) return 1;
        } else {
            double mx = fmax(fabs(q[0]), fmax(fabs(q[1]), fabs(q[2])));
            if (!(mx > 0.0)) return 1;
            s->S[i] = (int64_t)nearbyint((q[i] / mx) * 1048576.0);
        }
        if (snap_scalar(q[3 + i], m->C[i], m->g, &s->P00[i])) return 1;
        if (snap_scalar(q[6 + i], 0.0, m->g, &s->U[i])) return 1;
        if (snap_scalar(q[9 + i], 0.0, m->g, &s->V[i])) return 1;
    }
    return 0;
}

static int ray_points(const tetref_mesh* m, const tetref_geometry* g, int64_t id,
                      int64_t o[3], int64_t p[3]) {
    int64_t per = (int64_t)g->n_v * g->n_u;
    if (id < 0 || id >= per * g->n_angles) return 1;
    int a = (int)(id / per);
    int64_t rem = id % per;
    int64_t v = rem / g->n_u, u = rem % g->n_u;
    snapped_angle s;
    if (snap_angle(m, g, a, &s)) return 1;
    for (int i = 0; i < 3; ++i) {
        p[i] = s.P00[i] + u * s.U[i] + v * s.V[i];
        o[i] = (g->beam == 0) ? s.S[i] : p[i] - s.S[i];
        if (llabs(p[i]) > 2147483647LL || llabs(o[i]) > 2147483647LL) return 1;
    }
    if (o[0] == p[0] && o[1] == p[1] && o[2] == p[2]) return 1;
    return 0;
}

int tetref_ray_points(const tetref_mesh* m, const tetref_geometry* g, int64_t id,
                      int64_t o[3], int64_t p[3]) {
    return ray_points(m, g, id, o, p) ? fail(4, "bad ray / geometry") : 0;
}

/* ------------------------------------------------------------------ walk -- */
/* Is face k of tet t crossed with side sign `want` (-1 enter, +1 leave)? */
static int face_crossed(const tetref_mesh* m, int64_t t, int k, const int64_t o[3],
                        const int64_t p[3], int want) {
    const int64_t* a = m->v[m->tet[t][FACE[k][0]]];
    const int64_t* b = m->v[m->tet[t][FACE[k][1]]];
    const int64_t* c = m->v[m->tet[t][FACE[k][2]]];
    return tetref_side(o, p, a, b) == want && tetref_side(o, p, b, c) == want &&
           tetref_side(o, p, c, a) == want;
}

/* Reading R4: ray parameter of the plane of face k of tet t. */
static double face_t(const tetref_mesh* m, int64_t t, int k, const int64_t o[3],
                     const int64_t p[3]) {
    const int64_t* a = m->v[m->tet[t][FACE[k][0]]];
    const int64_t* b = m->v[m->tet[t][FACE[k][1]]];
    const int64_t* c = m->v[m->tet[t][FACE[k][2]]];
    i128 e1[3], e2[3], n[3];
    for (int i = 0; i < 3; ++i) { e1[i] = (i128)b[i] - a[i]; e2[i] = (i128)c[i] - a[i]; }
    n[0] = e1[1] * e2[2] - e1[2] * e2[1];
    n[1] = e1[2] * e2[0] - e1[0] * e2[2];
    n[2] = e1[0] * e2[1] - e1[1] * e2[0];
    i128 num = 0, den = 0;
    for (int i = 0; i < 3; ++i) {
        num += n[i] * ((i128)a[i] - o[i]);
        den += n[i] * ((i128)p[i] - o[i]);
    }
    return (double)num / (double)den; /* den != 0 for a crossed face */
}

typedef struct { int64_t crossings; int lost, stuck, hit; } walk_result;

/* Alg. 2 for one ray; visit(t, chord) is called for every element crossed. */
typedef void (*visit_fn)(void* ctx, int32_t t, double chord);

/* Step 1 of Alg. 2: the entering hull face, by scanning all of them
 * (PAPER.md:146-150).  Returns its tet (-1: the ray misses the mesh) and
 * sets *kin to the face; more than one entering face marks the ray lost. */
static int64_t entering_face(const tetref_mesh* m, const int64_t o[3], const int64_t p[3],
                             walk_result* r, int* kin) {
    int64_t t = -1;
    int n_enter = 0;
    for (int64_t h = 0; h < m->nb; ++h)
        if (face_crossed(m, m->hull[h][0], m->hull[h][1], o, p, -1)) {
            ++n_enter;
            t = m->hull[h][0];
            *kin = m->hull[h][1];
        }
    if (n_enter == 0) return -1;
    if (n_enter > 1) { r->lost = 1; return -1; }
    r->hit = 1;
    return t;
}

static int64_t entering_tet(const tetref_mesh* m, const int64_t o[3], const int64_t p[3],
                            walk_result* r) {
    int kin = -1;
    return entering_face(m, o, p, r, &kin);
}

static walk_result walk(const tetref_mesh* m, const int64_t o[3], const int64_t p[3],
                        visit_fn visit, void* ctx) {
    walk_result r = {0, 0, 0, 0};
    int kin = -1;
    int64_t t = entering_face(m, o, p, &r, &kin);
    if (t < 0) return r;                 /* "Return if i_now = -1" */
    double dx = (double)(p[0] - o[0]), dy = (double)(p[1] - o[1]), dz = (double)(p[2] - o[2]);
    double l = sqrt(dx * dx + dy * dy + dz * dz) * m->g; /* l = |R2-R1| */
    while (t >= 0) {
        if (r.crossings >= m->nt) { r.stuck = 1; return r; }
        /* step 2: the other intersected face (leaving) */
        int kout = -1, n_out = 0;
        for (int k = 0; k < 4; ++k)
            if (k != kin && face_crossed(m, t, k, o, p, +1)) { ++n_out; kout = k; }
        if (n_out != 1) { r.lost = 1; return r; }
        double t1 = face_t(m, t, kin, o, p), t2 = face_t(m, t, kout, o, p);
        double chord = l * (t2 > t1 ? t2 - t1 : 0.0);
        /* step 3 */
        visit(ctx, (int32_t)t, chord);
        r.crossings++;
        /* step 4: neighbour across the t2 face */
        int64_t n = m->nbr[t][kout];
        if (n < 0) break;
        int kn = -1;
        for (int k = 0; k < 4; ++k)
            if (m->nbr[n][k] == t) {
                /* the shared face: the node of n not on it is its local index */
                int on = 0;
                for (int j = 0; j < 4; ++j)
                    if (j != kout && m->tet[t][j] == m->tet[n][k]) on = 1;
                if (!on) kn = k;
            }
        if (kn < 0) { r.lost = 1; return r; }
        t = n;
        kin = kn;
    }
    return r;
}

/* ----------------------------------------------------------- operators -- */
typedef struct { const double* mu; double sum; } fwd_ctx;
static void fwd_visit(void* c, int32_t t, double chord) {
    fwd_ctx* f = (fwd_ctx*)c;
    f->sum += chord * f->mu[t];
}
typedef struct { double* x; double y; } bwd_ctx;
static void bwd_visit(void* c, int32_t t, double chord) {
    bwd_ctx* b = (bwd_ctx*)c;
    b->x[t] += chord * b->y;
}

static int check_geom(const tetref_mesh* m, const tetref_geometry* g) {
    if (!m || !g || !g->vecs || g->n_angles < 1 || g->n_v < 1 || g->n_u < 1 ||
        (g->beam != 0 && g->beam != 1))
        return fail(1, "bad geometry arguments");
    for (int a = 0; a < g->n_angles; ++a) {
        snapped_angle s;
        if (snap_angle(m, g, a, &s)) return fail(4, "geometry outside grid span");
    }
    return 0;
}

static int nthreads_of(int n) {
#ifdef _OPENMP
    return n > 0 ? n : omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

int tetref_project(const tetref_mesh* m, const tetref_geometry* g, const double* mu,
                   int64_t n_rays, const int64_t* ids, double* out, int nthreads,
                   tetref_stats* st) {
    int rc = check_geom(m, g);
    if (rc) return rc;
    int64_t total = (int64_t)g->n_angles * g->n_v * g->n_u;
    if (!ids) n_rays = total;
    int64_t hit = 0, cr = 0, lost = 0, stuck = 0, mx = 0, bad = 0;
    int nth = nthreads_of(nthreads);
#pragma omp parallel for schedule(dynamic, 16) num_threads(nth) \
    reduction(+ : hit, cr, lost, stuck, bad) reduction(max : mx)
    for (int64_t i = 0; i < n_rays; ++i) {
        int64_t o[3], p[3];
        if (ray_points(m, g, ids ? ids[i] : i, o, p)) { ++bad; continue; }
        fwd_ctx c = {mu, 0.0};
        walk_result r = walk(m, o, p, fwd_visit, &c);
        out[i] = c.sum;
        hit += r.hit; cr += r.crossings; lost += r.lost; stuck += r.stuck;
        if (r.crossings > mx) mx = r.crossings;
    }
    if (bad) return fail(4, "ray outside grid span");
    if (st) {
        st->rays = n_rays; st->rays_hit = hit; st->crossings = cr;
        st->lost = lost; st->stuck = stuck; st->max_crossings = mx;
    }
    return 0;
}

int tetref_backproject(const tetref_mesh* m, const tetref_geometry* g, const double* y,
                       int64_t n_rays, const int64_t* ids, double* x, int nthreads,
                       tetref_stats* st) {
    int rc = check_geom(m, g);
    if (rc) return rc;
    int64_t total = (int64_t)g->n_angles * g->n_v * g->n_u;
    if (!ids) n_rays = total;
    int nth = nthreads_of(nthreads);
    /* private per-thread accumulators merged in a fixed order */
    while (nth > 1 && (double)nth * m->nt * 8.0 > 4e9) --nth;
    double* buf = calloc((size_t)nth * m->nt, sizeof(double));
    if (!buf) return fail(5, "out of memory");
    int64_t hit = 0, cr = 0, lost = 0, stuck = 0, mx = 0, bad = 0;
#pragma omp parallel num_threads(nth) reduction(+ : hit, cr, lost, stuck, bad) \
    reduction(max : mx)
    {
        int me = 0;
#ifdef _OPENMP
        me = omp_get_thread_num();
#endif
        double* mine = buf + (size_t)me * m->nt;
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n_rays; ++i) {
            int64_t o[3], p[3];
            if (ray_points(m, g, ids ? ids[i] : i, o, p)) { ++bad; continue; }
            bwd_ctx c = {mine, y[i]};
            walk_result r = walk(m, o, p, bwd_visit, &c);
            hit += r.hit; cr += r.crossings; lost += r.lost; stuck += r.stuck;
            if (r.crossings > mx) mx = r.crossings;
        }
    }
    for (int th = 0; th < nth; ++th)
        for (int64_t t = 0; t < m->nt; ++t) x[t] += buf[(size_t)th * m->nt + t];
    free(buf);
    if (bad) return fail(4, "ray outside grid span");
    if (st) {
        st->rays = n_rays; st->rays_hit = hit; st->crossings = cr;
        st->lost = lost; st->stuck = stuck; st->max_crossings = mx;
    }
    return 0;
}

/* ------------------------------------------------ NEXT-1: Alg. 1 + Alg. 2 -- */
#define REAL double
#define SFX _f64
#include "tetref_mt.inc"
#undef REAL
#undef SFX
#define REAL float
#define SFX _f32
#include "tetref_mt.inc"
#undef REAL
#undef SFX

static walk_result mt_walk(const tetref_mesh* m, const int64_t o[3], const int64_t p[3],
                           const tetref_mt_options* opt, visit_fn visit, void* ctx,
                           int64_t* esc) {
    return opt->single ? mt_walk_f32(m, o, p, opt, visit, ctx, esc)
                       : mt_walk_f64(m, o, p, opt, visit, ctx, esc);
}

static int check_mt(const tetref_mt_options* opt) {
    if (!opt || !(opt->eps0 > 0) || !(opt->eps_growth > 1) || opt->max_escalations < 0)
        return fail(1, "bad MT options");
    return 0;
}

static void fill_mt_stats(tetref_mt_stats* st, int64_t n, int64_t hit, int64_t cr, int64_t lost,
                          int64_t stuck, int64_t mx, int64_t esc) {
    if (!st) return;
    st->rays = n; st->rays_hit = hit; st->crossings = cr; st->lost = lost;
    st->stuck = stuck; st->max_crossings = mx; st->escalations = esc;
}

int tetref_mt_project(const tetref_mesh* m, const tetref_geometry* g, const double* mu,
                      int64_t n_rays, const int64_t* ids, double* out,
                      const tetref_mt_options* opt, int nthreads, tetref_mt_stats* st) {
    int rc = check_geom(m, g);
    if (!rc) rc = check_mt(opt);
    if (rc) return rc;
    if (!ids) n_rays = (int64_t)g->n_angles * g->n_v * g->n_u;
    int64_t hit = 0, cr = 0, lost = 0, stuck = 0, mx = 0, bad = 0, esc = 0;
    int nth = nthreads_of(nthreads);
#pragma omp parallel for schedule(dynamic, 16) num_threads(nth) \
    reduction(+ : hit, cr, lost, stuck, bad, esc) reduction(max : mx)
    for (int64_t i = 0; i < n_rays; ++i) {
        int64_t o[3], p[3];
        if (ray_points(m, g, ids ? ids[i] : i, o, p)) { ++bad; continue; }
        fwd_ctx c = {mu, 0.0};
        walk_result r = mt_walk(m, o, p, opt, fwd_visit, &c, &esc);
        out[i] = c.sum;
        hit += r.hit; cr += r.crossings; lost += r.lost; stuck += r.stuck;
        if (r.crossings > mx) mx = r.crossings;
    }
    if (bad) return fail(4, "ray outside grid span");
    fill_mt_stats(st, n_rays, hit, cr, lost, stuck, mx, esc);
    return 0;
}

int tetref_mt_backproject(const tetref_mesh* m, const tetref_geometry* g, const double* y,
                          int64_t n_rays, const int64_t* ids, double* x,
                          const tetref_mt_options* opt, int nthreads, tetref_mt_stats* st) {
    int rc = check_geom(m, g);
    if (!rc) rc = check_mt(opt);
    if (rc) return rc;
    if (!ids) n_rays = (int64_t)g->n_angles * g->n_v * g->n_u;
    int nth = nthreads_of(nthreads);
    while (nth > 1 && (double)nth * m->nt * 8.0 > 4e9) --nth;
    double* buf = calloc((size_t)nth * m->nt, sizeof(double));
    if (!buf) return fail(5, "out of memory");
    int64_t hit = 0, cr = 0, lost = 0, stuck = 0, mx = 0, bad = 0, esc = 0;
#pragma omp parallel num_threads(nth) reduction(+ : hit, cr, lost, stuck, bad, esc) \
    reduction(max : mx)
    {
        int me = 0;
#ifdef _OPENMP
        me = omp_get_thread_num();
#endif
        double* mine = buf + (size_t)me * m->nt;
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n_rays; ++i) {
            int64_t o[3], p[3];
            if (ray_points(m, g, ids ? ids[i] : i, o, p)) { ++bad; continue; }
            bwd_ctx c = {mine, y[i]};
            walk_result r = mt_walk(m, o, p, opt, bwd_visit, &c, &esc);
            hit += r.hit; cr += r.crossings; lost += r.lost; stuck += r.stuck;
            if (r.crossings > mx) mx = r.crossings;
        }
    }
    for (int th = 0; th < nth; ++th)
        for (int64_t t = 0; t < m->nt; ++t) x[t] += buf[(size_t)th * m->nt + t];
    free(buf);
    if (bad) return fail(4, "ray outside grid span");
    fill_mt_stats(st, n_rays, hit, cr, lost, stuck, mx, esc);
    return 0;
}

typedef struct { int32_t* tets; double* chords; int64_t n, cap; } path_ctx;
static void path_visit(void* c, int32_t t, double chord) {
    path_ctx* p = (path_ctx*)c;
    if (p->n < p->cap) { p->tets[p->n] = t; p->chords[p->n] = chord; }
    p->n++;
}

int tetref_ray_path(const tetref_mesh* m, const tetref_geometry* g, int64_t id,
                    int64_t cap, int32_t* tets, double* chords, int64_t* n_out) {
    int rc = check_geom(m, g);
    if (rc) return rc;
    int64_t o[3], p[3];
    if (ray_points(m, g, id, o, p)) return fail(4, "bad ray id / geometry");
    path_ctx c = {tets, chords, 0, cap};
    walk_result r = walk(m, o, p, path_visit, &c);
    *n_out = c.n;
    if (r.lost) return fail(6, "lost ray");
    if (r.stuck) return fail(7, "stuck ray");
    return 0;
}
