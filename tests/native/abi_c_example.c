/* tests/native/abi_c_example.c -- the boundary used from plain C (no Python,
 * no torch): one tetrahedron, one parallel ray along +x through
 * (y, z) = (0.25, 0.25) -- the closed form of SPEC.md:152 (chord 0.5), also
 * pinned in the oracle (tests/test_oracle_mt_pins.py::
 * test_tetra_and_cube_closed_forms).  Host buffers throughout; a plan, its
 * projection and backprojection.  Prints one "key value" per line; exits 0
 * when every call returned a status (it never aborts). */
#include <stdio.h>

#include "../../include/tetproj.h"

int main(void) {
    const double verts[12] = {0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1};
    const int32_t tets[4] = {0, 1, 2, 3};
    const int32_t nbrs[4] = {-1, -1, -1, -1};
    const int32_t bfaces[8] = {0, 0, 0, 1, 0, 2, 0, 3};
    tet_mesh_t m = NULL;
    tet_status s = tet_mesh_create(verts, 4, tets, nbrs, 1, bfaces, 4, 0, TET_F_FIX_ORIENTATION, &m);
    printf("create %d\n", (int)s);
    if (s != TET_OK) {
        printf("error %s\n", tet_last_error());
        return 0;
    }
    /* parallel beam: ray direction | pixel (0,0) centre | u-step | v-step */
    const double vecs[12] = {1, 0, 0, -1, 0.25, 0.25, 0, 1, 0, 0, 0, 1};
    const tet_geometry g = {TET_BEAM_PARALLEL, 1, 1, 1, vecs};
    tet_plan_t p = NULL;
    s = tet_plan_create(m, &g, NULL, NULL, &p);
    printf("plan %d\n", (int)s);
    if (s != TET_OK) {
        printf("error %s\n", tet_last_error());
        tet_mesh_destroy(m);
        return 0;
    }
    const float mu = 2.0f, y = 3.0f;
    float proj = -1.0f, x = -1.0f;
    tet_stats st;
    s = tet_plan_project(p, &mu, &proj, NULL, &st);
    printf("project %d\nproj %.9g\ncrossings %llu\nlost %llu\n", (int)s, proj,
           (unsigned long long)st.crossings, (unsigned long long)st.lost);
    s = tet_plan_backproject(p, &y, &x, 0, NULL, &st);
    printf("backproject %d\nx %.9g\n", (int)s, x);
    s = tet_project(m, &g, &mu, &proj, NULL, NULL);   /* the plan-less call */
    printf("project_noplan %d\nproj_noplan %.9g\n", (int)s, proj);
    tet_plan_destroy(p, NULL);
    tet_mesh_destroy(m);
    return 0;
}
