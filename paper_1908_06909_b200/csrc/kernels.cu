// kernels.cu -- sm_100a kernels of libtetproj.
//
//   entry_setup_kernel / entry_small_kernel / entry_raster_kernel
//                     hull-entry finder: per (hull face,
//                     angle) item, exact affine side coefficients, then an
//                     exact test of every pixel in the face's detector
//                     footprint (a thread per small item, a warp per large
//                     one); writes entry[ray] = tet<<2 | k.  A plan
//                     (api.cu, tet_plan_create) keeps that map for its scan.
//   entry_bvh_kernel / entry_rtree_kernel
//                     the per-ray alternatives (binary BVH, the paper's
//                     R*-tree); same exact decision.
//   trace_kernel<B,..> ray walk (a4) + forward accumulate (a5, B=false) or
//                     backprojection scatter (a6, B=true).  Alg. 2 of the
//                     paper with exact sign decisions:
//                     walk_ray_ft (16-B face tags, default) or walk_ray
//                     (32-B records: exact-heavy scans, huge meshes).
//   mt_trace_kernel   the paper's own epsilon-MT traversal (NEXT-1 study).
//   gather / scatter  caller order <-> internal SFC order (K4).
//
// Exactness (R2-R4): side(a,b) = sign det[a-o, b-o, p-o] on the
// integer grid, symbolically perturbed.  The hot loop evaluates it in fp64
// in a per-ray shear frame (2 FMAs per side) and certifies the sign with a
// static error bound tau; only |side| <= tau falls back to an int128
// evaluation of the determinant and the 9-term SoS table.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <cmath>

#include "internal.h"

namespace tetproj {

typedef __int128 i128;

// Debug builds (-DTETPROJ_DEBUG, libtetproj_debug.so) trap on any gathered
// index outside its array: compute-sanitizer is unavailable on this pool, so
// the bounds are checked by the kernels themselves.
#ifdef TETPROJ_DEBUG
#define DBG_CHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define DBG_CHECK(cond) do { } while (0)
#endif

// Walker compile-time knobs (A/B builds, profiles/README.md): uniform frames
// in the backward walk; the forward walk's rare exact path as one call per
// step (1) or one call per uncertified sign (0).
#ifndef TRACE_BWD_UNI
#define TRACE_BWD_UNI 1
#endif
#ifndef TRACE_BWD_WY32
#define TRACE_BWD_WY32 1
#endif
#ifndef TRACE_BWD_VTX_SPLIT
#define TRACE_BWD_VTX_SPLIT 0
#endif
#ifndef TRACE_BWD_LATE_LOADS
#define TRACE_BWD_LATE_LOADS 1
#endif
#ifndef TRACE_FWD_LATE_LOADS
#define TRACE_FWD_LATE_LOADS 1
#endif
#ifndef TRACE_BWD_ONECALL
#define TRACE_BWD_ONECALL 0
#endif
#ifndef TRACE_PAR_UNI
#define TRACE_PAR_UNI 1
#endif
#ifndef TRACE_EMPTY_EXIT
#define TRACE_EMPTY_EXIT 1
#endif
#ifndef TRACE_HEAVY_KEEP_RAY
#define TRACE_HEAVY_KEEP_RAY 1
#endif
// exact-heavy scans on the FT16 walk too (1) or on the record walk (0)
#ifndef TRACE_HEAVY_FT
#define TRACE_HEAVY_FT 0
#endif
// early exit and shear-axis vote per WARP instead of per block: no block
// barrier at the start of the walk (c3 1.671e11 -> 1.678e11; 0 = per block)
#ifndef TRACE_WARP_VOTE
#define TRACE_WARP_VOTE 1
#endif
// footprints of at most this many pixels go to entry_small_kernel (thread
// per item); 0 sends every item to the warp raster.  c4a (36,300 hull faces
// of ~1 px at lattice pitch): entry 0.88 -> 0.34 ms per step at 32 px; c2
// (~50-px boxes) 0.58 -> 0.59, c3 unchanged; 128 / 256 px cost c2 0.75 / 1.02
#ifndef ENTRY_SMALL_PX
#define ENTRY_SMALL_PX 32u
#endif
#ifndef ENTRY_GUIDE
#define ENTRY_GUIDE 4u
#endif
#ifndef TRACE_BAND_ORDER
#define TRACE_BAND_ORDER 1
#endif
#ifndef TRACE_BAND_BYTES_PER_TET
#define TRACE_BAND_BYTES_PER_TET 32
#endif
// angles per band group of the backward walk on L2-exceeding meshes: 2 for
// round 1's record walk, 4 for the FT16 walk (c5 backward 558 -> 548 ms;
// 1: 591, 8: 552, 16: 558), profiles/README.md
// forward: all of a launch's angles per band (plain band order)
#ifndef TRACE_FWD_BAND_GROUP
#define TRACE_FWD_BAND_GROUP (1 << 20)
#endif
#ifndef TRACE_BWD_BAND_GROUP
#define TRACE_BWD_BAND_GROUP 4
#endif
#ifndef TRACE_EXACT_ONECALL
#define TRACE_EXACT_ONECALL 1
#endif


// ------------------------------------------------------------ exact -----
// Reading R2: sign of det[a-o, b-o, p-o] under o -> o + (d, d^2, d^4),
// p -> p + (d, d^2, d^4) + (d^8, d^16, d^32): first non-zero of
// [det, -(ExD)x, -(ExD)y, -(ExD)z, (AxB)x, -Ez, Ey, (AxB)y, -Ex].
__device__ __noinline__ int sos_side(long long ax, long long ay, long long az,
                                     long long bx, long long by, long long bz,
                                     long long ox, long long oy, long long oz,
                                     long long px, long long py, long long pz) {
    const long long Ax = ax - ox, Ay = ay - oy, Az = az - oz;   // |.| < 2^33
    const long long Bx = bx - ox, By = by - oy, Bz = bz - oz;
    const long long Dx = px - ox, Dy = py - oy, Dz = pz - oz;
    const long long Ex = bx - ax, Ey = by - ay, Ez = bz - az;
    const i128 cx = (i128)Ay * Bz - (i128)Az * By;
    const i128 cy = (i128)Az * Bx - (i128)Ax * Bz;
    const i128 cz = (i128)Ax * By - (i128)Ay * Bx;
    const i128 det = cx * Dx + cy * Dy + cz * Dz;
    if (det != 0) return det > 0 ? 1 : -1;
    const i128 ed0 = (i128)Ey * Dz - (i128)Ez * Dy;
    if (ed0 != 0) return ed0 > 0 ? -1 : 1;
    const i128 ed1 = (i128)Ez * Dx - (i128)Ex * Dz;
    if (ed1 != 0) return ed1 > 0 ? -1 : 1;
    const i128 ed2 = (i128)Ex * Dy - (i128)Ey * Dx;
    if (ed2 != 0) return ed2 > 0 ? -1 : 1;
    if (cx != 0) return cx > 0 ? 1 : -1;
    if (Ez != 0) return Ez > 0 ? -1 : 1;
    if (Ey != 0) return Ey > 0 ? 1 : -1;
    if (cy != 0) return cy > 0 ? 1 : -1;
    if (Ex != 0) return Ex > 0 ? -1 : 1;
    return 0;
}

struct RayPts {
    long long ox, oy, oz, px, py, pz;
};

__device__ __forceinline__ RayPts ray_points(const AngleGeom& G, int beam, int u, int v) {
    RayPts r;
    r.px = G.p00[0] + (long long)u * G.du[0] + (long long)v * G.dv[0];
    r.py = G.p00[1] + (long long)u * G.du[1] + (long long)v * G.dv[1];
    r.pz = G.p00[2] + (long long)u * G.du[2] + (long long)v * G.dv[2];
    if (beam == TET_BEAM_CONE) {
        r.ox = G.o[0]; r.oy = G.o[1]; r.oz = G.o[2];
    } else {
        r.ox = r.px - G.o[0]; r.oy = r.py - G.o[1]; r.oz = r.pz - G.o[2];
    }
    return r;
}

// Exact sign for vertex ids ia, ib of the ray (angle a, pixel u, v): rare path.
__device__ __noinline__ int exact_side_ids(const int4* __restrict__ vtx,
                                           const AngleGeom* __restrict__ ang, int beam,
                                           int a, int u, int v, int ia, int ib) {
    const AngleGeom G = ang[a];
    const RayPts r = ray_points(G, beam, u, v);
    const int4 A = __ldg(vtx + ia), B = __ldg(vtx + ib);
    return sos_side(A.x, A.y, A.z, B.x, B.y, B.z, r.ox, r.oy, r.oz, r.px, r.py, r.pz);
}

// The walker's rare exact path: the thread's own ray is recomputed from its
// grid position (same mapping as trace_kernel), so (a, u, v) need not stay
// live in registers across the walk loop.
// Walker blocks are BX x BY warp tiles of (1 << tw_log) x (32 >> tw_log) pixels.
// Block -> (tile column bx, tile row by, angle a) of a walk launch (grid =
// (tiles_u x tiles_v, angles)).  TRACE_BAND_ORDER: blocks are dispatched band
// by band -- a band is one row of tiles, roughly one z-slab of the mesh for
// a scan about z -- with all the launch's angles of a band before the next
// band, so the resident blocks share one slab of the mesh and its tags stay
// in L2 across angles (c5: angle by angle, each angle streamed the whole
// 360-MB mesh through L2, ~4 B of DRAM reads per crossing).
__device__ __forceinline__ void block_tile(int tiles_u, int group, int& bx, int& by, int& a) {
    // group = 0: angle by angle.  group = G > 0: angles in groups of G, and
    // within a group band by band (all G angles of a band before the next
    // band); G >= the launch's angles is plain band order.
    if (group > 0) {
        const unsigned L = blockIdx.y * gridDim.x + blockIdx.x;   // dispatch order
        const unsigned na = gridDim.y, tiles = gridDim.x;
        const unsigned G = min((unsigned)group, na);
        const unsigned full = na / G;                    // complete groups
        unsigned ag, g, Lg;
        if (L < full * G * tiles) {
            ag = L / (G * tiles);
            g = G;
            Lg = L - ag * G * tiles;
        } else {                                         // last, partial group
            ag = full;
            g = na - full * G;
            Lg = L - full * G * tiles;
        }
        const unsigned r = Lg / (unsigned)tiles_u;
        bx = (int)(Lg - r * (unsigned)tiles_u);
        a = (int)(ag * G + r % g);
        by = (int)(r / g);
    } else {
        bx = blockIdx.x % tiles_u;
        by = blockIdx.x / tiles_u;
        a = blockIdx.y;
    }
}

// tile_code = tw_log | group << 4 (the walk launch's tile width and block order)
// BAND (compile time): band-ordered launch, tile_code = tw_log | group << 4;
// otherwise tile_code = tw_log and the mapping reads blockIdx directly (the
// non-band kernels keep (a, bx, by) rematerialisable from blockIdx: with the
// runtime decode, c3 lost 1.5 % forward / 2.7 % backward to extra spills).
template <int BX, int BY, bool BAND>
__device__ __forceinline__ void thread_pixel(int nu, int tile_code, int& a, int& u, int& v) {
    const int tw_log = BAND ? (tile_code & 15) : tile_code;
    const int tw = 1 << tw_log, th = 32 >> tw_log;
    const int tiles_u = (nu + BX * tw - 1) / (BX * tw);
    int bx, by;
    if (BAND) {
        block_tile(tiles_u, tile_code >> 4, bx, by, a);
    } else {
        bx = blockIdx.x % tiles_u;
        by = blockIdx.x / tiles_u;
        a = blockIdx.y;
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    u = bx * BX * tw + (w % BX) * tw + (lane & (tw - 1));
    v = by * BY * th + (w / BX) * th + (lane >> tw_log);
}

// All the uncertified signs of one walker step in one call: bit k of the
// returned code is [side(apex, slot k) < 0], exact for the k in `mask`, taken
// from `neg` otherwise (one call per step keeps the caller-saved register
// traffic of the rare path to one save/restore).
template <int BX, int BY, bool BAND>
__device__ __noinline__ unsigned exact_neg_here(const int4* __restrict__ vtx,
                                                const AngleGeom* __restrict__ ang, int beam,
                                                int nu, int tw_log, unsigned mask, unsigned neg,
                                                int iap, int id0, int id1, int id2) {
    int a, u, v;
    thread_pixel<BX, BY, BAND>(nu, tw_log, a, u, v);
    const RayPts r = ray_points(ang[a], beam, u, v);
    const int4 A = __ldg(vtx + iap);
    const int ids[3] = {id0, id1, id2};
    for (int k = 0; k < 3; ++k) {
        if (!(mask >> k & 1u)) continue;
        const int4 B = __ldg(vtx + ids[k]);
        const int sg = sos_side(A.x, A.y, A.z, B.x, B.y, B.z, r.ox, r.oy, r.oz, r.px, r.py, r.pz);
        neg = (neg & ~(1u << k)) | (sg < 0 ? 1u << k : 0u);
    }
    return neg;
}

// The exact-heavy walk shape (128 registers) keeps its ray's grid points and
// passes them (TRACE_HEAVY_KEEP_RAY): no pixel decode, AngleGeom load or
// ray_points per call.
__device__ __noinline__ unsigned exact_neg_ray(const int4* __restrict__ vtx, long long ox,
                                               long long oy, long long oz, long long px,
                                               long long py, long long pz, unsigned mask,
                                               unsigned neg, int iap, int id0, int id1, int id2) {
    const int4 A = __ldg(vtx + iap);
    const int ids[3] = {id0, id1, id2};
    for (int k = 0; k < 3; ++k) {
        if (!(mask >> k & 1u)) continue;
        const int4 B = __ldg(vtx + ids[k]);
        const int sg = sos_side(A.x, A.y, A.z, B.x, B.y, B.z, ox, oy, oz, px, py, pz);
        neg = (neg & ~(1u << k)) | (sg < 0 ? 1u << k : 0u);
    }
    return neg;
}

// One uncertified sign (the backward walk calls this per sign: the wider
// exact_neg_here call makes it spill the RED weight in the loop).
template <int BX, int BY, bool BAND>
__device__ __noinline__ int exact_side_here(const int4* __restrict__ vtx,
                                            const AngleGeom* __restrict__ ang, int beam, int nu,
                                            int tw_log, int ia, int ib) {
    int a, u, v;
    thread_pixel<BX, BY, BAND>(nu, tw_log, a, u, v);
    return exact_side_ids(vtx, ang, beam, a, u, v, ia, ib);
}

// ------------------------------------------------------------ frame -----
// Shear frame of a ray (the projection along the ray onto the coordinate
// plane orthogonal to its dominant axis k):
//     A = X - o,  x' = A_k1 - (D_k1/D_k) A_k,  y' = A_k2 - (D_k2/D_k) A_k,  z' = A_k
// so that det[a-o, b-o, p-o] = D_k (x'_a y'_b - y'_a x'_b).  (k1,k2,k) is a
// cyclic permutation of (x,y,z), with k1,k2 swapped when D_k < 0, which makes
// side2() carry the sign of the determinant itself.  The computed side2() is
// within ~26 eps Amax^2 of det/D_k (Amax >= |X - o| for every vertex), far
// below tau = 2^-40 Amax^2.  z' of the crossing
// points gives the chord: |D|/D_k * dz' * g.
// Shear frame of one ray (dominant axis k, sigma = sign D_k):
//   z' = sigma X_k (absolute: chords only use differences), so z' grows along the ray
//   x' = (X_k1 - c1) - sx z',  sx = D_k1/|D_k|,  c1 = o_k1 - sx sigma o_k   (y' alike)
// i.e. x' = A_k1 - (D_k1/D_k) A_k with A = X - o: the ray is the z' axis and
// det[a-o, b-o, p-o] = D_k (x'_a y'_b - y'_a x'_b).  Error bound and tau: DESIGN.md §5.
struct Frame {
    double sx, sy;         // D_k1/|D_k|, D_k2/|D_k|
    double c1, c2;         // o_k1 - sx sigma o_k, o_k2 - sy sigma o_k
    double tau;            // sign-filter threshold
    double scale;          // |D|/|D_k| * g  (> 0)
    int k1, k2, k3;        // coordinate permutation
    int neg;               // sigma < 0
};

__device__ __forceinline__ double comp(long long x, long long y, long long z, int k) {
    return (double)(k == 0 ? x : (k == 1 ? y : z));
}

__device__ __forceinline__ void make_frame(const RayPts& r, double rmax, double g, Frame& F) {
    const long long Dx = r.px - r.ox, Dy = r.py - r.oy, Dz = r.pz - r.oz;
    const long long ax = Dx < 0 ? -Dx : Dx, ay = Dy < 0 ? -Dy : Dy, az = Dz < 0 ? -Dz : Dz;
    int k = 2;
    if (ax >= ay && ax >= az) k = 0;
    else if (ay >= az) k = 1;
    int k1 = k == 0 ? 1 : (k == 1 ? 2 : 0);
    int k2 = k == 0 ? 2 : (k == 1 ? 0 : 1);
    const double dk = comp(Dx, Dy, Dz, k);
    if (dk < 0) { const int tmp = k1; k1 = k2; k2 = tmp; }
    F.k1 = k1; F.k2 = k2; F.k3 = k;
    F.neg = dk < 0;
    const double adk = fabs(dk);
    F.sx = comp(Dx, Dy, Dz, k1) / adk;
    F.sy = comp(Dx, Dy, Dz, k2) / adk;
    const double so3 = F.neg ? -comp(r.ox, r.oy, r.oz, k) : comp(r.ox, r.oy, r.oz, k);
    F.c1 = fma(-F.sx, so3, comp(r.ox, r.oy, r.oz, k1));
    F.c2 = fma(-F.sy, so3, comp(r.ox, r.oy, r.oz, k2));
    const double ox = (double)r.ox, oy = (double)r.oy, oz = (double)r.oz;
    const double amax = sqrt(ox * ox + oy * oy + oz * oz) + rmax;
    F.tau = amax * amax * 0x1p-40;
    const double dx = (double)Dx, dy = (double)Dy, dz = (double)Dz;
    F.scale = sqrt(dx * dx + dy * dy + dz * dz) / adk * g;
}

// Branch-free selects (the ternary chains compiled to divergent branches).
__device__ __forceinline__ int selp(int a, int b, bool p) {
    int r;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\tselp.b32 %0, %1, %2, q;\n\t}"
        : "=r"(r) : "r"(a), "r"(b), "r"((int)p));
    return r;
}

__device__ __forceinline__ int icomp(const int4 v, int k) {
    return selp(v.x, selp(v.y, v.z, k == 1), k == 0);
}

// Per-ray streams (entry map, y, proj: 377 MB each per c3 step, touched once)
// go through L2 with the evict-first policy (ld/st .cs) so they do not
// displace the mesh's face tags (TRACE_STREAM_HINTS, A/B knob).
#ifndef TRACE_STREAM_HINTS
#define TRACE_STREAM_HINTS 1
#endif
template <class V>
__device__ __forceinline__ V ld_stream(const V* p) {
    if (TRACE_STREAM_HINTS) return __ldcs(p);
    return *p;
}
template <class V>
__device__ __forceinline__ void st_stream(V* p, V v) {
    if (TRACE_STREAM_HINTS) __stcs(p, v);
    else *p = v;
}

// Backprojection RED with an L2 evict-last policy on the accumulator lines
// (TRACE_RED_EVICT_LAST, A/B knob): on meshes whose tags exceed the L2 the
// accumulator competes with the tag stream.
#ifndef TRACE_RED_EVICT_LAST
#define TRACE_RED_EVICT_LAST 1
#endif
#ifndef TRACE_TAG_EVICT_LAST
#define TRACE_TAG_EVICT_LAST 0
#endif
// FT16 tag load, optionally with an L2 evict-last policy (A/B knob)
__device__ __forceinline__ int4 ld_tag(const int4* p) {
#if TRACE_TAG_EVICT_LAST
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    int4 r;
    asm volatile("ld.global.nc.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
    return r;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ void red_acc(double* p, double v) {
#if TRACE_RED_EVICT_LAST
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" :: "l"(p), "d"(v), "l"(pol) : "memory");
#else
    atomicAdd(p, v);
#endif
}

// reciprocal: MUFU approximation (~2^-23) + one fp64 Newton step (~2^-46);
// TRACE_RCP_NEWTON = 0 keeps the bare approximation (A/B knob)
#ifndef TRACE_RCP_NEWTON
#define TRACE_RCP_NEWTON 1
#endif
__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return TRACE_RCP_NEWTON ? r * fma(-x, r, 2.0) : r;
}

__device__ __forceinline__ void xform(const Frame& F, const int4 v, double& x, double& y,
                                      double& z) {
    const int zk = icomp(v, F.k3);
    z = (double)(F.neg ? -zk : zk);
    x = fma(-F.sx, z, (double)icomp(v, F.k1) - F.c1);
    y = fma(-F.sy, z, (double)icomp(v, F.k2) - F.c2);
}

// Compile-time axis variants of the shear frame: AX = 2*k + swap (k = shear
// axis, swap = D_k < 0) for AX < 6; AX = 6 is the generic per-ray frame.  A
// block uses a fixed variant when its tile's rays are all dominated by the
// same axis with the same sign (trace_kernel), which removes the per-vertex
// component selects and the permutation registers.
template <int AX>
struct Axis {
    static constexpr int k = AX >> 1;
    static constexpr int c1 = k == 0 ? 1 : (k == 1 ? 2 : 0);
    static constexpr int c2 = k == 0 ? 2 : (k == 1 ? 0 : 1);
    static constexpr int K1 = (AX & 1) ? c2 : c1;
    static constexpr int K2 = (AX & 1) ? c1 : c2;
};

template <int C>
__device__ __forceinline__ long long pick(long long x, long long y, long long z) {
    return C == 0 ? x : (C == 1 ? y : z);
}

template <int C>
__device__ __forceinline__ int pick4(const int4 v) {
    return C == 0 ? v.x : (C == 1 ? v.y : v.z);
}

// Frame with a FIXED axis (k, K1, K2); tau carries the (1 + |sx| + |sy|)^2
// growth of the shear coordinates when k is not the ray's dominant axis.
template <int AX>
__device__ __forceinline__ void make_frame_ax(const RayPts& r, double rmax, double g, Frame& F) {
    if constexpr (AX == 6) {
        make_frame(r, rmax, g, F);
    } else {
        using A = Axis<AX>;
        const long long Dx = r.px - r.ox, Dy = r.py - r.oy, Dz = r.pz - r.oz;
        // AX & 1 <=> D_k < 0 (the block vote guarantees the sign)
        const double adk = fabs((double)pick<A::k>(Dx, Dy, Dz));
        F.sx = (double)pick<A::K1>(Dx, Dy, Dz) / adk;
        F.sy = (double)pick<A::K2>(Dx, Dy, Dz) / adk;
        const double o3 = (double)pick<A::k>(r.ox, r.oy, r.oz);
        const double so3 = (AX & 1) ? -o3 : o3;
        F.c1 = fma(-F.sx, so3, (double)pick<A::K1>(r.ox, r.oy, r.oz));
        F.c2 = fma(-F.sy, so3, (double)pick<A::K2>(r.ox, r.oy, r.oz));
        F.neg = AX & 1;
        const double ox = (double)r.ox, oy = (double)r.oy, oz = (double)r.oz;
        const double amax = (sqrt(ox * ox + oy * oy + oz * oz) + rmax) *
                            (1.0 + fabs(F.sx) + fabs(F.sy)) * 0.5;
        F.tau = amax * amax * 0x1p-38;
        const double dx = (double)Dx, dy = (double)Dy, dz = (double)Dz;
        F.scale = sqrt(dx * dx + dy * dy + dz * dz) / adk * g;
        F.k1 = A::K1; F.k2 = A::K2; F.k3 = A::k;
    }
}

template <int AX>
__device__ __forceinline__ void xform_ax(const Frame& F, const int4 v, double& x, double& y,
                                         double& z) {
    if constexpr (AX == 6) {
        xform(F, v, x, y, z);
    } else {
        using A = Axis<AX>;
        const double zz = (double)pick4<A::k>(v);
        z = (AX & 1) ? -zz : zz;
        x = fma(-F.sx, z, (double)pick4<A::K1>(v) - F.c1);
        y = fma(-F.sy, z, (double)pick4<A::K2>(v) - F.c2);
    }
}

// Block-uniform half of the frame (one per angle, a __grid_constant__ kernel
// parameter indexed by blockIdx.y, so it lives in uniform registers and costs
// the walk loop no per-thread registers -- the per-ray frame spilled at the
// forward's 80-register cap):
//   cone (UNI = 1): the frame origin is the source S, shared by every ray of
//     the angle: z' = sigma (X_k - S_k), x' = (X_k1 - S_k1) - sx z' (y' alike);
//     per ray only sx, sy.  X - S is exact in fp64, so x' has one rounding.
//   parallel (UNI = 2): every ray has direction d: sx, sy, scale uniform;
//     per ray only c1, c2 (z' absolute as in the generic frame).
// tau is uniform: the host bounds (|o| + rmax) over the angle's rays and
// (1 + |sx| + |sy|)/2 <= 2.5 (the block vote admits |D_k1|, |D_k2| <= 2 |D_k|).
template <int AX, int UNI>
__device__ __forceinline__ void make_frame_uni(const RayPts& r, const UniFrame& U, Frame& F) {
    using A = Axis<AX>;
    if constexpr (UNI == 1) {
        const long long Dx = r.px - r.ox, Dy = r.py - r.oy, Dz = r.pz - r.oz;
        const double adk = fabs((double)pick<A::k>(Dx, Dy, Dz));
        F.sx = (double)pick<A::K1>(Dx, Dy, Dz) / adk;
        F.sy = (double)pick<A::K2>(Dx, Dy, Dz) / adk;
    } else {
        const double o3 = (double)pick<A::k>(r.ox, r.oy, r.oz);
        const double so3 = (AX & 1) ? -o3 : o3;
        F.c1 = fma(-U.q[0], so3, (double)pick<A::K1>(r.ox, r.oy, r.oz));
        F.c2 = fma(-U.q[1], so3, (double)pick<A::K2>(r.ox, r.oy, r.oz));
    }
}

template <int AX, int UNI>
__device__ __forceinline__ void xform_uni(const Frame& F, const UniFrame& U, const int4 v,
                                          double& x, double& y, double& z) {
    using A = Axis<AX>;
    if constexpr (UNI == 1) {
        const double zz = (double)pick4<A::k>(v) - U.q[A::k];
        z = (AX & 1) ? -zz : zz;
        x = fma(-F.sx, z, (double)pick4<A::K1>(v) - U.q[A::K1]);
        y = fma(-F.sy, z, (double)pick4<A::K2>(v) - U.q[A::K2]);
    } else {
        const double zz = (double)pick4<A::k>(v);
        z = (AX & 1) ? -zz : zz;
        x = fma(-U.q[0], z, (double)pick4<A::K1>(v) - F.c1);
        y = fma(-U.q[1], z, (double)pick4<A::K2>(v) - F.c2);
    }
}

__device__ __forceinline__ double side2(double xa, double ya, double xb, double yb) {
    return fma(xa, yb, -(ya * xb));
}

// Depth z' where the ray (the z' axis) crosses the face (slot 0, 1, 2):
// barycentric weights |side(1,2)|, |side(2,0)|, |side(0,1)| (all of one exact
// sign for a crossed face; |.| differs from the exact value only below tau),
// offsets from slot 0 for accuracy, 1/sum from the MUFU reciprocal refined by
// one fp64 Newton step (rel. error ~2^-40).  A face with all three weights 0
// (cannot happen with certified signs) returns `fallback`.
__device__ __forceinline__ double face_depth(double x0, double y0, double z0, double x1,
                                             double y1, double z1, double x2, double y2,
                                             double z2, double fallback, unsigned& n_exact) {
    const double w0 = fabs(side2(x1, y1, x2, y2)), w1 = fabs(side2(x2, y2, x0, y0)),
                 w2 = fabs(side2(x0, y0, x1, y1));
    const double sw = w0 + w1 + w2;
    if (sw > 0.0) return fma(fma(w1, z1 - z0, w2 * (z2 - z0)), rcp_nr(sw), z0);
    ++n_exact;
    return fallback;
}


__device__ __forceinline__ int sel4(int4 v, int k) {
    return selp(selp(v.x, v.y, k == 0), selp(v.z, v.w, k == 2), k < 2);
}

__device__ __forceinline__ int4 ldg_nc_v4(const int4* p) {
    return __ldg(p);  // ld.global.nc.v4: one 16-B request
}

// One 256-bit request (LDG.E.ENL2.256 on sm_100a) for a 32-B face-tag record.
__device__ __forceinline__ void ldg_rec256(const int4* p, int4& a, int4& b) {
    asm("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
        : "l"(p));
}

// warp-aggregated stats
__device__ __forceinline__ void add_stat(unsigned long long* st, int slot, unsigned v) {
    const unsigned s = __reduce_add_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(st + slot, (unsigned long long)s);
}

// ------------------------------------------------------- entry finder ----
// Direct det[A,B,D] (A=a-o, B=b-o, D=p-o exactly representable) with a
// Shewchuk-style static bound; exact SoS when inside the bound.
__device__ __forceinline__ int side_direct(const int4 a, const int4 b, const RayPts& r,
                                           unsigned& n_exact) {
    const double Ax = (double)(a.x - r.ox), Ay = (double)(a.y - r.oy), Az = (double)(a.z - r.oz);
    const double Bx = (double)(b.x - r.ox), By = (double)(b.y - r.oy), Bz = (double)(b.z - r.oz);
    const double Dx = (double)(r.px - r.ox), Dy = (double)(r.py - r.oy), Dz = (double)(r.pz - r.oz);
    const double cx = Ay * Bz - Az * By, cy = Az * Bx - Ax * Bz, cz = Ax * By - Ay * Bx;
    const double det = Dx * cx + Dy * cy + Dz * cz;
    const double perm = fabs(Dx) * (fabs(Ay * Bz) + fabs(Az * By)) +
                        fabs(Dy) * (fabs(Az * Bx) + fabs(Ax * Bz)) +
                        fabs(Dz) * (fabs(Ax * By) + fabs(Ay * Bx));
    const double bound = perm * 0x1p-48;
    if (det > bound) return 1;
    if (det < -bound) return -1;
    ++n_exact;
    return sos_side(a.x, a.y, a.z, b.x, b.y, b.z, r.ox, r.oy, r.oz, r.px, r.py, r.pz);
}

// Work item of the entry finder: one non-culled (hull face, angle) pair.
struct EntryItem {
    double c[3], al[3], be[3], bnd[3];  // side_e(u,v) = c + u al + v be, |error| <= bnd
    int ia, ib, ic;                     // face vertices (outward order)
    int a, u0, v0, bw, npx, code;       // angle, footprint box, tet<<2|k
    int pad[3];
};

// Kernel 1 (one thread per (hull face, angle)): cull the faces that every
// detector-corner ray leaves through, bound the face's detector footprint,
// and compute each edge side as an exact affine function of the pixel
// indices (int128, once per item):
//   cone:     side(u,v) = (P00 - S + uU + vV) . ((a-S) x (b-S))
//   parallel: side(u,v) = d . ((a+d) x (b+d)) + (P00 + uU + vV) . (d x (b-a))
// Rounded to double, side at any pixel of the box is within
// 4 eps (|c| + u1|al| + v1|be|) of the exact value (conversion + 2 FMAs).
__global__ void __launch_bounds__(128) entry_setup_kernel(
    const int4* __restrict__ tnode, const int4* __restrict__ vtx, const int2* __restrict__ hull,
    int nb, const AngleGeom* __restrict__ ang, const AngleAux* __restrict__ aux, int beam,
    int n_angles, int nv, int nu, EntryItem* __restrict__ items, unsigned* __restrict__ n_items,
    unsigned cap, unsigned small_px) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= nb * n_angles) return;
    const int h = idx % nb, a = idx / nb;
    const int2 hk = hull[h];
    const int4 nodes = __ldg(tnode + hk.x);
    const int k = hk.y;
    int ia, ib, ic;   // outward order of face k (opposite node k)
    if (k == 0)      { ia = nodes.y; ib = nodes.z; ic = nodes.w; }
    else if (k == 1) { ia = nodes.x; ib = nodes.w; ic = nodes.z; }
    else if (k == 2) { ia = nodes.x; ib = nodes.y; ic = nodes.w; }
    else             { ia = nodes.x; ib = nodes.z; ic = nodes.y; }
    const int4 V[3] = {__ldg(vtx + ia), __ldg(vtx + ib), __ldg(vtx + ic)};
    const AngleGeom G = ang[a];
    const AngleAux X = aux[a];
    // --- cull: every detector-corner ray leaves through this face's plane
    const double e1[3] = {(double)V[1].x - V[0].x, (double)V[1].y - V[0].y, (double)V[1].z - V[0].z};
    const double e2[3] = {(double)V[2].x - V[0].x, (double)V[2].y - V[0].y, (double)V[2].z - V[0].z};
    const double n[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                         e1[0] * e2[1] - e1[1] * e2[0]};
    const double nn = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    bool cull = true;
    for (int c = 0; c < 4 && cull; ++c) {
        const RayPts r = ray_points(G, beam, (c & 1) ? nu - 1 : 0, (c & 2) ? nv - 1 : 0);
        const double d[3] = {(double)(r.px - r.ox), (double)(r.py - r.oy), (double)(r.pz - r.oz)};
        const double dn = d[0] * n[0] + d[1] * n[1] + d[2] * n[2];
        const double dd = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        cull = dn > 1e-9 * dd * nn;
    }
    if (cull) return;
    // --- detector footprint (bounding box, 1 px margin)
    double umin = 1e300, umax = -1e300, vmin = 1e300, vmax = -1e300;
    bool full = false;
    for (int j = 0; j < 3; ++j) {
        const double P[3] = {(double)V[j].x, (double)V[j].y, (double)V[j].z};
        double Q[3];
        if (beam == TET_BEAM_CONE) {
            const double dX[3] = {P[0] - X.S[0], P[1] - X.S[1], P[2] - X.S[2]};
            const double den = dX[0] * X.N[0] + dX[1] * X.N[1] + dX[2] * X.N[2];
            const double num = (X.P00[0] - X.S[0]) * X.N[0] + (X.P00[1] - X.S[1]) * X.N[1] +
                               (X.P00[2] - X.S[2]) * X.N[2];
            const double lam = num / den;
            if (!(lam > 0) || !isfinite(lam)) { full = true; break; }
            for (int i = 0; i < 3; ++i) Q[i] = X.S[i] + lam * dX[i];
        } else {
            const double dN = X.S[0] * X.N[0] + X.S[1] * X.N[1] + X.S[2] * X.N[2];
            const double sc = ((P[0] - X.P00[0]) * X.N[0] + (P[1] - X.P00[1]) * X.N[1] +
                               (P[2] - X.P00[2]) * X.N[2]) / dN;
            for (int i = 0; i < 3; ++i) Q[i] = P[i] - sc * X.S[i];
        }
        const double w[3] = {Q[0] - X.P00[0], Q[1] - X.P00[1], Q[2] - X.P00[2]};
        const double uu = w[0] * X.Us[0] + w[1] * X.Us[1] + w[2] * X.Us[2];
        const double vv = w[0] * X.Vs[0] + w[1] * X.Vs[1] + w[2] * X.Vs[2];
        if (!isfinite(uu) || !isfinite(vv)) { full = true; break; }
        umin = fmin(umin, uu); umax = fmax(umax, uu);
        vmin = fmin(vmin, vv); vmax = fmax(vmax, vv);
    }
    int u0 = 0, u1 = nu - 1, v0 = 0, v1 = nv - 1;
    if (!full) {
        u0 = (int)fmax(0.0, floor(umin) - 1.0);
        v0 = (int)fmax(0.0, floor(vmin) - 1.0);
        u1 = (int)fmin((double)(nu - 1), ceil(umax) + 1.0);
        v1 = (int)fmin((double)(nv - 1), ceil(vmax) + 1.0);
    }
    if (u0 > u1 || v0 > v1) return;
    EntryItem it;
    for (int e = 0; e < 3; ++e) {
        const int4 E0 = V[e], E1 = V[e == 2 ? 0 : e + 1];
        i128 c, al, be;
        if (beam == TET_BEAM_CONE) {
            const i128 ax = (i128)E0.x - G.o[0], ay = (i128)E0.y - G.o[1], az = (i128)E0.z - G.o[2];
            const i128 bx = (i128)E1.x - G.o[0], by = (i128)E1.y - G.o[1], bz = (i128)E1.z - G.o[2];
            const i128 nx = ay * bz - az * by, ny = az * bx - ax * bz, nz = ax * by - ay * bx;
            c = (i128)(G.p00[0] - G.o[0]) * nx + (i128)(G.p00[1] - G.o[1]) * ny +
                (i128)(G.p00[2] - G.o[2]) * nz;
            al = (i128)G.du[0] * nx + (i128)G.du[1] * ny + (i128)G.du[2] * nz;
            be = (i128)G.dv[0] * nx + (i128)G.dv[1] * ny + (i128)G.dv[2] * nz;
        } else {
            const long long dx = G.o[0], dy = G.o[1], dz = G.o[2];
            const i128 ax = (i128)E0.x + dx, ay = (i128)E0.y + dy, az = (i128)E0.z + dz;
            const i128 bx = (i128)E1.x + dx, by = (i128)E1.y + dy, bz = (i128)E1.z + dz;
            const i128 ex = (i128)E1.x - E0.x, ey = (i128)E1.y - E0.y, ez = (i128)E1.z - E0.z;
            const i128 mx = dy * ez - dz * ey, my = dz * ex - dx * ez, mz = dx * ey - dy * ex;
            c = dx * (ay * bz - az * by) + dy * (az * bx - ax * bz) + dz * (ax * by - ay * bx) +
                (i128)G.p00[0] * mx + (i128)G.p00[1] * my + (i128)G.p00[2] * mz;
            al = (i128)G.du[0] * mx + (i128)G.du[1] * my + (i128)G.du[2] * mz;
            be = (i128)G.dv[0] * mx + (i128)G.dv[1] * my + (i128)G.dv[2] * mz;
        }
        it.c[e] = (double)c;
        it.al[e] = (double)al;
        it.be[e] = (double)be;
        it.bnd[e] = 0x1p-50 * (fabs(it.c[e]) + (double)u1 * fabs(it.al[e]) + (double)v1 * fabs(it.be[e]));
    }
    it.ia = ia; it.ib = ib; it.ic = ic;
    it.a = a; it.u0 = u0; it.v0 = v0; it.bw = u1 - u0 + 1;
    it.npx = (u1 - u0 + 1) * (v1 - v0 + 1);
    it.code = (hk.x << 2) | k;
    it.pad[0] = it.pad[1] = it.pad[2] = 0;
    // compacted item lists (order irrelevant: each ray has one entering
    // face): footprints of <= small_px pixels from the end of the array
    // (counter n_items[2]; one thread per item, entry_small_kernel), larger
    // ones from the front (counter n_items[0]; a warp per item)
    const unsigned act = __activemask();
    const bool small = (unsigned)it.npx <= small_px;
    const unsigned mask = __ballot_sync(act, small) ^ (small ? 0u : act);   // lanes of my kind
    const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
    unsigned slot = 0;
    if (lane == leader) slot = atomicAdd(n_items + (small ? 2 : 0), (unsigned)__popc(mask));
    slot = __shfl_sync(mask, slot, leader) + __popc(mask & ((1u << lane) - 1));
    items[small ? cap - 1 - slot : slot] = it;
}

__device__ __noinline__ bool exact_entering(const int4* __restrict__ vtx,
                                            const AngleGeom* __restrict__ ang, int beam, int a,
                                            int u, int v, int ia, int ib, int ic,
                                            unsigned& exact);

// Small footprints (beside the warp raster): one thread per (face, angle)
// item tests every pixel of its <= small_px-pixel box with the item's exact
// affine sides (certified by the bound, else int128 + SoS), the same test
// as the warp raster's dense pass; a warp per pixel-sized item (c4a's
// lattice hull) left most lanes idle.
__global__ void __launch_bounds__(128) entry_small_kernel(
    const int4* __restrict__ vtx, const AngleGeom* __restrict__ ang, int beam, int nv, int nu,
    const EntryItem* __restrict__ items, unsigned cap, const unsigned* __restrict__ n_small_p,
    int* __restrict__ entry, unsigned long long* __restrict__ stats) {
    const unsigned idx = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned conflicts = 0, exact = 0;
    if (idx < n_small_p[0]) {
        const EntryItem* it = items + (cap - 1 - idx);
        const double c0 = it->c[0], al0 = it->al[0], be0 = it->be[0], b0 = it->bnd[0];
        const double c1 = it->c[1], al1 = it->al[1], be1 = it->be[1], b1 = it->bnd[1];
        const double c2 = it->c[2], al2 = it->al[2], be2 = it->be[2], b2 = it->bnd[2];
        const int bw = it->bw, u0 = it->u0, v0 = it->v0, a = it->a, code = it->code;
        const int nrows = it->npx / bw;
        for (int r = 0; r < nrows; ++r) {
            const int v = v0 + r;
            const double fv = (double)v;
            const double r0 = fma(fv, be0, c0), r1 = fma(fv, be1, c1), r2 = fma(fv, be2, c2);
            for (int k = 0; k < bw; ++k) {
                const int u = u0 + k;
                const double fu = (double)u;
                const double sab = fma(fu, al0, r0);
                if (sab > b0) continue;
                const double sbc = fma(fu, al1, r1);
                if (sbc > b1) continue;
                const double sca = fma(fu, al2, r2);
                if (sca > b2) continue;
                if (sab >= -b0 || sbc >= -b1 || sca >= -b2) {
                    if (!exact_entering(vtx, ang, beam, a, u, v, it->ia, it->ib, it->ic, exact))
                        continue;
                }
                DBG_CHECK(u < nu && v < nv);
                const int old = atomicExch(entry + ((size_t)a * nv + v) * nu + u, code);
                conflicts += (old != -1);
            }
        }
    }
    const unsigned cs = __reduce_add_sync(0xffffffffu, conflicts);
    const unsigned es = __reduce_add_sync(0xffffffffu, exact);
    if ((threadIdx.x & 31) == 0) {
        if (cs) atomicAdd(stats + ST_CONFLICT, (unsigned long long)cs);
        if (es) atomicAdd(stats + ST_EXACT, (unsigned long long)es);
    }
}

// Rare path of the entry test: all three signs decided by side_direct (fp64
// static filter, else int128 + SoS).
__device__ __noinline__ bool exact_entering(const int4* __restrict__ vtx,
                                            const AngleGeom* __restrict__ ang, int beam, int a,
                                            int u, int v, int ia, int ib, int ic,
                                            unsigned& exact) {
    const RayPts r = ray_points(ang[a], beam, u, v);
    const int4 A = __ldg(vtx + ia), B = __ldg(vtx + ib), C = __ldg(vtx + ic);
    return side_direct(A, B, r, exact) == -1 && side_direct(B, C, r, exact) == -1 &&
           side_direct(C, A, r, exact) == -1;
}

// Conservative u-range of one row for one edge.  A pixel survives the
// per-pixel test only if the computed side f = c + u al + v be is <= bnd;
// the evaluation error is below bnd, so the exact value is <= 2 bnd, i.e.
// u al <= r := 2 bnd - c - v be.  r and r/al are rounded, so the range is
// widened by 1 px + the rounding error of r in pixels; a nearly u-parallel
// edge (error not below 2^20 px) does not narrow the row.  Widening only
// costs tests: every pixel inside is still tested exactly.
__device__ __forceinline__ void clip_row(double c, double al, double be, double bnd, double fv,
                                         int& lo, int& hi) {
    const double vb = fv * be;
    const double r = 2.0 * bnd - c - vb;
    const double aal = fabs(al);
    const double margin = 1.0 + 0x1p-50 * (2.0 * bnd + fabs(c) + fabs(vb)) / aal;
    if (!(margin < 0x1p20)) return;            // al == 0 or too ill-conditioned
    const double x = r / al;
    if (!(fabs(x) < 0x1p30)) {                 // far outside the detector
        if ((al > 0) == (x < 0)) { lo = 1; hi = 0; }
        return;
    }
    if (al > 0) hi = min(hi, (int)floor(x + margin));
    else        lo = max(lo, (int)ceil(x - margin));
}

// Kernel 2 (persistent grid, one warp per (face, angle) item): scanline
// rasterisation of the face's footprint box.  32 rows at a time, lane r
// clips row r against the three edge half-planes (conservatively), a warp
// scan packs the surviving pixels, and the lanes test them densely -- an
// entering test is side(a,b) = side(b,c) = side(c,a) = -1 for the
// outward-ordered face; the affine value certifies a sign when it clears
// the item's bound, otherwise the int128 + SoS path decides.  Writes
// entry[ray] = tet<<2 | k and counts conflicts (must be 0).
__global__ void __launch_bounds__(128, 8) entry_raster_kernel(
    const int4* __restrict__ vtx, const AngleGeom* __restrict__ ang, int beam, int nv, int nu,
    const EntryItem* __restrict__ items, const unsigned* __restrict__ n_items_p,
    unsigned* __restrict__ queue, int* __restrict__ entry, unsigned long long* __restrict__ stats) {
    const unsigned n_items = n_items_p[0];
    const int lane = threadIdx.x & 31;
    unsigned conflicts = 0, exact = 0;
    // Guided self-scheduling on one queue counter: a warp claims
    // max(1, remaining / (ENTRY_GUIDE x warps)) consecutive items per
    // atomic, "remaining" estimated from its own previous claim.  Footprints
    // vary by orders of magnitude: c2's ~270 k tiny items no longer pay one
    // atomic each (60 % of the raster's stall samples), c3's few large items
    // still go out one at a time once the queue runs low.
    const unsigned nwarps = gridDim.x * (blockDim.x >> 5);
    unsigned seen = 0;   // (lane 0) queue position at this warp's last claim
    for (;;) {
        unsigned start = 0, cnt = 0;
        if (lane == 0) {
            const unsigned rem = seen < n_items ? n_items - seen : 0u;
            cnt = ENTRY_GUIDE ? max(1u, rem / (ENTRY_GUIDE * nwarps)) : 1u;   // 0: one per claim
            start = atomicAdd(queue, cnt);
            seen = start + cnt;
        }
        start = __shfl_sync(0xffffffffu, start, 0);
        cnt = __shfl_sync(0xffffffffu, cnt, 0);
        if (start >= n_items) break;
        const unsigned end = min(start + cnt, n_items);
        for (unsigned item = start; item < end; ++item) {
        const EntryItem* it = items + item;
        const int npx = it->npx;
        const double c0 = it->c[0], al0 = it->al[0], be0 = it->be[0], b0 = it->bnd[0];
        const double c1 = it->c[1], al1 = it->al[1], be1 = it->be[1], b1 = it->bnd[1];
        const double c2 = it->c[2], al2 = it->al[2], be2 = it->be[2], b2 = it->bnd[2];
        const int bw = it->bw, u0 = it->u0, v0 = it->v0, a = it->a, code = it->code;
        const int nrows = npx / bw;
        for (int r0 = 0; r0 < nrows; r0 += 32) {
            int lo = u0, hi = u0 + bw - 1;
            if (r0 + lane < nrows) {
                const double fv = (double)(v0 + r0 + lane);
                clip_row(c0, al0, be0, b0, fv, lo, hi);
                clip_row(c1, al1, be1, b1, fv, lo, hi);
                clip_row(c2, al2, be2, b2, fv, lo, hi);
            } else {
                hi = lo - 1;
            }
            const int len = max(0, hi - lo + 1);
            int inc = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            const int total = __shfl_sync(0xffffffffu, inc, 31);
            const int exc = inc - len;
            for (int base = 0; base < total; base += 32) {
                const int i = base + lane;
                int j = 0;   // row of pixel i: number of rows whose inclusive end is <= i
#pragma unroll
                for (int st = 16; st; st >>= 1)
                    if (__shfl_sync(0xffffffffu, inc, j + st - 1) <= i) j += st;
                const int ej = __shfl_sync(0xffffffffu, exc, j);
                const int lj = __shfl_sync(0xffffffffu, lo, j);
                if (i >= total) continue;
                const int u = lj + (i - ej), v = v0 + r0 + j;
                const double fu = (double)u, fv = (double)v;
                const double sab = fma(fv, be0, fma(fu, al0, c0));
                if (sab > b0) continue;
                const double sbc = fma(fv, be1, fma(fu, al1, c1));
                if (sbc > b1) continue;
                const double sca = fma(fv, be2, fma(fu, al2, c2));
                if (sca > b2) continue;
                if (sab >= -b0 || sbc >= -b1 || sca >= -b2) {   // a sign the bound cannot certify
                    if (!exact_entering(vtx, ang, beam, a, u, v, it->ia, it->ib, it->ic, exact))
                        continue;
                }
                DBG_CHECK(u >= u0 && u < u0 + bw && u < nu && v >= 0 && v < nv);
                const int old = atomicExch(entry + ((size_t)a * nv + v) * nu + u, code);
                conflicts += (old != -1);
            }
        }
        }
    }
    if (conflicts) atomicAdd(stats + ST_CONFLICT, (unsigned long long)conflicts);
    if (exact) atomicAdd(stats + ST_EXACT, (unsigned long long)exact);
}

// Alternative entry finder (TET_ENTRY_BVH; NEXT-3): one thread per ray walks
// a BVH over the hull faces (the paper's per-ray tree search, PAPER.md:154-158,
// with a binary BVH instead of an R*-tree).  Boxes are float, rounded
// outward, tested in fp64 with a margin, so they never prune a face the ray
// meets; the entering test at the leaves is exact, and because the entering
// face is unique the search stops at the first one found.
__global__ void __launch_bounds__(128) entry_bvh_kernel(const int4* __restrict__ nodes,
                                                        const int4* __restrict__ faces,
                                                        const int4* __restrict__ vtx,
                                                        const AngleGeom* __restrict__ ang,
                                                        int beam, int nv, int nu,
                                                        int* __restrict__ entry,
                                                        unsigned long long* __restrict__ stats) {
    const int tiles_u = (nu + 15) >> 4;
    const int bx = blockIdx.x % tiles_u, by = blockIdx.x / tiles_u;
    const int a = blockIdx.y;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int u = bx * 16 + (w & 1) * 8 + (lane & 7);
    const int v = by * 8 + (w >> 1) * 4 + (lane >> 3);
    unsigned exact = 0;
    if (u < nu && v < nv) {
        const RayPts r = ray_points(ang[a], beam, u, v);
        const double o[3] = {(double)r.ox, (double)r.oy, (double)r.oz};
        const double d[3] = {(double)(r.px - r.ox), (double)(r.py - r.oy), (double)(r.pz - r.oz)};
        double inv[3];
        for (int i = 0; i < 3; ++i) inv[i] = 1.0 / d[i];   // +-inf for d = 0
        int stack[64];
        int sp = 0, found = -1;
        stack[sp++] = 0;
        while (sp > 0 && found < 0) {
            const int n = stack[--sp];
            const int4 q0 = __ldg(nodes + 2 * n), q1 = __ldg(nodes + 2 * n + 1);
            const float lo[3] = {__int_as_float(q0.x), __int_as_float(q0.y), __int_as_float(q0.z)};
            const float hi[3] = {__int_as_float(q0.w), __int_as_float(q1.x), __int_as_float(q1.y)};
            double tmin = -INFINITY, tmax = INFINITY;
            bool miss = false;
            for (int i = 0; i < 3; ++i) {
                const double m = 2.0 + 1e-9 * (fabs((double)lo[i]) + fabs(o[i]));
                const double l = (double)lo[i] - m, h = (double)hi[i] + m;
                if (d[i] == 0.0) {
                    miss |= o[i] < l || o[i] > h;
                } else {
                    const double t1 = (l - o[i]) * inv[i], t2 = (h - o[i]) * inv[i];
                    tmin = fmax(tmin, fmin(t1, t2));
                    tmax = fmin(tmax, fmax(t1, t2));
                }
            }
            if (miss || tmin > tmax + 1e-9 * (fabs(tmin) + fabs(tmax))) continue;
            if (q1.z < 0) {   // leaf
                const int first = -q1.z - 1, cnt = q1.w;
                for (int f = first; f < first + cnt; ++f) {
                    const int4 fc = __ldg(faces + f);
                    const int4 A = __ldg(vtx + fc.x), B = __ldg(vtx + fc.y), C = __ldg(vtx + fc.z);
                    if (side_direct(A, B, r, exact) == -1 && side_direct(B, C, r, exact) == -1 &&
                        side_direct(C, A, r, exact) == -1) {
                        found = fc.w;
                        break;
                    }
                }
            } else if (sp < 62) {
                stack[sp++] = q1.w;
                stack[sp++] = q1.z;
            }
        }
        if (found >= 0) entry[((size_t)a * nv + v) * nu + u] = found;
    }
    const unsigned s = __reduce_add_sync(0xffffffffu, exact);
    if (lane == 0 && s) atomicAdd(stats + ST_EXACT, (unsigned long long)s);
}

// The paper's initialisation (TET_ENTRY_RTREE): "an
// R*-tree is precomputed for the boundary elements ... To search the tree, a
// depth-first algorithm is implemented ... When a leaf node is reached in the
// search, all tetrahedra within that node are checked for intersection".
// One thread per ray; nodes of <= 10 children (rtree_host.cpp); child boxes
// tested like the BVH's (float, rounded outward, fp64 slab test with a
// margin, so no face the ray meets is pruned); faces tested exactly.  The
// paper keeps the leaf candidate with the minimum intersection parameter;
// with exact signs exactly one hull face is entering, so the search stops at
// it (reading R9).
__device__ __forceinline__ bool ray_box(const double o[3], const double inv[3], const double d[3],
                                        const float* lo, const float* hi) {
    double tmin = -INFINITY, tmax = INFINITY;
    for (int i = 0; i < 3; ++i) {
        const double m = 2.0 + 1e-9 * (fabs((double)lo[i]) + fabs(o[i]));
        const double l = (double)lo[i] - m, h = (double)hi[i] + m;
        if (d[i] == 0.0) {
            if (o[i] < l || o[i] > h) return false;
        } else {
            const double t1 = (l - o[i]) * inv[i], t2 = (h - o[i]) * inv[i];
            tmin = fmax(tmin, fmin(t1, t2));
            tmax = fmin(tmax, fmax(t1, t2));
        }
    }
    return !(tmin > tmax + 1e-9 * (fabs(tmin) + fabs(tmax)));
}

__global__ void __launch_bounds__(128) entry_rtree_kernel(const int* __restrict__ nodes,
                                                          const int4* __restrict__ faces,
                                                          const int4* __restrict__ vtx,
                                                          const AngleGeom* __restrict__ ang,
                                                          int beam, int nv, int nu,
                                                          int* __restrict__ entry,
                                                          unsigned long long* __restrict__ stats) {
    const int tiles_u = (nu + 15) >> 4;
    const int bx = blockIdx.x % tiles_u, by = blockIdx.x / tiles_u;
    const int a = blockIdx.y;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int u = bx * 16 + (w & 1) * 8 + (lane & 7);
    const int v = by * 8 + (w >> 1) * 4 + (lane >> 3);
    unsigned exact = 0;
    if (u < nu && v < nv) {
        const RayPts r = ray_points(ang[a], beam, u, v);
        const double o[3] = {(double)r.ox, (double)r.oy, (double)r.oz};
        const double d[3] = {(double)(r.px - r.ox), (double)(r.py - r.oy), (double)(r.pz - r.oz)};
        double inv[3];
        for (int i = 0; i < 3; ++i) inv[i] = 1.0 / d[i];   // +-inf for d = 0
        int stack[96];
        int sp = 0, found = -1;
        stack[sp++] = 0;                                   // root
        while (sp > 0 && found < 0) {
            const int* nd = nodes + 72 * stack[--sp];
            const int cnt = __ldg(nd), leaf = __ldg(nd + 1);
            const float* lo = reinterpret_cast<const float*>(nd + 12);
            const float* hi = reinterpret_cast<const float*>(nd + 42);
            float blo[3], bhi[3];
            if (leaf) {
                for (int c = 0; c < cnt && found < 0; ++c) {
                    for (int i = 0; i < 3; ++i) { blo[i] = __ldg(lo + 3 * c + i); bhi[i] = __ldg(hi + 3 * c + i); }
                    if (!ray_box(o, inv, d, blo, bhi)) continue;
                    const int4 fc = __ldg(faces + __ldg(nd + 2 + c));
                    const int4 A = __ldg(vtx + fc.x), B = __ldg(vtx + fc.y), C = __ldg(vtx + fc.z);
                    if (side_direct(A, B, r, exact) == -1 && side_direct(B, C, r, exact) == -1 &&
                        side_direct(C, A, r, exact) == -1)
                        found = fc.w;
                }
            } else {
                // depth first: children pushed in reverse so child 0 is searched first
                for (int c = cnt - 1; c >= 0; --c) {
                    for (int i = 0; i < 3; ++i) { blo[i] = __ldg(lo + 3 * c + i); bhi[i] = __ldg(hi + 3 * c + i); }
                    if (ray_box(o, inv, d, blo, bhi) && sp < 96) stack[sp++] = __ldg(nd + 2 + c);
                }
            }
        }
        if (found >= 0) entry[((size_t)a * nv + v) * nu + u] = found;
    }
    const unsigned s = __reduce_add_sync(0xffffffffu, exact);
    if (lane == 0 && s) atomicAdd(stats + ST_EXACT, (unsigned long long)s);
}

// ------------------------------------------------------------ walker ----
// float -> double at the point of use (volatile: nvcc would hoist a plain
// conversion of the loop-invariant weight out of the loop and keep -- at 64
// registers: spill -- the double)
__device__ __forceinline__ double f2d_here(float x) {
    double r;
    asm volatile("cvt.f64.f32 %0, %1;" : "=d"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ double f2d_here(double x) { return x; }

// Apex vertex gather.  Backward walk (64 registers): x, y and z as a 64-bit
// and a 32-bit load when TRACE_BWD_VTX_SPLIT -- the 128-bit load's register
// quad collided with the loop-carried tet id and nvcc copied a component out
// of it right after the load, stalling on it (ncu source view).
template <bool BACK>
__device__ __forceinline__ int4 ldg_vtx(const int4* p) {
    if (BACK && TRACE_BWD_VTX_SPLIT) {
        const int2 xy = __ldg(reinterpret_cast<const int2*>(p));
        const int z = __ldg(reinterpret_cast<const int*>(p) + 2);
        return make_int4(xy.x, xy.y, z, 0);
    }
    return __ldg(p);
}

// #{ids < x} for four distinct ids in [0, 2^31) (one of them may be x):
// [a < x] is the sign bit of a - x.  PTX, so that nvcc does not turn it back
// into compare + predicated-move chains.
__device__ __forceinline__ int rank4(int a, int b, int c, int d, int x) {
    int r;
    asm("{\n\t.reg .u32 p, q, s, t;\n\t"
        "sub.u32 p, %1, %5;\n\tsub.u32 q, %2, %5;\n\tsub.u32 s, %3, %5;\n\tsub.u32 t, %4, %5;\n\t"
        "shr.u32 p, p, 31;\n\tshr.u32 q, q, 31;\n\tshr.u32 s, s, 31;\n\tshr.u32 t, t, 31;\n\t"
        "add.u32 p, p, q;\n\tadd.u32 s, s, t;\n\tadd.u32 %0, p, s;\n\t}"
        : "=r"(r) : "r"(a), "r"(b), "r"(c), "r"(d), "r"(x));
    return r;
}

// j (dropped slot) per sign code neg = n0 | n1<<1 | n2<<2, 2 bits each; 3 = lost
constexpr unsigned kExitLUT = 3u | 2u << 2 | 0u << 4 | 0u << 6 | 1u << 8 | 2u << 10 | 1u << 12 |
                              3u << 14;

// [|a| <= t or |b| <= t or |c| <= t] as one predicate chain (keeps nvcc from
// rewriting it as an fp64 min with NaN fix-ups)
__device__ __forceinline__ bool any_abs_le(double a, double b, double c, double t) {
    unsigned r;
    asm("{\n\t.reg .pred q;\n\t.reg .f64 x, y, z;\n\t"
        "abs.f64 x, %1;\n\tabs.f64 y, %2;\n\tabs.f64 z, %3;\n\t"
        "setp.le.f64 q, x, %4;\n\tsetp.le.or.f64 q, y, %4, q;\n\t"
        "setp.le.or.f64 q, z, %4, q;\n\tselp.u32 %0, 1, 0, q;\n\t}"
        : "=r"(r) : "d"(a), "d"(b), "d"(c), "d"(t));
    return r != 0;
}


template <int AX, int UNI>
__device__ __forceinline__ void xf(const Frame& F, const UniFrame& U, const int4 v, double& x,
                                   double& y, double& z) {
    if constexpr (UNI == 0) xform_ax<AX>(F, v, x, y, z);
    else xform_uni<AX, UNI>(F, U, v, x, y, z);
}

// |D| / |D_k| * g (chord per unit of z')
template <int UNI>
__device__ __forceinline__ double ray_scale(const Frame& F, const UniFrame& U, double g) {
    if constexpr (UNI == 0) return F.scale;
    else if constexpr (UNI == 1) return sqrt(fma(F.sx, F.sx, fma(F.sy, F.sy, 1.0))) * g;
    else return U.scale;
}

// One thread per ray, 8x4-pixel warp tiles (16x8 per block).
// State: the entry face in three fixed slots k = 0,1,2 in cyclic order (shear
// coordinates x', y', z' and vertex id), the apex id `iap` (from the previous
// face tag) and the entry depth zin.  Per step the face tags of t and the
// apex vertex are gathered IN PARALLEL (the previous tag carried the apex
// id); the sign code of the three sides side(apex, slot k) picks the exit
// face, the rank of the dropped slot's vertex id among t's four ids gives the
// position of its tag, and the tag gives the next tet and its apex
// (DESIGN.md §5).
template <bool BACK, int AX, int UNI, int BX, int BY, bool LATE, bool BAND>
__device__ __forceinline__ void walk_ray(const UniFrame& U, const int4* __restrict__ rec, const int4* __restrict__ tnode,
                                         const int4* __restrict__ vtx,
                                         const AngleGeom* __restrict__ ang, int beam, int a, int u,
                                         int v, int nu, int tw_log, double rmax, double g,
                                         int max_steps, int nverts, int e, size_t rid,
                                         const float* __restrict__ mu,
                                         const float* __restrict__ y, double* __restrict__ acc,
                                         double& sum, unsigned& n_cross, unsigned& n_exact,
                                         unsigned& n_lost, unsigned& n_stuck) {
        const RayPts r = ray_points(ang[a], beam, u, v);
        Frame F;
        if constexpr (UNI == 0) make_frame_ax<AX>(r, rmax, g, F);
        else make_frame_uni<AX, UNI>(r, U, F);
        // chord = (z'_out - z'_in) * scale; scale is folded into y (back) or
        // applied once to the ray sum (forward)
#if TRACE_BWD_WY32
        // f32 weight: one register (at 64 registers the f64 weight spilled and
        // its local reload stalled every RED); relative error 2^-24
        const float wy = BACK ? (float)((double)ld_stream(y + rid) * ray_scale<UNI>(F, U, g)) : 0.f;
#else
        const double wy = BACK ? (double)y[rid] * ray_scale<UNI>(F, U, g) : 0.0;
#endif
        const double tau = UNI ? U.tau : F.tau;
        const int t0 = e >> 2, kin = e & 3;
        int t = t0;
        DBG_CHECK(t >= 0 && t < max_steps);
        const int4 nodes = __ldg(tnode + t);
        DBG_CHECK(nodes.x >= 0 && nodes.x < nverts && nodes.y >= 0 && nodes.y < nverts &&
                  nodes.z >= 0 && nodes.z < nverts && nodes.w >= 0 && nodes.w < nverts);
        // entry face = face kin in outward order (opposite node kin)
        int id0, id1, id2;
        if (kin == 0)      { id0 = nodes.y; id1 = nodes.z; id2 = nodes.w; }
        else if (kin == 1) { id0 = nodes.x; id1 = nodes.w; id2 = nodes.z; }
        else if (kin == 2) { id0 = nodes.x; id1 = nodes.y; id2 = nodes.w; }
        else               { id0 = nodes.x; id1 = nodes.z; id2 = nodes.y; }
        int iap = sel4(nodes, kin);
        double x0, y0, z0, x1, y1, z1, x2, y2, z2;
        xf<AX, UNI>(F, U, __ldg(vtx + id0), x0, y0, z0);
        xf<AX, UNI>(F, U, __ldg(vtx + id1), x1, y1, z1);
        xf<AX, UNI>(F, U, __ldg(vtx + id2), x2, y2, z2);
        unsigned n_exact_init = 0;
        double zin = face_depth(x0, y0, z0, x1, y1, z1, x2, y2, z2, (z0 + z1 + z2) * (1.0 / 3.0),
                                n_exact_init);
        int steps = 0;   // crossings done before this one
        // The gathers of step k+1 (face tags of the next tet, its apex vertex,
        // mu) can be issued as soon as step k's exit face is known, with step
        // k's chord / accumulation / slot update running while they are in
        // flight (TRACE_*_LATE_LOADS = 0), or after them (= 1, the default:
        // fewer live registers, so 8 blocks/SM without copies off the load).
        int4 ta, tb;
        ldg_rec256(rec + 2 * (size_t)t, ta, tb);             // face tags of t (32 B)
        float mut = 0.f;
        if (!BACK) mut = __ldg(mu + t);
        int4 X = __ldg(vtx + iap);                          // apex vertex (16 B)
        while (true) {
            double x3, y3, z3;
            xf<AX, UNI>(F, U, X, x3, y3, z3);
            const double p0 = side2(x3, y3, x0, y0);   // side(apex, slot k)
            const double p1 = side2(x3, y3, x1, y1);
            const double p2 = side2(x3, y3, x2, y2);
            // exit face (apex, slot i, slot i+1): the unique i with
            // sign p_i = -1 and sign p_{i+1} = +1
            // All three filters are evaluated in parallel (ILP); a sign that the
            // filter cannot certify is decided exactly (rare branch).  With
            // n_k = [sign p_k = -1]: i = 0 for (1,0,*), 1 for (*,1,0), 2 for
            // (0,*,1); (0,0,0) and (1,1,1) cannot occur for an entering ray.
            // certified iff |p| > tau; then the sign bit is the sign.  neg =
            // (n0, n1, n2) with n_k = [sign p_k = -1] as bits 0..2.
            unsigned neg = ((unsigned)__double2hiint(p0) >> 31) |
                           (((unsigned)__double2hiint(p1) >> 30) & 2u) |
                           (((unsigned)__double2hiint(p2) >> 29) & 4u);
            if (any_abs_le(p0, p1, p2, tau)) {
                const unsigned mask = (fabs(p0) <= tau ? 1u : 0u) | (fabs(p1) <= tau ? 2u : 0u) |
                                      (fabs(p2) <= tau ? 4u : 0u);
                if (TRACE_HEAVY_KEEP_RAY && !LATE) {   // the exact-heavy shape (early gathers)
                    neg = exact_neg_ray(vtx, r.ox, r.oy, r.oz, r.px, r.py, r.pz, mask, neg, iap, id0, id1, id2);
                } else if (BACK ? TRACE_BWD_ONECALL : TRACE_EXACT_ONECALL) {
                    neg = exact_neg_here<BX, BY, BAND>(vtx, ang, beam, nu, tw_log, mask, neg, iap, id0, id1, id2);
                } else {
                    const unsigned m = neg;
                    neg = 0;
                    neg |= (mask & 1u) ? (exact_side_here<BX, BY, BAND>(vtx, ang, beam, nu, tw_log, iap, id0) < 0 ? 1u : 0u) : (m & 1u);
                    neg |= (mask & 2u) ? (exact_side_here<BX, BY, BAND>(vtx, ang, beam, nu, tw_log, iap, id1) < 0 ? 2u : 0u) : (m & 2u);
                    neg |= (mask & 4u) ? (exact_side_here<BX, BY, BAND>(vtx, ang, beam, nu, tw_log, iap, id2) < 0 ? 4u : 0u) : (m & 4u);
                }
                n_exact += __popc(mask);
            }
            // exit face (apex, slot i, slot i+1) for the unique i with n_i = 1,
            // n_{i+1} = 0; it drops slot j = i+2.  j by table on neg:
            // 1,5 -> i=0, j=2;  2,3 -> i=1, j=0;  4,6 -> i=2, j=1;  0,7 -> lost (3)
            const int j = (int)((kExitLUT >> (2 * neg)) & 3u);
            // exit through the face opposite slot j = i+2; its tag is stored at
            // the rank of the dropped slot's vertex
            // id among t's four vertex ids (three slots + apex), mesh_host.cpp
            const int idj = selp(id0, selp(id1, id2, j == 1), j == 0);
            // ids are distinct and in [0, 2^31): [a < b] is the sign bit of a - b
            // (shift-adds, LEA.HI, instead of compare + predicated-move chains)
            const int L = rank4(id0, id1, id2, iap, idj);
            const int lo = selp(selp(ta.x, ta.z, L == 0), selp(tb.x, tb.z, L == 2), L < 2);
            const unsigned hi = (unsigned)selp(selp(ta.y, ta.w, L == 0), selp(tb.y, tb.w, L == 2), L < 2);
            const bool more = lo >= 0 && j != 3 && ++steps != max_steps;
            const int tcur = t;
            const bool d0 = j == 0, d1 = j == 1, d2 = j == 2;
            // the next step's gathers are issued after this step's chord and
            // accumulation (TRACE_*_LATE_LOADS).  Issued here, nvcc (64
            // registers) had to copy a component of the vertex quad out of
            // the load's destination right away -- a stall on the load that
            // the early issue was meant to hide (9 % of the backward's stall
            // samples); issued late, 32 warps/SM hide the latency instead
            constexpr bool late = LATE;
            if (!late && more) {
                t = lo;
                DBG_CHECK(t >= 0 && t < max_steps && (int)hi >= 0 && (int)hi < nverts);
                ldg_rec256(rec + 2 * (size_t)t, ta, tb);
                X = ldg_vtx<BACK>(vtx + (int)hi);
            }
            // ---- slot update: the apex takes the dropped slot j = i+2 (cyclic
            // order is preserved); s_{i+1} <- -p_{i+1}, s_{i+2} <- p_i.  The
            // slots are then the exit face = the next entry face.
            if (d0) { x0 = x3; y0 = y3; z0 = z3; id0 = iap; }
            if (d1) { x1 = x3; y1 = y3; z1 = z3; id1 = iap; }
            if (d2) { x2 = x3; y2 = y3; z2 = z3; id2 = iap; }
            // ---- chord of step k (overlaps the gathers of step k+1): depth of
            // the crossing point of the (updated) face, barycentric weights
            // |s12|, |s20|, |s01| -- symmetric in the slots, so no selects
            const double zout = face_depth(x0, y0, z0, x1, y1, z1, x2, y2, z2, zin, n_exact);
            // zout - zin >= 0 up to rounding; an exact zero-length crossing
            // may come out as -1e-16 R, which is harmless in the sum
            const double dz = zout - zin;
            if (BACK) {
                if (dz > 0.0) atomicAdd(acc + tcur, dz * f2d_here(wy));
            } else {
                sum = fma(dz, (double)mut, sum);
            }
            if (late && more) {
                t = lo;
                DBG_CHECK(t >= 0 && t < max_steps && (int)hi >= 0 && (int)hi < nverts);
                ldg_rec256(rec + 2 * (size_t)t, ta, tb);
                X = ldg_vtx<BACK>(vtx + (int)hi);
            }
            if (!more) {
                // hull exit (lo < 0), lost (no exit pattern; impossible with
                // exact signs) or stuck (max_steps crossings)
                const bool stuck = lo >= 0 && j != 3;
                n_lost += j == 3 ? 1u : 0u;
                n_stuck += stuck ? 1u : 0u;
                n_cross += (unsigned)steps + (stuck ? 0u : 1u);
                break;
            }
            // mu of the next tet: issued after this step's use so no second
            // register (and no copy that waits on the load) is needed; it is
            // consumed at the end of the next step
            if (!BACK) mut = __ldg(mu + t);
            zin = zout;
            iap = (int)hi;
        }
        if (!BACK) sum *= ray_scale<UNI>(F, U, g);
    }

// ---- FT16 walk: one dependent 16-B gather per step --------------------
// The tag of the exit face (mesh_host.cpp "FT16") carries the next tet, its
// apex vertex id AND the apex coordinates, so a step gathers one 16-B tag
// (plus mu in the forward walk) instead of a 32-B record and a 16-B vertex.
// Coordinates arrive scaled by 64 (the low 6 bits of each word carry apex-id
// bits), so this walk runs its shear frame in units of g/64: ray points and
// vertices x64, tau x4096, chord scale /64 (exact power-of-two scaling: every
// sign and rounding is that of the unscaled arithmetic).
constexpr int kFtShift = 6;
constexpr unsigned kFtHull = 0x3FFFFFFu;

__device__ __forceinline__ int4 ft_scaled(const int4 v) {
    return make_int4(v.x << kFtShift, v.y << kFtShift, v.z << kFtShift, 0);
}

__device__ __forceinline__ RayPts ft_scaled(RayPts r) {
    r.ox <<= kFtShift; r.oy <<= kFtShift; r.oz <<= kFtShift;
    r.px <<= kFtShift; r.py <<= kFtShift; r.pz <<= kFtShift;
    return r;
}

template <bool BACK, int AX, int UNI, int BX, int BY, bool BAND, bool KEEP>
__device__ __forceinline__ void walk_ray_ft(const UniFrame& Ug, const int4* __restrict__ tag,
                                            const int4* __restrict__ tnode,
                                            const int4* __restrict__ vtx,
                                            const AngleGeom* __restrict__ ang, int beam, int a,
                                            int u, int v, int nu, int tw_log, double rmax,
                                            double g, int max_steps, int nverts, int e,
                                            size_t rid, const float* __restrict__ mu,
                                            const float* __restrict__ y,
                                            double* __restrict__ acc, double& sum,
                                            unsigned& n_cross, unsigned& n_exact,
                                            unsigned& n_lost, unsigned& n_stuck) {
    const UniFrame& U = Ug;
    const RayPts r = ft_scaled(ray_points(ang[a], beam, u, v));
    const double gs = g * (1.0 / (1 << kFtShift));
    Frame F;
    if constexpr (UNI == 0) make_frame_ax<AX>(r, rmax * (1 << kFtShift), gs, F);
    else make_frame_uni<AX, UNI>(r, U, F);
#if TRACE_BWD_WY32
    const float wy = BACK ? (float)((double)ld_stream(y + rid) * ray_scale<UNI>(F, U, gs)) : 0.f;
#else
    const double wy = BACK ? (double)y[rid] * ray_scale<UNI>(F, U, gs) : 0.0;
#endif
    const double tau = UNI ? U.tau : F.tau;
    const int t0 = e >> 2, kin = e & 3;
    int t = t0;
    DBG_CHECK(t >= 0 && t < max_steps);
    const int4 nodes = __ldg(tnode + t);
    int id0, id1, id2;
    if (kin == 0)      { id0 = nodes.y; id1 = nodes.z; id2 = nodes.w; }
    else if (kin == 1) { id0 = nodes.x; id1 = nodes.w; id2 = nodes.z; }
    else if (kin == 2) { id0 = nodes.x; id1 = nodes.y; id2 = nodes.w; }
    else               { id0 = nodes.x; id1 = nodes.z; id2 = nodes.y; }
    int iap = sel4(nodes, kin);
    double x0, y0, z0, x1, y1, z1, x2, y2, z2;
    xf<AX, UNI>(F, U, ft_scaled(__ldg(vtx + id0)), x0, y0, z0);
    xf<AX, UNI>(F, U, ft_scaled(__ldg(vtx + id1)), x1, y1, z1);
    xf<AX, UNI>(F, U, ft_scaled(__ldg(vtx + id2)), x2, y2, z2);
    unsigned n_exact_init = 0;
    double zin = face_depth(x0, y0, z0, x1, y1, z1, x2, y2, z2, (z0 + z1 + z2) * (1.0 / 3.0),
                            n_exact_init);
    int steps = 0;
    float mut = 0.f;
    if (!BACK) mut = __ldg(mu + t);
    int4 X = ft_scaled(__ldg(vtx + iap));                   // apex of the entry tet
    while (true) {
        double x3, y3, z3;
        xf<AX, UNI>(F, U, X, x3, y3, z3);
        const double p0 = side2(x3, y3, x0, y0);   // side(apex, slot k)
        const double p1 = side2(x3, y3, x1, y1);
        const double p2 = side2(x3, y3, x2, y2);
        unsigned neg = ((unsigned)__double2hiint(p0) >> 31) |
                       (((unsigned)__double2hiint(p1) >> 30) & 2u) |
                       (((unsigned)__double2hiint(p2) >> 29) & 4u);
        if (any_abs_le(p0, p1, p2, tau)) {
            const unsigned mask = (fabs(p0) <= tau ? 1u : 0u) | (fabs(p1) <= tau ? 2u : 0u) |
                                  (fabs(p2) <= tau ? 4u : 0u);
            if (TRACE_HEAVY_KEEP_RAY && KEEP) {   // exact-heavy shape: the ray's (unscaled) grid points
                neg = exact_neg_ray(vtx, r.ox >> kFtShift, r.oy >> kFtShift, r.oz >> kFtShift,
                                    r.px >> kFtShift, r.py >> kFtShift, r.pz >> kFtShift, mask,
                                    neg, iap, id0, id1, id2);
            } else if (BACK ? TRACE_BWD_ONECALL : TRACE_EXACT_ONECALL) {
                neg = exact_neg_here<BX, BY, BAND>(vtx, ang, beam, nu, tw_log, mask, neg, iap, id0, id1, id2);
            } else {
                const unsigned m = neg;
                neg = 0;
                neg |= (mask & 1u) ? (exact_side_here<BX, BY, BAND>(vtx, ang, beam, nu, tw_log, iap, id0) < 0 ? 1u : 0u) : (m & 1u);
                neg |= (mask & 2u) ? (exact_side_here<BX, BY, BAND>(vtx, ang, beam, nu, tw_log, iap, id1) < 0 ? 2u : 0u) : (m & 2u);
                neg |= (mask & 4u) ? (exact_side_here<BX, BY, BAND>(vtx, ang, beam, nu, tw_log, iap, id2) < 0 ? 4u : 0u) : (m & 4u);
            }
            n_exact += __popc(mask);
        }
        const int j = (int)((kExitLUT >> (2 * neg)) & 3u);
        const int idj = selp(id0, selp(id1, id2, j == 1), j == 0);
        const int L = rank4(id0, id1, id2, iap, idj);
        // the exit face's tag: issued now, consumed after this step's chord
        const int4 tg = ld_tag(tag + 4 * (size_t)t + (j == 3 ? 0 : L));
        const int tcur = t;
        if (j == 0) { x0 = x3; y0 = y3; z0 = z3; id0 = iap; }
        if (j == 1) { x1 = x3; y1 = y3; z1 = z3; id1 = iap; }
        if (j == 2) { x2 = x3; y2 = y3; z2 = z3; id2 = iap; }
        const double zout = face_depth(x0, y0, z0, x1, y1, z1, x2, y2, z2, zin, n_exact);
        const double dz = zout - zin;
        if (BACK) {
            if (dz > 0.0) red_acc(acc + tcur, dz * f2d_here(wy));
        } else {
            sum = fma(dz, (double)mut, sum);
        }
        const unsigned n26 = (unsigned)tg.w & kFtHull;
        const bool more = n26 != kFtHull && j != 3 && ++steps != max_steps;
        if (!more) {
            const bool stuck = n26 != kFtHull && j != 3;
            n_lost += j == 3 ? 1u : 0u;
            n_stuck += stuck ? 1u : 0u;
            n_cross += (unsigned)steps + (stuck ? 0u : 1u);
            break;
        }
        t = (int)n26;
        if (!BACK) mut = __ldg(mu + t);
        X = make_int4(tg.x & ~63, tg.y & ~63, tg.z & ~63, 0);
        iap = (int)(((unsigned)tg.w >> 26) | (((unsigned)tg.x & 63u) << 6) |
                    (((unsigned)tg.y & 63u) << 12) | (((unsigned)tg.z & 63u) << 18));
        DBG_CHECK(t >= 0 && t < max_steps && iap >= 0 && iap < nverts);
        zin = zout;
    }
    if (!BACK) sum *= ray_scale<UNI>(F, U, gs);
}

template <bool BACK, int BX, int BY, int MINB, bool LATE, bool BAND, bool FT>
__global__ void __launch_bounds__(32 * BX * BY, MINB) trace_kernel(const int4* __restrict__ rec,
                                                          const int4* __restrict__ tnode,
                                                          const int4* __restrict__ vtx,
                                                          const AngleGeom* __restrict__ ang,
                                                          int beam, int nv, int nu, double rmax,
                                                          double g, int max_steps,
                                                          const int* __restrict__ entry,
                                                          const float* __restrict__ mu,
                                                          float* __restrict__ proj,
                                                          const float* __restrict__ y,
                                                          double* __restrict__ acc,
                                                          unsigned long long* __restrict__ stats,
                                                          int tw_log, int nverts,
                                                          const __grid_constant__ UniFrames UF) {
    // warp tile: (1 << tw_log) x (32 >> tw_log) pixels; block = BX x BY warp
    // tiles; the argument carries tw_log | group << 4 (thread_pixel)
    const int tile_code = tw_log;
    if (BAND) tw_log &= 15;
    const int tw = 1 << tw_log, th = 32 >> tw_log;
    const int tiles_u = (nu + BX * tw - 1) / (BX * tw);
    int bx, by, a;
    if (BAND) {
        block_tile(tiles_u, tile_code >> 4, bx, by, a);
    } else {
        bx = blockIdx.x % tiles_u;
        by = blockIdx.x / tiles_u;
        a = blockIdx.y;
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int u = bx * BX * tw + (w % BX) * tw + (lane & (tw - 1));
    const int v = by * BY * th + (w / BX) * th + (lane >> tw_log);
    const bool valid = u < nu && v < nv;
    const size_t rid = ((size_t)a * nv + v) * nu + u;
    const int e = valid ? ld_stream(entry + rid) : -1;
#if TRACE_WARP_VOTE
    if (!__any_sync(0xffffffffu, e >= 0)) {   // no ray of this warp enters the mesh
        if (!BACK && valid) st_stream(proj + rid, 0.f);
        return;
    }
#elif TRACE_EMPTY_EXIT
    // a block none of whose rays enters the mesh (outside the silhouette:
    // ~half of c3's blocks) writes its zero projections and leaves before
    // the axis vote and the statistics reductions
    if (!__syncthreads_or(e >= 0)) {
        if (!BACK && valid) st_stream(proj + rid, 0.f);
        return;
    }
#endif

    unsigned n_cross = 0, n_exact = 0, n_lost = 0, n_stuck = 0;
    double sum = 0.0;
    // Warp-uniform shear axis (block-uniform with TRACE_WARP_VOTE = 0): the
    // warp tile's centre ray decides; every ray of the warp must be dominated
    // (|D_k| >= max|D|/2) by that axis with the same sign (warp vote), else the
    // generic per-ray frame (variant 6) is used.
    int ax = 6;
    {
#if TRACE_WARP_VOTE
        const int uc = min(bx * BX * tw + (w % BX) * tw + tw / 2, nu - 1);   // the warp tile's centre
        const int vc = min(by * BY * th + (w / BX) * th + th / 2, nv - 1);
#else
        const int uc = min(bx * BX * tw + BX * tw / 2, nu - 1);
        const int vc = min(by * BY * th + BY * th / 2, nv - 1);
#endif
        const RayPts rc = ray_points(ang[a], beam, uc, vc);
        const long long cx = rc.px - rc.ox, cy = rc.py - rc.oy, cz = rc.pz - rc.oz;
        const long long ax_ = cx < 0 ? -cx : cx, ay_ = cy < 0 ? -cy : cy, az_ = cz < 0 ? -cz : cz;
        const int kc = (ax_ >= ay_ && ax_ >= az_) ? 0 : (ay_ >= az_ ? 1 : 2);
        const long long dkc = kc == 0 ? cx : (kc == 1 ? cy : cz);
        bool ok = true;
        if (e >= 0) {
            const RayPts r = ray_points(ang[a], beam, u, v);
            const long long dx = r.px - r.ox, dy = r.py - r.oy, dz = r.pz - r.oz;
            const long long dk = kc == 0 ? dx : (kc == 1 ? dy : dz);
            const long long adk = dk < 0 ? -dk : dk;
            const long long m = max(dx < 0 ? -dx : dx, max(dy < 0 ? -dy : dy, dz < 0 ? -dz : dz));
            ok = (dk < 0) == (dkc < 0) && 2 * adk >= m;
        }
#if TRACE_WARP_VOTE
        if (__all_sync(0xffffffffu, ok)) ax = 2 * kc + (dkc < 0 ? 1 : 0);
#else
        if (__syncthreads_and(ok)) ax = 2 * kc + (dkc < 0 ? 1 : 0);
#endif
        // parallel beam: the uniform shear was made for the angle's axis variant
        if (beam != TET_BEAM_CONE && ax != (int)UF.f[a].q[2]) ax = 6;
    }
    const UniFrame& U = UF.f[a];
    if (e >= 0) {
#define WALK(AXV, UNI) do { \
    if (FT) walk_ray_ft<BACK, AXV, UNI, BX, BY, BAND, !LATE>(U, rec, tnode, vtx, ang, beam, a, u, v, nu, tile_code, rmax, g, \
                                      max_steps, nverts, e, rid, mu, y, acc, sum, n_cross, n_exact, n_lost, n_stuck); \
    else walk_ray<BACK, AXV, UNI, BX, BY, LATE, BAND>(U, rec, tnode, vtx, ang, beam, a, u, v, nu, tile_code, rmax, g, \
                                      max_steps, \
                                      nverts, e, rid, mu, y, acc, sum, n_cross, n_exact, n_lost, \
                                      n_stuck); } while (0)
        // uniform frames (TRACE_BWD_UNI = 0: per-ray frame in the backward walk)
        // (one kernel per beam type spills the forward walk's frame: the
        // register allocation of this combined kernel is the measured best)
        const bool cone = beam == TET_BEAM_CONE;
        if (BACK && !TRACE_BWD_UNI) {
            switch (ax) {
                case 0: WALK(0, 0); break;
                case 1: WALK(1, 0); break;
                case 2: WALK(2, 0); break;
                case 3: WALK(3, 0); break;
                case 4: WALK(4, 0); break;
                case 5: WALK(5, 0); break;
                default: WALK(6, 0); break;
            }
        } else {
            constexpr int PU = TRACE_PAR_UNI ? 2 : 0;
            switch (ax) {
                case 0: if (cone) WALK(0, 1); else WALK(0, PU); break;
                case 1: if (cone) WALK(1, 1); else WALK(1, PU); break;
                case 2: if (cone) WALK(2, 1); else WALK(2, PU); break;
                case 3: if (cone) WALK(3, 1); else WALK(3, PU); break;
                case 4: if (cone) WALK(4, 1); else WALK(4, PU); break;
                case 5: if (cone) WALK(5, 1); else WALK(5, PU); break;
                default: WALK(6, 0); break;
            }
        }
#undef WALK
    }
    if (!BACK && valid) st_stream(proj + rid, (float)sum);
    add_stat(stats, ST_HIT, e >= 0 ? 1u : 0u);
    add_stat(stats, ST_CROSS, n_cross);
    add_stat(stats, ST_EXACT, n_exact);
    add_stat(stats, ST_LOST, n_lost);
    add_stat(stats, ST_STUCK, n_stuck);
    const unsigned mx = __reduce_max_sync(0xffffffffu, n_cross);
    if (lane == 0 && mx) atomicMax(stats + ST_MAXC, (unsigned long long)mx);
}

// ------------------------------------------- paper-faithful walker ------
// NEXT-1: the paper's own traversal, kept verbatim to measure
// the robustness gap -- Alg. 1 "Möller Trumbore with safety parameter eps"
// and Alg. 2 in precision T on world
// coordinates.  The first tet comes from the exact entry map (the paper's
// R*-tree initialisation is replaced); everything after it is
// the paper's method, including its failure modes.
// Single IEEE operations (never contracted into FMAs) in the order Alg. 1
// writes them, so the MT modes compute exactly what IEEE arithmetic in T
// computes for the paper's algorithm -- the single-precision failures of
// fig:singledouble are then reproducible operation for operation.
__device__ __forceinline__ double o_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double o_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double o_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double o_div(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double o_sqrt(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ float o_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float o_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float o_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float o_div(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float o_sqrt(float a) { return __fsqrt_rn(a); }

template <class T>
__device__ __forceinline__ T o_dot(const T a[3], const T b[3]) {
    return o_add(o_add(o_mul(a[0], b[0]), o_mul(a[1], b[1])), o_mul(a[2], b[2]));
}

template <class T>
__device__ __forceinline__ void o_cross(const T a[3], const T b[3], T c[3]) {
    c[0] = o_sub(o_mul(a[1], b[2]), o_mul(a[2], b[1]));
    c[1] = o_sub(o_mul(a[2], b[0]), o_mul(a[0], b[2]));
    c[2] = o_sub(o_mul(a[0], b[1]), o_mul(a[1], b[0]));
}

template <class T>
__device__ __forceinline__ bool mt_hit(const T r1[3], const T d[3], const T p1[3], const T p2[3],
                                       const T p3[3], T eps, T& t) {
    const T e1[3] = {o_sub(p2[0], p1[0]), o_sub(p2[1], p1[1]), o_sub(p2[2], p1[2])};
    const T e2[3] = {o_sub(p3[0], p1[0]), o_sub(p3[1], p1[1]), o_sub(p3[2], p1[2])};
    T q[3];
    o_cross(d, e2, q);                                         // q = d x E2
    const T a = o_dot(e1, q);
    if (a > T(-1e-8) && a < T(1e-8)) return false;            // "Check if its zero"
    const T f = o_div(T(1), a);
    const T s[3] = {o_sub(r1[0], p1[0]), o_sub(r1[1], p1[1]), o_sub(r1[2], p1[2])};
    const T u = o_mul(f, o_dot(s, q));
    if (u < -eps) return false;
    T r[3];
    o_cross(s, e1, r);                                         // r = s x E1
    const T v = o_mul(f, o_dot(d, r));   // printed "d x r": a dot (R2 reading)
    if (v < -eps || o_add(u, v) > o_add(T(1), eps)) return false;
    t = o_mul(f, o_dot(e2, r));
    return true;
}

template <class T>
__device__ __forceinline__ void world_vertex(const int4* __restrict__ vtx, int id, double g,
                                             const double C[3], T out[3]) {
    const int4 X = __ldg(vtx + id);
    out[0] = (T)fma((double)X.x, g, C[0]);
    out[1] = (T)fma((double)X.y, g, C[1]);
    out[2] = (T)fma((double)X.z, g, C[2]);
}

template <class T, bool BACK>
__global__ void __launch_bounds__(128) mt_trace_kernel(const int4* __restrict__ rec,
                                                       const int4* __restrict__ tnode,
                                                       const int4* __restrict__ vtx,
                                                       const AngleGeom* __restrict__ ang,
                                                       int beam, int nv, int nu, double g,
                                                       double cx, double cy, double cz,
                                                       int max_steps, double eps0,
                                                       double eps_growth, int max_esc,
                                                       const int* __restrict__ entry,
                                                       const float* __restrict__ mu,
                                                       float* __restrict__ proj,
                                                       const float* __restrict__ y,
                                                       double* __restrict__ acc,
                                                       unsigned long long* __restrict__ stats) {
    const int tiles_u = (nu + 15) >> 4;
    const int bx = blockIdx.x % tiles_u, by = blockIdx.x / tiles_u;
    const int a = blockIdx.y;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int u = bx * 16 + (w & 1) * 8 + (lane & 7);
    const int v = by * 8 + (w >> 1) * 4 + (lane >> 3);
    const bool valid = u < nu && v < nv;
    const size_t rid = ((size_t)a * nv + v) * nu + u;
    const int e = valid ? entry[rid] : -1;
    const double C[3] = {cx, cy, cz};
    unsigned n_cross = 0, n_lost = 0, n_stuck = 0, n_esc = 0;
    double sum = 0.0;
    if (e >= 0) {
        const RayPts rp = ray_points(ang[a], beam, u, v);
        const double R1d[3] = {fma((double)rp.ox, g, C[0]), fma((double)rp.oy, g, C[1]),
                               fma((double)rp.oz, g, C[2])};
        const double R2d[3] = {fma((double)rp.px, g, C[0]), fma((double)rp.py, g, C[1]),
                               fma((double)rp.pz, g, C[2])};
        const T R1[3] = {(T)R1d[0], (T)R1d[1], (T)R1d[2]};
        const T R2[3] = {(T)R2d[0], (T)R2d[1], (T)R2d[2]};
        const T d[3] = {o_sub(R2[0], R1[0]), o_sub(R2[1], R1[1]), o_sub(R2[2], R1[2])};
        const T l = o_sqrt(o_dot(d, d));                             // l = ||R2 - R1||
        const float yv = BACK ? y[rid] : 0.f;
        int t = e >> 2, prev = -1;
        int steps = 0;
        while (t >= 0) {
            DBG_CHECK(t >= 0);
            const int4 nd = __ldg(tnode + t);
            const int ids[4] = {nd.x, nd.y, nd.z, nd.w};
            T P[4][3];
            for (int k = 0; k < 4; ++k) world_vertex<T>(vtx, ids[k], g, C, P[k]);
            // while not Intersection: TetraRayIntersection(i_now, eps); eps *= 10
            T eps = (T)eps0;
            int esc = 0, nhit = 0, kmin = -1, kmax = -1;
            T tmin = 0, tmax = 0;
            while (true) {
                nhit = 0;
                for (int k = 0; k < 4; ++k) {   // the face opposite node k
                    const int i0 = k == 0 ? 1 : 0, i1 = k <= 1 ? 2 : 1, i2 = k <= 2 ? 3 : 2;
                    T th;
                    if (mt_hit<T>(R1, d, P[i0], P[i1], P[i2], eps, th)) {
                        // t1: the first face with the minimal t; t2: the last
                        // with the maximal t -- two hits at equal t come out
                        // in encounter order (R16)
                        if (nhit == 0 || th < tmin) { tmin = th; kmin = k; }
                        if (nhit == 0 || th >= tmax) { tmax = th; kmax = k; }
                        ++nhit;
                    }
                }
                if (nhit >= 2 || esc >= max_esc) break;
                eps = o_mul(eps, (T)eps_growth);
                ++esc;
            }
            n_esc += esc;
            if (nhit < 2) { ++n_lost; break; }                // the "black dots"
            const double chord = (double)o_mul(l, o_sub(tmax, tmin));   // l (t2 - t1)
            if (BACK) {
                if (chord > 0.0) atomicAdd(acc + t, chord * (double)yv);
            } else {
                sum = o_add(sum, o_mul(chord, (double)__ldg(mu + t)));
            }
            ++n_cross;
            // neighbour of the face where t2 happened; "if t2 = t1 check if they
            // need to be swapped": do not step back into the previous element
            // (face tags are stored by the rank of the opposite vertex id)
            const int4 r0 = __ldg(rec + 2 * (size_t)t), r1v = __ldg(rec + 2 * (size_t)t + 1);
            const int nb[4] = {r0.x, r0.z, r1v.x, r1v.z};
            auto rank = [&](int k) {
                int r = 0;
                for (int q = 0; q < 4; ++q) r += ids[q] < ids[k];
                return r;
            };
            int nxt = nb[rank(kmax)];
            if (tmax == tmin && nxt == prev && kmin != kmax) nxt = nb[rank(kmin)];
            prev = t;
            t = nxt;
            if (++steps >= max_steps) { ++n_stuck; break; }
        }
    }
    if (!BACK && valid) proj[rid] = (float)sum;
    add_stat(stats, ST_HIT, e >= 0 ? 1u : 0u);
    add_stat(stats, ST_CROSS, n_cross);
    add_stat(stats, ST_LOST, n_lost);
    add_stat(stats, ST_STUCK, n_stuck);
    add_stat(stats, ST_ESC, n_esc);
    const unsigned mx = __reduce_max_sync(0xffffffffu, n_cross);
    if (lane == 0 && mx) atomicMax(stats + ST_MAXC, (unsigned long long)mx);
}

cudaError_t launch_mt(const DevMesh& m, const LaunchChunk& c, bool back, bool single,
                      const MtOptions& o, const int* entry, const float* mu_int, float* proj,
                      const float* y, double* acc, unsigned long long* stats, cudaStream_t s) {
    const dim3 grid(((c.nu + 15) / 16) * ((c.nv + 7) / 8), c.n_angles);
    // loop detection for the MT modes: 10 ceil(T^(1/3)) + 100 elements per ray
    // (SPEC.md:315 reading) -- a straight line crosses O(T^(1/3)) elements
    const int steps = 10 * (int)ceil(cbrt((double)m.nt)) + 100;
#define MT_ARGS m.rec, m.tnode, m.vtx, c.ang, c.beam, c.nv, c.nu, m.g, m.C[0], m.C[1], m.C[2], \
                steps, o.eps0, o.eps_growth, o.max_escalations, entry, mu_int, proj, y, acc, stats
    if (single) {
        if (back) mt_trace_kernel<float, true><<<grid, 128, 0, s>>>(MT_ARGS);
        else mt_trace_kernel<float, false><<<grid, 128, 0, s>>>(MT_ARGS);
    } else {
        if (back) mt_trace_kernel<double, true><<<grid, 128, 0, s>>>(MT_ARGS);
        else mt_trace_kernel<double, false><<<grid, 128, 0, s>>>(MT_ARGS);
    }
#undef MT_ARGS
    return cudaGetLastError();
}

// ------------------------------------------------------------ permute ---
__global__ void gather_mu_kernel(const int* __restrict__ perm, const float* __restrict__ mu,
                                 float* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        DBG_CHECK(perm[i] >= 0 && perm[i] < n);
        out[i] = __ldg(mu + perm[i]);
    }
}

__global__ void scatter_x_kernel(const int* __restrict__ perm, const double* __restrict__ acc,
                                 float* __restrict__ x, int accumulate, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int j = perm[i];
        x[j] = accumulate ? (float)((double)x[j] + acc[i]) : (float)acc[i];
    }
}

__global__ void scatter_acc_kernel(const int* __restrict__ perm, const double* __restrict__ acc,
                                   double* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[perm[i]] += acc[i];
}

static int grid_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    return (int)(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

// ----------------------------------------------------------- launchers --
size_t entry_scratch_bytes(const DevMesh& m, int n_angles) {
    return sizeof(EntryItem) * (size_t)m.nb * n_angles + 256;
}

cudaError_t launch_entry_bvh(const DevMesh& m, const LaunchChunk& c, int* entry,
                             unsigned long long* stats, cudaStream_t s) {
    const dim3 grid((unsigned)(((c.nu + 15) / 16) * ((c.nv + 7) / 8)), (unsigned)c.n_angles);
    entry_bvh_kernel<<<grid, 128, 0, s>>>(m.bvh_nodes, m.bvh_faces, m.vtx, c.ang, c.beam, c.nv,
                                          c.nu, entry, stats);
    return cudaGetLastError();
}

cudaError_t launch_entry_rtree(const DevMesh& m, const LaunchChunk& c, int* entry,
                               unsigned long long* stats, cudaStream_t s) {
    const dim3 grid((unsigned)(((c.nu + 15) / 16) * ((c.nv + 7) / 8)), (unsigned)c.n_angles);
    entry_rtree_kernel<<<grid, 128, 0, s>>>(m.rtree, m.bvh_faces, m.vtx, c.ang, c.beam, c.nv,
                                            c.nu, entry, stats);
    return cudaGetLastError();
}

cudaError_t launch_entry(const DevMesh& m, const LaunchChunk& c, int* entry, void* scratch,
                         unsigned long long* stats, cudaStream_t s) {
    unsigned* n_items = (unsigned*)scratch;   // [0] large items, [1] queue, [2] small items
    EntryItem* items = (EntryItem*)((char*)scratch + 256);
    const long long n = (long long)m.nb * c.n_angles;
    cudaError_t e = cudaMemsetAsync(n_items, 0, 3 * sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    entry_setup_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(
        m.tnode, m.vtx, m.hull, (int)m.nb, c.ang, c.aux, c.beam, c.n_angles, c.nv, c.nu, items,
        n_items, (unsigned)n, ENTRY_SMALL_PX);
    if (ENTRY_SMALL_PX > 0)
        entry_small_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(
            m.vtx, c.ang, c.beam, c.nv, c.nu, items, (unsigned)n, n_items + 2, entry, stats);
    static const unsigned grid = [] {
        int dev = 0, sms = 148, per = 8;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, entry_raster_kernel, 128, 0);
        return (unsigned)(sms * (per > 0 ? per : 1));
    }();
    const unsigned blocks = (unsigned)std::min<long long>(grid, (n + 3) / 4);
    entry_raster_kernel<<<blocks, 128, 0, s>>>(m.vtx, c.ang, c.beam, c.nv, c.nu, items, n_items,
                                               n_items + 1, entry, stats);
    return cudaGetLastError();
}

// Warp pixel tile of the exact walker: (1 << tw_log) x (32 >> tw_log); default
// 8 x 4 (TETPROJ_TILE_W overrides for measurements).
static int tile_w_log() {
    static int v = [] {
        const char* e = getenv("TETPROJ_TILE_W");
        const int w = e ? atoi(e) : 8;
        return w == 4 ? 2 : w == 16 ? 4 : w == 32 ? 5 : w == 2 ? 1 : 3;
    }();
    return v;
}

static size_t l2_bytes() {
    static const size_t v = [] {
        int dev = 0, b = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&b, cudaDevAttrL2CacheSize, dev);
        return (size_t)(b > 0 ? b : 126 << 20);
    }();
    return v;
}

static dim3 trace_grid_w(const LaunchChunk& c, int tw_log, int bx, int by) {
    const int tw = 1 << tw_log, th = 32 >> tw_log;
    const unsigned tiles = (unsigned)(((c.nu + bx * tw - 1) / (bx * tw)) *
                                      ((c.nv + by * th - 1) / (by * th)));
    return dim3(tiles, (unsigned)c.n_angles);
}

#define TRACE_ARGS rec_or_tag, m.tnode, m.vtx, c.ang, c.beam, c.nv, c.nu, m.rmax, m.g, steps, entry, \
                   mu_int, proj, y, acc, stats

// Walker block shape (BX x BY warp tiles) and the blocks per SM it is compiled
// for (register cap 65536 / (32 BX BY MINB)): with the block-uniform frame and
// the next step's gathers issued late (TRACE_*_LATE_LOADS) both walks are
// fastest at 2x2 tiles, 8 blocks (64 registers, 32 warps/SM: the dependent
// gather chain wants latency hiding more than registers; profiles/README.md).
#ifndef TRACE_FWD_BX
#define TRACE_FWD_BX 2
#define TRACE_FWD_BY 2
#define TRACE_FWD_MINB 8
#endif
#ifndef TRACE_BWD_BX
#define TRACE_BWD_BX 2
#define TRACE_BWD_BY 2
#define TRACE_BWD_MINB 8
#endif
// Exact-heavy scans (a large share of the signs go to the int128 + SoS
// path, e.g. lattice rays through mesh vertices, c4a) run a second shape:
// fewer blocks, more registers, early gathers -- at 64 registers each
// noinline exact call saves and restores live state and the exact path
// itself spills (c4a 7.8e9 -> 4.6e9 crossings/s with the fast shape).
// api.cu picks it from the exact-fallback rate of the mesh's last call with
// statistics (LaunchChunk::exact_heavy).
template <bool BACK, bool HEAVY> struct TraceShape;
// MINB_FT: blocks per SM of the FT16 walk.  Its backward holds fewer live
// registers (no 32-B record, no vertex quad): 10 blocks at 48 registers
// (40 warps/SM) hide more of the RED traffic's latency than 8 at 64 (c3
// backward 32.96 -> 31.72 ms; 9 blocks 32.69, 11-12 blocks spill: 39.9;
// the forward prefers 8: 26.6 vs 29.6 ms at 10), profiles/README.md.
#ifndef TRACE_FT_BWD_MINB
#define TRACE_FT_BWD_MINB 10
#endif
// ... and of the band-ordered backward (meshes beyond half the L2, c5): 8
// blocks at 64 registers (c5 backward 545 ms at 10, 530 at 9, 526 at 8, 558
// at 7, 568 at 6; c3's angle-ordered backward stays at 10: 30.4 vs 30.9 ms
// at 9), profiles/README.md
#ifndef TRACE_FT_BWD_BAND_MINB
#define TRACE_FT_BWD_BAND_MINB 8
#endif
template <> struct TraceShape<false, false> {
    static constexpr int BX = TRACE_FWD_BX, BY = TRACE_FWD_BY, MINB = TRACE_FWD_MINB;
    static constexpr int MINB_FT = TRACE_FWD_MINB, MINB_FT_BAND = MINB_FT;
    static constexpr bool LATE = TRACE_FWD_LATE_LOADS;
};
template <> struct TraceShape<true, false> {
    static constexpr int BX = TRACE_BWD_BX, BY = TRACE_BWD_BY, MINB = TRACE_BWD_MINB;
    static constexpr int MINB_FT = TRACE_FT_BWD_MINB, MINB_FT_BAND = TRACE_FT_BWD_BAND_MINB;
    static constexpr bool LATE = TRACE_BWD_LATE_LOADS;
};
#ifndef TRACE_HEAVY_FWD_MINB
#define TRACE_HEAVY_FWD_MINB 4
#endif
template <> struct TraceShape<false, true> {
    static constexpr int BX = 2, BY = 2, MINB = TRACE_HEAVY_FWD_MINB, MINB_FT = MINB,
                         MINB_FT_BAND = MINB;
    static constexpr bool LATE = false;
};
#ifndef TRACE_HEAVY_BWD_MINB
#define TRACE_HEAVY_BWD_MINB 4
#endif
template <> struct TraceShape<true, true> {
    static constexpr int BX = 2, BY = 2, MINB = TRACE_HEAVY_BWD_MINB, MINB_FT = MINB,
                         MINB_FT_BAND = MINB;
    static constexpr bool LATE = false;
};

// Host half of make_frame_uni: the block-uniform frame of each angle, in
// grid units / `sc` (sc = 64 for the FT16 walk, whose coordinates are x64).
static void make_uni_frames(const DevMesh& m, const LaunchChunk& c, UniFrames& U, double sc) {
    for (int a = 0; a < c.n_angles; ++a) {
        const AngleGeom& G = c.host_ang[a];
        UniFrame& f = U.f[a];
        if (c.beam == TET_BEAM_CONE) {
            double n2 = 0;
            for (int i = 0; i < 3; ++i) {
                f.q[i] = (double)G.o[i] * sc;
                n2 += f.q[i] * f.q[i];
            }
            // |X - S| <= |S| + rmax;  (1 + |sx| + |sy|) / 2 <= 2.5
            const double amax = (std::sqrt(n2) + m.rmax * sc) * 2.5;
            f.tau = amax * amax * 0x1p-38;
            f.scale = 0;
        } else {
            // the axis variant the block vote picks for direction d (trace_kernel)
            const long long* d = G.o;
            const long long ax_ = std::llabs(d[0]), ay_ = std::llabs(d[1]), az_ = std::llabs(d[2]);
            const int k = (ax_ >= ay_ && ax_ >= az_) ? 0 : (ay_ >= az_ ? 1 : 2);
            const int AX = 2 * k + (d[k] < 0 ? 1 : 0);
            const int c1 = (k + 1) % 3, c2 = (k + 2) % 3;
            const int K1 = (AX & 1) ? c2 : c1, K2 = (AX & 1) ? c1 : c2;
            const double adk = std::fabs((double)d[k]);
            f.q[0] = (double)d[K1] / adk;
            f.q[1] = (double)d[K2] / adk;
            f.q[2] = (double)AX;
            // |o| over the detector (o = P - d, convex in (u, v): corners)
            double omax = 0;
            for (int cv = 0; cv < 2; ++cv)
                for (int cu = 0; cu < 2; ++cu) {
                    const long long u = cu ? c.nu - 1 : 0, v = cv ? c.nv - 1 : 0;
                    double n2 = 0;
                    for (int i = 0; i < 3; ++i) {
                        const double o = (double)(G.p00[i] + u * G.du[i] + v * G.dv[i] - d[i]);
                        n2 += o * o;
                    }
                    omax = std::max(omax, std::sqrt(n2));
                }
            const double amax = (omax + m.rmax) * sc * (1.0 + std::fabs(f.q[0]) + std::fabs(f.q[1])) * 0.5;
            f.tau = amax * amax * 0x1p-38;
            const double dx = (double)d[0], dy = (double)d[1], dz = (double)d[2];
            f.scale = std::sqrt(dx * dx + dy * dy + dz * dz) / adk * (m.g / sc);
        }
    }
}

template <bool BACK, bool HEAVY>
static void launch_trace(const DevMesh& m, const LaunchChunk& c, const int* entry,
                         const float* mu_int, float* proj, const float* y, double* acc,
                         unsigned long long* stats, cudaStream_t s) {
    using S = TraceShape<BACK, HEAVY>;
    const int steps = (int)(m.nt < 0x7fffffff ? m.nt : 0x7fffffff);
    const int twl = tile_w_log();
    // band-ordered blocks (block_tile) for a mesh whose tag records do not
    // fit in half the L2 (c5: 337 MB): all the launch's angles per band in
    // the forward walk; angle pairs in the backward walk -- rays of many
    // angles through the same slab at once make its f64 REDs collide (full
    // band order: c3 backward 34.8 -> 52.9 ms).  L2-resident meshes keep
    // angle order (c3 forward 27.1 -> 27.3 ms with bands).
    const bool big = TRACE_BAND_ORDER && (size_t)m.nt * TRACE_BAND_BYTES_PER_TET > l2_bytes() / 2;
    const int group = big ? (BACK ? TRACE_BWD_BAND_GROUP : TRACE_FWD_BAND_GROUP) : 0;
    const int tile_code = twl | group << 4;
    static thread_local UniFrames U;   // 10 KB: copied into the launch parameters
    // FT16 walk (coordinates x64), except for exact-heavy scans: there the
    // rec walk's shape measured faster (c4a 9.32e9 vs 8.98e9 crossings/s)
    const bool ft = m.tag16 != nullptr && (!HEAVY || TRACE_HEAVY_FT);
    make_uni_frames(m, c, U, ft ? (double)(1 << kFtShift) : 1.0);
    auto kern = ft ? (big ? trace_kernel<BACK, S::BX, S::BY, S::MINB_FT_BAND, S::LATE, true, true>
                          : trace_kernel<BACK, S::BX, S::BY, S::MINB_FT, S::LATE, false, true>)
                   : (big ? trace_kernel<BACK, S::BX, S::BY, S::MINB, S::LATE, true, false>
                          : trace_kernel<BACK, S::BX, S::BY, S::MINB, S::LATE, false, false>);
    const int4* rec_or_tag = ft ? m.tag16 : m.rec;

    if (m.l2_window_bytes == 0) {
        kern<<<trace_grid_w(c, twl, S::BX, S::BY), 32 * S::BX * S::BY, 0, s>>>(TRACE_ARGS, tile_code,
                                                                               (int)m.nv, U);
        return;
    }
    // L2 persistence hint for the face-tag records (per launch; the caller's
    // stream attributes are not touched): hits persist, misses stream.
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = trace_grid_w(c, twl, S::BX, S::BY);
    cfg.blockDim = dim3(32 * S::BX * S::BY);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow.base_ptr = (void*)rec_or_tag;   // the table this walk gathers
    attr[0].val.accessPolicyWindow.num_bytes = m.l2_window_bytes;
    attr[0].val.accessPolicyWindow.hitRatio = (float)m.l2_hit_ratio;
    attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, TRACE_ARGS,
                       tile_code, (int)m.nv, U);
}

cudaError_t launch_forward(const DevMesh& m, const LaunchChunk& c, const int* entry,
                           const float* mu_int, float* proj, unsigned long long* stats,
                           cudaStream_t s) {
    if (c.n_angles > kUniMaxAngles) return cudaErrorInvalidValue;   // api.cu chunks by it
    if (c.exact_heavy) launch_trace<false, true>(m, c, entry, mu_int, proj, nullptr, nullptr, stats, s);
    else launch_trace<false, false>(m, c, entry, mu_int, proj, nullptr, nullptr, stats, s);
    return cudaGetLastError();
}

cudaError_t launch_backward(const DevMesh& m, const LaunchChunk& c, const int* entry,
                            const float* y, double* acc, unsigned long long* stats,
                            cudaStream_t s) {
    if (c.n_angles > kUniMaxAngles) return cudaErrorInvalidValue;   // api.cu chunks by it
    if (c.exact_heavy) launch_trace<true, true>(m, c, entry, nullptr, nullptr, y, acc, stats, s);
    else launch_trace<true, false>(m, c, entry, nullptr, nullptr, y, acc, stats, s);
    return cudaGetLastError();
}

cudaError_t launch_gather_mu(const DevMesh& m, const float* mu, float* mu_int, cudaStream_t s) {
    gather_mu_kernel<<<grid_for(m.nt), 256, 0, s>>>(m.perm, mu, mu_int, m.nt);
    return cudaGetLastError();
}

cudaError_t launch_scatter_x(const DevMesh& m, const double* acc, float* x, int accumulate,
                             cudaStream_t s) {
    scatter_x_kernel<<<grid_for(m.nt), 256, 0, s>>>(m.perm, acc, x, accumulate, m.nt);
    return cudaGetLastError();
}

cudaError_t launch_scatter_acc(const DevMesh& m, const double* acc, double* out,
                               cudaStream_t s) {
    scatter_acc_kernel<<<grid_for(m.nt), 256, 0, s>>>(m.perm, acc, out, m.nt);
    return cudaGetLastError();
}

}  // namespace tetproj
