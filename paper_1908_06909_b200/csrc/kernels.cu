// kernels.cu -- sm_100a kernels of libtetproj.
//
//   entry_kernel      hull-entry finder: per (hull face,
//                     angle) block, exact test of every pixel in the face's
//                     detector footprint; writes entry[ray] = tet<<2 | k.
//   trace_kernel<B>   ray walk (a4) + forward accumulate (a5, B=false) or
//                     backprojection scatter (a6, B=true).  Alg. 2 of the
//                     paper with exact sign decisions.
//   gather / scatter  caller order <-> internal SFC order (K4).
//
// Exactness (R2-R4): side(a,b) = sign det[a-o, b-o, p-o] on the
// integer grid, symbolically perturbed.  The hot loop evaluates it in fp64
// in a per-ray orthonormal frame (2 FMAs per side) and certifies the sign
// with a static error bound tau; only |side| <= tau falls back to an int128
// evaluation of the determinant and the 9-term SoS table.
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace tetproj {

typedef __int128 i128;

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

// ------------------------------------------------------------ frame -----
struct Frame {
    double e1x, e1y, e1z, e2x, e2y, e2z, e3x, e3y, e3z;
    double oe1, oe2, oe3;
    double tau;
};

// Orthonormal frame with e3 = (p-o)/|p-o|; x,y of a point give
// det[a-o,b-o,p-o]/|p-o| = x_a y_b - y_a x_b.  tau bounds the rounding error
// of that 2x2 determinant for every vertex |X| <= rmax.
__device__ __forceinline__ void make_frame(const RayPts& r, double rmax, Frame& F) {
    const double Dx = (double)(r.px - r.ox), Dy = (double)(r.py - r.oy), Dz = (double)(r.pz - r.oz);
    const double inv = rsqrt(Dx * Dx + Dy * Dy + Dz * Dz);
    F.e3x = Dx * inv; F.e3y = Dy * inv; F.e3z = Dz * inv;
    const double ax = fabs(F.e3x), ay = fabs(F.e3y), az = fabs(F.e3z);
    double tx, ty, tz;
    if (ax <= ay && ax <= az) { tx = 0.0; ty = F.e3z; tz = -F.e3y; }
    else if (ay <= az)        { tx = -F.e3z; ty = 0.0; tz = F.e3x; }
    else                      { tx = F.e3y; ty = -F.e3x; tz = 0.0; }
    const double it = rsqrt(tx * tx + ty * ty + tz * tz);
    F.e1x = tx * it; F.e1y = ty * it; F.e1z = tz * it;
    F.e2x = F.e3y * F.e1z - F.e3z * F.e1y;
    F.e2y = F.e3z * F.e1x - F.e3x * F.e1z;
    F.e2z = F.e3x * F.e1y - F.e3y * F.e1x;
    const double ox = (double)r.ox, oy = (double)r.oy, oz = (double)r.oz;
    F.oe1 = ox * F.e1x + oy * F.e1y + oz * F.e1z;
    F.oe2 = ox * F.e2x + oy * F.e2y + oz * F.e2z;
    F.oe3 = ox * F.e3x + oy * F.e3y + oz * F.e3z;
    const double amax = sqrt(ox * ox + oy * oy + oz * oz) + rmax;
    F.tau = amax * amax * 0x1p-40;
}

__device__ __forceinline__ void xform(const Frame& F, const int4 v, double& x, double& y,
                                      double& z) {
    const double X = (double)v.x, Y = (double)v.y, Z = (double)v.z;
    x = fma(X, F.e1x, fma(Y, F.e1y, fma(Z, F.e1z, -F.oe1)));
    y = fma(X, F.e2x, fma(Y, F.e2y, fma(Z, F.e2z, -F.oe2)));
    z = fma(X, F.e3x, fma(Y, F.e3y, fma(Z, F.e3z, -F.oe3)));
}

__device__ __forceinline__ double side2(double xa, double ya, double xb, double yb) {
    return fma(xa, yb, -(ya * xb));
}

__device__ __forceinline__ int sel4(int4 v, int k) {
    return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
}

__device__ __forceinline__ int4 ldg_nc_v4(const int4* p) {
    int4 r;
    asm volatile("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
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

__global__ void __launch_bounds__(256) entry_kernel(const int4* __restrict__ rec,
                                                    const int4* __restrict__ vtx,
                                                    const int2* __restrict__ hull,
                                                    const AngleGeom* __restrict__ ang,
                                                    const AngleAux* __restrict__ aux, int beam,
                                                    int nv, int nu, int* __restrict__ entry,
                                                    unsigned long long* __restrict__ stats) {
    const int h = blockIdx.x, a = blockIdx.y;
    const int2 hk = hull[h];
    const int4 nodes = ldg_nc_v4(rec + 2 * (size_t)hk.x);
    const int k = hk.y;
    // outward order of face k (opposite node k)
    int ia, ib, ic;
    if (k == 0)      { ia = nodes.y; ib = nodes.z; ic = nodes.w; }
    else if (k == 1) { ia = nodes.x; ib = nodes.w; ic = nodes.z; }
    else if (k == 2) { ia = nodes.x; ib = nodes.y; ic = nodes.w; }
    else             { ia = nodes.x; ib = nodes.z; ic = nodes.y; }
    const int4 A = __ldg(vtx + ia), B = __ldg(vtx + ib), C = __ldg(vtx + ic);
    const AngleGeom G = ang[a];
    const AngleAux X = aux[a];
    // --- cull: every detector-corner ray leaves through this face's plane
    const double e1[3] = {(double)B.x - A.x, (double)B.y - A.y, (double)B.z - A.z};
    const double e2[3] = {(double)C.x - A.x, (double)C.y - A.y, (double)C.z - A.z};
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
    const int4 V3[3] = {A, B, C};
    for (int j = 0; j < 3; ++j) {
        const double P[3] = {(double)V3[j].x, (double)V3[j].y, (double)V3[j].z};
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
            const double s = ((P[0] - X.P00[0]) * X.N[0] + (P[1] - X.P00[1]) * X.N[1] +
                              (P[2] - X.P00[2]) * X.N[2]) / dN;
            for (int i = 0; i < 3; ++i) Q[i] = P[i] - s * X.S[i];
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
    const int bw = u1 - u0 + 1;
    const long long npx = (long long)bw * (v1 - v0 + 1);
    const int code = (hk.x << 2) | k;
    unsigned conflicts = 0, exact = 0;
    for (long long i = threadIdx.x; i < npx; i += blockDim.x) {
        const int u = u0 + (int)(i % bw), v = v0 + (int)(i / bw);
        const RayPts r = ray_points(G, beam, u, v);
        // entering iff side(a,b) = side(b,c) = side(c,a) = -1 (outward order)
        if (side_direct(A, B, r, exact) != -1) continue;
        if (side_direct(B, C, r, exact) != -1) continue;
        if (side_direct(C, A, r, exact) != -1) continue;
        const int old = atomicExch(entry + ((size_t)a * nv + v) * nu + u, code);
        conflicts += (old != -1);
    }
    if (conflicts) atomicAdd(stats + ST_CONFLICT, (unsigned long long)conflicts);
    if (exact) atomicAdd(stats + ST_EXACT, (unsigned long long)exact);
}

// ------------------------------------------------------------ walker ----
template <bool BACK>
__global__ void __launch_bounds__(128) trace_kernel(const int4* __restrict__ rec,
                                                    const int4* __restrict__ vtx,
                                                    const AngleGeom* __restrict__ ang, int beam,
                                                    int nv, int nu, double rmax, double g,
                                                    long long max_steps,
                                                    const int* __restrict__ entry,
                                                    const float* __restrict__ mu,
                                                    float* __restrict__ proj,
                                                    const float* __restrict__ y,
                                                    double* __restrict__ acc,
                                                    unsigned long long* __restrict__ stats) {
    // 16x8 pixel tile per block, 8x4 per warp
    const int tiles_u = (nu + 15) >> 4;
    const int bx = blockIdx.x % tiles_u, by = blockIdx.x / tiles_u;
    const int a = blockIdx.y;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int u = bx * 16 + (w & 1) * 8 + (lane & 7);
    const int v = by * 8 + (w >> 1) * 4 + (lane >> 3);
    const bool valid = u < nu && v < nv;
    const size_t rid = ((size_t)a * nv + v) * nu + u;
    const int e = valid ? entry[rid] : -1;

    unsigned n_cross = 0, n_exact = 0, n_lost = 0, n_stuck = 0;
    double sum = 0.0;
    if (e >= 0) {
        const AngleGeom G = ang[a];
        const RayPts r = ray_points(G, beam, u, v);
        Frame F;
        make_frame(r, rmax, F);
        const float yv = BACK ? y[rid] : 0.f;
        int t = e >> 2, kin = e & 3;
        int4 nodes = ldg_nc_v4(rec + 2 * (size_t)t);
        int ia, ib, ic;
        if (kin == 0)      { ia = nodes.y; ib = nodes.z; ic = nodes.w; }
        else if (kin == 1) { ia = nodes.x; ib = nodes.w; ic = nodes.z; }
        else if (kin == 2) { ia = nodes.x; ib = nodes.y; ic = nodes.w; }
        else               { ia = nodes.x; ib = nodes.z; ic = nodes.y; }
        double xa, ya, za, xb, yb, zb, xc, yc, zc;
        xform(F, __ldg(vtx + ia), xa, ya, za);
        xform(F, __ldg(vtx + ib), xb, yb, zb);
        xform(F, __ldg(vtx + ic), xc, yc, zc);
        // entry face sides (exact signs are all -1: certified by the entry finder)
        double sab = side2(xa, ya, xb, yb), sbc = side2(xb, yb, xc, yc), sca = side2(xc, yc, xa, ya);
        double zin;
        {
            const double wa = fmax(-sbc, 0.0), wb = fmax(-sca, 0.0), wc = fmax(-sab, 0.0);
            const double sw = wa + wb + wc;
            zin = sw > 0 ? (wa * za + wb * zb + wc * zc) / sw : (za + zb + zc) * (1.0 / 3.0);
        }
        long long steps = 0;
        while (true) {
            const int4 tags = ldg_nc_v4(rec + 2 * (size_t)t + 1);
            float mut = 0.f;
            if (!BACK) mut = __ldg(mu + t);
            const int iap = sel4(nodes, kin);  // apex: node opposite the entry face
            double x3, y3, z3;
            xform(F, __ldg(vtx + iap), x3, y3, z3);
            const double pa = side2(x3, y3, xa, ya);
            const double pb = side2(x3, y3, xb, yb);
            const double pc = side2(x3, y3, xc, yc);
            // exit: the unique i with sign(p_i) = -1 and sign(p_{i+1}) = +1
            int sa = pa > F.tau ? 1 : pa < -F.tau ? -1 : 0;
            if (!sa) { sa = exact_side_ids(vtx, ang, beam, a, u, v, iap, ia); ++n_exact; }
            int i;
            if (sa < 0) {
                int sb = pb > F.tau ? 1 : pb < -F.tau ? -1 : 0;
                if (!sb) { sb = exact_side_ids(vtx, ang, beam, a, u, v, iap, ib); ++n_exact; }
                i = sb > 0 ? 0 : 1;
                if (i == 1 && pc < -F.tau) ++n_lost;   // (-,-,-) is impossible
            } else {
                int sc = pc > F.tau ? 1 : pc < -F.tau ? -1 : 0;
                if (!sc) { sc = exact_side_ids(vtx, ang, beam, a, u, v, iap, ic); ++n_exact; }
                i = sc < 0 ? 2 : 1;
                if (i == 1 && pb > F.tau) ++n_lost;    // (+,+,+) is impossible
            }
            // exit face (apex, Q, R), opposite vertex O; weights of the crossing
            // point: w_apex = -s(Q,R), w_Q = -s(R,apex) = p_R, w_R = -s(apex,Q) = -p_Q
            int iq, ir, io;
            double xq, yq, zq, xr, yr, zr, sqr, pq, pr;
            if (i == 0)      { iq = ia; ir = ib; io = ic; xq = xa; yq = ya; zq = za; xr = xb; yr = yb; zr = zb; sqr = sab; pq = pa; pr = pb; }
            else if (i == 1) { iq = ib; ir = ic; io = ia; xq = xb; yq = yb; zq = zb; xr = xc; yr = yc; zr = zc; sqr = sbc; pq = pb; pr = pc; }
            else             { iq = ic; ir = ia; io = ib; xq = xc; yq = yc; zq = zc; xr = xa; yr = ya; zr = za; sqr = sca; pq = pc; pr = pa; }
            const double wP = fmax(-sqr, 0.0), wQ = fmax(pr, 0.0), wR = fmax(-pq, 0.0);
            const double sw = wP + wQ + wR;
            double zout;
            if (sw > 0.0) {
                // offset from the apex; 1/sw from the fp32 reciprocal refined by
                // one fp64 Newton step (rel. error ~2^-46)
                double rin = (double)__frcp_rn((float)sw);
                rin = rin * fma(-sw, rin, 2.0);
                zout = fma(fma(wQ, zq - z3, wR * (zr - z3)), rin, z3);
            } else {
                zout = zin;
                ++n_exact;
            }
            const double chord = fmax(zout - zin, 0.0) * g;
            if (BACK) {
                if (chord > 0.0) atomicAdd(acc + t, chord * (double)yv);
            } else {
                sum = fma(chord, (double)mut, sum);
            }
            ++n_cross;
            // neighbour across the exit face = the face opposite O
            const int lo = nodes.x == io ? 0 : nodes.y == io ? 1 : nodes.z == io ? 2 : 3;
            const int tag = sel4(tags, lo);
            if (tag < 0) break;
            if (++steps >= max_steps) { ++n_stuck; break; }
            t = tag >> 2;
            kin = tag & 3;
            nodes = ldg_nc_v4(rec + 2 * (size_t)t);
            ia = iap; ib = iq; ic = ir;
            xa = x3; ya = y3; za = z3;
            xb = xq; yb = yq; zb = zq;
            xc = xr; yc = yr; zc = zr;
            sab = pq; sbc = sqr; sca = -pr;
            zin = zout;
        }
    }
    if (!BACK && valid) proj[rid] = (float)sum;
    add_stat(stats, ST_RAYS, valid ? 1u : 0u);
    add_stat(stats, ST_HIT, e >= 0 ? 1u : 0u);
    add_stat(stats, ST_CROSS, n_cross);
    add_stat(stats, ST_EXACT, n_exact);
    add_stat(stats, ST_LOST, n_lost);
    add_stat(stats, ST_STUCK, n_stuck);
    const unsigned mx = __reduce_max_sync(0xffffffffu, n_cross);
    if (lane == 0 && mx) atomicMax(stats + ST_MAXC, (unsigned long long)mx);
}

// ------------------------------------------------------------ permute ---
__global__ void gather_mu_kernel(const int* __restrict__ perm, const float* __restrict__ mu,
                                 float* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = __ldg(mu + perm[i]);
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
cudaError_t launch_entry(const DevMesh& m, const LaunchChunk& c, int* entry,
                         unsigned long long* stats, cudaStream_t s) {
    dim3 grid((unsigned)m.nb, (unsigned)c.n_angles);
    entry_kernel<<<grid, 256, 0, s>>>(m.rec, m.vtx, m.hull, c.ang, c.aux, c.beam, c.nv, c.nu,
                                      entry, stats);
    return cudaGetLastError();
}

static dim3 trace_grid(const LaunchChunk& c) {
    const unsigned tiles = (unsigned)(((c.nu + 15) / 16) * ((c.nv + 7) / 8));
    return dim3(tiles, (unsigned)c.n_angles);
}

cudaError_t launch_forward(const DevMesh& m, const LaunchChunk& c, const int* entry,
                           const float* mu_int, float* proj, unsigned long long* stats,
                           cudaStream_t s) {
    trace_kernel<false><<<trace_grid(c), 128, 0, s>>>(m.rec, m.vtx, c.ang, c.beam, c.nv, c.nu,
                                                      m.rmax, m.g, (long long)m.nt, entry,
                                                      mu_int, proj, nullptr, nullptr, stats);
    return cudaGetLastError();
}

cudaError_t launch_backward(const DevMesh& m, const LaunchChunk& c, const int* entry,
                            const float* y, double* acc, unsigned long long* stats,
                            cudaStream_t s) {
    trace_kernel<true><<<trace_grid(c), 128, 0, s>>>(m.rec, m.vtx, c.ang, c.beam, c.nv, c.nu,
                                                     m.rmax, m.g, (long long)m.nt, entry,
                                                     nullptr, nullptr, y, acc, stats);
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
