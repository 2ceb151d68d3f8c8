// pair.cuh -- per-pair geometry on the device.
//
// For voxel r = (0, y, z) and pixel r' = (x_d, y_d, det_z), s = r' - r:
//   G_od   = s_z / |s|^3
//   theta  : sin(theta) = |r x s| / (|r||s|),  cos(theta) = r^.s^
//            sin(theta/2) = sin(theta) / (2 cos(theta/2)),
//            cos(theta/2) = sqrt((1 + cos theta)/2)  -- half-angle forms, no
//            cancellation at small theta (K2 "angle conditioning")
//   dtheta = atan(p |x^ x s| / (|s|^2 - p^2/4))           PAPER.md:609 (closed form
//            of the angle between s +- (p/2) x^, reading R6)
//   T      = mask bit at the ray's crossing of z = mask_z  PAPER.md:648, reading R8
//   P      = G_so G_od dtheta (1 + cos^2 theta) cos(theta/2)   (C_E folded into c_k)
#pragma once
#include "internal.h"

namespace cacsi {

__device__ __forceinline__ float fast_sqrt(float x) { return x * rsqrtf(fmaxf(x, 1e-30f)); }

// T(r, r') in {0, 1} by the exact fp64 rule of reading R8: same op order as
// the definition, no FMA contraction (__d*_rn intrinsics), on the fp64 centre
// tables.  Bit-identical to the definition.
__device__ __forceinline__ bool mask_exact(const Params &p, int v, int q) {
    const double t = p.vt64[v], yr = p.vy64[v];
    const double xd = p.dx64[q], yd = p.dy64[q];
    const double px = __dmul_rn(t, xd);
    const double py = __dadd_rn(yr, __dmul_rn(t, __dsub_rn(yd, yr)));
    const double gx = floor(__ddiv_rn(__dsub_rn(px, p.m0x), p.mask_pitch64));
    const double gy = floor(__ddiv_rn(__dsub_rn(py, p.m0y), p.mask_pitch64));
    if (!(gx >= 0.0 && gy >= 0.0 && gx < (double)p.mask_nx && gy < (double)p.mask_ny)) return false;
    const int ix = (int)gx, iy = (int)gy;
    const uint32_t w = __ldg(p.maskbits + (size_t)ix * p.mask_words + (iy >> 5));
    return (w >> (iy & 31)) & 1u;
}

// fp32 fast path of T: u = (t/p) x + const per axis, cell = floor(u).  *near is
// set when u lies within p.mask_guard cells of a cell edge (4x the fp32 error bound
// of u derived at create from the geometry's extents, at least kMaskGuard; DESIGN.md
// 4.1); the result is then undefined and the caller must use mask_exact.  Kept branch-free so batched callers stay
// converged; the exact re-tests run in a separate pass.
__device__ __forceinline__ bool mask_fast(const Params &p, const VoxelRec &vr, float2 d, bool &near) {
    const float ux = fmaf(vr.tq, d.x, p.ax);
    const float uy = fmaf(vr.tq, d.y, vr.ay);
    const float fx = floorf(ux), fy = floorf(uy);
    near = fabsf(ux - fx - 0.5f) > 0.5f - p.mask_guard || fabsf(uy - fy - 0.5f) > 0.5f - p.mask_guard;
    const int ix = (int)fx, iy = (int)fy;
    if ((unsigned)ix >= (unsigned)p.mask_nx || (unsigned)iy >= (unsigned)p.mask_ny) return false;
    const uint32_t w = __ldg(p.maskbits + (size_t)ix * p.mask_words + (iy >> 5));
    return (w >> (iy & 31)) & 1u;
}

__device__ __forceinline__ bool mask_open(const Params &p, int v, int q, const VoxelRec &vr, float2 d) {
    bool near;
    const bool o = mask_fast(p, vr, d, near);
    return near ? mask_exact(p, v, q) : o;
}

// P (without C_E) and sin(theta/2) of one pair.  angular = false (scatter-angle
// interpolation): P = G_so G_od dtheta only -- the spectral-angular factor
// (1 + cos^2 theta) cos(theta/2) then lives in the tabulated rows.
__device__ __forceinline__ void pair_geom(const Params &p, const VoxelRec &vr, float2 d, float &P, float &sh,
                                          bool angular = true) {
    const float sx = d.x, sy = d.y - vr.y, sz = vr.sz;
    const float syz2 = fmaf(sy, sy, sz * sz);
    const float s2 = fmaf(sx, sx, syz2);
    const float rs = rsqrtf(s2);
    const float rs2 = rs * rs;
    const float god = sz * rs * rs2;                         // G_od
    const float e1 = fmaf(vr.ry, p.det_z, -vr.rz * d.y);     // (r x s)_x / |r|
    const float sin_t = fast_sqrt(fmaf(e1, e1, sx * sx)) * rs;
    const float cos_t = fmaf(vr.ry, sy, vr.rz * sz) * rs;
    const float h = fmaf(0.5f, cos_t, 0.5f);                 // cos^2(theta/2)
    const float rh = rsqrtf(h);
    const float ch = h * rh;
    sh = 0.5f * sin_t * rh;
    // dtheta = atan(x), x = p sqrt(sy^2+sz^2) / (|s|^2 - p^2/4); x <= kAtanXMax (checked
    // at create) so atan(x) = x (1 - x^2/3) to x^4/5 < 1e-8 and 1/(s2 - p^2/4) = rs2 (1 + p^2/4 rs2)
    const float x = p.pitch_d * fast_sqrt(syz2) * rs2 * fmaf(p.quarter_p2, rs2, 1.0f);
    const float dth = x * fmaf(-0.33333334f * x, x, 1.0f);
    P = angular ? vr.gso * god * dth * fmaf(cos_t, cos_t, 1.0f) * ch : vr.gso * god * dth;
}

// Scatter angle of a pair in fp64 from the fp64 centre tables, the plain
// definition atan2(|r x s|, r . s) (the oracle's formula), for
// decisions that must not depend on fp32 rounding (SAI cell boundaries).
__device__ __forceinline__ double theta64(const Params &p, int v, int q) {
    const double y = p.vy64[v], z = p.vz64[v];
    const double sx = p.dx64[q], sy = __dsub_rn(p.dy64[q], y), sz = __dsub_rn(p.det_z64, z);
    const double c0 = __dsub_rn(__dmul_rn(y, sz), __dmul_rn(z, sy));
    const double c1 = __dmul_rn(z, sx), c2 = -__dmul_rn(y, sx);
    const double cr = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(c0, c0), __dmul_rn(c1, c1)), __dmul_rn(c2, c2)));
    return atan2(cr, __dadd_rn(__dmul_rn(y, sy), __dmul_rn(z, sz)));
}

// Energies whose u_k = alpha_k sh - q_min/dq can fall inside (-1, nq): a
// superset [klo, khi] (the clamp in the term loop zeroes the extras).
__device__ __forceinline__ void k_range(const Params &p, float sh, int &klo, int &khi) {
    if (p.uniform_e) {
        const float inv = __frcp_rn(sh);
        const float lo = fminf((fmaf(p.klo_num, inv, -p.a0)) * p.inv_da, 1e8f);
        const float hi = fminf((fmaf(p.khi_num, inv, -p.a0)) * p.inv_da, 1e8f);
        klo = max(0, (int)floorf(lo));
        khi = min(p.ne - 1, (int)ceilf(hi));
    } else {
        klo = 0;
        khi = p.ne - 1;
    }
}

// Hat-basis lookup coordinates of u' = u - 1/2 clamped to [-3/2, nq - 1/2]:
// n = round(u') in [-2, nq], tt = u' - n in [-1/2, 1/2].  Rounding by the
// 1.5*2^23 trick (no F2I); ties are harmless because the interpolant is
// continuous (either neighbour gives the same value).
__device__ __forceinline__ int hat_coord(const Params &p, float alpha, float sh, float &tt) {
    float u = fmaf(alpha, sh, p.nb);
    u = fminf(fmaxf(u, -1.5f), p.qm);
    const float vm = u + kMagic;
    tt = u - (vm - kMagic);
    return __float_as_int(vm) - kMagicBits;
}

}  // namespace cacsi
