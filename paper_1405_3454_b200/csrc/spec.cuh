// spec.cuh — the speculative pre-filter region of Step 3,
// __host__ __device__ code shared by the seed kernel (which builds the
// region), K1 (which tests points against it), the verification (Step 2) and
// the host-side test hooks.
//
// PAPER.md §2 Step 3 discards the points strictly inside the
// polygon P of the Step-1 extremes.  P is only known after the whole Step-1
// pass, so the paper (and round 1 of this build) reads every point a second
// time.  Here K1 already sets aside every point that is NOT certainly inside a
// region D built from a small sample before K1 starts; once P is known, D is
// checked to lie strictly inside P, rigorously.  If it does, the points K1 set
// aside ("candidates") are the only ones Step 3 has to classify: every other
// point is strictly inside D, hence strictly inside P, hence discarded — the
// survivors are exactly the paper's.  If the check fails, Step 3 streams every
// point as before.  The output never depends on D.
//
// D is the disk |p - c|^2 < r2min around a float centre c, tested as the K2
// inner disk is: (dx, dy) = RN32(p - c), d2 = RN32(RN32(dx^2) + RN32(dy^2))
// < r2min, so |p - c|^2 < r2min (1 + 2^-20) (d2 >= |p - c|^2 (1 - 4u), u =
// 2^-24, r2min >= 2^-90: no underflow) -- or the closed axis-aligned box
// [bx0, bx1] x [by0, by1], whichever covers more of the seed's polygon.  The
// disk is strictly inside P iff c is and every edge line of P is farther than
// sqrt(r2min (1 + 2^-20)) from c (binary64 with error bounds); the closed box
// iff its four float corners are (exact predicate, P convex).
#pragma once

#include <cmath>

#include "exact.cuh"

namespace cudapre {
namespace spec {

#if defined(__CUDACC__)
#define SPEC_HD __host__ __device__ __forceinline__
#else
#define SPEC_HD inline
#endif

constexpr double kGuard = 1.0 / 64.0;   // bucket guard (same as the K2 sector tables, geom.cuh)
// the seed ring is shrunk towards its centre by 0.8 m^(-1/3) for m sample
// points (clamped to [0.4 %, 3 %]): 0.8 % for the 10^6-point sample of 2e9
// points, 1.5 % for 1.6e5 (10^7 points)
SPEC_HD double shrink(double m) {
    const double e = 0.8 / cbrt(m > 1.0 ? m : 1.0);
    return e < 0.004 ? 0.004 : (e > 0.03 ? 0.03 : e);
}
constexpr float kR2Lo = 0x1p-90f;       // usable radii: r2 in [2^-90, 2^120]
constexpr float kR2Hi = 0x1p+120f;

// ---- heuristics (the seed kernel's region; plain binary64, no rigour needed)
// squared distance from (cx, cy) to the nearest edge line of the CCW ring
// (qx, qy)[0..m) (c inside), times (1 - 2^-10), rounded down; -1 if unusable
SPEC_HD float ring_r2(const double* qx, const double* qy, int m, double cx, double cy) {
    double best = INFINITY;
    for (int j = 0; j < m; ++j) {
        const int k = j + 1 == m ? 0 : j + 1;
        const double ex = qx[k] - qx[j], ey = qy[k] - qy[j];
        const double num = ex * (cy - qy[j]) - ey * (cx - qx[j]);   // > 0 inside
        const double d2 = num * num / (ex * ex + ey * ey);
        if (!(num > 0.0)) return -1.0f;
        if (d2 < best) best = d2;
    }
    const double r2 = best * (1.0 - 0x1p-10);
    if (!(r2 >= (double)kR2Lo) || !(r2 <= (double)kR2Hi)) return -1.0f;
    float f = (float)r2;
    if ((double)f > r2) f = nextafterf(f, 0.0f);
    return f;
}
SPEC_HD bool ring_contains(const double* qx, const double* qy, int m, double px, double py) {
    for (int j = 0; j < m; ++j) {
        const int k = j + 1 == m ? 0 : j + 1;
        if ((qx[k] - qx[j]) * (py - qy[j]) - (qy[k] - qy[j]) * (px - qx[j]) <= 0.0) return false;
    }
    return true;
}

// ---- the verification (rigorous)
// The disk |p - c|^2 < r2 (1 + 2^-20) lies strictly inside the CCW ring
// v[0..nv] (v[nv] = v[0], strictly convex, c strictly inside): for every edge
// a -> b, num = orient(a, b, c) and len2 = |b - a|^2 in binary64 (no FMA; the
// x* helpers) with |err(num)| <= 2^-50 (|t1| + |t2|) (Shewchuk's bound for
// binary64 inputs, 3u + 16u^2) and len2 within a factor (1 +- 2^-50); the
// distance num / sqrt(len2) exceeds the radius iff (num - err)^2 > r2 (1 +
// 2^-20) len2 (1 + 2^-49) (1 + 2^-48) with num - err > 0, each side evaluated
// with a relative slack far above its own rounding.
SPEC_HD bool disk_inside(const float* vx, const float* vy, int nv, float cx, float cy, float r2) {
    if (!(r2 > 0.0f)) return true;
    const double R2 = xmul((double)r2, 1.0 + 0x1p-20);
    for (int j = 0; j < nv; ++j) {
        const double ex = xsub((double)vx[j + 1], (double)vx[j]), ey = xsub((double)vy[j + 1], (double)vy[j]);
        const double t1 = xmul(ex, xsub((double)cy, (double)vy[j]));
        const double t2 = xmul(ey, xsub((double)cx, (double)vx[j]));
        const double err = xmul(xadd(xabs(t1), xabs(t2)), 0x1p-50);
        const double lo = xsub(xsub(t1, t2), err);
        if (!(lo > 0.0)) return false;
        const double len2 = xadd(xmul(ex, ex), xmul(ey, ey));
        const double lhs = xmul(xmul(lo, lo), 1.0 - 0x1p-48);
        const double rhs = xmul(xmul(R2, len2), 1.0 + 0x1p-46);
        if (!(lhs > rhs)) return false;
    }
    return true;
}

// K1 / K2 bucket of a point relative to the centre (the K2 sector arithmetic,
// DESIGN.md §6.2): d2 = RN32(RN32(dx^2)+RN32(dy^2)) and b = round(256 pa)
// from one approximate reciprocal, clamped to [0, CUDAPRE_SECTORS].
#if defined(__CUDACC__)
__device__ __forceinline__ float rcp_approx_f(float a) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    return r;
}
__device__ __forceinline__ unsigned sector_bucket(float dx, float dy) {
    const float t = __fmul_rn(dy, rcp_approx_f(__fadd_rn(fabsf(dx), fabsf(dy))));
    const bool pos = dx >= 0.0f;
    const float v = __fmaf_rn(t, pos ? 256.0f : -256.0f, pos ? 8388864.0f : 8389376.0f);   // 2^23 + 256 pa
    return min(__float_as_uint(v) - 0x4B000000u, (unsigned)CUDAPRE_SECTORS);
}
#endif

}  // namespace spec
}  // namespace cudapre
