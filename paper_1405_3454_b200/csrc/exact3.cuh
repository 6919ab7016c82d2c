// exact3.cuh — exact orient3d sign for float inputs, host and device
// (the 3D extension; DESIGN.md §3 reading B6, §6.5).
//
// orient3d(a, b, c, d) = det[b-a; c-a; d-a] (rows) = ((b-a) x (c-a)) . (d-a):
// positive when d lies on the side the right-handed normal of (a, b, c)
// points to.
//
// Stage 1 (Shewchuk's orient3d stage A, in binary64): the differences are
// rounded, then the 3x3 determinant is evaluated naively; its error is at
// most (7u + 56u^2) * permanent, u = 2^-53, where the permanent is the same
// expression with every term replaced by its absolute value.  The bound
// assumes neither overflow nor underflow: float inputs give differences in
// (2^-149 multiples, < 2^129), products of three >= 2^-447 or 0 and < 2^387,
// all inside binary64's normal range.  2^-49 * permanent covers the bound and
// the rounding of the permanent itself.
// Stage 2 (exact): by multilinearity det(b-a, c-a, d-a) = det(b,c,d) -
// det(a,c,d) - det(b,a,d) - det(b,c,a), 24 signed products x*y*z of input
// floats.  x*y is exact in binary64 (48 significant bits); (x*y)*z = hi + lo
// exactly with hi = RN(x*y*z) and lo = fma(x*y, z, -hi) (TwoProduct; lo is
// representable because the product has <= 72 significant bits and no
// underflow).  The 48 components are summed into a non-overlapping expansion
// (Knuth TwoSum, grow-expansion, zero elimination); the most significant
// nonzero component carries the exact sign.
//
// No fused multiply-add may be formed except the explicit TwoProduct fma:
// device code uses __d*_rn intrinsics, host code is compiled with
// -ffp-contract=off (build.py).
#pragma once

#include <cmath>

#include "exact.cuh"

namespace cudapre {

CUDAPRE_HD double xfma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
    return __fma_rn(a, b, c);
#else
    return std::fma(a, b, c);
#endif
}

// Stage 2, out of line on the device (rare path).
#if defined(__CUDACC__)
__host__ __device__ __noinline__
#else
inline
#endif
int orient3d_exact(const float* a, const float* b, const float* c, const float* d) {
    // rows of the four 3x3 determinants and their signs
    const float* R[4][3] = {{b, c, d}, {a, c, d}, {b, a, d}, {b, c, a}};
    const double sg[4] = {1.0, -1.0, -1.0, -1.0};
    // the six permutations of (0,1,2) with their parity
    const int P[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    const double ps[6] = {1.0, -1.0, -1.0, 1.0, 1.0, -1.0};
    double e[48];
    int ne = 0;
    for (int t = 0; t < 4; ++t)
        for (int q = 0; q < 6; ++q) {
            const double xy = xmul((double)R[t][0][P[q][0]], (double)R[t][1][P[q][1]]);   // exact
            const double z = (double)R[t][2][P[q][2]];
            const double hi = xmul(xy, z);
            const double lo = xfma(xy, z, -hi);
            const double s = xmul(sg[t], ps[q]);
            const double comp[2] = {xmul(s, lo), xmul(s, hi)};   // s = +-1: exact
            for (int h = 0; h < 2; ++h) {
                double qv = comp[h];
                if (qv == 0.0) continue;
                int w = 0;
                for (int j = 0; j < ne; ++j) {   // grow-expansion with zero elimination
                    double err;
                    two_sum(qv, e[j], qv, err);
                    if (err != 0.0) e[w++] = err;
                }
                if (qv != 0.0) e[w++] = qv;
                ne = w;
            }
        }
    for (int j = ne - 1; j >= 0; --j) {
        if (e[j] > 0) return 1;
        if (e[j] < 0) return -1;
    }
    return 0;
}

CUDAPRE_HD int orient3d_sign_f(const float* a, const float* b, const float* c, const float* d) {
    const double ux = xsub(b[0], a[0]), uy = xsub(b[1], a[1]), uz = xsub(b[2], a[2]);
    const double vx = xsub(c[0], a[0]), vy = xsub(c[1], a[1]), vz = xsub(c[2], a[2]);
    const double wx = xsub(d[0], a[0]), wy = xsub(d[1], a[1]), wz = xsub(d[2], a[2]);
    const double uyvz = xmul(uy, vz), uzvy = xmul(uz, vy);
    const double uzvx = xmul(uz, vx), uxvz = xmul(ux, vz);
    const double uxvy = xmul(ux, vy), uyvx = xmul(uy, vx);
    const double det = xadd(xadd(xmul(wx, xsub(uyvz, uzvy)), xmul(wy, xsub(uzvx, uxvz))),
                            xmul(wz, xsub(uxvy, uyvx)));
    const double perm = xadd(xadd(xmul(xabs(wx), xadd(xabs(uyvz), xabs(uzvy))),
                                  xmul(xabs(wy), xadd(xabs(uzvx), xabs(uxvz)))),
                             xmul(xabs(wz), xadd(xabs(uxvy), xabs(uyvx))));
    const double bound = xmul(perm, 0x1p-49);
    if (det > bound) return 1;
    if (det < -bound) return -1;
    return orient3d_exact(a, b, c, d);
}

}  // namespace cudapre
