// exact.cuh — exact orientation sign for float inputs, usable on host and device.
//
// orient(a, b, c) = (bx-ax)(cy-ay) - (by-ay)(cx-ax)
//                 = bx*cy - bx*ay - ax*cy - by*cx + by*ax + ay*cx      (ax*ay cancels)
// (reading A11: the sign must be exact).  Each of the six terms is
// a product of two floats, which is exact in binary64 (<= 48-bit significand,
// exponent in [-298, 256]: no overflow, no underflow).  Their sum is first
// evaluated naively with a forward error bound; only if the bound cannot
// decide the sign is the exact sum formed as a non-overlapping floating-point
// expansion (Knuth TwoSum, grow-expansion), whose most significant non-zero
// component carries the exact sign.  TwoSum is exact under round-to-nearest
// without overflow, and the sum of six terms < 2^259 cannot overflow.
//
// No fused multiply-add may be formed here: device code uses the explicit
// __dmul_rn/__dadd_rn intrinsics, host code is compiled with
// -ffp-contract=off (see build.py).
#pragma once

#if defined(__CUDACC__)
#define CUDAPRE_HD __host__ __device__ __forceinline__
#else
#define CUDAPRE_HD inline
#endif

namespace cudapre {

CUDAPRE_HD double xmul(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
CUDAPRE_HD double xadd(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
CUDAPRE_HD double xsub(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}
CUDAPRE_HD double xabs(double a) { return a < 0 ? -a : a; }

// s + err == a + b exactly (Knuth TwoSum, 6 flops, any magnitudes).
CUDAPRE_HD void two_sum(double a, double b, double& s, double& err) {
    s = xadd(a, b);
    double bb = xsub(s, a);
    double aa = xsub(s, bb);
    err = xadd(xsub(a, aa), xsub(b, bb));
}

CUDAPRE_HD int orient_sign_f(float ax, float ay, float bx, float by, float cx, float cy) {
    const double t[6] = {
        xmul((double)bx, (double)cy), -xmul((double)bx, (double)ay),
        -xmul((double)ax, (double)cy), -xmul((double)by, (double)cx),
        xmul((double)by, (double)ax), xmul((double)ay, (double)cx)};
    // naive sum with a forward error bound: |fl(sum) - sum| <= 5 u sum|t_i| (1+5u),
    // u = 2^-53; 2^-49 covers it with margin.
    double s = t[0], mag = xabs(t[0]);
    for (int i = 1; i < 6; ++i) {
        s = xadd(s, t[i]);
        mag = xadd(mag, xabs(t[i]));
    }
    const double bound = xmul(mag, 0x1p-49);
    if (s > bound) return 1;
    if (s < -bound) return -1;
    // exact: grow a non-overlapping expansion e[0..ne) (increasing magnitude)
    double e[6];
    int ne = 0;
    for (int i = 0; i < 6; ++i) {
        double q = t[i];
        for (int j = 0; j < ne; ++j) {
            double h;
            two_sum(q, e[j], q, h);
            e[j] = h;
        }
        e[ne++] = q;
    }
    for (int j = ne - 1; j >= 0; --j) {
        if (e[j] > 0) return 1;
        if (e[j] < 0) return -1;
    }
    return 0;
}

// The same exact sign, with a float32 filter in front (Shewchuk's orient2d
// stage A in single precision): det = (ax-cx)(by-cy) - (ay-cy)(bx-cx) has
// |fl(det) - det| <= (3e + 16e^2)(|dl| + |dr|) for e = 2^-24 without
// underflow; subnormal differences are exact and a subnormal product is off by
// <= 2^-150, which the 2^-140 term covers; any overflow fails the finiteness
// test.  Used where one thread runs many predicates in a row (the Step-2
// builders): the result is the exact sign either way.
CUDAPRE_HD float xfsub(float a, float b) {
#if defined(__CUDA_ARCH__)
    return __fsub_rn(a, b);
#else
    return a - b;
#endif
}
CUDAPRE_HD float xfmul(float a, float b) {
#if defined(__CUDA_ARCH__)
    return __fmul_rn(a, b);
#else
    return a * b;
#endif
}
CUDAPRE_HD float xfadd(float a, float b) {
#if defined(__CUDA_ARCH__)
    return __fadd_rn(a, b);
#else
    return a + b;
#endif
}
CUDAPRE_HD int orient_sign_filtered(float ax, float ay, float bx, float by, float cx, float cy) {
    const float dl = xfmul(xfsub(ax, cx), xfsub(by, cy));
    const float dr = xfmul(xfsub(ay, cy), xfsub(bx, cx));
    const float det = xfsub(dl, dr);
    const float sum = xfadd(dl < 0 ? -dl : dl, dr < 0 ? -dr : dr);
    const float bound = xfadd(xfmul(0x1p-22f, sum), 0x1p-140f);   // 4e > 3e + 16e^2 + the bound's own roundings
    if (bound < 0x1p+127f) {   // finite (NaN / inf fail the comparison)
        if (det > bound) return 1;
        if (det < -bound) return -1;
    }
    return orient_sign_f(ax, ay, bx, by, cx, cy);
}

}  // namespace cudapre
