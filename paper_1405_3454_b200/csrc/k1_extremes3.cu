// k1_extremes3.cu — Step 1 of the 3D extension (PAPER.md P:115 with
// P:33-35; DESIGN.md §3 B1-B2, §6.5) as ONE streaming pass over HBM.
//
// Slot 6k+{minX, maxX, minY, maxY, minZ, maxZ} of the frame rotated by angle
// k about z: X_k = RN(RN(x c_k) + RN(y s_k)), Y_k = RN(RN(y c_k) - RN(x s_k))
// in binary64 without FMA, Z = z; lowest index on ties.  Distinct keys: the
// 4 angle-0 keys (x, y themselves: RN(x*1 + y*0) = x), the 2 z keys, and 4
// per further angle.
//
// Per point (12 bytes, read once as part of a 48-byte quad):
//   * angle-0 and z keys: exact float compares, strict improvement (a lane
//     visits its points in ascending index order);
//   * every key is screened against the warp's threshold T (a float on the
//     safe side of the exact key of a point already reduced: redux.sync over
//     the lanes' exact states, refreshed whenever a lane took the exact path);
//     axis keys exactly (x, y, z are the keys), rotated keys with the 2D
//     kernel's margin (k1_extremes.cu header: |Xf - X_k| <
//     m = RN32(fma(|x|+|y|, 2^-20, 2^-120))), here the quad's largest m
//     folded into the thresholds once per quad.  Ties are never pruned,
//     NaN / Inf are always candidates (the exact path flags them).
// Lane states -> warp (shuffles) -> block partial -> last-block finalize
// (ticket) that expands the 4*nang+2 distinct keys into the 6*nang slots.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "internal3.h"

#ifndef K13_AHEAD
#define K13_AHEAD 4   // L2 prefetch distance, in warp steps (2: +0.8 %, 8: +20 % time; r02_experiments.md)
#endif

namespace cudapre {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned kNone = 0xffffffffu;

__device__ __forceinline__ unsigned enc_f(float f) {
    const unsigned b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float dec_f(unsigned e) {
    return __uint_as_float((e & 0x80000000u) ? (e & 0x7fffffffu) : ~e);
}

// (k, i) strictly better than (K, I) for the slot direction; lowest index on ties
__device__ __forceinline__ bool lex_better(double k, unsigned i, double K, unsigned I, bool mx) {
    return mx ? (k > K || (k == K && i < I)) : (k < K || (k == K && i < I));
}

// L2 prefetch of [p, p + bytes) (cp.async.bulk.prefetch; 16-B aligned, bytes % 16 == 0)
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

struct Quad {
    float v[12];   // x0 y0 z0 x1 y1 z1 ...
};

template <bool VEC>
__device__ __forceinline__ void load_quad(const float* __restrict__ pts, unsigned q, unsigned n, Quad& Q,
                                          unsigned& valid) {
    const unsigned i0 = 4u * q;
    valid = i0 >= n ? 0u : (n - i0 >= 4u ? 4u : n - i0);
    if (VEC && valid == 4u) {
        const float4* s = reinterpret_cast<const float4*>(pts) + 3u * q;
        const float4 a = __ldg(s), b = __ldg(s + 1), c = __ldg(s + 2);
        Q.v[0] = a.x, Q.v[1] = a.y, Q.v[2] = a.z, Q.v[3] = a.w;
        Q.v[4] = b.x, Q.v[5] = b.y, Q.v[6] = b.z, Q.v[7] = b.w;
        Q.v[8] = c.x, Q.v[9] = c.y, Q.v[10] = c.z, Q.v[11] = c.w;
    } else {
#pragma unroll
        for (int j = 0; j < 12; ++j) Q.v[j] = (unsigned)(j / 3) < valid ? __ldg(pts + 3ull * i0 + j) : 0.0f;
        if (valid > 0u)   // pad the tail with copies of the quad's first point (no effect on any key)
#pragma unroll
            for (int j = 3; j < 12; ++j)
                if ((unsigned)(j / 3) >= valid) Q.v[j] = Q.v[j % 3];
    }
}

template <int NANG>
struct Lane {
    static constexpr int R = 4 * (NANG - 1);
    static constexpr int RR = R > 0 ? R : 1;
    static constexpr int D = 6 + R;   // distinct keys: x, x, y, y, z, z, then 4 per further angle
    float ak[6];        // exact float keys of the axis slots (min x, max x, min y, max y, min z, max z)
    unsigned ai[6];
    double rk[RR];      // exact binary64 keys of the rotated slots
    unsigned ri[RR];
    float T[D];         // warp thresholds (float, on the safe side of a reduced point's exact key)
};

template <int NANG>
__device__ __forceinline__ void lane_init(Lane<NANG>& L) {
#pragma unroll
    for (int s = 0; s < 6; ++s) {
        L.ak[s] = (s & 1) ? -INFINITY : INFINITY;
        L.ai[s] = kNone;
    }
#pragma unroll
    for (int s = 0; s < Lane<NANG>::RR; ++s) {
        L.rk[s] = (s & 1) ? -INFINITY : INFINITY;
        L.ri[s] = kNone;
    }
#pragma unroll
    for (int s = 0; s < Lane<NANG>::D; ++s) L.T[s] = (s & 1) ? -INFINITY : INFINITY;
}

// exact update of every key of one point (cold path; a lane's points arrive in
// ascending index order, so strict improvement keeps the lowest index)
template <int NANG>
__device__ __forceinline__ void exact_point(Lane<NANG>& L, float x, float y, float z, unsigned i,
                                            const K13Params& p, unsigned& bad) {
    if (!(fabsf(x) <= FLT_MAX && fabsf(y) <= FLT_MAX && fabsf(z) <= FLT_MAX)) {
        bad = 1u;
        return;
    }
    const float av[6] = {x, x, y, y, z, z};
#pragma unroll
    for (int s = 0; s < 6; ++s)
        if ((s & 1) ? av[s] > L.ak[s] : av[s] < L.ak[s]) L.ak[s] = av[s], L.ai[s] = i;
    const double xd = x, yd = y;
#pragma unroll
    for (int k = 1; k < NANG; ++k) {
        const double X = __dadd_rn(__dmul_rn(xd, p.c[k]), __dmul_rn(yd, p.s[k]));
        const double Y = __dsub_rn(__dmul_rn(yd, p.c[k]), __dmul_rn(xd, p.s[k]));
        const double kv[4] = {X, X, Y, Y};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int s = 4 * (k - 1) + r;
            if ((r & 1) ? kv[r] > L.rk[s] : kv[r] < L.rk[s]) L.rk[s] = kv[r], L.ri[s] = i;
        }
    }
}

// warp thresholds from the lanes' exact states: max slots take the largest
// float <= some lane's key, min slots the smallest float >= some lane's key
template <int NANG>
__device__ __forceinline__ void refresh(Lane<NANG>& L) {
#pragma unroll
    for (int s = 0; s < 6; ++s)
        L.T[s] = dec_f((s & 1) ? __reduce_max_sync(kFull, enc_f(L.ak[s])) : __reduce_min_sync(kFull, enc_f(L.ak[s])));
#pragma unroll
    for (int s = 0; s < Lane<NANG>::R; ++s) {
        if (s & 1) {
            L.T[6 + s] = dec_f(__reduce_max_sync(kFull, enc_f(__double2float_rd(L.rk[s]))));
        } else {
            L.T[6 + s] = dec_f(__reduce_min_sync(kFull, enc_f(__double2float_ru(L.rk[s]))));
        }
    }
}

// One quad: screen all four points — the axis keys exactly in float, the
// rotated keys against thresholds widened by the quad's largest margin
// mq = max_e RN32(fma(|x_e|+|y_e|, 2^-20, 2^-120)) >= each point's m (a point
// whose exact key ties or beats T has Xf < T + m <= T + mq, so Xf <= RN(T +
// mq): never pruned).  A candidate sends the whole quad through the exact
// path.  Unordered compares make NaN / Inf candidates, which the exact path
// flags.
template <int NANG>
__device__ __forceinline__ void fold_quad(Lane<NANG>& L, const Quad& Q, unsigned valid, unsigned i0,
                                          const K13Params& p, unsigned& bad, unsigned& nexact) {
    bool c = false;
    float am = 0.0f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float x = Q.v[3 * e], y = Q.v[3 * e + 1], z = Q.v[3 * e + 2];
        c |= !(x > L.T[0]) | !(x < L.T[1]) | !(y > L.T[2]) | !(y < L.T[3]) | !(z > L.T[4]) | !(z < L.T[5]);
        am = fmaxf(am, __fadd_rn(fabsf(x), fabsf(y)));
    }
    if (NANG > 1) {
        const float mq = __fmaf_rn(am, 0x1p-20f, 0x1p-120f);
#pragma unroll
        for (int k = 1; k < NANG; ++k) {
            const float* T = &L.T[6 + 4 * (k - 1)];
            const float t0 = __fadd_rn(T[0], mq), t1 = __fsub_rn(T[1], mq);
            const float t2 = __fadd_rn(T[2], mq), t3 = __fsub_rn(T[3], mq);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float x = Q.v[3 * e], y = Q.v[3 * e + 1];
                const float X = __fmaf_rn(x, p.cf[k], __fmul_rn(y, p.sf[k]));
                const float Y = __fmaf_rn(y, p.cf[k], __fmul_rn(x, p.nsf[k]));
                c |= !(X > t0) | !(X < t1) | !(Y > t2) | !(Y < t3);
            }
        }
    }
    c &= valid != 0u;
    if (__any_sync(kFull, c)) {
        if (c) {
#pragma unroll
            for (int e = 0; e < 4; ++e)   // static indices: the quad stays in registers
                if ((unsigned)e < valid)
                    exact_point<NANG>(L, Q.v[3 * e], Q.v[3 * e + 1], Q.v[3 * e + 2], i0 + e, p, bad);
            nexact += valid;
        }
        refresh<NANG>(L);
    }
}

template <int NANG, bool VEC>
__global__ void __launch_bounds__(kK13Threads, NANG >= 8 ? 1 : 2) k1_extremes3(const __grid_constant__ K13Params p) {
    constexpr int R = Lane<NANG>::R;
    constexpr int D = 6 + R;   // distinct keys
    __shared__ double s_key[kK13Threads / 32][D];
    __shared__ unsigned s_idx[kK13Threads / 32][D];
    __shared__ bool s_last;

    Lane<NANG> L;
    lane_init<NANG>(L);
    unsigned bad = 0, nexact = 0;
    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const unsigned nq = p.n / 4u + ((p.n & 3u) != 0u);   // ceil(n / 4) without wrapping near 2^32
    const unsigned gwarps = gridDim.x * (kK13Threads / 32);
    const unsigned gw = blockIdx.x * (kK13Threads / 32) + warp;
    // warp-uniform loop: each warp takes kK13Quads*32 consecutive quads per
    // step; lane 0 prefetches the warp's range kAhead steps ahead into L2
    // (16-B aligned input only), which doubles the bytes in flight at no
    // register cost
    constexpr unsigned kStep = 32u * kK13Quads;
    constexpr int kAhead = K13_AHEAD;
    const unsigned gstep = gwarps * kStep;
    if (VEC && lane == 0)
        for (int a = 1; a < kAhead; ++a) {
            const unsigned qa = gw * kStep + a * gstep;
            if (qa + kStep <= p.n / 4u) prefetch_l2(p.pts + 12ull * qa, 48u * kStep);
        }
    for (unsigned qb = gw * kStep; qb < nq; qb += gstep) {
        if (VEC && lane == 0) {
            const unsigned qa = qb + kAhead * gstep;
            if (qa < qb) {
                // wrapped past 2^32: beyond the end of the input (n < 2^32), nothing to prefetch
            } else if (qa + kStep <= p.n / 4u) {
                prefetch_l2(p.pts + 12ull * qa, 48u * kStep);
            }
        }
        Quad Q[kK13Quads];
        unsigned valid[kK13Quads];
#pragma unroll
        for (int u = 0; u < kK13Quads; ++u)
            load_quad<VEC>(p.pts, qb + u * 32u + lane, p.n, Q[u], valid[u]);
#pragma unroll
        for (int u = 0; u < kK13Quads; ++u)
            fold_quad<NANG>(L, Q[u], valid[u], 4u * (qb + u * 32u + lane), p, bad, nexact);
    }

    // lane -> warp (lexicographic), distinct key d: 0..5 axis, 6.. rotated
#pragma unroll
    for (int d = 0; d < D; ++d) {
        double k = d < 6 ? (double)L.ak[d < 6 ? d : 0] : L.rk[d >= 6 ? d - 6 : 0];
        unsigned i = d < 6 ? L.ai[d < 6 ? d : 0] : L.ri[d >= 6 ? d - 6 : 0];
        const bool mx = (d & 1) != 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double k2 = __shfl_xor_sync(kFull, k, o);
            const unsigned i2 = __shfl_xor_sync(kFull, i, o);
            if (i2 != kNone && (i == kNone || lex_better(k2, i2, k, i, mx))) k = k2, i = i2;
        }
        if (lane == 0) {
            s_key[warp][d] = k;
            s_idx[warp][d] = i;
        }
    }
    bad = __reduce_or_sync(kFull, bad);
    nexact = __reduce_add_sync(kFull, nexact);
    if (lane == 0) {
        if (bad) atomicOr(&p.ws->k1_nonfinite, 1u);
        if (nexact) atomicAdd(&p.ws->k1_exact, nexact);
    }
    __syncthreads();
    if (threadIdx.x < D) {   // warp -> block partial
        const int d = threadIdx.x;
        double k = s_key[0][d];
        unsigned i = s_idx[0][d];
        for (int w = 1; w < kK13Threads / 32; ++w)
            if (s_idx[w][d] != kNone && (i == kNone || lex_better(s_key[w][d], s_idx[w][d], k, i, d & 1)))
                k = s_key[w][d], i = s_idx[w][d];
        p.partials[(size_t)blockIdx.x * kMax3Slots + d] = K13Partial{k, i, 0u};
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&p.ws->k1_ticket, 1u) == gridDim.x - 1u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // last block: partials -> result (6*nang slots)
    cudapre3_extremes_t* out = &p.ws->result;
    if (threadIdx.x < D) {
        const int d = threadIdx.x;
        double k = 0.0;
        unsigned i = kNone;
        for (unsigned b = 0; b < gridDim.x; ++b) {
            const K13Partial* q = &p.partials[(size_t)b * kMax3Slots + d];
            const double qk = __ldcg(&q->key);
            const unsigned qi = __ldcg(&q->idx);
            if (qi != kNone && (i == kNone || lex_better(qk, qi, k, i, d & 1))) k = qk, i = qi;
        }
        s_idx[0][d] = i;
    }
    __syncthreads();
    if (threadIdx.x < 6 * p.nang) {
        const int slot = threadIdx.x, kk = slot / 6, r = slot % 6;
        const int d = r >= 4 ? r : (kk == 0 ? r : 6 + 4 * (kk - 1) + r);
        const unsigned i = s_idx[0][d];
        if (i == kNone) {
            out->idx[slot] = -1;
            out->key[slot] = 0.0;
            out->pt[slot] = cudapre_pt3{0.f, 0.f, 0.f};
        } else {
            const float x = p.pts[3ull * i], y = p.pts[3ull * i + 1], z = p.pts[3ull * i + 2];
            const double xd = x, yd = y;
            double key;
            if (r >= 4) {
                key = (double)z;
            } else if (r < 2) {
                key = __dadd_rn(__dmul_rn(xd, p.c[kk]), __dmul_rn(yd, p.s[kk]));
            } else {
                key = __dsub_rn(__dmul_rn(yd, p.c[kk]), __dmul_rn(xd, p.s[kk]));
            }
            out->idx[slot] = p.base + (long long)i;
            out->key[slot] = key;
            out->pt[slot] = cudapre_pt3{x, y, z};
        }
    }
    if (threadIdx.x == 0) {
        out->nang = p.nang;
        out->nonfinite = (int)atomicExch(&p.ws->k1_nonfinite, 0u);
        out->n = p.n;
        out->exact_points = atomicExch(&p.ws->k1_exact, 0u);
        p.ws->k1_ticket = 0u;
    }
    if (threadIdx.x < CUDAPRE_MAX_ANGLES) {
        out->c[threadIdx.x] = threadIdx.x < (unsigned)p.nang ? p.c[threadIdx.x] : 0.0;
        out->s[threadIdx.x] = threadIdx.x < (unsigned)p.nang ? p.s[threadIdx.x] : 0.0;
    }
}

template <int NANG>
int launch_n(const K13Params& p, void* stream) {
    const unsigned nq = p.n / 4u + ((p.n & 3u) != 0u);   // ceil(n / 4) without wrapping near 2^32
    const unsigned per_block = kK13Threads * kK13Quads;
    unsigned blocks = (nq + per_block - 1) / per_block;
    const unsigned cap = (unsigned)device_sm_count() * 2u;
    if (blocks > cap) blocks = cap;
    if (blocks > (unsigned)kMaxK13Blocks) blocks = kMaxK13Blocks;
    if (blocks == 0) blocks = 1;
    cudaStream_t s = (cudaStream_t)stream;
    if (p.vec)
        k1_extremes3<NANG, true><<<blocks, kK13Threads, 0, s>>>(p);
    else
        k1_extremes3<NANG, false><<<blocks, kK13Threads, 0, s>>>(p);
    return (int)cudaGetLastError();
}

}  // namespace

int launch_extremes3(const K13Params& p, void* stream, int* launches) {
    int rc;
    switch (p.nang) {
        case 1: rc = launch_n<1>(p, stream); break;
        case 2: rc = launch_n<2>(p, stream); break;
        case 3: rc = launch_n<3>(p, stream); break;
        case 4: rc = launch_n<4>(p, stream); break;
        case 8: rc = launch_n<8>(p, stream); break;
        default: return (int)cudaErrorInvalidValue;
    }
    *launches += 1;
    return rc;
}

}  // namespace cudapre
