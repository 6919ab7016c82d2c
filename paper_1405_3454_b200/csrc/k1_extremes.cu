// k1_extremes.cu — Step 1 of CudaPre (§2 Step 1; SPEC.md
// S:126-134) as ONE streaming pass over HBM on sm_100a.
//
// The paper materialises three rotated copies and runs Thrust min/max
// reductions over four point sets.  Here each rotation is a
// projection, so a single kernel reads every point once (8 B/point, 128-bit
// loads of two points) and reduces all 4*nang (key, index) pairs:
//
//   exact key   X_k = RN(RN(x c_k) + RN(y s_k)),  Y_k = RN(RN(y c_k) - RN(x s_k))
//               in binary64 without FMA (readings A3, A6), lowest index
//               wins equal keys (A7).
//
// FP64 per point would exceed the HBM-rate issue budget, so
// the hot loop SCREENS in float32 with a rigorous margin and only candidates
// take the exact binary64 path:
//
//   Xf = RN32(x*cf + RN32(y*sf)) (one fma), m = RN32(fma(|x|+|y|, 2^-20, 2^-120))
//   |Xf - X_k| <= 3.0000004 * 2^-24 (|x|+|y|) + 2^-149 < m
//   point is a candidate for max-slot s iff NOT(RN(Xf + m) <  T_s)
//                        for min-slot s iff NOT(RN(Xf - m) >  T_s)
//   where T_s is a float that is <= (max slot) / >= (min slot) the exact key
//   of a point already in the reduction.  Rounding is monotone, so a point
//   whose exact key ties or beats T_s is always a candidate; ties are never
//   pruned; NaN/Inf inputs are always candidates (unordered compares).
//   Angle 0 (c=1, s=0) keys are the coordinates themselves: exact float tests.
//
// Before the screen, a per-warp PRE-SCREEN disk (centre and radius derived
// from the warp's thresholds, rigorous margin: a point strictly inside it
// cannot tie or beat any slot) lets most points of a dense set skip the 4 *
// nang screens; the others go to a per-warp queue screened in full 32-lane
// batches.  Input: 16-B aligned data is streamed by a dedicated producer warp
// (cp.async.bulk, 4 x 16 KiB ring, full / empty mbarriers) into shared
// memory, so no register holds data in flight (8-byte aligned input:
// register double-buffered 128-bit loads instead).
// Thresholds start from a tiny seed kernel (float-only lower/upper bounds of
// a sample, combined with atomicMax on an order-preserving encoding) so the
// exact path stays rare from the first iteration on.  Candidates update a
// per-warp state in shared memory (one lane at a time, lexicographic (key,
// index) compare — correct for any arrival order); the state then tightens
// the warp's thresholds.  Warp states -> block partial -> last-block
// finalize (threadfence + ticket) -> 32 slots of (global idx, key, point).
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "internal.h"
#include "tma.cuh"

namespace cudapre {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned kNoIdx = 0xffffffffu;

__device__ __forceinline__ float4 ld_stream(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

// Load the point pair q = (2q, 2q+1); v1 false if 2q+1 >= n.  VEC: 16-B aligned base.
template <bool VEC>
__device__ __forceinline__ float4 load_pair(const float* pts, unsigned q, unsigned n, bool& v0,
                                            bool& v1) {
    const unsigned i0 = 2u * q;
    v0 = i0 < n;
    v1 = i0 + 1u < n;
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    if (v1) {
        if (VEC) {
            r = ld_stream(reinterpret_cast<const float4*>(pts) + q);
        } else {
            const float2 a = __ldg(reinterpret_cast<const float2*>(pts) + i0);
            const float2 b = __ldg(reinterpret_cast<const float2*>(pts) + i0 + 1);
            r = make_float4(a.x, a.y, b.x, b.y);
        }
    } else if (v0) {
        const float2 a = __ldg(reinterpret_cast<const float2*>(pts) + i0);
        r = make_float4(a.x, a.y, 0.f, 0.f);
    }
    return r;
}

// order-preserving float <-> uint (for atomicMax); 0 never encodes a real float
__device__ __forceinline__ unsigned enc_f(float f) {
    const unsigned b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float dec_f(unsigned e) {
    return __uint_as_float((e & 0x80000000u) ? (e & 0x7fffffffu) : ~e);
}

__device__ __forceinline__ bool is_max_slot(int s) { return (s & 1) != 0; }

// (k, i) strictly better than (K, I) for the slot direction; lowest index on ties
__device__ __forceinline__ bool lex_better(double k, unsigned i, double K, unsigned I, bool mx) {
    return mx ? (k > K || (k == K && i < I)) : (k < K || (k == K && i < I));
}

template <int NANG>
__device__ __forceinline__ bool screen1(float x, float y, const float (&T)[4 * NANG],
                                        const K1Params& p);

template <int NANG>
struct WarpState {
    double key[4 * NANG];
    unsigned idx[4 * NANG];
    float4 stage[kK1Unroll];   // the candidate lane's points, for the cold exact path
    unsigned stage_q[kK1Unroll];
    unsigned stage_n;          // valid points in stage (remainder iterations)
};

// exact binary64 keys of (x, y) folded into a warp state (one lane at a time)
template <int NANG>
__device__ __forceinline__ void exact_update(WarpState<NANG>& st, float x, float y, unsigned i,
                                             const K1Params& p) {
    if (!isfinite(x) || !isfinite(y)) {
        atomicOr(&p.ws->k1_nonfinite, 1u);
        return;
    }
    const double xd = (double)x, yd = (double)y;
#pragma unroll
    for (int k = 0; k < NANG; ++k) {
        const double X = __dadd_rn(__dmul_rn(xd, p.c[k]), __dmul_rn(yd, p.s[k]));
        const double Y = __dsub_rn(__dmul_rn(yd, p.c[k]), __dmul_rn(xd, p.s[k]));
        const double kv[4] = {X, X, Y, Y};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int s = 4 * k + r;
            if (lex_better(kv[r], i, st.key[s], st.idx[s], r & 1)) {
                st.key[s] = kv[r];
                st.idx[s] = i;
            }
        }
    }
}

// float screen of one point against thresholds T (see file header)
template <int NANG>
__device__ __forceinline__ bool screen1(float x, float y, const float (&T)[4 * NANG],
                                        const K1Params& p) {
    bool c = !(x > T[0]) | !(x < T[1]) | !(y > T[2]) | !(y < T[3]);
    const float m = __fmaf_rn(__fadd_rn(fabsf(x), fabsf(y)), 0x1p-20f, 0x1p-120f);
#pragma unroll
    for (int k = 1; k < NANG; ++k) {
        const float X = __fmaf_rn(x, p.cf[k], __fmul_rn(y, p.sf[k]));
        const float Y = __fmaf_rn(y, p.cf[k], __fmul_rn(x, p.nsf[k]));
        c |= !(__fsub_rn(X, m) > T[4 * k + 0]) | !(__fadd_rn(X, m) < T[4 * k + 1]) |
             !(__fsub_rn(Y, m) > T[4 * k + 2]) | !(__fadd_rn(Y, m) < T[4 * k + 3]);
    }
    return c;
}

// packed screen of a pair of points (x0,y0),(x1,y1) = v, both valid
template <int NANG>
__device__ __forceinline__ bool screen2(const float4 v, const float (&T)[4 * NANG],
                                        const K1Params& p) {
    bool c = !(v.x > T[0]) | !(v.x < T[1]) | !(v.y > T[2]) | !(v.y < T[3]) |
             !(v.z > T[0]) | !(v.z < T[1]) | !(v.w > T[2]) | !(v.w < T[3]);
    if (NANG > 1) {
        const float2 xx = make_float2(v.x, v.z), yy = make_float2(v.y, v.w);
        const float2 ab = make_float2(__fadd_rn(fabsf(v.x), fabsf(v.y)), __fadd_rn(fabsf(v.z), fabsf(v.w)));
        const float2 m = __ffma2_rn(ab, make_float2(0x1p-20f, 0x1p-20f), make_float2(0x1p-120f, 0x1p-120f));
        const float2 nm = __ffma2_rn(ab, make_float2(-0x1p-20f, -0x1p-20f), make_float2(-0x1p-120f, -0x1p-120f));
#pragma unroll
        for (int k = 1; k < NANG; ++k) {
            const float2 cf = make_float2(p.cf[k], p.cf[k]);
            const float2 X = __ffma2_rn(xx, cf, __fmul2_rn(yy, make_float2(p.sf[k], p.sf[k])));
            const float2 Y = __ffma2_rn(yy, cf, __fmul2_rn(xx, make_float2(p.nsf[k], p.nsf[k])));
            const float2 Xl = __fadd2_rn(X, nm), Xh = __fadd2_rn(X, m);
            const float2 Yl = __fadd2_rn(Y, nm), Yh = __fadd2_rn(Y, m);
            c |= !(Xl.x > T[4 * k + 0]) | !(Xl.y > T[4 * k + 0]) | !(Xh.x < T[4 * k + 1]) |
                 !(Xh.y < T[4 * k + 1]) | !(Yl.x > T[4 * k + 2]) | !(Yl.y > T[4 * k + 2]) |
                 !(Yh.x < T[4 * k + 3]) | !(Yh.y < T[4 * k + 3]);
        }
    }
    return c;
}

// Cold path: fold the staged points of ONE lane (those passing the screen)
// into the warp state.  Not unrolled: one copy of the exact code.
template <int NANG>
__device__ __forceinline__ void exact_staged(WarpState<NANG>& st, const float (&T)[4 * NANG],
                                             const K1Params& p) {
    unsigned hits = 0;
#pragma unroll 1
    for (int j = 0; j < 2 * kK1Unroll; ++j) {
        const float4 v = st.stage[j >> 1];
        const unsigned i = 2u * st.stage_q[j >> 1] + (unsigned)(j & 1);
        const float x = (j & 1) ? v.z : v.x;
        const float y = (j & 1) ? v.w : v.y;
        if (i < p.n && screen1<NANG>(x, y, T, p)) {
            exact_update<NANG>(st, x, y, i, p);
            ++hits;
        }
    }
    atomicAdd(&p.ws->k1_exact, hits);
}

// thresholds <- the warp state (rounded to the safe side) and the seed
template <int NANG>
__device__ __forceinline__ void refresh_thresholds(float (&T)[4 * NANG], const WarpState<NANG>& st) {
#pragma unroll
    for (int s = 0; s < 4 * NANG; ++s) {
        if (st.idx[s] == kNoIdx) continue;
        if (is_max_slot(s))
            T[s] = fmaxf(T[s], __double2float_rd(st.key[s]));
        else
            T[s] = fminf(T[s], __double2float_ru(st.key[s]));
    }
}

// Pre-screen disk: with c = centre of the angle-0 thresholds
// and slack_s = T_s - key_s(c) (max slots) / key_s(c) - T_s (min slots), a
// point with |p - c| < rho = min_s slack_s (1 - 2^-10) - (|cx|+|cy|) 2^-17
// - 2^-100 cannot pass the float screen of any slot (the screen margin m,
// the binary64 key rounding and ulp(T_s) are all absorbed by the two
// relative terms).  The kernel tests d2 = RN(RN(dx^2)+RN(dy^2)) < rho2 with
// (dx, dy) = RN(p - c); d2 >= |p-c|^2 (1 - 4u) and rho2 <= rho^2 (1 - 2^-16).
// rho2 = -1 disables the pre-screen (no seed yet, or no positive slack).
template <int NANG>
__device__ __forceinline__ void prescreen_params(const float (&T)[4 * NANG], const K1Params& p,
                                                 float& cx, float& cy, float& rho2) {
    cx = __fmul_rn(__fadd_rn(T[0], T[1]), 0.5f);
    cy = __fmul_rn(__fadd_rn(T[2], T[3]), 0.5f);
    rho2 = -1.0f;
    if (!isfinite(cx) || !isfinite(cy)) return;
    double smin = INFINITY;
#pragma unroll
    for (int k = 0; k < NANG; ++k) {
        const double px = __dadd_rn(__dmul_rn((double)cx, p.c[k]), __dmul_rn((double)cy, p.s[k]));
        const double py = __dsub_rn(__dmul_rn((double)cy, p.c[k]), __dmul_rn((double)cx, p.s[k]));
        smin = fmin(smin, __dsub_rn(px, (double)T[4 * k + 0]));
        smin = fmin(smin, __dsub_rn((double)T[4 * k + 1], px));
        smin = fmin(smin, __dsub_rn(py, (double)T[4 * k + 2]));
        smin = fmin(smin, __dsub_rn((double)T[4 * k + 3], py));
    }
    const double ac = __dadd_rn(fabs((double)cx), fabs((double)cy));
    const double rho = __dsub_rn(__dsub_rn(__dmul_rn(smin, 1.0 - 0x1p-10), __dmul_rn(ac, 0x1p-17)), 0x1p-100);
    if (!(rho > 0.0) || !isfinite(rho)) return;
    const double r2 = fmin(__dmul_rn(__dmul_rn(rho, rho), 1.0 - 0x1p-16), 0x1p126);
    if (r2 < 0x1p-100) return;
    rho2 = __double2float_rd(r2);
}

// ---------------------------------------------------------------- seed kernel
// Float-only bounds over sample chunks spread evenly over the input:
//   max slot: a float <= the exact key of some sampled point  (RD(Xf - m))
//   min slot: a float >= the exact key of some sampled point  (RU(Xf + m))
template <int NANG, bool VEC>
__global__ void __launch_bounds__(kSeedThreads) k1_seed(const K1Params p) {
    constexpr int NS = 4 * NANG;
    float L[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) L[s] = is_max_slot(s) ? -INFINITY : INFINITY;
    const unsigned npairs = p.n / 2u + (p.n & 1u);   // (n + 1) / 2 without wrapping at 2^32-1
    const unsigned chunk_pairs = kSeedThreads;
    const unsigned span = npairs > chunk_pairs ? npairs - chunk_pairs : 0u;
    for (unsigned c = blockIdx.x; c < p.seed_chunks; c += gridDim.x) {
        const unsigned q0 = p.seed_chunks > 1
                                ? (unsigned)(((unsigned long long)c * span) / (p.seed_chunks - 1))
                                : 0u;
        const unsigned q = q0 + threadIdx.x;
        bool v0, v1;
        const float4 v = load_pair<VEC>(p.pts, q, p.n, v0, v1);
        const float px[2] = {v.x, v.z}, py[2] = {v.y, v.w};
        const bool ok[2] = {v0, v1};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (!ok[h]) continue;
            const float x = px[h], y = py[h];
            L[0] = fminf(L[0], x);
            L[1] = fmaxf(L[1], x);
            L[2] = fminf(L[2], y);
            L[3] = fmaxf(L[3], y);
            const float m = __fmaf_rn(__fadd_rn(fabsf(x), fabsf(y)), 0x1p-20f, 0x1p-120f);
#pragma unroll
            for (int k = 1; k < NANG; ++k) {
                const float X = __fmaf_rn(x, p.cf[k], __fmul_rn(y, p.sf[k]));
                const float Y = __fmaf_rn(y, p.cf[k], __fmul_rn(x, p.nsf[k]));
                L[4 * k + 0] = fminf(L[4 * k + 0], __fadd_ru(X, m));
                L[4 * k + 1] = fmaxf(L[4 * k + 1], __fsub_rd(X, m));
                L[4 * k + 2] = fminf(L[4 * k + 2], __fadd_ru(Y, m));
                L[4 * k + 3] = fmaxf(L[4 * k + 3], __fsub_rd(Y, m));
            }
        }
    }
    __shared__ float red[kSeedThreads / 32][NS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        float v = L[s];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float w = __shfl_xor_sync(kFull, v, o);
            v = is_max_slot(s) ? fmaxf(v, w) : fminf(v, w);
        }
        if (lane == 0) red[warp][s] = v;
    }
    __syncthreads();
    if (threadIdx.x < NS) {
        const int s = threadIdx.x;
        float v = red[0][s];
        for (int w = 1; w < kSeedThreads / 32; ++w)
            v = is_max_slot(s) ? fmaxf(v, red[w][s]) : fminf(v, red[w][s]);
        if (is_max_slot(s)) {
            if (v > -INFINITY) atomicMax(&p.ws->seed[s], enc_f(v));
        } else {
            if (v < INFINITY) atomicMax(&p.ws->seed[s], ~enc_f(v));
        }
    }
}

// ---------------------------------------------------------------- main kernel
// TMA: one extra (producer) warp
template <int NANG, bool VEC, bool TMA>
__global__ void __launch_bounds__(kK1Threads + (TMA ? 32 : 0), 2) k1_extremes(const K1Params p) {
    constexpr int NS = 4 * NANG;
    constexpr int kWarps = kK1Threads / 32;
    __shared__ WarpState<NANG> sst[kWarps];
    __shared__ float sqx[kWarps][kK1Queue], sqy[kWarps][kK1Queue];
    __shared__ unsigned sqi[kWarps][kK1Queue];
    __shared__ bool s_last;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    WarpState<NANG>& st = sst[warp < (unsigned)kWarps ? warp : 0u];   // (TMA producer warp: unused)

    // thresholds from the seed (0 = no seed)
    float T[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const unsigned e = p.ws->seed[s];
        if (is_max_slot(s))
            T[s] = e ? dec_f(e) : -INFINITY;
        else
            T[s] = e ? dec_f(~e) : INFINITY;
    }
    if (lane < NS && warp < (unsigned)kWarps) {
        st.key[lane] = is_max_slot(lane) ? -INFINITY : INFINITY;
        st.idx[lane] = kNoIdx;
    }
    __syncwarp();
    float pcx, pcy, prho2;
    prescreen_params<NANG>(T, p, pcx, pcy, prho2);
    unsigned qcount = 0;   // this warp's queued points (uniform)

    const unsigned npairs = p.n / 2u + (p.n & 1u);   // (n + 1) / 2 without wrapping at 2^32-1
    const unsigned stride = gridDim.x * kK1Threads * kK1Unroll;
    unsigned q0 = blockIdx.x * (kK1Threads * kK1Unroll) + threadIdx.x;
    // full iterations: every pair valid (2q+1 < n  <=>  q < n/2)
    const unsigned full_pairs = p.n / 2u;
    // Full iterations (every pair valid), software-pipelined: the next
    // iteration's 4 x 128-bit loads are issued before this one is screened.
    // Loop conditions use the warp's lane-0 pair so all lanes agree.
    auto full = [&](unsigned q) {
        return (q - lane) + 31u + (kK1Unroll - 1) * kK1Threads < full_pairs;
    };
    auto load_full = [&](float4 (&dst)[kK1Unroll], unsigned q) {
#pragma unroll
        for (int u = 0; u < kK1Unroll; ++u) {
            if (VEC) {
                dst[u] = ld_stream(reinterpret_cast<const float4*>(p.pts) + q + u * kK1Threads);
            } else {
                bool a, b;
                dst[u] = load_pair<false>(p.pts, q + u * kK1Threads, p.n, a, b);
            }
        }
    };
    // Screen queued points in full 32-lane batches (all of them if `all`):
    // float screen, then the rare candidates' exact binary64 update (cold).
    auto drain = [&](bool all) {
        const unsigned nb = all ? qcount : (qcount & ~31u);
        for (unsigned base = 0; base < nb; base += 32) {
            const unsigned e = base + lane;
            bool cand = false;
            float x = 0.f, y = 0.f;
            unsigned i = 0;
            if (e < nb) {
                x = sqx[warp][e];
                y = sqy[warp][e];
                i = sqi[warp][e];
                cand = screen1<NANG>(x, y, T, p);
            }
            unsigned mask = __ballot_sync(kFull, cand);
            if (mask) {
                const unsigned hits = __popc(mask);
                while (mask) {
                    const unsigned l = __ffs(mask) - 1;
                    mask &= mask - 1;
                    if (lane == l) exact_update<NANG>(st, x, y, i, p);
                    __syncwarp();
                }
                if (lane == 0) atomicAdd(&p.ws->k1_exact, hits);
                refresh_thresholds<NANG>(T, st);
                prescreen_params<NANG>(T, p, pcx, pcy, prho2);
            }
        }
        const unsigned rem = qcount - nb;   // < 32: move to the front
        float rx = 0.f, ry = 0.f;
        unsigned ri = 0;
        if (lane < rem) {
            rx = sqx[warp][nb + lane];
            ry = sqy[warp][nb + lane];
            ri = sqi[warp][nb + lane];
        }
        __syncwarp();
        if (lane < rem) {
            sqx[warp][lane] = rx;
            sqy[warp][lane] = ry;
            sqi[warp][lane] = ri;
        }
        __syncwarp();
        qcount = rem;
    };
    // Pre-screen 4 pairs against the warp's disk; queue the rest.
    auto process = [&](const float4 (&v)[kK1Unroll], unsigned qb) {
        unsigned needy = 0u;   // bit b = 2u + h
        const float2 nc = make_float2(-pcx, -pcy);
#pragma unroll
        for (int u = 0; u < kK1Unroll; ++u) {
            const float2 d0 = __fmul2_rn(__fadd2_rn(make_float2(v[u].x, v[u].y), nc), __fadd2_rn(make_float2(v[u].x, v[u].y), nc));
            const float2 d1 = __fmul2_rn(__fadd2_rn(make_float2(v[u].z, v[u].w), nc), __fadd2_rn(make_float2(v[u].z, v[u].w), nc));
            needy |= ((__fadd_rn(d0.x, d0.y) < prho2) ? 0u : 1u) << (2 * u);
            needy |= ((__fadd_rn(d1.x, d1.y) < prho2) ? 0u : 2u) << (2 * u);
        }
        const unsigned nq = __popc(needy);
        unsigned incl = nq;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(kFull, incl, o);
            if (lane >= (unsigned)o) incl += t;
        }
        const unsigned qtotal = __shfl_sync(kFull, incl, 31);
        if (qtotal) {
            unsigned j = qcount + incl - nq;
#pragma unroll
            for (int b = 0; b < 2 * kK1Unroll; ++b) {
                if ((needy >> b) & 1u) {
                    const float4 w = v[b >> 1];
                    sqx[warp][j] = (b & 1) ? w.z : w.x;
                    sqy[warp][j] = (b & 1) ? w.w : w.y;
                    sqi[warp][j] = 2u * (qb + (b >> 1) * kK1Threads) + (unsigned)(b & 1);
                }
                j += (needy >> b) & 1u;
            }
            qcount += qtotal;
            __syncwarp();
            if (qcount >= 32u) drain(false);
        }
    };
    if constexpr (TMA) {
        // Chunks of kK1StagePairs pairs (16 KiB) stream through a kK1Stages-deep
        // shared-memory ring filled by cp.async.bulk (TMA): a dedicated producer
        // warp (warp kWarps, one lane) issues chunk i once every compute warp
        // has released stage i % kK1Stages ("empty" mbarrier, kWarps arrivals);
        // compute warps wait on the stage's transaction-counting "full"
        // mbarrier.  No block-wide barrier in the loop.  Chunk c goes to block
        // c % gridDim.x.
        extern __shared__ __align__(128) float4 ring[];
        __shared__ unsigned long long fullb[kK1Stages], emptyb[kK1Stages];
        const unsigned nchunks = full_pairs / kK1StagePairs;
        const unsigned mine =
            blockIdx.x < nchunks ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0u;
        if (threadIdx.x == 0) {
            for (int k = 0; k < kK1Stages; ++k) {
                mbar_init(&fullb[k], 1u);
                mbar_init(&emptyb[k], (unsigned)kWarps);
            }
            mbar_fence_init();
        }
        __syncthreads();
        const unsigned a_full = smem_u32(&fullb[0]), a_empty = smem_u32(&emptyb[0]), a_ring = smem_u32(ring);
        if (warp == (unsigned)kWarps) {
            if (lane == 0) {
                const float4* src = reinterpret_cast<const float4*>(p.pts);
                for (unsigned i = 0; i < mine; ++i) {
                    const unsigned sidx = i % kK1Stages;
                    if (i >= (unsigned)kK1Stages) mbar_sleep_wait(a_empty + 8u * sidx, ((i / kK1Stages) - 1u) & 1u);
                    mbar_expect_tx_a(a_full + 8u * sidx, kK1StagePairs * 16u);
                    bulk_g2s_a(a_ring + sidx * (kK1StagePairs * 16u),
                               src + (size_t)(blockIdx.x + i * gridDim.x) * kK1StagePairs, kK1StagePairs * 16u,
                               a_full + 8u * sidx);
                }
            }
        } else {
            for (unsigned i = 0; i < mine; ++i) {
                const unsigned sidx = i % kK1Stages;
                mbar_sleep_wait(a_full + 8u * sidx, (i / kK1Stages) & 1u);
                float4 v[kK1Unroll];
#pragma unroll
                for (int u = 0; u < kK1Unroll; ++u) v[u] = ring[sidx * kK1StagePairs + u * kK1Threads + threadIdx.x];
                __syncwarp();
                if (lane == 0) mbar_arrive_a(a_empty + 8u * sidx);   // data now in registers
                process(v, (blockIdx.x + i * gridDim.x) * kK1StagePairs + threadIdx.x);
            }
        }
        q0 = nchunks * kK1StagePairs + blockIdx.x * (kK1Threads * kK1Unroll) + threadIdx.x;
    } else if (full(q0)) {
        // registers: the next iteration's 4 x 128-bit loads are issued before
        // this one is screened
        float4 v[kK1Unroll];
        load_full(v, q0);
        while (true) {
            const unsigned qn = q0 + stride;
            const bool more = full(qn);
            float4 vn[kK1Unroll];
            if (more) load_full(vn, qn);
            process(v, q0);
            q0 = qn;
            if (!more) break;
#pragma unroll
            for (int u = 0; u < kK1Unroll; ++u) v[u] = vn[u];
        }
    }
    if (!TMA || warp < (unsigned)kWarps) {   // (TMA: the producer warp has no warp state)
    drain(true);
    // remainder (guarded)
    for (; q0 - lane < npairs; q0 += stride) {
        float4 v[kK1Unroll];
        bool va[kK1Unroll], vb[kK1Unroll];
#pragma unroll
        for (int u = 0; u < kK1Unroll; ++u) {
            const unsigned q = q0 + u * kK1Threads;
            v[u] = load_pair<VEC>(p.pts, q < npairs ? q : 0u, q < npairs ? p.n : 0u, va[u], vb[u]);
        }
        bool cand = false;
#pragma unroll
        for (int u = 0; u < kK1Unroll; ++u)
            cand |= (va[u] && screen1<NANG>(v[u].x, v[u].y, T, p)) ||
                    (vb[u] && screen1<NANG>(v[u].z, v[u].w, T, p));
        unsigned mask = __ballot_sync(kFull, cand);
        while (mask) {
            const unsigned l = __ffs(mask) - 1;
            mask &= mask - 1;
            if (lane == l) {
#pragma unroll
                for (int u = 0; u < kK1Unroll; ++u) {
                    st.stage[u] = v[u];
                    st.stage_q[u] = q0 + u * kK1Threads;   // out-of-range pairs: i >= n, skipped
                }
                exact_staged<NANG>(st, T, p);
            }
            __syncwarp();
        }
        if (__any_sync(kFull, cand)) refresh_thresholds<NANG>(T, st);
    }
    }

    // ---- warp states -> block partial
    __syncthreads();
    if (threadIdx.x < NS) {
        const int s = threadIdx.x;
        const bool mx = is_max_slot(s);
        double K = sst[0].key[s];
        unsigned I = sst[0].idx[s];
        for (int w = 1; w < kWarps; ++w) {
            if (sst[w].idx[s] != kNoIdx && (I == kNoIdx || lex_better(sst[w].key[s], sst[w].idx[s], K, I, mx))) {
                K = sst[w].key[s];
                I = sst[w].idx[s];
            }
        }
        K1Partial& part = p.partials[blockIdx.x * CUDAPRE_MAX_SLOTS + s];
        part.key = K;
        part.idx = I;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned t = atomicAdd(&p.ws->k1_ticket, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;

    // ---- last block: reduce all block partials, write the result, reset
    __threadfence();
    cudapre_extremes_t* outs[2] = {&p.ws->result, p.d_out};
    for (int s = warp; s < NS && warp < (unsigned)kWarps; s += kWarps) {
        const bool mx = is_max_slot(s);
        double K = mx ? -INFINITY : INFINITY;
        unsigned I = kNoIdx;
        for (unsigned b = lane; b < gridDim.x; b += 32) {
            const K1Partial* q = &p.partials[b * CUDAPRE_MAX_SLOTS + s];
            const double k2 = __ldcg(&q->key);
            const unsigned i2 = __ldcg(&q->idx);
            if (i2 != kNoIdx && (I == kNoIdx || lex_better(k2, i2, K, I, mx))) {
                K = k2;
                I = i2;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double k2 = __shfl_down_sync(kFull, K, o);
            const unsigned i2 = __shfl_down_sync(kFull, I, o);
            if (i2 != kNoIdx && (I == kNoIdx || lex_better(k2, i2, K, I, mx))) {
                K = k2;
                I = i2;
            }
        }
        if (lane == 0) {
            cudapre_pt pt = {0.f, 0.f};
            if (I != kNoIdx) {
                const float2 q = __ldg(reinterpret_cast<const float2*>(p.pts) + I);
                pt.x = q.x;
                pt.y = q.y;
            }
            for (int o = 0; o < 2; ++o) {
                if (!outs[o]) continue;
                outs[o]->idx[s] = (I == kNoIdx) ? -1ll : p.base + (long long)I;
                outs[o]->key[s] = K;
                outs[o]->pt[s] = pt;
            }
        }
    }
    if (threadIdx.x < 32) {
        const unsigned nf = __ldcg(&p.ws->k1_nonfinite);
        for (int o = 0; o < 2; ++o) {
            if (!outs[o]) continue;
            if (threadIdx.x < CUDAPRE_MAX_ANGLES) {
                const int k = threadIdx.x;
                outs[o]->c[k] = k < p.nang ? p.c[k] : 0.0;
                outs[o]->s[k] = k < p.nang ? p.s[k] : 0.0;
            }
            if (threadIdx.x >= (unsigned)NS) {   // unused slots
                outs[o]->idx[threadIdx.x] = -1;
                outs[o]->key[threadIdx.x] = 0.0;
                outs[o]->pt[threadIdx.x] = cudapre_pt{0.f, 0.f};
            }
            if (threadIdx.x == 0) {
                outs[o]->nang = p.nang;
                outs[o]->nonfinite = nf ? 1 : 0;
                outs[o]->n = (long long)p.n;
                outs[o]->exact_points = (long long)__ldcg(&p.ws->k1_exact);
            }
        }
        __syncwarp();
        if (threadIdx.x < CUDAPRE_MAX_SLOTS) p.ws->seed[threadIdx.x] = 0u;
        if (threadIdx.x == 0) {
            p.ws->k1_ticket = 0u;
            p.ws->k1_nonfinite = 0u;
            p.ws->k1_exact = 0u;
            p.ws->lb_rounds = 0u;   // Step-3 diagnostics count from here
            p.ws->lb_spins = 0u;
        }
    }
}

template <int NANG, bool VEC, bool TMA>
cudaError_t launch_t(const K1Params& p, cudaStream_t s, int* launches) {
    static std::once_flag once[kMaxDevices];
    static int cap[kMaxDevices];
    const int smem = TMA ? kK1Stages * kK1StagePairs * 16 : 0;
    const int k1_blocks = per_device(once, cap, [&] {
        if (TMA)
            cudaFuncSetAttribute(k1_extremes<NANG, VEC, TMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1_extremes<NANG, VEC, TMA>,
                                                      kK1Threads + (TMA ? 32 : 0), smem);
        int b = per_sm * device_sm_count();
        return b > kMaxK1Blocks ? kMaxK1Blocks : (b < 1 ? 1 : b);
    });
    const int seed_blocks = 2 * device_sm_count();
    const unsigned long long npairs = (p.n + 1ull) / 2ull;
    unsigned blocks = (unsigned)((npairs + kK1Threads * kK1Unroll - 1) / (kK1Threads * kK1Unroll));
    if (blocks > (unsigned)k1_blocks) blocks = (unsigned)k1_blocks;
    if (blocks < 1) blocks = 1;
    if (p.seed_chunks) {
        const unsigned sb = p.seed_chunks < (unsigned)seed_blocks ? p.seed_chunks : (unsigned)seed_blocks;
        k1_seed<NANG, VEC><<<sb, kSeedThreads, 0, s>>>(p);
        ++*launches;
    }
    k1_extremes<NANG, VEC, TMA><<<blocks, kK1Threads + (TMA ? 32 : 0), smem, s>>>(p);
    ++*launches;
    return cudaGetLastError();
}

template <int NANG>
cudaError_t launch_n(const K1Params& p, int vec16, cudaStream_t s, int* launches) {
    // 16-B aligned input streams through the TMA ring; 8-B aligned input uses
    // register loads (cp.async.bulk needs 16-B aligned sources).
    if (vec16) return launch_t<NANG, true, true>(p, s, launches);
    return launch_t<NANG, false, false>(p, s, launches);
}

}  // namespace

int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    return dev;
}

int device_sm_count() {
    static std::once_flag once[kMaxDevices];
    static int sms[kMaxDevices];
    return per_device(once, sms, [] {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, current_device());
        return v > 0 ? v : 148;
    });
}

int launch_extremes(const K1Params& p, int vec16, void* stream, int* launches) {
    cudaStream_t s = (cudaStream_t)stream;
    switch (p.nang) {
        case 1: return (int)launch_n<1>(p, vec16, s, launches);
        case 2: return (int)launch_n<2>(p, vec16, s, launches);
        case 3: return (int)launch_n<3>(p, vec16, s, launches);
        case 4: return (int)launch_n<4>(p, vec16, s, launches);
        case 8: return (int)launch_n<8>(p, vec16, s, launches);
        default: return (int)cudaErrorInvalidValue;
    }
}

}  // namespace cudapre
