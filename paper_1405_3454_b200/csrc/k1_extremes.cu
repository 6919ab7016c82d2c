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
// memory, so no register holds data in flight (CUDAPRE_K1_TMA=0: register
// double-buffered 128-bit loads instead).
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
#include "spec.cuh"
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
// fixc: keep the caller's centre (the pre-filter region's, DESIGN.md §6.6:
// the argument holds for any centre) instead of the thresholds' midpoint.
template <int NANG>
__device__ __forceinline__ void prescreen_params(const float (&T)[4 * NANG], const K1Params& p,
                                                 float& cx, float& cy, float& rho2, bool fixc = false) {
    if (!fixc) {
        cx = __fmul_rn(__fadd_rn(T[0], T[1]), 0.5f);
        cy = __fmul_rn(__fadd_rn(T[2], T[3]), 0.5f);
    }
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
// SPEC: also the sample point with the best float key per slot (the "seed
// picks"); the last block to finish builds the pre-filter region from them
// (build_region).
template <int NANG>
__device__ void build_region(const K1Params& p);

template <int NANG, bool VEC, bool SPEC>
__global__ void __launch_bounds__(kSeedThreads) k1_seed(const K1Params p) {
    constexpr int NS = 4 * NANG;
    float L[NS];
    float BK[SPEC ? NS : 1];      // best float key per slot (SPEC)
    unsigned BI[SPEC ? NS : 1];   // its local index
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        L[s] = is_max_slot(s) ? -INFINITY : INFINITY;
        if (SPEC) {
            BK[s] = L[s];
            BI[s] = kNoIdx;
        }
    }
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
            const unsigned i = 2u * q + (unsigned)h;
            L[0] = fminf(L[0], x);
            L[1] = fmaxf(L[1], x);
            L[2] = fminf(L[2], y);
            L[3] = fmaxf(L[3], y);
            if (SPEC) {
                const float kv[4] = {x, x, y, y};
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    if ((r & 1) ? kv[r] > BK[r] : kv[r] < BK[r]) BK[r] = kv[r], BI[r] = i;
            }
            const float m = __fmaf_rn(__fadd_rn(fabsf(x), fabsf(y)), 0x1p-20f, 0x1p-120f);
#pragma unroll
            for (int k = 1; k < NANG; ++k) {
                const float X = __fmaf_rn(x, p.cf[k], __fmul_rn(y, p.sf[k]));
                const float Y = __fmaf_rn(y, p.cf[k], __fmul_rn(x, p.nsf[k]));
                L[4 * k + 0] = fminf(L[4 * k + 0], __fadd_ru(X, m));
                L[4 * k + 1] = fmaxf(L[4 * k + 1], __fsub_rd(X, m));
                L[4 * k + 2] = fminf(L[4 * k + 2], __fadd_ru(Y, m));
                L[4 * k + 3] = fmaxf(L[4 * k + 3], __fsub_rd(Y, m));
                if (SPEC) {
                    const float kv[4] = {X, X, Y, Y};
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int s = 4 * k + r;
                        if ((r & 1) ? kv[r] > BK[s] : kv[r] < BK[s]) BK[s] = kv[r], BI[s] = i;
                    }
                }
            }
        }
    }
    __shared__ float red[kSeedThreads / 32][NS];
    __shared__ unsigned long long redp[kSeedThreads / 32][SPEC ? NS : 1];
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
        if (SPEC) {   // (order-preserving key << 32) | index; 0 = none
            unsigned long long e = 0;
            if (BI[s] != kNoIdx) {
                const unsigned ek = is_max_slot(s) ? enc_f(BK[s]) : ~enc_f(BK[s]);
                e = ((unsigned long long)ek << 32) | BI[s];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long w = __shfl_xor_sync(kFull, e, o);
                e = w > e ? w : e;
            }
            if (lane == 0) redp[warp][s] = e;
        }
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
        if (SPEC) {
            unsigned long long e = redp[0][s];
            for (int w = 1; w < kSeedThreads / 32; ++w) e = redp[w][s] > e ? redp[w][s] : e;
            if (e) atomicMax(&p.ws->seed_pick[s], e);
        }
    }
    if (SPEC) {   // last block out builds the pre-filter region
        __shared__ bool s_last;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) s_last = atomicAdd(&p.ws->seed_ticket, 1u) == gridDim.x - 1;
        __syncthreads();
        if (s_last) {
            __threadfence();
            build_region<NANG>(p);
        }
    }
}

// The pre-filter region D (spec.cuh) from the seed picks:
// their convex hull (plain binary64 monotone chain: D only has to be a good
// guess, the Step-2 verification makes it safe), centre = vertex mean,
// shrunk towards it by ~ the sample's angular resolution (spec::shrink), then
// the largest disk around the centre and the largest centred axis-aligned box
// inside the shrunk ring; D is the one covering more area.  Thread 0 of the
// last seed block.
template <int NANG>
__device__ void build_region(const K1Params& p) {
    constexpr int NS = 4 * NANG;
    if (threadIdx.x != 0) return;
    SpecPage* sp = p.sp;
    double px[NS], py[NS];
    int m = 0;
    bool ok = true;
    for (int s = 0; s < NS; ++s) {
        const unsigned long long e = __ldcg(&p.ws->seed_pick[s]);
        p.ws->seed_pick[s] = 0ull;   // (reset for the next call)
        if (!e) {
            ok = false;
            continue;
        }
        const float2 q = __ldg(reinterpret_cast<const float2*>(p.pts) + (unsigned)(e & 0xffffffffu));
        if (!isfinite(q.x) || !isfinite(q.y)) ok = false;
        // insertion sort by (x, y), dropping duplicates
        bool dup = false;
        for (int t = 0; t < m; ++t) dup |= (px[t] == (double)q.x && py[t] == (double)q.y);
        if (dup) continue;
        int j = m;
        while (j > 0 && (px[j - 1] > q.x || (px[j - 1] == q.x && py[j - 1] > q.y))) {
            px[j] = px[j - 1];
            py[j] = py[j - 1];
            --j;
        }
        px[j] = q.x;
        py[j] = q.y;
        ++m;
    }
    // monotone chain (CCW), strict turns
    double hx[2 * NS + 1], hy[2 * NS + 1];
    int k = 0;
    for (int i = 0; i < m && ok; ++i) {
        while (k >= 2 && (hx[k - 1] - hx[k - 2]) * (py[i] - hy[k - 2]) - (hy[k - 1] - hy[k - 2]) * (px[i] - hx[k - 2]) <= 0.0)
            --k;
        hx[k] = px[i], hy[k] = py[i], ++k;
    }
    for (int i = m - 2, t = k + 1; i >= 0 && ok; --i) {
        while (k >= t && (hx[k - 1] - hx[k - 2]) * (py[i] - hy[k - 2]) - (hy[k - 1] - hy[k - 2]) * (px[i] - hx[k - 2]) <= 0.0)
            --k;
        hx[k] = px[i], hy[k] = py[i], ++k;
    }
    const int nv = ok && m >= 3 ? k - 1 : 0;
    sp->nv_seed = (unsigned)nv;
    p.ws->seed_ticket = 0u;
    float r2 = -1.0f, box[4] = {1.f, -1.f, 1.f, -1.f};
    float fx = 0.f, fy = 0.f;
    bool use_box = false;
    if (nv >= 3) {
        // centre: the midpoint of the ring's bounding box (the angle-0 picks) --
        // also the K1 pre-screen centre, which wants it close to the data's
        double lx = INFINITY, ly = INFINITY, ux = -INFINITY, uy = -INFINITY;
        for (int j = 0; j < nv; ++j)
            lx = fmin(lx, hx[j]), ux = fmax(ux, hx[j]), ly = fmin(ly, hy[j]), uy = fmax(uy, hy[j]);
        fx = (float)(0.5 * (lx + ux)), fy = (float)(0.5 * (ly + uy));
        lx = ly = INFINITY, ux = uy = -INFINITY;
        const double eps = spec::shrink(fmin((double)p.seed_chunks * (2.0 * kSeedThreads), (double)p.n));
        for (int j = 0; j < nv; ++j) {   // shrink towards the (float) centre
            hx[j] = fx + (1.0 - eps) * (hx[j] - fx);
            hy[j] = fy + (1.0 - eps) * (hy[j] - fy);
            lx = fmin(lx, hx[j]), ux = fmax(ux, hx[j]), ly = fmin(ly, hy[j]), uy = fmax(uy, hy[j]);
        }
        if (isfinite(fx) && isfinite(fy) && spec::ring_contains(hx, hy, nv, fx, fy)) {
            r2 = spec::ring_r2(hx, hy, nv, fx, fy);
            // largest t in [0, 1]: the ring's bounding box scaled by t towards the
            // centre, [fx - t (fx - lx), fx + t (ux - fx)] x [fy - t (fy - ly), fy + t (uy - fy)], inside
            double lo = 0.0, hi = 1.0;
            for (int it = 0; it < 24; ++it) {
                const double t = 0.5 * (lo + hi);
                const double x0 = fx - t * (fx - lx), x1 = fx + t * (ux - fx);
                const double y0 = fy - t * (fy - ly), y1 = fy + t * (uy - fy);
                const bool in = spec::ring_contains(hx, hy, nv, x0, y0) && spec::ring_contains(hx, hy, nv, x1, y0) &&
                                spec::ring_contains(hx, hy, nv, x1, y1) && spec::ring_contains(hx, hy, nv, x0, y1);
                (in ? lo : hi) = t;
            }
            if (lo > 0.0) {
                box[0] = (float)(fx - lo * (fx - lx)), box[1] = (float)(fx + lo * (ux - fx));
                box[2] = (float)(fy - lo * (fy - ly)), box[3] = (float)(fy + lo * (uy - fy));
                const double barea = (double)(box[1] - box[0]) * (double)(box[3] - box[2]);
                use_box = box[0] < box[1] && box[2] < box[3] && barea > 3.14159 * fmax((double)r2, 0.0);
            }
        }
    }
    const bool on = use_box || r2 > 0.0f;
    sp->cx = fx;
    sp->cy = fy;
    sp->r2min = r2;
    sp->use_box = use_box ? 1 : 0;
    for (int j = 0; j < 4; ++j) sp->box[j] = box[j];
    sp->overflow = 0u;
    sp->candidates = 0ull;
    sp->on = 0;
    sp->enabled = on ? 1 : 0;
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
    // spec: per warp, two record images being built / stored by a bulk copy
    __shared__ __align__(16) unsigned char srec[TMA ? kWarps : 1][1][TMA ? kRecBytes : 16];
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
    // Spec mode (TMA ring only): the pre-filter region D
    // (the disk d2 < r2min around its centre, or its box, whichever the seed
    // found larger) shares its centre with the pre-screen, so one d2 serves
    // both tests.  Each lane writes its points outside D straight into the
    // chunk's record at the slots a warp scan of their counts gives.
    const bool spec = TMA && p.spec && p.sp->enabled;
    float scx = 0.f, scy = 0.f, sr2min = -1.f, sbx0 = 1.f, sbx1 = -1.f, sby0 = 1.f, sby1 = -1.f;
    int sbox = 0;
    if (spec) {
        scx = p.sp->cx;
        scy = p.sp->cy;
        sr2min = p.sp->r2min;
        sbox = p.sp->use_box;
        sbx0 = p.sp->box[0], sbx1 = p.sp->box[1], sby0 = p.sp->box[2], sby1 = p.sp->box[3];
    }
    float pcx = scx, pcy = scy, prho2;
    prescreen_params<NANG>(T, p, pcx, pcy, prho2, spec);
    unsigned qcount = 0;   // this warp's queued points (uniform)
    unsigned ncand = 0;    // spec: candidates written (diagnostic)

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
                prescreen_params<NANG>(T, p, pcx, pcy, prho2, spec);
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
    auto process = [&](const float4 (&v)[kK1Unroll], unsigned qb, const float2* stage2) {
        unsigned needy = 0u;   // bit b = 2u + h
        unsigned keep = 0u;    // spec: bit b = outside the pre-filter region (NaN: outside)
        const float2 nc = make_float2(-pcx, -pcy);
#pragma unroll
        for (int u = 0; u < kK1Unroll; ++u) {
            const float2 e0 = __fadd2_rn(make_float2(v[u].x, v[u].y), nc);
            const float2 e1 = __fadd2_rn(make_float2(v[u].z, v[u].w), nc);
            const float2 d0 = __fmul2_rn(e0, e0), d1 = __fmul2_rn(e1, e1);
            const float q0 = __fadd_rn(d0.x, d0.y), q1 = __fadd_rn(d1.x, d1.y);
            needy |= ((q0 < prho2) ? 0u : 1u) << (2 * u);
            needy |= ((q1 < prho2) ? 0u : 2u) << (2 * u);
            if (spec) {
                const bool in0 = sbox ? (v[u].x >= sbx0) & (v[u].x <= sbx1) & (v[u].y >= sby0) & (v[u].y <= sby1)
                                      : q0 < sr2min;
                const bool in1 = sbox ? (v[u].z >= sbx0) & (v[u].z <= sbx1) & (v[u].w >= sby0) & (v[u].w <= sby1)
                                      : q1 < sr2min;
                keep |= (in0 ? 0u : 1u) << (2 * u);
                keep |= (in1 ? 0u : 2u) << (2 * u);
            }
        }
        if (spec) {
            // the chunk's record (this warp's 256 points): slots by a warp scan of
            // the lanes' counts; each lane copies its points from the ring stage
            // into the warp's record image in shared memory (a loop over its
            // points outside D only), one bulk copy stores the image
            const unsigned nk = __popc(keep);
            unsigned kinc = nk;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned t = __shfl_up_sync(kFull, kinc, o);
                if (lane >= (unsigned)o) kinc += t;
            }
            const unsigned ktotal = __shfl_sync(kFull, kinc, 31);
            const unsigned chunk = qb >> 10;
            unsigned char* img = srec[warp][0];
            if (ktotal) {
                unsigned slot = kinc - nk;
                for (unsigned kb = keep; kb; kb &= kb - 1, ++slot) {
                    const unsigned b = __ffs(kb) - 1;
                    if (slot < (unsigned)kRecSlots) {
                        img[slot] = (unsigned char)(((b >> 1) << 6) | (lane << 1) | (b & 1));   // (u << 6) | offset
                        reinterpret_cast<float2*>(img + kRecMetaBytes)[slot] =
                            stage2[2u * ((b >> 1) * kK1Threads + threadIdx.x) + (b & 1)];
                    }
                }
                __syncwarp();
                // the image's used bytes, 16 per lane, coalesced
                const unsigned m = ktotal > (unsigned)kRecSlots ? 0u : ktotal;
                const unsigned nq = (kRecMetaBytes + 8u * m + 15u) / 16u;
                uint4* dst = reinterpret_cast<uint4*>(p.records + ((size_t)chunk * kWarps + warp) * kRecBytes);
                for (unsigned q = lane; q < nq; q += 32) dst[q] = reinterpret_cast<const uint4*>(img)[q];
                __syncwarp();
            }
            if (lane == 0) {
                p.rcount[(size_t)chunk * kWarps + warp] = (unsigned char)(ktotal > (unsigned)kRecSlots ? kRecOverflow : ktotal);
                if (ktotal > (unsigned)kRecSlots) atomicAdd(&p.sp->overflow, 1u);
            }
            ncand += ktotal;
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
                // data now in registers (spec: the record copies read the stage: release after)
                if (!spec && lane == 0) mbar_arrive_a(a_empty + 8u * sidx);
                const unsigned chunk = blockIdx.x + i * gridDim.x;
                process(v, chunk * kK1StagePairs + threadIdx.x,
                        reinterpret_cast<const float2*>(&ring[sidx * kK1StagePairs]));
                if (spec) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive_a(a_empty + 8u * sidx);
                }
            }
        }
        q0 = nchunks * kK1StagePairs + blockIdx.x * (kK1Threads * kK1Unroll) + threadIdx.x;
        if (spec && lane == 0 && ncand) atomicAdd(&p.sp->candidates, (unsigned long long)ncand);
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
            process(v, q0, nullptr);
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
            if (threadIdx.x == 0 && o == 0 && p.sp) {   // what the records describe (token; none if tok_n = 0)
                SpecPage* sp = p.sp;
                const bool on = TMA && p.spec && sp->enabled;
                sp->tok_pts = p.pts;
                sp->tok_base = p.base;
                sp->rec_chunks = (p.n / 2u) / (unsigned)kK1StagePairs;
                sp->tok_n = on ? (unsigned long long)p.n : 0ull;
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
        // spec (16-B aligned TMA path, <= 4 angles): the seed also builds the
        // pre-filter region
        bool spec_seed = false;
        if constexpr (TMA && NANG <= 4) {
            if (p.spec) {
                k1_seed<NANG, VEC, true><<<sb, kSeedThreads, 0, s>>>(p);
                spec_seed = true;
            }
        }
        if (!spec_seed) k1_seed<NANG, VEC, false><<<sb, kSeedThreads, 0, s>>>(p);
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
