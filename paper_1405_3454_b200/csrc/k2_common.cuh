// k2_common.cuh — device helpers shared by the two Step-3 kernels
// (k2_filter.cu: register path; k2_filter_tma.cu: TMA-ring path).  Internal
// linkage: each translation unit gets its own copy.
#pragma once

#include <cuda_runtime.h>

#include "exact.cuh"
#include "internal.h"

namespace cudapre {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned kFlagA = 1u;   // tile aggregate available
constexpr unsigned kFlagP = 2u;   // inclusive prefix available
constexpr unsigned kEpochMask = 0x3fffffffu;

__device__ __forceinline__ float4 ld_stream(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void st_status(unsigned long long* a, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}

template <bool VEC>
__device__ __forceinline__ float4 load_pair(const float* pts, unsigned q, unsigned n) {
    const unsigned i0 = 2u * q;
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i0 + 1u < n) {
        if (VEC) {
            r = ld_stream(reinterpret_cast<const float4*>(pts) + q);
        } else {
            const float2 a = __ldg(reinterpret_cast<const float2*>(pts) + i0);
            const float2 b = __ldg(reinterpret_cast<const float2*>(pts) + i0 + 1);
            r = make_float4(a.x, a.y, b.x, b.y);
        }
    } else if (i0 < n) {
        const float2 a = __ldg(reinterpret_cast<const float2*>(pts) + i0);
        r = make_float4(a.x, a.y, 0.f, 0.f);
    }
    return r;
}

// The part of K2Geom the per-point tests read, copied into shared memory at
// block start (uniform addresses: broadcast loads).  The sector tables are
// copied separately by the kernels that use them.
struct GeomLite {
    int nv, mode, fast, pad;
    float bx0, bx1, by0, by1, ox, oy, r2, e2max;
    float A[CUDAPRE_MAX_SLOTS], B[CUDAPRE_MAX_SLOTS], C[CUDAPRE_MAX_SLOTS];
    float vx[CUDAPRE_MAX_SLOTS + 1], vy[CUDAPRE_MAX_SLOTS + 1];
};
// cooperative copy (all threads of the block; a barrier must follow)
__device__ __forceinline__ void load_geom_lite(GeomLite& s, const K2Geom* __restrict__ g, unsigned tid,
                                               unsigned nthreads) {
    if (tid == 0) {
        s.nv = g->nv;
        s.mode = g->mode;
        s.fast = g->fast;
        s.bx0 = g->bx0;
        s.bx1 = g->bx1;
        s.by0 = g->by0;
        s.by1 = g->by1;
        s.ox = g->ox;
        s.oy = g->oy;
        s.r2 = g->r2;
        s.e2max = g->e2max;
    }
    for (unsigned j = tid; j < (unsigned)CUDAPRE_MAX_SLOTS; j += nthreads) {
        s.A[j] = g->A[j];
        s.B[j] = g->B[j];
        s.C[j] = g->C[j];
    }
    for (unsigned j = tid; j <= (unsigned)CUDAPRE_MAX_SLOTS; j += nthreads) {
        s.vx[j] = g->vx[j];
        s.vy[j] = g->vy[j];
    }
}

__device__ __noinline__ bool exact_inside(const GeomLite& G, float x, float y) {
    for (int j = 0; j < G.nv; ++j)
        if (orient_sign_f(G.vx[j], G.vy[j], G.vx[j + 1], G.vy[j + 1], x, y) <= 0) return false;
    return true;
}

// Certainly strictly inside (inner box or inner disk; both proven on the host).
// Disk: (dx, dy) = RN((x, y) - (ox, oy)) in one FADD2, squares in one FMUL2,
// d2 = RN(dx^2 + dy^2) >= true d^2 (1 - 4u) — the bound DESIGN.md §6.2 uses.
// Bitwise (not short-circuit) logic: no branches.
__device__ __forceinline__ bool fast_inside(const GeomLite& G, float x, float y) {
    const float2 d = __fadd2_rn(make_float2(x, y), make_float2(-G.ox, -G.oy));
    const float2 d2 = __fmul2_rn(d, d);
    const bool in_disk = __fadd_rn(d2.x, d2.y) < G.r2;
    const bool in_box = (x >= G.bx0) & (x <= G.bx1) & (y >= G.by0) & (y <= G.by1);
    return in_disk | in_box;
}

// Survivor test for a point the fast tests could not decide (true = keep).
// EDGES: compile-time edge count; the builder pads edges nv..31 with
// A = B = 0, C = +inf (never the minimum), so the loop fully unrolls.
template <int EDGES>
__device__ __forceinline__ bool queue_keep(const GeomLite& G, float x, float y) {
    if (G.mode == 1) return true;
    if (G.mode == 2) return !exact_inside(G, x, y);
    float mn = INFINITY;
#pragma unroll
    for (int j = 0; j < EDGES; ++j) mn = fminf(mn, __fmaf_rn(G.A[j], x, __fmaf_rn(G.B[j], y, G.C[j])));
    if (mn > 0.0f) return false;
    if (__fadd_rn(mn, G.e2max) < 0.0f) return true;
    return !exact_inside(G, x, y);
}

// Out-of-line copy for kernels where the all-edge loop is a rare path: inlined,
// the compiler hoists its loads onto the common path.
template <int EDGES>
__device__ __noinline__ bool queue_keep_rare(const GeomLite& G, float x, float y) {
    return queue_keep<EDGES>(G, x, y);
}

// look-back loads per lane: first round / later rounds (A/B-measured)
#ifndef K2_LB_FIRST
#define K2_LB_FIRST 2
#endif
#ifndef K2_LB_NEXT
#define K2_LB_NEXT 8
#endif
// ---------------------------------------------------------------- look-back
// Status word of super-tile t: [epoch:30 | flag:2 | count:32] at
// status[t * kStatusStride] (one per 128-byte line).  publish() writes it with
// one relaxed 64-bit store; resolve() (warp 0) walks back 256
// predecessors per round (8 loads in flight per lane) summing aggregates up to
// the nearest inclusive prefix.  Because resolve(t) runs one tile-time after
// t's own aggregate was published (deferred, see the kernel), every
// predecessor's aggregate is normally already there: no spinning.
__device__ __forceinline__ void publish(const K2Params& p, unsigned tile, unsigned flag,
                                        unsigned long long value, unsigned epoch) {
    st_status(&p.status[(size_t)tile * kStatusStride], ((unsigned long long)(epoch & kEpochMask) << 34) |
                                   ((unsigned long long)flag << 32) | (value & 0xffffffffull));
}

// rounds / spins: diagnostic counters kept in registers by the caller and
// added to the workspace once per block (a per-tile atomic on one address
// is itself a hot spot).
__device__ __forceinline__ unsigned long long resolve(const K2Params& p, unsigned tile,
                                                      unsigned epoch, unsigned lane,
                                                      unsigned& rounds, unsigned& spins) {
    constexpr int kPer = K2_LB_NEXT;   // loads per lane in later rounds
    int per = K2_LB_FIRST;              // ... and in the first (the nearest prefix is usually close)
    const unsigned long long PF = (unsigned long long)kFlagP << 32;
    const unsigned long long E = (unsigned long long)(epoch & kEpochMask) << 34;
    unsigned long long ex = 0;
    long long pred = (long long)tile - 1;
    while (pred >= 0) {
        unsigned long long w[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const long long t = pred - (long long)(per * (int)lane + k);
            w[k] = (k < per && t >= 0) ? ld_status(&p.status[(size_t)t * kStatusStride]) : (E | PF);
        }
        int kp = per;
        bool inval = false;
        unsigned long long sum = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            if (k >= per) break;
            const unsigned flag =
                ((unsigned)(w[k] >> 34) == (epoch & kEpochMask)) ? (unsigned)((w[k] >> 32) & 3u) : 0u;
            if (kp == per) {
                if (flag == 0u) inval = true;
                sum += w[k] & 0xffffffffull;
                if (flag == kFlagP) kp = k;
            }
        }
        const unsigned pmask = __ballot_sync(kFull, kp < per);
        const unsigned imask = __ballot_sync(kFull, inval);
        const unsigned lim = pmask ? (unsigned)(__ffs(pmask) - 1) : 31u;
        const unsigned need = (lim == 31u) ? kFull : ((2u << lim) - 1u);
        ++rounds;
        if (imask & need) {
            ++spins;
            __nanosleep(128);
            continue;
        }
        unsigned long long v = (lane <= lim) ? sum : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        ex += v;
        if (pmask) break;
        pred -= 32 * per;
        per = kPer;
    }
    return ex;
}

}  // namespace
}  // namespace cudapre
