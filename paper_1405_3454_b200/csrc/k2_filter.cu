// k2_filter.cu — Step 3 of CudaPre (§2 Step 3; SPEC.md
// S:71-79) as ONE streaming pass on sm_100a: classify every point
// against the filter polygon and stream-compact the survivors in ascending
// index order (A15), with a single-pass decoupled look-back scan.
//
// Classification (exact semantics, A11/A12): point p is DISCARDED iff
// orient(v_j, v_j+1, p) > 0 for every ring edge j.  Fast paths, all proven
// conservative in DESIGN.md §6.2:
//   1. inner box (4 float compares): the closed box lies strictly inside the
//      ring (checked exactly on the host)              -> discard
//   2. g_j = fma(A_j, x, fma(B_j, y, C'_j)) with C'_j = C_j - E_j, where E_j
//      bounds |float evaluation - exact orient| over the data bounding box:
//      min_j g_j > 0                                   -> discard
//      RN(min_j g_j + 2 max_j E_j) < 0                 -> keep
//   3. otherwise (|orient| within ~E of 0: a few points per million) the exact
//      orientation predicate (exact.cuh) on every edge.
// The polygon (<= 32 vertices, coefficients, box) is a __grid_constant__
// kernel parameter: warp-uniform reads served from the constant bank — the
// paper stages it in shared memory.
//
// Compaction: persistent blocks take 2048-point tiles from an atomic ticket
// (so every predecessor tile is already running: no deadlock), prefetch the
// next tile before the current one's look-back, and write each warp's
// survivors as one contiguous run (warp ballots + a 32-entry block scan).
// Tile status words carry a 30-bit epoch so the workspace never needs a
// memset; the last block out resets the counters and bumps the epoch.
#include <cuda_runtime.h>

#include <cstdint>

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

__device__ __noinline__ bool exact_inside(const K2Params& p, float x, float y) {
    for (int j = 0; j < p.nv; ++j)
        if (orient_sign_f(p.vx[j], p.vy[j], p.vx[j + 1], p.vy[j + 1], x, y) <= 0) return false;
    return true;
}

// true = survivor (not strictly inside the ring)
__device__ __forceinline__ bool keep_point(const K2Params& p, float x, float y) {
    if (p.mode == 1) return true;
    if (p.mode == 2) return !exact_inside(p, x, y);
    if (x >= p.bx0 && x <= p.bx1 && y >= p.by0 && y <= p.by1) return false;
    float mn = INFINITY;
    for (int j = 0; j < p.nv; ++j) mn = fminf(mn, __fmaf_rn(p.A[j], x, __fmaf_rn(p.B[j], y, p.C[j])));
    if (mn > 0.0f) return false;
    if (__fadd_rn(mn, p.e2max) < 0.0f) return true;
    return !exact_inside(p, x, y);
}

// Decoupled look-back by warp 0: returns the exclusive prefix of `tile`.
__device__ __forceinline__ unsigned long long lookback(const K2Params& p, unsigned tile,
                                                       unsigned total, unsigned epoch,
                                                       unsigned lane) {
    unsigned long long* st = p.status;
    const unsigned long long E = (unsigned long long)(epoch & kEpochMask) << 34;
    if (tile == 0) {
        if (lane == 0) st_status(&st[0], E | ((unsigned long long)kFlagP << 32) | total);
        return 0ull;
    }
    if (lane == 0) st_status(&st[tile], E | ((unsigned long long)kFlagA << 32) | total);
    unsigned long long ex = 0;
    long long pred = (long long)tile - 1;
    while (true) {
        const long long t = pred - (long long)lane;
        unsigned long long w = (t >= 0) ? ld_status(&st[t]) : (E | ((unsigned long long)kFlagP << 32));
        const unsigned flag = ((unsigned)(w >> 34) == (epoch & kEpochMask)) ? (unsigned)((w >> 32) & 3u) : 0u;
        const unsigned pmask = __ballot_sync(kFull, flag == kFlagP);
        const unsigned inval = __ballot_sync(kFull, flag == 0u);
        const unsigned lim = pmask ? (unsigned)(__ffs(pmask) - 1) : 31u;
        const unsigned need = (lim == 31u) ? kFull : ((2u << lim) - 1u);
        if (inval & need) {
            __nanosleep(20);
            continue;
        }
        unsigned long long v = (lane <= lim) ? (w & 0xffffffffull) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        ex += v;
        if (pmask) break;
        pred -= 32;
    }
    if (lane == 0) st_status(&st[tile], E | ((unsigned long long)kFlagP << 32) | (ex + total));
    return ex;
}

template <bool VEC>
__global__ void __launch_bounds__(kK2Threads) k2_filter(const __grid_constant__ K2Params p) {
    constexpr int kWarps = kK2Threads / 32;
    static_assert(kWarps * kK2Items == 32, "block scan assumes 32 (item, warp) groups");
    __shared__ unsigned s_next;
    __shared__ unsigned s_counts[32];
    __shared__ unsigned s_offs[32];
    __shared__ unsigned long long s_prefix;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned epoch = *(volatile unsigned*)&p.ws->epoch;

    if (threadIdx.x == 0) s_next = atomicAdd(&p.ws->k2_ticket, 1u);
    __syncthreads();
    unsigned tile = s_next;
    float4 v[kK2Items];
    if (tile < p.num_tiles) {
#pragma unroll
        for (int u = 0; u < kK2Items; ++u)
            v[u] = load_pair<VEC>(p.pts, tile * kK2TilePairs + u * kK2Threads + threadIdx.x, p.n);
    }
    while (tile < p.num_tiles) {
        const unsigned qbase = tile * kK2TilePairs + threadIdx.x;
        bool k0[kK2Items], k1[kK2Items];
        unsigned pre[kK2Items];
#pragma unroll
        for (int u = 0; u < kK2Items; ++u) {
            const unsigned i0 = 2u * (qbase + u * kK2Threads);
            k0[u] = (i0 < p.n) && keep_point(p, v[u].x, v[u].y);
            k1[u] = (i0 + 1u < p.n) && keep_point(p, v[u].z, v[u].w);
            const unsigned b0 = __ballot_sync(kFull, k0[u]);
            const unsigned b1 = __ballot_sync(kFull, k1[u]);
            pre[u] = __popc(b0 & lt) + __popc(b1 & lt);
            if (lane == 0) s_counts[u * kWarps + warp] = __popc(b0) + __popc(b1);
        }
        if (threadIdx.x == 0) s_next = atomicAdd(&p.ws->k2_ticket, 1u);
        __syncthreads();
        const unsigned next = s_next;
        float4 vn[kK2Items];
        if (next < p.num_tiles) {   // prefetch the next tile during the look-back
#pragma unroll
            for (int u = 0; u < kK2Items; ++u)
                vn[u] = load_pair<VEC>(p.pts, next * kK2TilePairs + u * kK2Threads + threadIdx.x, p.n);
        }
        if (warp == 0) {
            const unsigned c = s_counts[lane];
            unsigned incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(kFull, incl, o);
                if (lane >= (unsigned)o) incl += y;
            }
            s_offs[lane] = incl - c;
            const unsigned total = __shfl_sync(kFull, incl, 31);
            const unsigned long long ex = lookback(p, tile, total, epoch, lane);
            if (lane == 0) {
                s_prefix = ex;
                if (tile == p.num_tiles - 1) p.ws->count = ex + total;
            }
        }
        __syncthreads();
        const unsigned long long ex = s_prefix;
#pragma unroll
        for (int u = 0; u < kK2Items; ++u) {
            const unsigned i0 = 2u * (qbase + u * kK2Threads);
            unsigned long long pos = ex + s_offs[u * kWarps + warp] + pre[u];
            if (k0[u]) {
                if (pos < p.capacity) {
                    p.out_idx[pos] = p.base + (long long)i0;
                    if (p.out_pts) reinterpret_cast<float2*>(p.out_pts)[pos] = make_float2(v[u].x, v[u].y);
                }
                ++pos;
            }
            if (k1[u] && pos < p.capacity) {
                p.out_idx[pos] = p.base + (long long)(i0 + 1u);
                if (p.out_pts) reinterpret_cast<float2*>(p.out_pts)[pos] = make_float2(v[u].z, v[u].w);
            }
        }
        __syncthreads();   // s_counts / s_offs / s_prefix reuse
        tile = next;
#pragma unroll
        for (int u = 0; u < kK2Items; ++u) v[u] = vn[u];
    }
    // last block out resets the ticket and bumps the epoch (all blocks have
    // read `epoch` and taken their final ticket before incrementing k2_done)
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned d = atomicAdd(&p.ws->k2_done, 1u);
        if (d == gridDim.x - 1) {
            unsigned e = (epoch + 1u) & kEpochMask;
            if (e == 0u) e = 1u;
            p.ws->k2_ticket = 0u;
            p.ws->k2_done = 0u;
            p.ws->epoch = e;
            __threadfence();
        }
    }
}

template <bool VEC>
cudaError_t launch_t(const K2Params& p, cudaStream_t s, int* launches) {
    static int max_blocks = 0;
    if (!max_blocks) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2_filter<VEC>, kK2Threads, 0);
        max_blocks = (per_sm > 0 ? per_sm : 1) * device_sm_count();
    }
    unsigned blocks = p.num_tiles < (unsigned)max_blocks ? p.num_tiles : (unsigned)max_blocks;
    if (blocks < 1) blocks = 1;
    k2_filter<VEC><<<blocks, kK2Threads, 0, s>>>(p);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace

int launch_filter(const K2Params& p, int vec16, void* stream, int* launches) {
    cudaStream_t s = (cudaStream_t)stream;
    return vec16 ? (int)launch_t<true>(p, s, launches) : (int)launch_t<false>(p, s, launches);
}

}  // namespace cudapre
