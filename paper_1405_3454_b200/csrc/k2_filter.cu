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
constexpr unsigned kStash = 256;   // per-warp survivor coordinates kept in smem per super-tile

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

// Certainly strictly inside (inner box or inner disk; both proven on the host).
__device__ __forceinline__ bool fast_inside(const K2Params& p, float x, float y) {
    const bool in_box = x >= p.bx0 && x <= p.bx1 && y >= p.by0 && y <= p.by1;
    const float dx = __fsub_rn(x, p.ox), dy = __fsub_rn(y, p.oy);
    const bool in_disk = __fmaf_rn(dx, dx, __fmul_rn(dy, dy)) < p.r2;
    return in_box || in_disk;
}

// Survivor test for a point the fast tests could not decide (true = keep).
// EDGES: compile-time edge count; the host pads edges nv..EDGES-1 with
// A = B = 0, C = +inf (never the minimum), so the loop fully unrolls and the
// coefficients are constant-bank operands of the FFMAs.
template <int EDGES>
__device__ __forceinline__ bool queue_keep(const K2Params& p, float x, float y) {
    if (p.mode == 2) return !exact_inside(p, x, y);
    float mn = INFINITY;
#pragma unroll
    for (int j = 0; j < EDGES; ++j) mn = fminf(mn, __fmaf_rn(p.A[j], x, __fmaf_rn(p.B[j], y, p.C[j])));
    if (mn > 0.0f) return false;
    if (__fadd_rn(mn, p.e2max) < 0.0f) return true;
    return !exact_inside(p, x, y);
}

// Decoupled look-back by warp 0, 256 predecessors per round (8 per lane,
// loads in flight together): returns the exclusive prefix of super-tile `tile`.
// At HBM speed ~50 super-tiles complete per microsecond, so the look-back
// window must be wide or the chain of inclusive prefixes serialises.
__device__ __forceinline__ unsigned long long lookback(const K2Params& p, unsigned tile,
                                                       unsigned total, unsigned epoch,
                                                       unsigned lane) {
    constexpr int kPer = 8;
    unsigned long long* st = p.status;
    const unsigned long long E = (unsigned long long)(epoch & kEpochMask) << 34;
    const unsigned long long PF = (unsigned long long)kFlagP << 32;
    if (tile == 0) {
        if (lane == 0) st_status(&st[0], E | PF | total);
        return 0ull;
    }
    if (lane == 0) st_status(&st[tile], E | ((unsigned long long)kFlagA << 32) | total);
    unsigned long long ex = 0;
    long long pred = (long long)tile - 1;
    while (true) {
        unsigned long long w[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const long long t = pred - (long long)(kPer * lane + k);
            w[k] = (t >= 0) ? ld_status(&st[t]) : (E | PF);
        }
        // lane-local: nearest P among its 8 (k = 0 is the nearest), validity, sum
        int kp = kPer;
        bool inval = false;
        unsigned long long sum = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const unsigned flag =
                ((unsigned)(w[k] >> 34) == (epoch & kEpochMask)) ? (unsigned)((w[k] >> 32) & 3u) : 0u;
            if (kp == kPer) {
                if (flag == 0u) inval = true;
                sum += w[k] & 0xffffffffull;
                if (flag == kFlagP) kp = k;
            }
        }
        const unsigned pmask = __ballot_sync(kFull, kp < kPer);
        const unsigned imask = __ballot_sync(kFull, inval);
        const unsigned lim = pmask ? (unsigned)(__ffs(pmask) - 1) : 31u;
        const unsigned need = (lim == 31u) ? kFull : ((2u << lim) - 1u);
        if (imask & need) {
            __nanosleep(32);
            continue;
        }
        unsigned long long v = (lane <= lim) ? sum : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        ex += v;
        if (pmask) break;
        pred -= 32 * kPer;
    }
    if (lane == 0) st_status(&st[tile], E | PF | (ex + total));
    return ex;
}

// One super-tile = kK2Sub sub-tiles of kK2SubPairs point pairs.
//   pass A: stream the sub-tiles (register double buffer), classify, keep the
//           per-(sub-tile, item, warp) ballots in shared memory;
//   scan:   256 counts -> exclusive offsets inside the super-tile;
//   look-back (warp 0) -> global offset; the next super-tile's first
//           sub-tile is already in flight;
//   pass B: survivors' int64 indices (+ float2 re-read from L2, just streamed)
//           written as contiguous runs per (sub-tile, item, warp).
template <bool VEC, int EDGES>
__global__ void __launch_bounds__(kK2Threads, 2) k2_filter(const __grid_constant__ K2Params p) {
    constexpr int kWarps = kK2Threads / 32;
    constexpr int kGroups = kK2Sub * kK2Items * kWarps;   // 256 ballot groups per super-tile
    static_assert(kGroups == kK2Threads, "one scan entry per thread");
    __shared__ unsigned s_mask[kGroups][2];
    __shared__ float2 s_stash[kWarps][kStash];
    __shared__ float2 s_qxy[kWarps][2 * kK2Items * 32];         // undecided points
    __shared__ unsigned char s_qslot[kWarps][2 * kK2Items * 32]; // owner lane * 8 + bit
    __shared__ unsigned s_res[kWarps][2 * kK2Items];             // keep bits back to owners
    __shared__ unsigned s_off[kGroups];
    __shared__ unsigned s_wsum[kWarps];
    __shared__ unsigned s_next;
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
        const unsigned tbase = tile * kK2TilePairs;
        unsigned wc = 0;   // this warp's survivors so far in the super-tile (stash cursor)
        // ---- pass A
#pragma unroll 1
        for (int sub = 0; sub < kK2Sub; ++sub) {
            const unsigned qbase = tbase + sub * kK2SubPairs + threadIdx.x;
            float4 vn[kK2Items];
            if (sub + 1 < kK2Sub) {
#pragma unroll
                for (int u = 0; u < kK2Items; ++u)
                    vn[u] = load_pair<VEC>(p.pts, qbase + kK2SubPairs + u * kK2Threads, p.n);
            }
            // fast tests for the lane's 8 points: bit b = 2u + h
            unsigned keep = 0u, needy = 0u;
#pragma unroll
            for (int u = 0; u < kK2Items; ++u) {
                const unsigned i0 = 2u * (qbase + u * kK2Threads);
                const unsigned valid = (i0 < p.n ? 1u : 0u) | (i0 + 1u < p.n ? 2u : 0u);
                if (p.mode == 1) {
                    keep |= valid << (2 * u);
                } else {
                    const unsigned in = (p.mode == 0 && fast_inside(p, v[u].x, v[u].y) ? 1u : 0u) |
                                        (p.mode == 0 && fast_inside(p, v[u].z, v[u].w) ? 2u : 0u);
                    needy |= (valid & ~in) << (2 * u);
                }
            }
            // undecided points -> per-warp queue, tested with full lanes
            const unsigned nq = __popc(needy);
            unsigned incl = nq;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(kFull, incl, o);
                if (lane >= (unsigned)o) incl += y;
            }
            const unsigned qtotal = __shfl_sync(kFull, incl, 31);
            if (qtotal) {
                if (lane < 2 * kK2Items) s_res[warp][lane] = 0u;
                unsigned j = incl - nq;
#pragma unroll
                for (int b = 0; b < 2 * kK2Items; ++b) {
                    if ((needy >> b) & 1u) {
                        const float4 w = v[b >> 1];
                        s_qxy[warp][j] = (b & 1) ? make_float2(w.z, w.w) : make_float2(w.x, w.y);
                        s_qslot[warp][j] = (unsigned char)(lane * 8u + (unsigned)b);
                        ++j;
                    }
                }
                __syncwarp();
                for (unsigned base = 0; base < qtotal; base += 32) {
                    const unsigned e = base + lane;
                    if (e < qtotal) {
                        const float2 q = s_qxy[warp][e];
                        if (queue_keep<EDGES>(p, q.x, q.y)) {
                            const unsigned sl = s_qslot[warp][e];
                            atomicOr(&s_res[warp][sl & 7u], 1u << (sl >> 3));
                        }
                    }
                }
                __syncwarp();
#pragma unroll
                for (int b = 0; b < 2 * kK2Items; ++b) keep |= ((s_res[warp][b] >> lane) & 1u) << b;
                __syncwarp();
            }
#pragma unroll
            for (int u = 0; u < kK2Items; ++u) {
                const bool k0 = (keep >> (2 * u)) & 1u, k1 = (keep >> (2 * u + 1)) & 1u;
                const unsigned b0 = __ballot_sync(kFull, k0);
                const unsigned b1 = __ballot_sync(kFull, k1);
                if (lane == 0) {
                    const int g = (sub * kK2Items + u) * kWarps + warp;
                    s_mask[g][0] = b0;
                    s_mask[g][1] = b1;
                }
                if (p.out_pts && (b0 | b1)) {   // stash survivors' coordinates (pass B order)
                    const unsigned r0 = wc + __popc(b0 & lt) + __popc(b1 & lt);
                    if (k0 && r0 < kStash) s_stash[warp][r0] = make_float2(v[u].x, v[u].y);
                    if (k1 && r0 + k0 < kStash) s_stash[warp][r0 + k0] = make_float2(v[u].z, v[u].w);
                }
                wc += __popc(b0) + __popc(b1);
            }
            if (sub + 1 < kK2Sub) {
#pragma unroll
                for (int u = 0; u < kK2Items; ++u) v[u] = vn[u];
            }
        }
        // The next ticket is taken only now, so a tile is never held while its
        // block is still busy with an earlier one (that made successors' look-
        // backs wait a whole tile time and the delays cascade).
        if (threadIdx.x == 0) s_next = atomicAdd(&p.ws->k2_ticket, 1u);
        __syncthreads();
        const unsigned next = s_next;
        if (next < p.num_tiles) {   // prefetch the next super-tile's first sub-tile
#pragma unroll
            for (int u = 0; u < kK2Items; ++u)
                v[u] = load_pair<VEC>(p.pts, next * kK2TilePairs + u * kK2Threads + threadIdx.x, p.n);
        }
        // ---- block exclusive scan of the 256 group counts (group order = index order)
        {
            const unsigned c = __popc(s_mask[threadIdx.x][0]) + __popc(s_mask[threadIdx.x][1]);
            unsigned incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(kFull, incl, o);
                if (lane >= (unsigned)o) incl += y;
            }
            if (lane == 31) s_wsum[warp] = incl;
            __syncthreads();
            unsigned wpre = 0, total = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const unsigned x = s_wsum[w];
                wpre += (w < (int)warp) ? x : 0u;
                total += x;
            }
            s_off[threadIdx.x] = wpre + incl - c;
            if (warp == 0) {
                const unsigned long long ex = lookback(p, tile, total, epoch, lane);
                if (lane == 0) {
                    s_prefix = ex;
                    if (tile == p.num_tiles - 1) p.ws->count = ex + total;
                }
            }
        }
        __syncthreads();
        // ---- pass B: coordinates come from the stash (global re-read only on overflow)
        const unsigned long long ex = s_prefix;
        wc = 0;
#pragma unroll 1
        for (int sub = 0; sub < kK2Sub; ++sub) {
#pragma unroll
            for (int u = 0; u < kK2Items; ++u) {
                const int g = (sub * kK2Items + u) * kWarps + warp;
                const unsigned b0 = s_mask[g][0], b1 = s_mask[g][1];
                if ((b0 | b1) == 0u) continue;
                const bool k0 = (b0 >> lane) & 1u, k1 = (b1 >> lane) & 1u;
                const unsigned r0 = __popc(b0 & lt) + __popc(b1 & lt);
                unsigned long long pos = ex + s_off[g] + r0;
                const unsigned q = tbase + sub * kK2SubPairs + u * kK2Threads + threadIdx.x;
                const unsigned i0 = 2u * q;
                if (k0 | k1) {
                    float2 a = make_float2(0.f, 0.f), b = a;
                    if (p.out_pts) {
                        const unsigned s0 = wc + r0;
                        if (k0) a = s0 < kStash ? s_stash[warp][s0]
                                                : __ldcg(reinterpret_cast<const float2*>(p.pts) + i0);
                        if (k1) b = s0 + k0 < kStash ? s_stash[warp][s0 + k0]
                                                     : __ldcg(reinterpret_cast<const float2*>(p.pts) + i0 + 1);
                    }
                    if (k0) {
                        if (pos < p.capacity) {
                            p.out_idx[pos] = p.base + (long long)i0;
                            if (p.out_pts) reinterpret_cast<float2*>(p.out_pts)[pos] = a;
                        }
                        ++pos;
                    }
                    if (k1 && pos < p.capacity) {
                        p.out_idx[pos] = p.base + (long long)(i0 + 1u);
                        if (p.out_pts) reinterpret_cast<float2*>(p.out_pts)[pos] = b;
                    }
                }
                wc += __popc(b0) + __popc(b1);
            }
        }
        __syncthreads();   // shared arrays are reused by the next super-tile
        tile = next;
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

template <bool VEC, int EDGES>
cudaError_t launch_t(const K2Params& p, cudaStream_t s, int* launches) {
    static int max_blocks = 0;
    if (!max_blocks) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2_filter<VEC, EDGES>, kK2Threads, 0);
        max_blocks = (per_sm > 0 ? per_sm : 1) * device_sm_count();
    }
    unsigned blocks = p.num_tiles < (unsigned)max_blocks ? p.num_tiles : (unsigned)max_blocks;
    if (blocks < 1) blocks = 1;
    k2_filter<VEC, EDGES><<<blocks, kK2Threads, 0, s>>>(p);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace

int launch_filter(const K2Params& p, int vec16, void* stream, int* launches) {
    cudaStream_t s = (cudaStream_t)stream;
    if (p.nv <= 16)
        return vec16 ? (int)launch_t<true, 16>(p, s, launches) : (int)launch_t<false, 16>(p, s, launches);
    return vec16 ? (int)launch_t<true, 32>(p, s, launches) : (int)launch_t<false, 32>(p, s, launches);
}

}  // namespace cudapre
