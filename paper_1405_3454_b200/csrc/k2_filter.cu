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
#include <cstdlib>

#include "k2_common.cuh"

namespace cudapre {
namespace {

// ---------------------------------------------------------------- kernel
// Per-super-tile state, double buffered: pass B of tile k-1 runs after pass A
// of tile k.
struct alignas(16) SurvEntry {
    float x, y;
    unsigned idx;    // local point index
    unsigned meta;   // (group << 6) | (owner lane << 1) | pair element
};

constexpr int kK2Warps = kK2Threads / 32;
constexpr int kGroups = kK2Sub * kK2Items * kK2Warps;   // 256 ballot groups per super-tile
constexpr unsigned kList = 128;                          // per-warp survivor list per super-tile
constexpr int kQueue = 2 * kK2Items * 32;                // per-warp undecided-point queue

struct TileState {
    unsigned mask[kGroups][2];     // keep ballots (element 0 / 1 of each pair)
    unsigned off[kGroups];         // exclusive offset of each group inside the super-tile
    unsigned wcnt[kK2Warps];       // survivors per warp
    unsigned total;
    SurvEntry list[kK2Warps][kList];
};
struct K2Smem {
    TileState ts[2];
    float2 qxy[kK2Warps][kQueue];
    unsigned char qslot[kK2Warps][kQueue];
    unsigned char own[kK2Warps][32];   // keep bits returned to each owner lane
    unsigned wsum[kK2Warps];
    unsigned next;
    unsigned done;   // warps done with pass A of the current super-tile (the first one resolves)
    unsigned long long prefix;
    GeomLite geo;   // polygon scalars + coefficients (copied from p.g)
};

// Pass B of a resolved super-tile: write indices (+ coordinates).
__device__ __forceinline__ void emit(const K2Params& p, const TileState& ts, unsigned tbase,
                                     unsigned long long ex, unsigned warp, unsigned lane,
                                     unsigned lt) {
    const unsigned wc = ts.wcnt[warp];
    if (wc <= kList) {   // sparse: the compact list, full lanes
        for (unsigned r = lane; r < wc; r += 32) {
            const SurvEntry e = ts.list[warp][r];
            const unsigned g = e.meta >> 6, ol = (e.meta >> 1) & 31u, h = e.meta & 1u;
            const unsigned m0 = ts.mask[g][0], m1 = ts.mask[g][1], olt = (1u << ol) - 1u;
            const unsigned rig = __popc(m0 & olt) + __popc(m1 & olt) + (h ? ((m0 >> ol) & 1u) : 0u);
            const unsigned long long pos = ex + ts.off[g] + rig;
            if (pos < p.capacity) {
                p.out_idx[pos] = p.base + (long long)e.idx;
                if (p.out_pts) reinterpret_cast<float2*>(p.out_pts)[pos] = make_float2(e.x, e.y);
            }
        }
        return;
    }
    // dense: every group of this warp; coordinates re-read (L2-resident)
#pragma unroll 1
    for (int sub = 0; sub < kK2Sub; ++sub) {
#pragma unroll
        for (int u = 0; u < kK2Items; ++u) {
            const int g = (sub * kK2Items + u) * kK2Warps + warp;
            const unsigned b0 = ts.mask[g][0], b1 = ts.mask[g][1];
            const bool k0 = (b0 >> lane) & 1u, k1 = (b1 >> lane) & 1u;
            if (!(k0 | k1)) continue;
            unsigned long long pos = ex + ts.off[g] + __popc(b0 & lt) + __popc(b1 & lt);
            const unsigned i0 = 2u * (tbase + sub * kK2SubPairs + u * kK2Threads + threadIdx.x);
            if (k0) {
                if (pos < p.capacity) {
                    p.out_idx[pos] = p.base + (long long)i0;
                    if (p.out_pts)
                        reinterpret_cast<float2*>(p.out_pts)[pos] =
                            __ldcg(reinterpret_cast<const float2*>(p.pts) + i0);
                }
                ++pos;
            }
            if (k1 && pos < p.capacity) {
                p.out_idx[pos] = p.base + (long long)(i0 + 1u);
                if (p.out_pts)
                    reinterpret_cast<float2*>(p.out_pts)[pos] =
                        __ldcg(reinterpret_cast<const float2*>(p.pts) + i0 + 1);
            }
        }
    }
}

// One super-tile = kK2Sub sub-tiles of kK2SubPairs point pairs (128 KiB).
//   pass A(k):   stream + classify tile k, ballots and survivor list into
//                ts[k&1]; warp 0, once done with its share, resolves tile
//                k-1 (exclusive prefix by look-back, its predecessors published
//                long ago; publishes its inclusive prefix) while the other
//                warps finish; block scan; publish tile k's aggregate;
//   pass B(k-1): write tile k-1's survivors.
// The next tile's ticket is taken after pass A(k) and its first sub-tile is
// prefetched into registers before resolve/pass B.
template <bool VEC, int EDGES>
__global__ void __launch_bounds__(kK2Threads, 2) k2_filter(const __grid_constant__ K2Params p) {
    static_assert(kGroups == kK2Threads, "one scan entry per thread");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K2Smem& S = *reinterpret_cast<K2Smem*>(smem_raw);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned epoch = *(volatile unsigned*)&p.ws->epoch;

    load_geom_lite(S.geo, p.g, threadIdx.x, kK2Threads);
    if (threadIdx.x == 0) {
        S.done = 0u;
        S.next = atomicAdd(&p.ws->k2_ticket, 1u);
    }
    __syncthreads();
    const int mode = S.geo.mode;
    unsigned tile = S.next;
    unsigned pend = 0xffffffffu;   // super-tile awaiting resolve + pass B
    unsigned lb_rounds = 0, lb_spins = 0;   // look-back diagnostics of the warps that resolved
    float4 v[kK2Items];
    if (tile < p.num_tiles) {
#pragma unroll
        for (int u = 0; u < kK2Items; ++u)
            v[u] = load_pair<VEC>(p.pts, tile * kK2TilePairs + u * kK2Threads + threadIdx.x, p.n);
    }
    for (unsigned k = 0;; ++k) {
        const bool have = tile < p.num_tiles;
        TileState& cur = S.ts[k & 1];
        TileState& prv = S.ts[(k & 1) ^ 1];
        const unsigned tbase = tile * kK2TilePairs;
        if (have) {
            // ---------------- pass A
            const bool full_tile = mode == 0 && 2ull * (tbase + kK2TilePairs) <= (unsigned long long)p.n;
            unsigned wc = 0;
#pragma unroll 1
            for (int sub = 0; sub < kK2Sub; ++sub) {
                const unsigned qbase = tbase + sub * kK2SubPairs + threadIdx.x;
                float4 vn[kK2Items];
                if (sub + 1 < kK2Sub) {
#pragma unroll
                    for (int u = 0; u < kK2Items; ++u) {
                        const unsigned q = qbase + kK2SubPairs + u * kK2Threads;
                        vn[u] = (VEC && full_tile) ? ld_stream(reinterpret_cast<const float4*>(p.pts) + q)
                                                   : load_pair<VEC>(p.pts, q, p.n);
                    }
                }
                unsigned keep = 0u, needy = 0u;   // bit b = 2u + h
                if (full_tile) {
#pragma unroll
                    for (int u = 0; u < kK2Items; ++u) {
                        const unsigned in = (fast_inside(S.geo, v[u].x, v[u].y) ? 1u : 0u) |
                                            (fast_inside(S.geo, v[u].z, v[u].w) ? 2u : 0u);
                        needy |= (3u & ~in) << (2 * u);
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < kK2Items; ++u) {
                        const unsigned i0 = 2u * (qbase + u * kK2Threads);
                        const unsigned valid = (i0 < p.n ? 1u : 0u) | (i0 + 1u < p.n ? 2u : 0u);
                        if (mode == 1) {
                            keep |= valid << (2 * u);
                        } else {
                            const unsigned in =
                                (mode == 0 && fast_inside(S.geo, v[u].x, v[u].y) ? 1u : 0u) |
                                (mode == 0 && fast_inside(S.geo, v[u].z, v[u].w) ? 2u : 0u);
                            needy |= (valid & ~in) << (2 * u);
                        }
                    }
                }
                // Undecided points -> per-warp queue, tested with full lanes.
                // Survivors are always queued points (fast paths only discard),
                // so the survivor list is built here, in the queue pass.
                const unsigned nq = __popc(needy);
                unsigned incl = nq;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned y = __shfl_up_sync(kFull, incl, o);
                    if (lane >= (unsigned)o) incl += y;
                }
                const unsigned qtotal = __shfl_sync(kFull, incl, 31);
                if (qtotal) {
                    S.own[warp][lane] = 0;
                    unsigned j = incl - nq;
                    for (unsigned m = needy; m; m &= m - 1) {
                        const unsigned b = __ffs(m) - 1;
                        const float4 w = (b >> 1) == 0 ? v[0] : (b >> 1) == 1 ? v[1] : (b >> 1) == 2 ? v[2] : v[3];
                        S.qxy[warp][j] = (b & 1) ? make_float2(w.z, w.w) : make_float2(w.x, w.y);
                        S.qslot[warp][j] = (unsigned char)(lane * 8u + b);
                        ++j;
                    }
                    __syncwarp();
                    for (unsigned base = 0; base < qtotal; base += 32) {
                        const unsigned e = base + lane;
                        bool kp = false;
                        float2 q = make_float2(0.f, 0.f);
                        unsigned sl = 0;
                        if (e < qtotal) {
                            q = S.qxy[warp][e];
                            sl = S.qslot[warp][e];
                            kp = queue_keep<EDGES>(S.geo, q.x, q.y);
                        }
                        const unsigned kb = __ballot_sync(kFull, kp);
                        if (kp) {
                            const unsigned ol = sl >> 3, bb = sl & 7u, u = bb >> 1, h = bb & 1u;
                            atomicOr(reinterpret_cast<unsigned*>(&S.own[warp][ol & ~3u]),
                                     (1u << bb) << (8u * (ol & 3u)));
                            const unsigned r = wc + __popc(kb & lt);
                            if (r < kList) {
                                const unsigned g = (sub * kK2Items + u) * kK2Warps + warp;
                                cur.list[warp][r] = SurvEntry{
                                    q.x, q.y, 2u * (qbase - lane + ol + u * kK2Threads) + h,
                                    (g << 6) | (ol << 1) | h};
                            }
                        }
                        wc += __popc(kb);
                    }
                    __syncwarp();
                    keep |= S.own[warp][lane];
                }
                if (qtotal || mode == 1) {
#pragma unroll
                    for (int u = 0; u < kK2Items; ++u) {
                        const unsigned b0 = __ballot_sync(kFull, (keep >> (2 * u)) & 1u);
                        const unsigned b1 = __ballot_sync(kFull, (keep >> (2 * u + 1)) & 1u);
                        if (lane == 0) {
                            const unsigned g = (sub * kK2Items + u) * kK2Warps + warp;
                            cur.mask[g][0] = b0;
                            cur.mask[g][1] = b1;
                        }
                        if (mode == 1) wc += __popc(b0) + __popc(b1);   // list unused: dense pass B
                    }
                } else if (lane < kK2Items) {
                    const unsigned g = (sub * kK2Items + lane) * kK2Warps + warp;
                    cur.mask[g][0] = 0u;
                    cur.mask[g][1] = 0u;
                }
                if (sub + 1 < kK2Sub) {
#pragma unroll
                    for (int u = 0; u < kK2Items; ++u) v[u] = vn[u];
                }
            }
            if (lane == 0) cur.wcnt[warp] = (mode == 1) ? kList + 1u : wc;
            // the first warp done with its pass A resolves the pending
            // super-tile now, while the other warps finish theirs (its
            // aggregate went out a tile ago), rather than between two barriers
            // with every warp waiting
            unsigned first = 0;
            if (lane == 0) first = atomicAdd(&S.done, 1u) == 0u;
            first = __shfl_sync(kFull, first, 0);
            if (first && pend != 0xffffffffu) {   // resolve the pending super-tile (see above)
                unsigned long long ex = 0;
                if (pend != 0) {
                    ex = resolve(p, pend, epoch, lane, lb_rounds, lb_spins);
                    if (lane == 0) {
                        publish(p, pend, kFlagP, ex + prv.total, epoch);
                        if (pend == p.num_tiles - 1) p.ws->count = ex + prv.total;
                    }
                }
                if (lane == 0) S.prefix = ex;
            }
            // next ticket only now: a tile is never held while its block is busy
            if (threadIdx.x == 0) S.next = atomicAdd(&p.ws->k2_ticket, 1u);
            __syncthreads();
            // ---------------- block scan of the 256 group counts (group order = index order)
            {
                const unsigned c = __popc(cur.mask[threadIdx.x][0]) + __popc(cur.mask[threadIdx.x][1]);
                unsigned incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned y = __shfl_up_sync(kFull, incl, o);
                    if (lane >= (unsigned)o) incl += y;
                }
                if (lane == 31) S.wsum[warp] = incl;
                __syncthreads();
                unsigned wpre = 0, total = 0;
#pragma unroll
                for (int w = 0; w < kK2Warps; ++w) {
                    const unsigned x = S.wsum[w];
                    wpre += (w < (int)warp) ? x : 0u;
                    total += x;
                }
                cur.off[threadIdx.x] = wpre + incl - c;
                if (threadIdx.x == 0) {
                    S.done = 0u;   // (counted again after the coming barriers)
                    cur.total = total;
                    if (tile == 0) {   // first tile: its inclusive prefix is known now
                        publish(p, 0, kFlagP, total, epoch);
                        if (p.num_tiles == 1) p.ws->count = total;
                    } else {
                        publish(p, tile, kFlagA, total, epoch);
                    }
                }
            }
        } else {
            if (warp == 0 && pend != 0xffffffffu) {   // resolve the pending super-tile (see above)
                unsigned long long ex = 0;
                if (pend != 0) {
                    ex = resolve(p, pend, epoch, lane, lb_rounds, lb_spins);
                    if (lane == 0) {
                        publish(p, pend, kFlagP, ex + prv.total, epoch);
                        if (pend == p.num_tiles - 1) p.ws->count = ex + prv.total;
                    }
                }
                if (lane == 0) S.prefix = ex;
            }
            if (threadIdx.x == 0) S.next = 0xffffffffu;
        }
        __syncthreads();
        const unsigned next = have ? S.next : 0xffffffffu;
        if (next < p.num_tiles) {   // prefetch the next super-tile's first sub-tile
#pragma unroll
            for (int u = 0; u < kK2Items; ++u)
                v[u] = load_pair<VEC>(p.pts, next * kK2TilePairs + u * kK2Threads + threadIdx.x, p.n);
        }
        // ---------------- pass B of the pending super-tile (resolved by warp 0 above)
        if (pend != 0xffffffffu) emit(p, prv, pend * kK2TilePairs, S.prefix, warp, lane, lt);
        __syncthreads();   // prv is reused by the next pass A
        if (!have) break;
        pend = tile;
        tile = next;
    }
    // last block out resets the ticket and bumps the epoch (all blocks have
    // read `epoch` and taken their final ticket before incrementing k2_done)
    if (lane == 0) {   // (any warp may have resolved some super-tiles)
        if (lb_rounds) atomicAdd(&p.ws->lb_rounds, lb_rounds);
        if (lb_spins) atomicAdd(&p.ws->lb_spins, lb_spins);
    }
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
    static std::once_flag once[kMaxDevices];
    static int cap[kMaxDevices];
    const int smem = (int)sizeof(K2Smem);
    const int max_blocks = per_device(once, cap, [&] {
        cudaFuncSetAttribute(k2_filter<VEC, EDGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2_filter<VEC, EDGES>, kK2Threads, smem);
        return (per_sm > 0 ? per_sm : 1) * device_sm_count();
    });
    unsigned blocks = p.num_tiles < (unsigned)max_blocks ? p.num_tiles : (unsigned)max_blocks;
    if (blocks < 1) blocks = 1;
    k2_filter<VEC, EDGES><<<blocks, kK2Threads, smem, s>>>(p);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace

// 16-B aligned input: the warp-specialised TMA-ring kernel (handles every ring
// mode); 8-B aligned input: this register-loading kernel.
int launch_filter(const K2Params& p, int vec16, void* stream, int* launches) {
    if (vec16) return launch_filter_tma(p, stream, launches);
    cudaStream_t s = (cudaStream_t)stream;
    if (p.edges <= 16) return (int)launch_t<false, 16>(p, s, launches);
    return (int)launch_t<false, 32>(p, s, launches);
}

}  // namespace cudapre
