// k2_filter_tma.cu — Step 3 of CudaPre (§2 Step 3; SPEC.md
// S:156-164), TMA-ring variant for 16-byte aligned input (mode 0).
//
// Same classification and ordered compaction as k2_filter.cu (see its header
// and DESIGN.md §6.2), but the points never pass through registers on their
// way in: one elected thread streams 16 KiB sub-tiles global -> shared with
// cp.async.bulk (SASS UBLKCP) into a kNst-deep ring of stages, each guarded by
// a transaction-counting "full" mbarrier and a per-warp "empty" mbarrier.
// Warps read their 8 points per sub-tile with LDS.128; undecided points are
// queued as 1-byte slots that point back into the stage, so the queue pass,
// the survivor list and the coordinates all come from shared memory.
//
// Per super-tile (8 sub-tiles, 128 KiB, one ticket):
//   pass A(k)    classify, queue, ballots + survivor list into ts[k&1];
//                block scan; publish the aggregate (tile 0: its prefix);
//   resolve(k-1) decoupled look-back one tile-time later (no spinning);
//   pass B(k-1)  write the survivors' int64 indices + float2 points.
// The producer takes the next super-tile's ticket when the ring first needs
// it (sub-tile 8 - kNst + 1 of pass A) so loads never stall at the boundary.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "k2_common.cuh"
#include "tma.cuh"

namespace cudapre {
namespace {

constexpr int kW = kK2Threads / 32;                  // 8 warps
constexpr int kG = kK2Sub * kK2Items * kW;           // 256 ballot groups per super-tile
constexpr unsigned kNone = 0xffffffffu;
constexpr unsigned kProd = kK2Threads - 32;          // producer thread: lane 0 of the last warp

struct SurvT {
    float x, y;
    unsigned meta;   // (group << 6) | (owner lane << 1) | pair element
};

template <unsigned kL>
struct TileT {
    unsigned mask[kG][2];   // keep ballots, group g = (sub*kK2Items + u)*kW + warp
    unsigned off[kG];       // exclusive offset of each group inside the super-tile
    unsigned wcnt[kW];      // survivors per warp
    unsigned total;
    SurvT list[kW][kL];
};

template <int kNst, unsigned kL>
struct SmemT {
    float4 ring[kNst][kK2SubPairs];
    unsigned long long full[kNst];
    unsigned long long empty[kNst];
    TileT<kL> ts[2];
    unsigned char qslot[kW][2 * kK2Items * 32];
    unsigned char own[kW][32];
    float sr2[CUDAPRE_SECTORS + 1];    // sector inner radii^2 (copied from the parameters;
    float sro2[CUDAPRE_SECTORS + 1];   // divergent parameter-space reads serialise)
    unsigned wsum[kW];
    unsigned next;
    unsigned long long prefix;
};

// Sector test: pseudo-angle bucket of p around (ox, oy) by
// one approximate reciprocal; strictly inside if |p - o|^2 < sr2[bucket].
// The host's buckets carry a 1/64-bucket guard band, far above the bucket
// error of this arithmetic (< 2^-12 bucket); NaN/Inf map to a clamped bucket
// and fail the comparison.
__device__ __forceinline__ float rcp_approx(float a) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    return r;
}
// 0 = strictly inside, 1 = strictly outside, 2 = undecided
__device__ __forceinline__ int sector_class(const float* sr2, const float* sro2, float x, float y,
                                            float ox, float oy) {
    const float2 d = __fadd2_rn(make_float2(x, y), make_float2(-ox, -oy));
    const float2 q = __fmul2_rn(d, d);
    const float d2 = __fadd_rn(q.x, q.y);
    const float t = __fmul_rn(d.y, rcp_approx(__fadd_rn(fabsf(d.x), fabsf(d.y))));
    const bool pos = d.x >= 0.0f;
    const float v = __fmaf_rn(t, pos ? 256.0f : -256.0f, pos ? 8388864.0f : 8389376.0f);   // 2^23 + 256 pa
    const unsigned b = min(__float_as_uint(v) - 0x4B000000u, (unsigned)CUDAPRE_SECTORS);
    return d2 < sr2[b] ? 0 : (d2 > sro2[b] ? 1 : 2);
}

// global point index of a survivor entry
__device__ __forceinline__ unsigned entry_index(unsigned tbase, unsigned meta) {
    const unsigned g = meta >> 6, ol = (meta >> 1) & 31u, h = meta & 1u;
    const unsigned q = tbase + (g >> 5) * kK2SubPairs + ((g >> 3) & 3u) * kK2Threads + (g & 7u) * 32u + ol;
    return 2u * q + h;
}

template <unsigned kL>
__device__ __forceinline__ void emit_t(const K2Params& p, const TileT<kL>& ts, unsigned tbase,
                                       unsigned long long ex, unsigned warp, unsigned lane,
                                       unsigned lt) {
    const unsigned wc = ts.wcnt[warp];
    if (wc <= kL) {
        for (unsigned r = lane; r < wc; r += 32) {
            const SurvT e = ts.list[warp][r];
            const unsigned g = e.meta >> 6, ol = (e.meta >> 1) & 31u, h = e.meta & 1u;
            const unsigned m0 = ts.mask[g][0], m1 = ts.mask[g][1], olt = (1u << ol) - 1u;
            const unsigned rig = __popc(m0 & olt) + __popc(m1 & olt) + (h ? ((m0 >> ol) & 1u) : 0u);
            const unsigned long long pos = ex + ts.off[g] + rig;
            if (pos < p.capacity) {
                p.out_idx[pos] = p.base + (long long)entry_index(tbase, e.meta);
                if (p.out_pts) reinterpret_cast<float2*>(p.out_pts)[pos] = make_float2(e.x, e.y);
            }
        }
        return;
    }
    // dense (list overflow): every group of this warp, coordinates re-read (L2)
#pragma unroll 1
    for (int sub = 0; sub < kK2Sub; ++sub) {
#pragma unroll
        for (int u = 0; u < kK2Items; ++u) {
            const int g = (sub * kK2Items + u) * kW + warp;
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

// bytes of full point pairs of sub-tile `sub` of super-tile `tile` in memory
__device__ __forceinline__ unsigned sub_bytes(unsigned tile, unsigned sub, unsigned full_pairs) {
    const unsigned qs = tile * kK2TilePairs + sub * kK2SubPairs;
    if (qs >= full_pairs) return 0u;
    const unsigned np = full_pairs - qs;
    return (np >= (unsigned)kK2SubPairs ? (unsigned)kK2SubPairs : np) * 16u;
}

// CFG 0: 4-stage ring, 128-entry lists, 2 blocks/SM (default);
// CFG 1: 3-stage ring, 64-entry lists, 3 blocks/SM (<= 85 registers).
template <int CFG> struct K2Cfg;
template <> struct K2Cfg<0> { static constexpr int kNst = 4; static constexpr unsigned kL = 128; static constexpr int kMinB = 2; };
template <> struct K2Cfg<1> { static constexpr int kNst = 3; static constexpr unsigned kL = 64; static constexpr int kMinB = 3; };

template <int EDGES, int CFG>
__global__ void __launch_bounds__(kK2Threads, K2Cfg<CFG>::kMinB) k2_filter_tma(const __grid_constant__ K2Params p) {
    static_assert(kG == kK2Threads, "one scan entry per thread");
    constexpr int kNst = K2Cfg<CFG>::kNst;
    constexpr unsigned kL = K2Cfg<CFG>::kL;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SmemT<kNst, kL>& S = *reinterpret_cast<SmemT<kNst, kL>*>(smem_raw);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned epoch = *(volatile unsigned*)&p.ws->epoch;
    const unsigned full_pairs = p.n / 2u;
    const bool odd = (p.n & 1u) != 0u;
    const float4* src = reinterpret_cast<const float4*>(p.pts);

    // producer state (thread 0 only)
    unsigned issued = 0, pk = 0, ptile = kNone, pnext = kNone;
    auto produce = [&](unsigned upto) {   // issue sequences < upto
        while (issued < upto) {
            const unsigned kk = issued / kK2Sub;
            unsigned t;
            if (kk == pk) {
                t = ptile;
            } else {   // kk == pk + 1: the next super-tile, ticket taken on first need
                if (pnext == kNone) {
                    pnext = atomicAdd(&p.ws->k2_ticket, 1u);
                    S.next = pnext;
                }
                t = pnext;
            }
            if (t >= p.num_tiles) return;
            const unsigned bytes = sub_bytes(t, issued % kK2Sub, full_pairs);
            if (bytes == 0u) return;
            const unsigned st = issued % kNst;
            if (issued >= (unsigned)kNst) mbar_wait(&S.empty[st], ((issued / kNst) - 1u) & 1u);
            mbar_expect_tx(&S.full[st], bytes);
            bulk_g2s(&S.ring[st][0], src + (size_t)t * kK2TilePairs + (issued % kK2Sub) * kK2SubPairs,
                     bytes, &S.full[st]);
            ++issued;
        }
    };

    const float ox = p.ox, oy = p.oy;
    for (int i = threadIdx.x; i <= CUDAPRE_SECTORS; i += kK2Threads) {
        S.sr2[i] = p.sr2[i];
        S.sro2[i] = p.sro2[i];
    }
    if (threadIdx.x == kProd) {
        for (int k = 0; k < kNst; ++k) {
            mbar_init(&S.full[k], 1u);
            mbar_init(&S.empty[k], (unsigned)kW);
        }
        mbar_fence_init();
        ptile = atomicAdd(&p.ws->k2_ticket, 1u);
        S.next = ptile;
        produce(kNst);
    }
    __syncthreads();
    unsigned tile = S.next;
    unsigned pend = kNone;
    unsigned lb_rounds = 0, lb_spins = 0;   // warp 0's look-back diagnostics
    for (unsigned k = 0;; ++k) {
        const bool have = tile < p.num_tiles;
        TileT<kL>& cur = S.ts[k & 1];
        TileT<kL>& prv = S.ts[(k & 1) ^ 1];
        const unsigned tbase = tile * kK2TilePairs;
        if (have) {
            // ---------------- pass A
            unsigned wc = 0;
#pragma unroll 1
            for (int sub = 0; sub < kK2Sub; ++sub) {
                const unsigned seq = k * kK2Sub + sub;
                const unsigned qs = tbase + sub * kK2SubPairs;
                const unsigned bytes = sub_bytes(tile, sub, full_pairs);
                const unsigned npairs_here = bytes / 16u;
                if (threadIdx.x == kProd) produce(seq + kNst);
                const float4* stg = S.ring[seq % kNst];
                if (bytes) mbar_wait(&S.full[seq % kNst], (seq / kNst) & 1u);
                unsigned needy = 0u;   // bit b = 2u + h
                if (p.debug == 1) {   // perf experiment only: skeleton, no classification
#pragma unroll
                    for (int u = 0; u < kK2Items; ++u) {
                        const float4 v = stg[u * kK2Threads + threadIdx.x];
                        needy |= (v.x == 12345.0f ? 1u : 0u) << (2 * u);
                    }
                } else if (npairs_here == (unsigned)kK2SubPairs) {
#pragma unroll
                    for (int u = 0; u < kK2Items; ++u) {
                        const float4 v = stg[u * kK2Threads + threadIdx.x];
                        const unsigned in = (fast_inside(p, v.x, v.y) ? 1u : 0u) | (fast_inside(p, v.z, v.w) ? 2u : 0u);
                        needy |= (3u & ~in) << (2 * u);
                    }
                } else {   // last super-tile only: ragged end
#pragma unroll
                    for (int u = 0; u < kK2Items; ++u) {
                        const unsigned pr = u * kK2Threads + threadIdx.x;
                        const unsigned q = qs + pr;
                        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                        unsigned valid = 0u;
                        if (pr < npairs_here) {
                            v = stg[pr];
                            valid = 3u;
                        } else if (odd && q == full_pairs) {
                            const float2 a = __ldg(reinterpret_cast<const float2*>(p.pts) + 2u * q);
                            v = make_float4(a.x, a.y, 0.f, 0.f);
                            valid = 1u;
                        }
                        const unsigned in = (fast_inside(p, v.x, v.y) ? 1u : 0u) | (fast_inside(p, v.z, v.w) ? 2u : 0u);
                        needy |= (valid & ~in) << (2 * u);
                    }
                }
                // undecided points -> per-warp queue of slots into the stage
                const unsigned nq = __popc(needy);
                unsigned incl = nq;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned y = __shfl_up_sync(kFull, incl, o);
                    if (lane >= (unsigned)o) incl += y;
                }
                const unsigned qtotal = __shfl_sync(kFull, incl, 31);
                unsigned keep = 0u;
                if (qtotal) {
                    S.own[warp][lane] = 0;
                    unsigned j = incl - nq;
#pragma unroll
                    for (int b = 0; b < 2 * kK2Items; ++b) {   // converged, predicated stores
                        if ((needy >> b) & 1u) S.qslot[warp][j] = (unsigned char)(lane * 8u + b);
                        j += (needy >> b) & 1u;
                    }
                    __syncwarp();
                    for (unsigned base = 0; base < qtotal; base += 32) {
                        const unsigned e = base + lane;
                        bool kp = false;
                        float2 q = make_float2(0.f, 0.f);
                        unsigned sl = 0;
                        if (e < qtotal) {
                            sl = S.qslot[warp][e];
                            const unsigned ol = sl >> 3, b = sl & 7u;
                            const unsigned pr = (b >> 1) * kK2Threads + warp * 32u + ol;
                            if (pr < npairs_here) {
                                const float4* cell = &stg[pr];
                                q = (b & 1u) ? make_float2(cell->z, cell->w) : make_float2(cell->x, cell->y);
                            } else {   // the unpaired last point
                                q = __ldg(reinterpret_cast<const float2*>(p.pts) + 2u * (qs + pr));
                            }
                            const int sc = sector_class(S.sr2, S.sro2, q.x, q.y, ox, oy);
                            kp = sc == 1 || (sc == 2 && queue_keep<EDGES>(p, q.x, q.y));
                        }
                        const unsigned kb = __ballot_sync(kFull, kp);
                        if (kp) {
                            const unsigned ol = sl >> 3, b = sl & 7u;
                            atomicOr(reinterpret_cast<unsigned*>(&S.own[warp][ol & ~3u]), (1u << b) << (8u * (ol & 3u)));
                            const unsigned r = wc + __popc(kb & lt);
                            if (r < kL) {
                                const unsigned g = (sub * kK2Items + (b >> 1)) * kW + warp;
                                cur.list[warp][r] = SurvT{q.x, q.y, (g << 6) | (ol << 1) | (b & 1u)};
                            }
                        }
                        wc += __popc(kb);
                    }
                    __syncwarp();
                    keep = S.own[warp][lane];
#pragma unroll
                    for (int u = 0; u < kK2Items; ++u) {
                        const unsigned b0 = __ballot_sync(kFull, (keep >> (2 * u)) & 1u);
                        const unsigned b1 = __ballot_sync(kFull, (keep >> (2 * u + 1)) & 1u);
                        if (lane == 0) {
                            const unsigned g = (sub * kK2Items + u) * kW + warp;
                            cur.mask[g][0] = b0;
                            cur.mask[g][1] = b1;
                        }
                    }
                } else if (lane < (unsigned)kK2Items) {
                    const unsigned g = (sub * kK2Items + lane) * kW + warp;
                    cur.mask[g][0] = 0u;
                    cur.mask[g][1] = 0u;
                }
                __syncwarp();
                if (bytes && lane == 0) mbar_arrive(&S.empty[seq % kNst]);
            }
            if (lane == 0) cur.wcnt[warp] = wc;
            if (threadIdx.x == kProd) {
                if (pnext == kNone) {   // short last tile: ticket not taken yet
                    pnext = atomicAdd(&p.ws->k2_ticket, 1u);
                    S.next = pnext;
                }
                // refill the stage just released so the ring stays full through
                // the scan / look-back / pass B that follow
                produce((k + 1) * kK2Sub + kNst);
            }
        }
        __syncthreads();   // pass A done everywhere
        const unsigned next = have ? S.next : kNone;
        unsigned c = 0, inc = 0;
        if (have) {   // block scan of the 256 group counts (group order = index order)
            c = __popc(cur.mask[threadIdx.x][0]) + __popc(cur.mask[threadIdx.x][1]);
            inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(kFull, inc, o);
                if (lane >= (unsigned)o) inc += y;
            }
            if (lane == 31) S.wsum[warp] = inc;
        }
        __syncthreads();
        if (have) {   // offsets + publish this tile's aggregate (tile 0: its prefix)
            unsigned wpre = 0, total = 0;
#pragma unroll
            for (int w = 0; w < kW; ++w) {
                const unsigned x = S.wsum[w];
                wpre += (w < (int)warp) ? x : 0u;
                total += x;
            }
            cur.off[threadIdx.x] = wpre + inc - c;
            if (threadIdx.x == 0) {
                cur.total = total;
                if (tile == 0) {
                    publish(p, 0, kFlagP, total, epoch);
                    if (p.num_tiles == 1) p.ws->count = total;
                } else {
                    publish(p, tile, kFlagA, total, epoch);
                }
            }
        }
        // ---------------- resolve + pass B of the pending super-tile: one
        // tile-time after its aggregate was published, so its predecessors
        // have published theirs (no spinning); the next super-tile's first
        // sub-tiles are already in flight in the ring.
        if (pend != kNone) {
            if (warp == 0) {
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
            __syncthreads();
            emit_t(p, prv, pend * kK2TilePairs, S.prefix, warp, lane, lt);
        }
        __syncthreads();   // prv is reused by the next pass A
        if (!have) break;
        pend = tile;
        tile = next;
        if (threadIdx.x == kProd) {   // producer moves to the next super-tile
            pk += 1;
            ptile = pnext;
            pnext = kNone;
        }
    }
    if (threadIdx.x == 0) {
        if (lb_rounds) atomicAdd(&p.ws->lb_rounds, lb_rounds);
        if (lb_spins) atomicAdd(&p.ws->lb_spins, lb_spins);
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

template <int EDGES, int CFG>
cudaError_t launch_tma_t(const K2Params& p, cudaStream_t s, int* launches) {
    static int max_blocks = 0;
    const int smem = (int)sizeof(SmemT<K2Cfg<CFG>::kNst, K2Cfg<CFG>::kL>);
    if (!max_blocks) {
        cudaFuncSetAttribute(k2_filter_tma<EDGES, CFG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2_filter_tma<EDGES, CFG>, kK2Threads, smem);
        max_blocks = (per_sm > 0 ? per_sm : 1) * device_sm_count();
    }
    unsigned blocks = p.num_tiles < (unsigned)max_blocks ? p.num_tiles : (unsigned)max_blocks;
    if (blocks < 1) blocks = 1;
    k2_filter_tma<EDGES, CFG><<<blocks, kK2Threads, smem, s>>>(p);
    ++*launches;
    return cudaGetLastError();
}

int k2_cfg() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("CUDAPRE_K2_CFG");
        v = e ? atoi(e) : 0;
        if (v < 0 || v > 1) v = 0;
    }
    return v;
}

}  // namespace

int launch_filter_tma(const K2Params& p, void* stream, int* launches) {
    cudaStream_t s = (cudaStream_t)stream;
    if (k2_cfg() == 1)
        return p.nv <= 16 ? (int)launch_tma_t<16, 1>(p, s, launches) : (int)launch_tma_t<32, 1>(p, s, launches);
    return p.nv <= 16 ? (int)launch_tma_t<16, 0>(p, s, launches) : (int)launch_tma_t<32, 0>(p, s, launches);
}

}  // namespace cudapre
