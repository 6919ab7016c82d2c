// k2_filter_tma.cu — Step 3 of CudaPre (§2 Step 3; SPEC.md
// S:156-164), TMA-ring variant for 16-byte aligned input (mode 0).
//
// Same classification and ordered compaction contract as k2_filter.cu (see
// its header and DESIGN.md §6.2), organised so that the common path costs as
// few instructions per point as possible:
//
//  * Warp roles (kW compute warps + 2): a PRODUCER warp (lane 0) takes
//    super-tile tickets (the next one while issuing the current one) and
//    streams 16 KiB sub-tiles global -> shared with cp.async.bulk (SASS
//    UBLKCP) into a kNst-deep ring guarded by a transaction-counting "full"
//    mbarrier and an "empty" mbarrier the compute warps release; an EMIT warp
//    does the ordered compaction's bookkeeping (group scan, look-back,
//    publish) and writes the survivors; the compute warps classify (and
//    write their own lists when the emit warp falls behind).  After set-up
//    there is no block barrier.
//  * Ownership: compute warp w owns the contiguous 256 points [256w, 256w+256)
//    of each sub-tile, lane l the eight points 8l..8l+7 (four float4 pairs,
//    read in a rotated order that keeps LDS.128 conflict-free).  The groups of
//    the ordered compaction are the 8 * kW (sub-tile, warp) chunks, in index
//    order.
//  * Pass A: one fast test per point (inner disk or inner box, whichever the
//    host found larger; a warp-uniform switch).  Points it cannot decide are
//    queued in INDEX order (lane prefix of the per-lane counts by four
//    bit-sliced ballots, then each lane writes its own), so the per-warp
//    survivor list comes out sorted and a survivor's rank inside its group is
//    its list position minus the group's start: no per-group ballots.
//  * Queue pass: sector table (inner/outer radius of the bucket), then for
//    the thin undecided band the 1-2 edges the bucket's rays can exit through
//    (coefficients in shared memory), then the exact predicate.  Survivors go
//    to a per-warp list of the super-tile's buffer (triple-buffered; a list
//    that overflows spills to the block's global scratch).
//  * Per super-tile k: each compute warp signals "tile done"; the last one
//    publishes the tile's aggregate (a packed shared-memory atomic of warps
//    done and survivor total).  The emit warp then scans the 8 * kW group
//    counts of k, resolves the PREVIOUS super-tile's prefix (decoupled
//    look-back one tile-time after its aggregate went out: no spinning),
//    publishes its inclusive prefix, posts the exclusive one ("resolved")
//    and writes the survivors (index + float2) list by list.  A compute warp
//    that needs its list buffer back (three tiles later) before the emit warp
//    got to its list claims the list and writes it itself, so dense inputs
//    are written by all warps, sparse ones off the compute warps' path.
#include <cuda_runtime.h>

#include <cstdint>

#include "k2_common.cuh"
#include "tma.cuh"

namespace cudapre {
namespace {

// kW compute warps per block.  A warp chunk is always 256 points; a sub-tile
// is kW chunks, a super-tile 8 sub-tiles.  (10 compute warps measured the
// same as 8, profiles/r01_experiments.md, and round 2 at 2 blocks/SM with
// 80 registers: no better, r02_experiments.md.)
constexpr int kW = 8;
constexpr int kGroups = kK2Sub * kW;                 // groups (sub, warp) per super-tile
constexpr unsigned kChunkPairs = 128;                // 256 points per warp chunk
constexpr unsigned kSubPairsT = kW * kChunkPairs;    // pairs per sub-tile (16 KiB at 8 warps)
constexpr unsigned kTilePairsT = kK2Sub * kSubPairsT;
constexpr int kGroupsPerLane = (kGroups + 31) / 32;
constexpr unsigned kNone = 0xffffffffu;
constexpr unsigned kBlock = kW * 32 + 64;            // compute warps + producer warp + emit warp
constexpr unsigned kProdWarp = kW, kEmitWarp = kW + 1;
constexpr int kBufs = kK2Bufs;                       // survivor-list buffers (tiles in flight)

// 4-stage ring, 96-entry lists (~110 KB of shared memory, 2 blocks per SM).
// Overflowing lists spill to global scratch, so the list size only trades
// shared memory for traffic (a 3-stage ring with 128-entry lists measured the
// same, profiles/r01_experiments.md).
constexpr int kNst = 4;
constexpr unsigned kL = 96;

using SurvT = SurvEntry;   // meta = (sub << 8) | loc, loc = 8*lane + k = point offset in the warp chunk
static_assert(kK2Bufs == 3 && kK2WarpPts == kK2Sub * 2 * (int)kChunkPairs && kW <= kK2MaxWarps, "layout");

struct TileT {
    SurvT list[kW][kL];                 // per-warp survivors in index order
    unsigned lstart[kW][kK2Sub + 1];    // list position where (warp, sub) starts; [kK2Sub] = total
    unsigned off[kGroups];              // exclusive offset of group sub*kW + warp in the super-tile
    unsigned total;
    unsigned tile;                      // super-tile id (kNone: end of work)
    unsigned long long ex;              // exclusive prefix of the super-tile (emit warp -> compute warps)
};

struct SmemT {
    float4 ring[kNst][kSubPairsT];
    unsigned long long full[kNst];
    unsigned long long empty[kNst];
    TileT ts[kBufs];
    unsigned long long tile_done[kBufs];   // compute warps -> emit warp (count kW)
    unsigned long long resolved[kBufs];    // emit warp -> compute warps: off[] and ex are ready (count 1)
    unsigned claim[kBufs][kW];             // list (buffer, warp) of local tile j claimed for writing: j + 1
    unsigned emitted[kBufs][kW];           // ... written by the emit warp: j + 1
    unsigned long long agg[kBufs];         // (compute warps done << 32) | survivors so far
    unsigned char qslot[kW][8 * 32];
    float2 sec[CUDAPRE_SECTORS + 1];               // {inner r^2, outer r^2} per bucket
    unsigned short sedge[CUDAPRE_SECTORS + 1];     // candidate exit edges per bucket
    float4 edge[CUDAPRE_MAX_SLOTS];                // {A, B, C', 0} (C' already lowered by E_j)
    GeomLite geo;                                  // scalars, coefficients, ring (rare paths)
    unsigned stile[kNst];   // super-tile id of the sub-tile-0 stage (kNone = end)
};

__device__ __forceinline__ unsigned ld_acquire_s(const unsigned* a) {
    unsigned v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(a)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_s(unsigned* a, unsigned v) {
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(a)), "r"(v) : "memory");
}
// warp-uniform: did this warp win list (b, w) of local tile tag - 1?
__device__ __forceinline__ bool claim_list(unsigned* c, unsigned tag, unsigned lane) {
    unsigned won = 0;
    if (lane == 0) won = atomicMax(c, tag) < tag;
    return __shfl_sync(kFull, won, 0) != 0u;
}

__device__ __forceinline__ float rcp_approx(float a) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    return r;
}

// Keep decision for a point the pass-A test could not decide (true = keep).
// Sector test: pseudo-angle bucket of p around (ox, oy) by one
// approximate reciprocal; strictly inside if |p - o|^2 < inner[b], strictly
// outside if > outer[b] (the host's buckets carry a 1/64-bucket guard band,
// far above this arithmetic's bucket error < 2^-12).  In between, p's ray exits
// through one of the bucket's candidate edges, so "inside" = inside those
// edges; float lines with the error margin E_j folded into C' decide unless
// |g| is within 2 Emax, then the exact predicate over the whole ring.
// Mode 1 (degenerate ring: keep everything) and mode 2 (coefficients out of
// float range: exact predicate only) take the uniform early exits.
template <int EDGES>
__device__ __forceinline__ bool classify_queued(const SmemT& S, int mode, float ox, float oy,
                                                float e2max, float x, float y) {
    if (mode != 0) return mode == 1 ? true : !exact_inside(S.geo, x, y);
    const float2 d = __fadd2_rn(make_float2(x, y), make_float2(-ox, -oy));
    const float2 q = __fmul2_rn(d, d);
    const float d2 = __fadd_rn(q.x, q.y);
    const float t = __fmul_rn(d.y, rcp_approx(__fadd_rn(fabsf(d.x), fabsf(d.y))));
    const bool pos = d.x >= 0.0f;
    const float v = __fmaf_rn(t, pos ? 256.0f : -256.0f, pos ? 8388864.0f : 8389376.0f);   // 2^23 + 256 pa
    const unsigned b = min(__float_as_uint(v) - 0x4B000000u, (unsigned)CUDAPRE_SECTORS);
    const float2 rr = S.sec[b];
    if (d2 < rr.x) return false;
    if (d2 > rr.y) return true;
    const unsigned se = S.sedge[b];
    if (se == 0xffffu) return queue_keep_rare<EDGES>(S.geo, x, y);
    const float4 e0 = S.edge[se & 0xffu], e1 = S.edge[se >> 8];
    const float mn = fminf(__fmaf_rn(e0.x, x, __fmaf_rn(e0.y, y, e0.z)),
                           __fmaf_rn(e1.x, x, __fmaf_rn(e1.y, y, e1.z)));
    if (mn > 0.0f) return false;
    if (__fadd_rn(mn, e2max) < 0.0f) return true;
    return !exact_inside(S.geo, x, y);
}

// inner box, closed (proven strictly inside by the builder)
__device__ __forceinline__ bool in_box(float bx0, float bx1, float by0, float by1, float x, float y) {
    return (x >= bx0) & (x <= bx1) & (y >= by0) & (y <= by1);
}
// inner disk: RN(RN(dx^2) + RN(dy^2)) < r2 (DESIGN.md §6.2 bound)
__device__ __forceinline__ bool in_disk(float ox, float oy, float r2, float x, float y) {
    const float2 d = __fadd2_rn(make_float2(x, y), make_float2(-ox, -oy));
    const float2 d2 = __fmul2_rn(d, d);
    return __fadd_rn(d2.x, d2.y) < r2;
}

// bytes of full point pairs of sub-tile `sub` of super-tile `tile` in memory
__device__ __forceinline__ unsigned sub_bytes(unsigned tile, unsigned sub, unsigned full_pairs) {
    const unsigned qs = tile * kTilePairsT + sub * kSubPairsT;
    if (qs >= full_pairs) return 0u;
    const unsigned np = full_pairs - qs;
    return (np >= (unsigned)kSubPairsT ? (unsigned)kSubPairsT : np) * 16u;
}

// point index (relative to the super-tile) of chunk offset loc of (sub, warp)
__device__ __forceinline__ unsigned chunk_point(unsigned sub, unsigned warp, unsigned loc) {
    return sub * (2u * kSubPairsT) + warp * (2u * kChunkPairs) + loc;
}

// compute warp `warp` writes its own survivors of super-tile `tile` from the
// tile's exclusive prefix ex: list entries [0, kL) from shared memory, the
// overflow [kL, wc) from the warp's global scratch (written by this warp's
// lanes before a __syncwarp)
template <int kU>
__device__ __forceinline__ void emit_t(const K2Params& p, const TileT& ts, const SurvT* ovf, unsigned tile,
                                       unsigned long long ex, unsigned warp, unsigned lane) {
    const unsigned long long tpt = (unsigned long long)tile * (2u * kTilePairsT);
    float2* out_pts = reinterpret_cast<float2*>(p.out_pts);
    const unsigned wc = ts.lstart[warp][kK2Sub];
    for (unsigned r0 = 0; r0 < wc; r0 += 32 * kU) {
        SurvT e[kU];
#pragma unroll
        for (int k = 0; k < kU; ++k) {
            const unsigned r = r0 + 32u * k + lane;
            if (r < wc) {
                if (r < kL) {
                    e[k] = ts.list[warp][r];
                } else {
                    const SurvT* q = ovf + (r - kL);
                    e[k].x = __ldcg(&q->x);
                    e[k].y = __ldcg(&q->y);
                    e[k].meta = __ldcg(&q->meta);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < kU; ++k) {
            const unsigned r = r0 + 32u * k + lane;
            if (r >= wc) break;
            const unsigned sub = e[k].meta >> 8, loc = e[k].meta & 0xffu;
            const unsigned long long pos = ex + ts.off[sub * kW + warp] + (r - ts.lstart[warp][sub]);
            if (pos < p.capacity) {
                p.out_idx[pos] = p.base + (long long)(tpt + chunk_point(sub, warp, loc));
                if (out_pts) out_pts[pos] = make_float2(e[k].x, e[k].y);
            }
        }
    }
}


template <int EDGES>
__global__ void __launch_bounds__(kBlock, 2) k2_filter_tma(const __grid_constant__ K2Params p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SmemT& S = *reinterpret_cast<SmemT*>(smem_raw);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned epoch = *(volatile unsigned*)&p.ws->epoch;
    const unsigned full_pairs = p.n / 2u;
    const bool odd = (p.n & 1u) != 0u;
    // list-overflow scratch of (this block, buffer b, warp w): sbase + (b*kW + w)*kK2WarpPts
    SurvT* const sbase = p.scratch + (size_t)blockIdx.x * (kBufs * kW * kK2WarpPts);

    for (int i = threadIdx.x; i <= CUDAPRE_SECTORS; i += kBlock) {
        S.sec[i] = make_float2(p.g->sr2[i], p.g->sro2[i]);
        S.sedge[i] = p.g->sedge[i];
    }
    if (threadIdx.x < (unsigned)CUDAPRE_MAX_SLOTS)
        S.edge[threadIdx.x] = make_float4(p.g->A[threadIdx.x], p.g->B[threadIdx.x], p.g->C[threadIdx.x], 0.0f);
    load_geom_lite(S.geo, p.g, threadIdx.x, kBlock);
    if (threadIdx.x == 0) {
        for (int k = 0; k < kNst; ++k) {
            mbar_init(&S.full[k], 1u);
            mbar_init(&S.empty[k], (unsigned)kW);
        }
        for (int k = 0; k < kBufs; ++k) {
            mbar_init(&S.tile_done[k], (unsigned)kW);
            mbar_init(&S.resolved[k], 1u);
            for (int w = 0; w < kW; ++w) S.claim[k][w] = S.emitted[k][w] = 0u;
            S.agg[k] = 0ull;
        }
        mbar_fence_init();
    }
    __syncthreads();   // the only whole-block barrier
    // shared-window addresses of the mbarriers and the ring (hot loops use these)
    const unsigned a_full = smem_u32(&S.full[0]), a_empty = smem_u32(&S.empty[0]);
    const unsigned a_done = smem_u32(&S.tile_done[0]), a_res = smem_u32(&S.resolved[0]);
    const unsigned a_ring = smem_u32(&S.ring[0][0]);

    // ================================================================ producer warp
    // Lane 0 takes super-tile tickets (the next one while issuing the current
    // one, so the atomic's latency is hidden), streams every sub-tile of each
    // into the ring (zero-byte sub-tiles past the end complete their phase by a
    // plain arrive) and tags the stage of sub-tile 0 with the tile id.  After
    // the last ticket it publishes kNone in the next stage: the end marker.
    if (warp == kProdWarp) {
        if (lane == 0) {
            const float4* src = reinterpret_cast<const float4*>(p.pts);
            unsigned seq = 0;
            unsigned t = atomicAdd(&p.ws->k2_ticket, 1u);
            for (;;) {
                const bool valid = t < p.num_tiles;
                const unsigned tn = valid ? atomicAdd(&p.ws->k2_ticket, 1u) : kNone;
#pragma unroll 1
                for (int sub = 0; sub < (valid ? kK2Sub : 1); ++sub, ++seq) {
                    const unsigned st = seq % kNst;
                    if (seq >= (unsigned)kNst) mbar_sleep_wait(a_empty + 8u * st, ((seq / kNst) - 1u) & 1u);
                    if (sub == 0) S.stile[st] = valid ? t : kNone;
                    const unsigned bytes = valid ? sub_bytes(t, sub, full_pairs) : 0u;
                    if (bytes) {
                        mbar_expect_tx_a(a_full + 8u * st, bytes);
                        bulk_g2s_a(a_ring + st * (16u * kSubPairsT), src + (size_t)t * kTilePairsT + sub * kSubPairsT,
                                   bytes, a_full + 8u * st);
                    } else {
                        mbar_arrive_a(a_full + 8u * st);
                    }
                }
                if (!valid) break;
                t = tn;
            }
        }
        return;
    }

    // ================================================================ emit warp
    // Per super-tile k (list buffer k % kBufs), once all compute warps are done
    // with it (the last of them has published the tile's aggregate; tile 0:
    // its inclusive prefix): scan its 64 group counts; then resolve the
    // PREVIOUS super-tile (decoupled look-back one tile-time after its
    // aggregate went out: no spinning), publish its inclusive prefix and hand
    // its exclusive prefix to the compute warps ("resolved"), which write the
    // survivors.
    if (warp == kEmitWarp) {
        unsigned lb_rounds = 0, lb_spins = 0;
        unsigned pend = kNone, pbuf = 0;
        for (unsigned k = 0;; ++k) {
            const unsigned bi = k % kBufs;
            TileT& cur = S.ts[bi];
            mbar_sleep_wait(a_done + 8u * bi, (k / kBufs) & 1u);
            const unsigned tile = cur.tile;
            if (tile != kNone) {
                // lane l owns groups g = l*kGroupsPerLane + i (g = sub*kW + w, index order)
                unsigned c[kGroupsPerLane], mine = 0;
#pragma unroll
                for (int i = 0; i < kGroupsPerLane; ++i) {
                    const unsigned g = lane * kGroupsPerLane + i;
                    c[i] = 0u;
                    if (g < (unsigned)kGroups) {
                        const unsigned sub = g / kW, w = g % kW;
                        c[i] = cur.lstart[w][sub + 1] - cur.lstart[w][sub];
                    }
                    mine += c[i];
                }
                unsigned inc = mine;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned y = __shfl_up_sync(kFull, inc, o);
                    if (lane >= (unsigned)o) inc += y;
                }
                unsigned run = inc - mine;
#pragma unroll
                for (int i = 0; i < kGroupsPerLane; ++i) {
                    const unsigned g = lane * kGroupsPerLane + i;
                    if (g < (unsigned)kGroups) cur.off[g] = run;
                    run += c[i];
                }
                const unsigned total = __shfl_sync(kFull, inc, 31);
                if (lane == 0) {
                    cur.total = total;
                }
                __syncwarp();
            }
            if (pend != kNone) {
                TileT& prv = S.ts[pbuf];
                unsigned long long ex = 0;
                if (pend != 0) {
                    ex = resolve(p, pend, epoch, lane, lb_rounds, lb_spins);
                    if (lane == 0) {
                        publish(p, pend, kFlagP, ex + prv.total, epoch);
                        if (pend == p.num_tiles - 1) p.ws->count = ex + prv.total;
                    }
                }
                if (lane == 0) {
                    prv.ex = ex;
                    mbar_arrive_a(a_res + 8u * pbuf);   // release: ex and off[] before the phase flips
                }
                // write the lists no compute warp has claimed (a compute warp that
                // needs its buffer back before this warp got to its list writes
                // it itself: dense inputs, where one writer is the bottleneck)
#pragma unroll 1
                for (unsigned w = 0; w < (unsigned)kW; ++w) {
                    if (!claim_list(&S.claim[pbuf][w], k, lane)) continue;   // tag: local tile k-1, + 1
                    emit_t<4>(p, prv, sbase + (size_t)(pbuf * kW + w) * kK2WarpPts, pend, ex, w, lane);
                    __syncwarp();
                    if (lane == 0) st_release_s(&S.emitted[pbuf][w], k);
                }
            }
            if (tile == kNone) break;
            pend = tile;
            pbuf = bi;
        }
        if (lane == 0) {
            if (lb_rounds) atomicAdd(&p.ws->lb_rounds, lb_rounds);
            if (lb_spins) atomicAdd(&p.ws->lb_spins, lb_spins);
            __threadfence();
            const unsigned d = atomicAdd(&p.ws->k2_done, 1u);
            if (d == gridDim.x - 1) {   // last block out: reset the tickets, bump the epoch
                unsigned e = (epoch + 1u) & kEpochMask;
                if (e == 0u) e = 1u;
                p.ws->k2_ticket = 0u;
                p.ws->k2_done = 0u;
                p.ws->epoch = e;
                __threadfence();
            }
        }
        return;
    }

    // ================================================================ compute warps
    // Pass A only: classify each sub-tile from the ring, build the per-warp
    // survivor lists of super-tile k in buffer k % kBufs, signal the emit warp,
    // go on with the next super-tile.  No block-wide barriers.
    const int fast = S.geo.fast, mode = S.geo.mode;
    const float gox = S.geo.ox, goy = S.geo.oy, gr2 = S.geo.r2, ge2 = S.geo.e2max;
    const float gbx0 = S.geo.bx0, gbx1 = S.geo.bx1, gby0 = S.geo.by0, gby1 = S.geo.by1;
    const unsigned rot = (lane >> 1) & 3u;
    // make sure this warp's list of local super-tile j (buffer j % kBufs,
    // global id t) has been written: normally the emit warp has done it; else
    // wait until the tile is resolved and write it here unless the emit warp
    // claims it first (then, if `wait`, until it is done)
    auto emit_own = [&](unsigned j, unsigned t, bool wait) {
        const unsigned bj = j % kBufs, tag = j + 1u;
        if (ld_acquire_s(&S.emitted[bj][warp]) == tag) return;
        mbar_sleep_wait(a_res + 8u * bj, (j / kBufs) & 1u);
        if (claim_list(&S.claim[bj][warp], tag, lane)) {
            emit_t<2>(p, S.ts[bj], sbase + (size_t)(bj * kW + warp) * kK2WarpPts, t, S.ts[bj].ex, warp, lane);
        } else if (wait) {
            while (ld_acquire_s(&S.emitted[bj][warp]) != tag) __nanosleep(64);
        }
    };
    unsigned seq = 0, t1 = 0, t2 = 0, t3 = 0;   // global ids of local super-tiles k-1, k-2, k-3
    unsigned k = 0;
    for (;; ++k) {
        const unsigned bi = k % kBufs;
        TileT& cur = S.ts[bi];
        mbar_sleep_wait(a_full + 8u * (seq % kNst), (seq / kNst) & 1u);
        const unsigned tile = S.stile[seq % kNst];
        const bool have = tile != kNone;
        if (have && k >= (unsigned)kBufs) {
            emit_own(k - kBufs, t3, true);   // frees this warp's part of buffer bi
            __syncwarp();
        }
        if (have) {
            unsigned wc = 0;
            SurvT* const wscr = sbase + (size_t)(bi * kW + warp) * kK2WarpPts;
#pragma unroll 1
            for (int sub = 0; sub < kK2Sub; ++sub, ++seq) {
                const unsigned st = seq % kNst;
                const unsigned bytes = sub_bytes(tile, sub, full_pairs);
                const unsigned np = bytes / 16u;   // full pairs of this sub-tile in memory
                const float4* chunk = &S.ring[st][warp * kChunkPairs];
                mbar_sleep_wait(a_full + 8u * st, (seq / kNst) & 1u);
                // lane l owns the chunk's points loc = 8l + k (k = 0..7), read as
                // four 16-B pairs in the rotated order j -> (j + rot) & 3, so the
                // eight lanes of each quarter-warp hit eight distinct 16-B bank
                // groups (conflict-free LDS.128).  Bit j of m holds pair
                // (j + rot) & 3; one rotate at the end puts point k at bit k.
                unsigned needy = 0u;   // bit k: point 8*lane + k not decided by the fast test
                if (np == (unsigned)kSubPairsT) {
                    if (fast == 0) {
                        unsigned m = 0u;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const float4 v = chunk[lane * 4u + ((j + rot) & 3u)];
                            m |= (in_disk(gox, goy, gr2, v.x, v.y) ? 0u : 1u) << (2 * j);
                            m |= (in_disk(gox, goy, gr2, v.z, v.w) ? 0u : 2u) << (2 * j);
                        }
                        needy = ((m << (2u * rot)) | (m >> (8u - 2u * rot))) & 0xffu;
                    } else if (fast == 1) {
                        unsigned m = 0u;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const float4 v = chunk[lane * 4u + ((j + rot) & 3u)];
                            m |= (in_box(gbx0, gbx1, gby0, gby1, v.x, v.y) ? 0u : 1u) << (2 * j);
                            m |= (in_box(gbx0, gbx1, gby0, gby1, v.z, v.w) ? 0u : 2u) << (2 * j);
                        }
                        needy = ((m << (2u * rot)) | (m >> (8u - 2u * rot))) & 0xffu;
                    } else {   // no fast test (degenerate / exact-only rings): queue everything
                        needy = 0xffu;
                    }
                } else {   // last super-tile only: ragged end (+ the unpaired last point)
                    const unsigned qs = tile * kTilePairsT + sub * kSubPairsT;   // first pair of the sub-tile
                    const float2* chunk2 = reinterpret_cast<const float2*>(chunk);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const unsigned pt = warp * (2u * kChunkPairs) + lane * 8u + k;   // point in the sub-tile
                        bool valid = false;
                        float2 v = make_float2(0.f, 0.f);
                        if (pt < 2u * np) {
                            v = chunk2[lane * 8u + k];
                            valid = true;
                        } else if (odd && 2u * qs + pt == 2u * full_pairs) {
                            v = __ldg(reinterpret_cast<const float2*>(p.pts) + 2u * full_pairs);
                            valid = true;
                        }
                        needy |= (valid && !fast_inside(S.geo, v.x, v.y) ? 1u : 0u) << k;
                    }
                }
                // ---- index-ordered queue: slot of loc = 8l + k = (needy points of
                //      lanes < l) + (needy points of lane l below k).  The lane
                //      prefix of the counts (0..8, four bits) by bit-sliced ballots.
                if (lane == 0) cur.lstart[warp][sub] = wc;
                const unsigned cnt = __popc(needy);
                unsigned slot = 0, qtotal = 0;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const unsigned bb = __ballot_sync(kFull, (cnt >> b) & 1u);
                    slot += __popc(bb & lt) << b;
                    qtotal += __popc(bb) << b;
                }
                for (unsigned m = needy; m; m &= m - 1u)
                    S.qslot[warp][slot++] = (unsigned char)(lane * 8u + (__ffs(m) - 1));
                if (qtotal) {
                    __syncwarp();
                    for (unsigned base = 0; base < qtotal; base += 32) {
                        const unsigned e = base + lane;
                        bool kp = false;
                        float2 q = make_float2(0.f, 0.f);
                        unsigned loc = 0;
                        if (e < qtotal) {
                            loc = S.qslot[warp][e];
                            const unsigned pt = warp * (2u * kChunkPairs) + loc;   // point in the sub-tile
                            if (pt < 2u * np) {
                                q = reinterpret_cast<const float2*>(&S.ring[st][0])[pt];
                            } else {   // the unpaired last point
                                q = __ldg(reinterpret_cast<const float2*>(p.pts) + 2u * full_pairs);
                            }
                            kp = classify_queued<EDGES>(S, mode, gox, goy, ge2, q.x, q.y);
                        }
                        const unsigned kb = __ballot_sync(kFull, kp);
                        if (kp) {
                            const unsigned r = wc + __popc(kb & lt);
                            const SurvT e{q.x, q.y, ((unsigned)sub << 8) | loc};
                            if (r < kL) cur.list[warp][r] = e;
                            else wscr[r - kL] = e;   // overflow: global scratch
                        }
                        wc += __popc(kb);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive_a(a_empty + 8u * st);
            }
            if (lane == 0) cur.lstart[warp][kK2Sub] = wc;
        }
        if (warp == 0 && lane == 0) cur.tile = have ? tile : kNone;
        __syncwarp();
        if (lane == 0) {
            if (have) {
                // the last compute warp done with the tile publishes its aggregate
                // at once: other blocks' look-backs never wait on this block's
                // emit warp (a late aggregate stalls every later tile's look-back)
                const unsigned wc = cur.lstart[warp][kK2Sub];
                const unsigned long long old = atomicAdd(&S.agg[bi], (1ull << 32) | wc);
                if ((unsigned)(old >> 32) == (unsigned)kW - 1u) {
                    const unsigned total = (unsigned)old + wc;
                    S.agg[bi] = 0ull;   // next use: 3 tiles later, after tile_done / buf_free
                    if (tile == 0) {
                        publish(p, 0, kFlagP, total, epoch);
                        if (p.num_tiles == 1) p.ws->count = total;
                    } else {
                        publish(p, tile, kFlagA, total, epoch);
                    }
                }
            }
            mbar_arrive_a(a_done + 8u * bi);
        }
        if (!have) break;
        t3 = t2;
        t2 = t1;
        t1 = tile;
    }
    // the end marker went out as local tile k: help with the last (up to)
    // kBufs super-tiles, resolved once their successor's tile_done arrived
#pragma unroll 1
    for (unsigned i = 0; i < 3u; ++i) {
        if (k + i >= 3u) emit_own(k + i - 3u, t3, false);
        t3 = t2;
        t2 = t1;
    }
}

template <int EDGES>
cudaError_t launch_tma_t(const K2Params& p, cudaStream_t s, int* launches) {
    static std::once_flag once[kMaxDevices];
    static int cap[kMaxDevices];
    const int smem = (int)sizeof(SmemT);
    const int max_blocks = per_device(once, cap, [&] {
        cudaFuncSetAttribute(k2_filter_tma<EDGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2_filter_tma<EDGES>, kBlock, smem);
        return (per_sm > 0 ? per_sm : 1) * device_sm_count();
    });
    unsigned blocks = p.num_tiles < (unsigned)max_blocks ? p.num_tiles : (unsigned)max_blocks;
    if (blocks > p.scratch_blocks) blocks = p.scratch_blocks;   // one overflow scratch area per block
    if (blocks < 1) return cudaErrorInvalidValue;               // (workspace checked by the caller)
    k2_filter_tma<EDGES><<<blocks, kBlock, smem, s>>>(p);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace

int launch_filter_tma(const K2Params& p_in, void* stream, int* launches) {
    cudaStream_t s = (cudaStream_t)stream;
    K2Params p = p_in;   // this kernel's super-tiles: kTilePairsT pairs
    p.num_tiles = (unsigned)((2ull * kTilePairsT - 1 + p.n) / (2ull * kTilePairsT));
    return p.edges <= 16 ? (int)launch_tma_t<16>(p, s, launches) : (int)launch_tma_t<32>(p, s, launches);
}

}  // namespace cudapre
