// k2_spec.cu — Step 3 of CudaPre (§2 Step 3) over K1's
// candidate records: the speculative pre-filter (spec.cuh).
//
// k_spec_verify (one block) decides, after Step 2, whether the pre-filter
// region D that K1 used lies strictly inside the Step-2 ring (exact / rigorous
// predicates; spec.cuh).  If it does, every point K1 did not set aside is
// strictly inside the ring and is discarded, and Step 3 only has to classify
// the candidates: k2_filter_spec below.  Otherwise the streaming K2
// (k2_filter_tma.cu) reads every point as in the paper; each kernel exits at
// once when the other one is selected, so both are always launched and the
// choice stays on the device (no host round trip, CUDA-graph friendly).
//
// k2_filter_spec: tiles of up to 64 chunks (131072 points; the tile-status
// array of the streaming K2, whose tiles are 8 chunks, has room for them),
// assigned statically (tile = block + k * grid).  Warp w classifies the
// records (chunk j, w) of a tile, 8 at a time: their candidates are numbered
// across the 8 records and taken 32 per pass (full lanes), every load of the
// 8 records in flight at once; a record that overflowed (or a chunk K1 did
// not cover: the ragged end) is re-read from the input and classified point
// by point.  Survivors set bits in 64-bit masks, one per 64-point group g =
// 32 j + 8 u + w (index order); a survivor's rank in its group is popc(mask
// below it), so the order of the candidates in a record does not matter.
// Ordered compaction: block scan of the group counts, decoupled look-back
// deferred by one tile (tile k-1 is resolved and written after tile k's
// classification, so its predecessors have published), the writes done by
// all 8 warps (the candidates re-read from L2, the masks say which survive).
#include <cuda_runtime.h>

#include <cstdint>

#include "k2_common.cuh"
#include "spec.cuh"
#include "tma.cuh"

namespace cudapre {
namespace {

constexpr int kSW = 8;                                   // compute warps per block (= K1's warps per chunk)
constexpr int kSThreads = kSW * 32 + 32;                 // + one producer warp
constexpr int kSChunks = 8;                              // chunks per tile (16384 points = the streaming K2's super-tile)
constexpr int kSRecs = kSChunks * kSW;                   // records per tile (64)
constexpr int kSTilePts = kSChunks * kRecChunkPts;
constexpr int kSGroups = kSChunks * 32;                  // 64-point groups per tile
constexpr int kSStages = 3;                              // tiles in the ring: written out / classified / loading
constexpr unsigned kSStageBytes = 18432;                 // packed records of a tile (more: the rest re-read raw)
static_assert(kSTilePts == kK2TilePts, "tile status shared with the streaming K2");
static_assert(kSGroups == kSW * 32, "one group per compute thread in the scan");

struct alignas(128) SStage {
    unsigned char rec[kSStageBytes];          // the used part of each record (metas, entries), packed
    unsigned short roff[kSRecs];              // record r = j * 8 + w at rec + roff[r]
    unsigned char cnt[kSRecs];                // its count; kRecOverflow: re-read from the input
    unsigned tile;                            // the tile in the stage (kSNone: no more tiles)
};
constexpr unsigned kSNone = 0xffffffffu;

constexpr unsigned kSList = 96;               // survivors per warp and tile in shared memory (more: scratch)
constexpr unsigned kSListMax = kSChunks * kRecSlots;   // at most (448)

struct SSmem {
    SStage st[kSStages];
    unsigned long long full[kSStages], empty[kSStages];   // producer <-> classification
    unsigned long long agg[2], exr[2];        // tile aggregate published / tile prefix resolved
    unsigned mask[2][kSGroups][2];            // survivors of group g = 32 j + 8 u + w (bit = offset), lo / hi
    unsigned off[2][kSGroups];                // exclusive offset of group g in its tile
    SurvEntry list[2][kSW][kSList];           // survivors from records: x, y, (j << 8) | meta
    unsigned nlist[2][kSW];
    unsigned long long raw[2];                // bit j * 8 + w: record re-read from the input
    unsigned total[2];
    unsigned long long ex[2];
    unsigned tile[2];
    float2 sec[CUDAPRE_SECTORS + 1];
    unsigned short sedge[CUDAPRE_SECTORS + 1];
    float4 edge[CUDAPRE_MAX_SLOTS];
    GeomLite geo;
    unsigned wsum[kSW];
    unsigned tab[kSW][kSListMax];             // a warp's candidates of the tile: (j << 24) | (slot << 16) | roff
};

__device__ __forceinline__ void mbar_expect_tx_only(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(unsigned bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred P1;\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n selp.u32 %0, 1, 0, P1;\n }"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}

// barrier of the 8 compute warps only (the producer warp is elsewhere)
__device__ __forceinline__ void bar_compute() { asm volatile("bar.sync 1, %0;" ::"n"(kSW * 32) : "memory"); }

// keep decision for a point (true = survives): the streaming K2's queued-point
// test (inner disk, sector table -> candidate edges -> exact), which is exact
template <int EDGES>
__device__ __forceinline__ bool classify(const SSmem& S, float x, float y) {
    const GeomLite& G = S.geo;
    const float2 d = __fadd2_rn(make_float2(x, y), make_float2(-G.ox, -G.oy));
    const float2 q = __fmul2_rn(d, d);
    const float d2 = __fadd_rn(q.x, q.y);
    if (d2 < G.r2) return false;   // inner disk (G.mode == 0 here: the verification requires it)
    const unsigned b = spec::sector_bucket(d.x, d.y);
    const float2 rr = S.sec[b];
    if (d2 < rr.x) return false;
    if (d2 > rr.y) return true;
    const unsigned se = S.sedge[b];
    if (se == 0xffffu) return queue_keep_rare<EDGES>(G, x, y);
    const float4 e0 = S.edge[se & 0xffu], e1 = S.edge[se >> 8];
    const float mn = fminf(__fmaf_rn(e0.x, x, __fmaf_rn(e0.y, y, e0.z)),
                           __fmaf_rn(e1.x, x, __fmaf_rn(e1.y, y, e1.z)));
    if (mn > 0.0f) return false;
    if (__fadd_rn(mn, G.e2max) < 0.0f) return true;
    return !exact_inside(G, x, y);
}

static_assert(2 * kSW * kSListMax * sizeof(SurvEntry) <= kK2ScratchPerBlock, "list overflow scratch");

// the 8 points (u = 0..3, h = 0..1) of lane `lane` of record (chunk c, warp w):
// local indices 2 (1024 c + 256 u + 32 w + lane) + h; valid bit 2u+h if < n
__device__ __forceinline__ unsigned load_raw(const K2Params& p, unsigned c, unsigned w, unsigned lane,
                                             float4 (&v)[4]) {
    unsigned valid = 0;
    const unsigned full_pairs = p.n / 2u;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const unsigned q = c * (unsigned)(kRecChunkPts / 2) + 256u * u + 32u * w + lane;
        v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (q < full_pairs) {
            v[u] = __ldcg(reinterpret_cast<const float4*>(p.pts) + q);
            valid |= 3u << (2 * u);
        } else if (2u * q < p.n) {
            const float2 a = __ldcg(reinterpret_cast<const float2*>(p.pts) + 2u * q);
            v[u] = make_float4(a.x, a.y, 0.f, 0.f);
            valid |= 1u << (2 * u);
        }
    }
    return valid;
}

template <int EDGES>
__global__ void __launch_bounds__(kSThreads, 2) k2_filter_spec(const __grid_constant__ K2Params p) {
    if (!p.sp || !p.sp->on) return;   // the streaming K2 does Step 3 (uniform)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SSmem& S = *reinterpret_cast<SSmem*>(smem_raw);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned epoch = *(volatile unsigned*)&p.ws->epoch;
    const unsigned rec_chunks = (unsigned)p.sp->rec_chunks;
    const unsigned nchunks = (unsigned)(((unsigned long long)p.n + kRecChunkPts - 1) / kRecChunkPts);

    for (int i = tid; i <= CUDAPRE_SECTORS; i += kSThreads) {
        S.sec[i] = make_float2(p.g->sr2[i], p.g->sro2[i]);
        S.sedge[i] = p.g->sedge[i];
    }
    if (tid < (unsigned)CUDAPRE_MAX_SLOTS) S.edge[tid] = make_float4(p.g->A[tid], p.g->B[tid], p.g->C[tid], 0.0f);
    load_geom_lite(S.geo, p.g, tid, kSThreads);
    if (tid == 0) {
        for (int k = 0; k < kSStages; ++k) {
            mbar_init(&S.full[k], 1u);
            mbar_init(&S.empty[k], 1u);
        }
        for (int k = 0; k < 2; ++k) {
            mbar_init(&S.agg[k], 1u);
            mbar_init(&S.exr[k], 1u);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const unsigned a_full = smem_u32(&S.full[0]), a_empty = smem_u32(&S.empty[0]);
    const unsigned a_agg = smem_u32(&S.agg[0]), a_exr = smem_u32(&S.exr[0]);

    // ================================================================ producer warp
    // (1) tile k (= block + k * grid) -> stage k % 3: the used part of each of
    // its 64 records (metas + count entries), packed, one bulk copy per record
    // (lane l: records l and l + 32), their counts and offsets, two tiles
    // ahead of the classification; (2) the decoupled look-back of tile k once
    // its aggregate is out (the compute warps write it out one tile later).
    if (warp == (unsigned)kSW) {
        // tiles from a global ticket (claimed in order, so a tile's predecessors
        // publish first: short look-backs); the next tile is claimed, and its
        // counts loaded, while the current one is issued
        auto claim = [&]() -> unsigned {
            unsigned t = 0;
            if (lane == 0) t = atomicAdd(&p.ws->k2_ticket, 1u);
            t = __shfl_sync(kFull, t, 0);
            return t < p.num_tiles ? t : kSNone;
        };
        auto cnt_of = [&](unsigned tile, unsigned r) -> unsigned {   // count byte of record r of tile
            if (tile == kSNone) return 0u;
            const unsigned c = tile * kSChunks + r / kSW;
            if (c >= nchunks) return 0u;
            if (c >= rec_chunks) return kRecOverflow;
            return (unsigned)__ldcg(p.rcount + (size_t)c * kSW + (r % kSW));
        };
        unsigned ntile = claim();
        unsigned nxt[2] = {cnt_of(ntile, lane), cnt_of(ntile, lane + 32)};
        auto issue = [&](unsigned k) -> unsigned {   // the next claimed tile into stage k % 3
            const unsigned tile = ntile;
            const unsigned s = k % kSStages;
            unsigned cc[2] = {nxt[0], nxt[1]};
            if (tile != kSNone) {
                ntile = claim();
                nxt[0] = cnt_of(ntile, lane);
                nxt[1] = cnt_of(ntile, lane + 32);
            }
            unsigned sz[2];
#pragma unroll
            for (int h = 0; h < 2; ++h)
                sz[h] = (cc[h] == kRecOverflow || cc[h] == 0u) ? 0u : ((kRecMetaBytes + 8u * cc[h] + 15u) & ~15u);
            unsigned inc0 = sz[0], inc1 = sz[1];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y0 = __shfl_up_sync(kFull, inc0, o), y1 = __shfl_up_sync(kFull, inc1, o);
                if (lane >= (unsigned)o) inc0 += y0, inc1 += y1;
            }
            const unsigned t0 = __shfl_sync(kFull, inc0, 31);
            const unsigned o0 = inc0 - sz[0], o1 = t0 + inc1 - sz[1];
            // records past the stage's capacity are re-read from the input
            if (o0 + sz[0] > kSStageBytes) sz[0] = 0, cc[0] = kRecOverflow;
            if (o1 + sz[1] > kSStageBytes) sz[1] = 0, cc[1] = kRecOverflow;
            const unsigned total = __reduce_add_sync(kFull, sz[0] + sz[1]);
            if (k >= (unsigned)kSStages)
                while (!mbar_try_wait(a_empty + 8u * s, ((k / kSStages) - 1u) & 1u)) __nanosleep(128);
            SStage& T = S.st[s];
            T.cnt[lane] = (unsigned char)cc[0];
            T.cnt[lane + 32] = (unsigned char)cc[1];
            T.roff[lane] = (unsigned short)o0;
            T.roff[lane + 32] = (unsigned short)o1;
            if (lane == 0) T.tile = tile;
            if (lane == 0 && total) mbar_expect_tx_only(a_full + 8u * s, total);
            __syncwarp();
            const unsigned c0 = tile * kSChunks;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const unsigned r = lane + 32u * h;
                if (sz[h])
                    bulk_g2s_a(smem_u32(T.rec) + (h ? o1 : o0),
                               p.records + ((size_t)(c0 + r / kSW) * kSW + r % kSW) * kRecBytes, sz[h],
                               a_full + 8u * s);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_a(a_full + 8u * s);
            return tile;
        };
        unsigned lb_rounds = 0, lb_spins = 0;
        unsigned tiles[kSStages] = {kSNone, kSNone, kSNone};   // tile of issue k at [k % 3]
        unsigned nissued = 0;
        for (; nissued < 2u; ++nissued) {
            tiles[nissued] = issue(nissued);
            if (tiles[nissued] == kSNone) { ++nissued; break; }
        }
        for (unsigned k = 0;; ++k) {
            const unsigned tile = tiles[k % kSStages];
            if (tile == kSNone) break;
            if (nissued == k + 2 && tiles[(k + 1) % kSStages] != kSNone) {
                tiles[nissued % kSStages] = issue(nissued);
                ++nissued;
            }
            const unsigned b = k & 1u;
            while (!mbar_try_wait(a_agg + 8u * b, (k >> 1) & 1u)) __nanosleep(64);
            unsigned long long ex = 0;
            if (tile != 0) {
                ex = resolve(p, tile, epoch, lane, lb_rounds, lb_spins);
                if (lane == 0) {
                    publish(p, tile, kFlagP, ex + S.total[b], epoch);
                    if (tile == p.num_tiles - 1) p.ws->count = ex + S.total[b];
                }
            }
            if (lane == 0) {
                S.ex[b] = ex;
                mbar_arrive_a(a_exr + 8u * b);
            }
        }
        if (lane == 0) {
            if (lb_rounds) atomicAdd(&p.ws->lb_rounds, lb_rounds);
            if (lb_spins) atomicAdd(&p.ws->lb_spins, lb_spins);
        }
        return;
    }

    // ================================================================ compute warps
    // per tile k: classification (survivor masks, per-warp survivor lists),
    // scan of the 256 group counts, the aggregate; then the write-out of tile
    // k - 1, whose prefix the producer warp has resolved meanwhile
    SurvEntry* const sbase = p.scratch + (size_t)blockIdx.x * (2 * kSW * kSListMax);
    bool more = true;
    for (unsigned k = 0;; ++k) {
        const unsigned b = k & 1u, s = k % kSStages;
        unsigned tile = kSNone;
        if (more) {
            S.mask[b][tid][0] = 0u;
            S.mask[b][tid][1] = 0u;
            if (tid == 0) S.raw[b] = 0ull;
            while (!mbar_try_wait(a_full + 8u * s, (k / kSStages) & 1u)) __nanosleep(32);
            tile = S.st[s].tile;
            more = tile != kSNone;
        }
        if (more) {
            const unsigned c0 = tile * kSChunks;
            bar_compute();
            if (tid == 0) S.tile[b] = tile;
            // ---------------------------------------------------------------- classification
            const SStage& T = S.st[s];
            SurvEntry* const ovf = sbase + (size_t)(b * kSW + warp) * kSListMax;
            // this warp's 8 records (j, warp): their candidates numbered across the
            // records (lane j < 8 lists record j's), then taken 32 per pass
            unsigned cj = 0, rawj = 0;
            if (lane < (unsigned)kSChunks) cj = T.cnt[lane * kSW + warp];
            rawj = __ballot_sync(kFull, lane < (unsigned)kSChunks && cj == kRecOverflow);
            if (cj == kRecOverflow) cj = 0;
            unsigned cinc = cj;
#pragma unroll
            for (int o = 1; o < kSChunks; o <<= 1) {
                const unsigned y = __shfl_up_sync(kFull, cinc, o);
                if (lane >= (unsigned)o) cinc += y;
            }
            const unsigned ctot = __shfl_sync(kFull, cinc, kSChunks - 1);
            if (lane < (unsigned)kSChunks) {
                const unsigned ro = T.roff[lane * kSW + warp];
                for (unsigned t = 0, e = cinc - cj; t < cj; ++t, ++e) S.tab[warp][e] = (lane << 24) | (t << 16) | ro;
            }
            __syncwarp();
            unsigned wl = 0;
            for (unsigned q0 = 0; q0 < ctot; q0 += 32) {
                const unsigned q = q0 + lane;
                bool kp = false;
                float2 pt = make_float2(0.f, 0.f);
                unsigned mt = 0, j = 0;
                if (q < ctot) {
                    const unsigned tv = S.tab[warp][q];
                    const unsigned slot = (tv >> 16) & 0xffu, ro = tv & 0xffffu;
                    j = tv >> 24;
                    pt = reinterpret_cast<const float2*>(T.rec + ro + kRecMetaBytes)[slot];
                    mt = T.rec[ro + slot];
                    kp = classify<EDGES>(S, pt.x, pt.y);
                }
                const unsigned kb = __ballot_sync(kFull, kp);
                if (kp) {
                    const unsigned g = j * 32 + (mt >> 6) * 8 + warp, loc = mt & 63u;
                    atomicOr(&S.mask[b][g][loc >> 5], 1u << (loc & 31u));
                    const unsigned e = wl + __popc(kb & lt);
                    const SurvEntry se{pt.x, pt.y, (j << 8) | mt};
                    if (e < kSList) S.list[b][warp][e] = se;
                    else ovf[e - kSList] = se;
                }
                wl += __popc(kb);
            }
            // overflowed records, records past the stage and chunks without records: every point
            for (unsigned rb = rawj; rb; rb &= rb - 1) {
                const unsigned j = __ffs(rb) - 1;
                float4 v[4];
                const unsigned valid = load_raw(p, c0 + j, warp, lane, v);
                unsigned long long bits[4] = {0, 0, 0, 0};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (!((valid >> (2 * u + h)) & 1u)) continue;
                        const float x = h ? v[u].z : v[u].x, y = h ? v[u].w : v[u].y;
                        if (!fast_inside(S.geo, x, y) && queue_keep_rare<EDGES>(S.geo, x, y))
                            bits[u] |= 1ull << (2 * lane + h);
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const unsigned lo = __reduce_or_sync(kFull, (unsigned)bits[u]);
                    const unsigned hi = __reduce_or_sync(kFull, (unsigned)(bits[u] >> 32));
                    if (lane == 0) {
                        S.mask[b][j * 32 + u * 8 + warp][0] = lo;
                        S.mask[b][j * 32 + u * 8 + warp][1] = hi;
                    }
                }
            }
            if (lane == 0) {
                S.nlist[b][warp] = wl;
                if (rawj) {
                    unsigned long long rm = 0;
                    for (unsigned j = 0; j < (unsigned)kSChunks; ++j)
                        if ((rawj >> j) & 1u) rm |= 1ull << (j * kSW + warp);
                    atomicOr(&S.raw[b], rm);
                }
            }
            if (wl > kSList) __threadfence_block();   // (scratch entries before the barrier)
            bar_compute();   // all warps done with stage s: the producer may refill it
            if (tid == 0) mbar_arrive_a(a_empty + 8u * s);
            // ---------------------------------------------------------------- scan of the 256 groups
            const unsigned gc = __popc(S.mask[b][tid][0]) + __popc(S.mask[b][tid][1]);
            unsigned inc = gc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(kFull, inc, o);
                if (lane >= (unsigned)o) inc += y;
            }
            if (lane == 31) S.wsum[warp] = inc;
            bar_compute();
            unsigned wbase = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < kSW; ++w) {
                const unsigned v = S.wsum[w];
                wbase += (unsigned)w < warp ? v : 0u;
                tot += v;
            }
            S.off[b][tid] = wbase + inc - gc;
            if (tid == 0) {
                S.total[b] = tot;
                if (tile == 0) {
                    publish(p, 0, kFlagP, tot, epoch);
                    if (p.num_tiles == 1) p.ws->count = tot;
                } else {
                    publish(p, tile, kFlagA, tot, epoch);
                }
                mbar_arrive_a(a_agg + 8u * b);   // the producer resolves this tile's prefix
            }
        }
        // ---------------------------------------------------------------- write-out of tile k - 1
        if (k > 0) {
            const unsigned pk = k - 1, pb = pk & 1u;
            const unsigned prev = S.tile[pb];
            while (!mbar_try_wait(a_exr + 8u * pb, (pk >> 1) & 1u)) __nanosleep(32);
            const unsigned long long ex = S.ex[pb];
            const unsigned long long tbase = (unsigned long long)prev * kSTilePts;
            float2* out_pts = reinterpret_cast<float2*>(p.out_pts);
            const SurvEntry* ovf = sbase + (size_t)(pb * kSW + warp) * kSListMax;
            const unsigned n = S.nlist[pb][warp];
            for (unsigned r = lane; r < n; r += 32) {
                SurvEntry e;
                if (r < kSList) {
                    e = S.list[pb][warp][r];
                } else {
                    const SurvEntry* q = ovf + (r - kSList);
                    e.x = __ldcg(&q->x);
                    e.y = __ldcg(&q->y);
                    e.meta = __ldcg(&q->meta);
                }
                const unsigned j = e.meta >> 8, u = (e.meta >> 6) & 3u, loc = e.meta & 63u;
                const unsigned g = j * 32 + u * 8 + warp;
                const unsigned long long gm = ((unsigned long long)S.mask[pb][g][1] << 32) | S.mask[pb][g][0];
                const unsigned long long pos = ex + S.off[pb][g] + __popcll(gm & ((1ull << loc) - 1ull));
                if (pos < p.capacity) {
                    p.out_idx[pos] = p.base + (long long)(tbase + j * kRecChunkPts + u * 512 + warp * 64 + loc);
                    if (out_pts) out_pts[pos] = make_float2(e.x, e.y);
                }
            }
            const unsigned long long rawb = S.raw[pb];
            for (unsigned j = 0; j < (unsigned)kSChunks; ++j) {
                if (!((rawb >> (j * kSW + warp)) & 1ull)) continue;
                const unsigned c = prev * kSChunks + j;
                float4 v[4];
                load_raw(p, c, warp, lane, v);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const unsigned g = j * 32 + u * 8 + warp;
                    const unsigned long long gm = ((unsigned long long)S.mask[pb][g][1] << 32) | S.mask[pb][g][0];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const unsigned loc = 2 * lane + h;
                        if (!((gm >> loc) & 1ull)) continue;
                        const unsigned long long pos = ex + S.off[pb][g] + __popcll(gm & ((1ull << loc) - 1ull));
                        if (pos < p.capacity) {
                            p.out_idx[pos] = p.base + (long long)((unsigned long long)c * kRecChunkPts + u * 512 +
                                                                  warp * 64 + loc);
                            if (out_pts) out_pts[pos] = h ? make_float2(v[u].z, v[u].w) : make_float2(v[u].x, v[u].y);
                        }
                    }
                }
            }
        }
        bar_compute();   // buffers (k - 1) & 1 are free for tile k + 1
        if (!more) break;
    }
    if (tid == 0) {
        __threadfence();
        const unsigned d = atomicAdd(&p.ws->k2_done, 1u);
        if (d == gridDim.x - 1) {   // last block out: reset the ticket, bump the epoch
            unsigned e = (epoch + 1u) & kEpochMask;
            if (e == 0u) e = 1u;
            p.ws->k2_ticket = 0u;
            p.ws->k2_done = 0u;
            p.ws->epoch = e;
            __threadfence();
        }
    }
}

// ---------------------------------------------------------------- verification
constexpr int kVThreads = 32;

__global__ void __launch_bounds__(kVThreads) k_spec_verify(const K2Geom* __restrict__ g, SpecPage* sp,
                                                         const float* pts, unsigned long long n, long long base) {
    const unsigned lane = threadIdx.x;
    // the records describe this input (token), the ring is a proper one, and
    // few records overflowed (else the streaming K2 is the faster choice)
    bool ok = sp->enabled && sp->tok_n != 0ull && sp->tok_n == n && sp->tok_pts == pts && sp->tok_base == base &&
              g->mode == 0 && g->nv >= 3 && 64ull * sp->overflow <= 8ull * sp->rec_chunks;
    const int nv = g->nv;
    if (ok) {
        const float cx = sp->cx, cy = sp->cy;
        // the centre strictly inside the ring (exact): one edge per lane
        bool in = true;
        for (int j = lane; j < nv; j += 32)
            in &= orient_sign_f(g->vx[j], g->vy[j], g->vx[j + 1], g->vy[j + 1], cx, cy) > 0;
        if (sp->use_box) {   // the closed box: its 4 float corners strictly inside (exact)
            const float bx[4] = {sp->box[0], sp->box[1], sp->box[1], sp->box[0]};
            const float by[4] = {sp->box[2], sp->box[2], sp->box[3], sp->box[3]};
            for (int t = lane; t < 4 * nv; t += 32) {
                const int j = t >> 2, q = t & 3;
                in &= orient_sign_f(g->vx[j], g->vy[j], g->vx[j + 1], g->vy[j + 1], bx[q], by[q]) > 0;
            }
        } else if (lane == 0) {   // the disk: every edge line farther than its radius (rigorous)
            in &= spec::disk_inside(g->vx, g->vy, nv, cx, cy, sp->r2min);
        }
        ok = __all_sync(0xffffffffu, in);
    }
    if (lane == 0) {
        sp->on = ok ? 1 : 0;
        sp->tok_n = 0ull;   // records are consumed by at most one Step 3
    }
}

}  // namespace

int launch_spec_verify(const K2Geom* g, SpecPage* sp, const float* pts, unsigned long long n, long long base,
                       void* stream, int* launches) {
    k_spec_verify<<<1, kVThreads, 0, (cudaStream_t)stream>>>(g, sp, pts, n, base);
    ++*launches;
    return (int)cudaGetLastError();
}

int launch_filter_spec(const K2Params& p_in, void* stream, int* launches) {
    cudaStream_t s = (cudaStream_t)stream;
    K2Params p = p_in;
    p.num_tiles = (unsigned)(((unsigned long long)p.n + kSTilePts - 1) / kSTilePts);
    static std::once_flag once[kMaxDevices];
    static int cap[kMaxDevices];
    const int smem = (int)sizeof(SSmem);
    static_assert(sizeof(SSmem) <= 110 * 1024, "two blocks per SM");
    const int max_blocks = per_device(once, cap, [&] {
        cudaFuncSetAttribute(k2_filter_spec<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k2_filter_spec<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2_filter_spec<16>, kSThreads, smem);
        return (per_sm > 0 ? per_sm : 1) * device_sm_count();
    });
    unsigned blocks = p.num_tiles < (unsigned)max_blocks ? p.num_tiles : (unsigned)max_blocks;
    if (blocks > p.scratch_blocks) blocks = p.scratch_blocks;   // one list-overflow scratch area per block
    if (blocks < 1) return (int)cudaErrorInvalidValue;
    if (p.edges <= 16)
        k2_filter_spec<16><<<blocks, kSThreads, smem, s>>>(p);
    else
        k2_filter_spec<32><<<blocks, kSThreads, smem, s>>>(p);
    ++*launches;
    return (int)cudaGetLastError();
}

}  // namespace cudapre
