// k2_filter3.cu — Step 3 of the 3D extension ("Those points
// locating inside the convex polyhedron must be interior points, and can be
// directly discarded"; DESIGN.md §3 B5, §6.5) as ONE streaming pass:
// classify every point against the polyhedron and stream-compact the
// survivors in ascending index order.
//
// Classification (exact semantics): p is DISCARDED iff orient3d(f, p) > 0
// for every facet plane f.  With the centre o strictly inside (checked
// exactly on the host), the ray from o through p leaves the polyhedron
// through a facet whose face contains the ray's direction; p is strictly
// inside iff it is strictly inside that facet.  The direction d = RN(p - o)
// selects one of 6144 cube-map cells (major axis, sign, and the two other
// components over the major one on a 32 x 32 grid; one approximate
// reciprocal), and the host lists, per cell, every facet whose face meets the
// cell's direction pyramid widened by a guard far larger than the kernel's
// rounding — about 1.2 of ~32 on average.  Lists of up to
// 3 are tested branch-free (unused slots: a plane that always says
// "inside"); longer lists and undecided tests go to a warp-cooperative pass
// (the whole warp splits one point's candidate facets and votes):
//   g = fma(A, x, fma(B, y, fma(C, z, D))), |g - orient3d| <= E over the
//   data bounding box:   g < -E on any candidate -> keep;  g > E on all ->
//   discard;  otherwise the exact orient3d (exact3.cuh) on the undecided ones.
// A direction too short for the reciprocal (or NaN) takes every facet.
// Compaction: persistent blocks take tiles of kK23Quads * 1024 points from an
// atomic ticket; each thread classifies kK23Quads quads; packed (two 16-bit
// halves per word) block scans order the survivors; the first warp done
// classifying a tile takes the next ticket and resolves the PREVIOUS tile's
// exclusive prefix by a decoupled look-back over epoch-tagged status words
// (one per 128-byte line) while the others still classify — deferred by one
// tile, so it never waits, and off the barrier-to-barrier path; survivors'
// int64 index (+ xyz) are staged in shared memory and written in order with
// coalesced stores.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "exact3.cuh"
#include "internal3.h"

namespace cudapre {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned kFlagA = 1u;
constexpr unsigned kFlagP = 2u;
constexpr unsigned kEpochMask = 0x3fffffffu;
constexpr int kWarps = kK23Threads / 32;
// look-back loads per lane: first round / later rounds (A/B-measured)
#ifndef K23_LB_FIRST
#define K23_LB_FIRST 2
#endif
#ifndef K23_LB_NEXT
#define K23_LB_NEXT 2
#endif

struct Smem3 {
    unsigned clist[kCells];
    float4 pl[kMax3Facets + 1];
    float pe[kMax3Facets + 1];
    float fv[kMax3Facets][9];
    unsigned long long all;
    float ox, oy, oz;
    int mode;
    unsigned wsum[kK23Quads / 2][kWarps];
    unsigned wbase[2][kK23Quads / 2][kWarps];
    unsigned tile[2];
    unsigned total[2][kK23Quads / 2];
    unsigned long long ex;
    unsigned done;   // warps done classifying the current tile (the first one resolves)
    // the previous tile's survivors, compacted in order: tile-local index + xyz
    unsigned sidx[kK23TilePts];
    float spts[3 * kK23TilePts];
};

__device__ __forceinline__ void st_status(unsigned long long* a, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ void publish(const K23Params& p, unsigned tile, unsigned flag, unsigned long long v,
                                        unsigned epoch) {
    st_status(&p.status[(size_t)tile * kStatus3Stride],
              ((unsigned long long)(epoch & kEpochMask) << 34) | ((unsigned long long)flag << 32) |
                  (v & 0xffffffffull));
}

// exclusive prefix of `tile` (warp 0): walk back 32*8 predecessors per round,
// summing aggregates up to the nearest inclusive prefix.
__device__ unsigned long long resolve(const K23Params& p, unsigned tile, unsigned epoch, unsigned lane) {
    constexpr int kPer = K23_LB_NEXT;   // loads per lane in later rounds
    int per = K23_LB_FIRST;             // ... and in the first (the nearest prefix is usually close)
    const unsigned long long PF = (unsigned long long)kFlagP << 32;
    const unsigned long long E = (unsigned long long)(epoch & kEpochMask) << 34;
    unsigned long long ex = 0;
    long long pred = (long long)tile - 1;
    while (pred >= 0) {
        unsigned long long w[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const long long t = pred - (long long)(per * (int)lane + k);
            w[k] = (k < per && t >= 0) ? ld_status(&p.status[(size_t)t * kStatus3Stride]) : (E | PF);
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
        if (imask & need) {
            __nanosleep(64);
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

__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ float rcp_approx(float a) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    return r;
}

// Fast test of one point: 0 = discard, 1 = keep, 2 = slow (a long candidate
// list, an undecided plane test, or no cell); `cw` then holds the cell's list
// word (kNoCell: every facet) for the warp-cooperative pass (cell_mask).
constexpr unsigned kNoCell = 0xffffffffu;
__device__ __forceinline__ int classify_fast(const Smem3& g, float x, float y, float z, unsigned& cw) {
    const float dx = __fsub_rn(x, g.ox), dy = __fsub_rn(y, g.oy), dz = __fsub_rn(z, g.oz);
    const float ax = fabsf(dx), ay = fabsf(dy), az = fabsf(dz);
    const bool xm = ax >= ay && ax >= az;
    const bool ym = !xm && ay >= az;
    const float m = xm ? dx : (ym ? dy : dz);
    const float u = xm ? dy : (ym ? dz : dx);
    const float v = xm ? dz : (ym ? dx : dy);
    const float am = fabsf(m);
    const float r = __fmul_rn(rcp_approx(am), 0.5f * kCellG);
    const float fu = fminf(fmaxf(__fmaf_rn(u, r, 0.5f * kCellG), 0.0f), kCellG - 0.5f);
    const float fv = fminf(fmaxf(__fmaf_rn(v, r, 0.5f * kCellG), 0.0f), kCellG - 0.5f);
    const int face = (xm ? 0 : (ym ? 2 : 4)) + (m < 0.0f ? 1 : 0);
    const int cell = (face * kCellG + (int)fu) * kCellG + (int)fv;
    const bool ok = am >= 0x1p-100f;   // false for NaN and for directions too short for the reciprocal
    const unsigned w = g.clist[ok ? cell : 0];
    cw = ok ? w : kNoCell;
    if (!ok || (w >> 24) > (unsigned)kCellSlots) return 2;   // long list (or no cell)
    bool out = false, unsure = false;
#pragma unroll
    for (int k = 0; k < kCellSlots; ++k) {   // branch-free: unused slots test the dummy plane
        const unsigned t = (w >> (8 * k)) & 0xffu;
        const float4 P = g.pl[t];
        const float E = g.pe[t];
        const float val = __fmaf_rn(P.x, x, __fmaf_rn(P.y, y, __fmaf_rn(P.z, z, P.w)));
        out |= val < -E;
        unsure |= !(val > E);
    }
    return out ? 1 : (unsure ? 2 : 0);
}

// the candidate facets of a cell list word (for the slow pass)
__device__ __forceinline__ unsigned long long cell_mask(const Smem3& g, const K3Geom* __restrict__ G, unsigned w) {
    if (w == kNoCell) return g.all;
    if ((w >> 24) > (unsigned)kCellSlots) {
        const unsigned li = w & 0xffffffu;
        return li != kNoLong ? __ldg(&G->lmask[li]) : g.all;
    }
    unsigned long long m = 0;
#pragma unroll
    for (int k = 0; k < kCellSlots; ++k) {
        const unsigned t = (w >> (8 * k)) & 0xffu;
        if (t < (unsigned)kMax3Facets) m |= 1ull << t;
    }
    return m;
}

// The slow decision for one point, by the whole warp (x, y, z, mask uniform):
// lane j takes the j-th candidate facet — float test, exact orient3d when the
// float test cannot decide — and the warp votes.  Non-finite points are kept.
__device__ __noinline__ bool slow_coop(const Smem3& g, float x, float y, float z, unsigned long long mask,
                                       unsigned lane, unsigned* nexact) {
    bool out = !(fabsf(x) <= FLT_MAX && fabsf(y) <= FLT_MAX && fabsf(z) <= FLT_MAX);
    const unsigned lo = (unsigned)mask, hi = (unsigned)(mask >> 32);
    const int nlo = __popc(lo), n = nlo + __popc(hi);
    const float q[3] = {x, y, z};
    for (int base = 0; base < n && !out; base += 32) {
        const int j = base + (int)lane;
        if (j < n) {
            const int t = j < nlo ? (int)__fns(lo, 0, j + 1) : 32 + (int)__fns(hi, 0, j - nlo + 1);
            const float4 P = g.pl[t];
            const float E = g.pe[t];
            const float val = __fmaf_rn(P.x, x, __fmaf_rn(P.y, y, __fmaf_rn(P.z, z, P.w)));
            if (val < -E) {
                out = true;
            } else if (!(val > E)) {
                ++*nexact;
                const float* f = g.fv[t];
                out = orient3d_sign_f(f, f + 3, f + 6, q) <= 0;
            }
        }
        out = __any_sync(kFull, out);
    }
    return out;
}

template <bool VEC>
__device__ __forceinline__ unsigned load_quad(const float* __restrict__ pts, unsigned q, unsigned n, float (&v)[12]) {
    const unsigned i0 = 4u * q;
    const unsigned valid = i0 >= n ? 0u : (n - i0 >= 4u ? 4u : n - i0);
    if (VEC && valid == 4u) {
        const float4* s = reinterpret_cast<const float4*>(pts) + 3u * q;
        const float4 a = __ldg(s), b = __ldg(s + 1), c = __ldg(s + 2);
        v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y;
        v[6] = b.z, v[7] = b.w, v[8] = c.x, v[9] = c.y, v[10] = c.z, v[11] = c.w;
    } else {
#pragma unroll
        for (int j = 0; j < 12; ++j) v[j] = (unsigned)(j / 3) < valid ? __ldg(pts + 3ull * i0 + j) : 0.0f;
    }
    return valid;
}

// Stage one quad's survivors (coordinates v) at tile-local positions from pos on.
__device__ __forceinline__ void stage(Smem3& g, const float (&v)[12], unsigned bits, unsigned local_q,
                                      unsigned pos) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if ((bits >> e) & 1u) {
            g.sidx[pos] = 4u * local_q + e;
            g.spts[3 * pos] = v[3 * e], g.spts[3 * pos + 1] = v[3 * e + 1], g.spts[3 * pos + 2] = v[3 * e + 2];
            ++pos;
        }
    }
}

template <bool VEC>
__global__ void __launch_bounds__(kK23Threads, kK23BlocksPerSM) k2_filter3(const __grid_constant__ K23Params p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem3& g = *reinterpret_cast<Smem3*>(smem_raw);
    const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const K3Geom* G = p.g;
    for (int t = tid; t < kCells; t += kK23Threads) g.clist[t] = G->clist[t];
    const int nf = G->nf;
    for (int t = tid; t <= kMax3Facets; t += kK23Threads)
        if (t < nf || t == kDummyFacet) {
            g.pl[t] = G->pl[t];
            g.pe[t] = G->pe[t];
        }
    for (int t = tid; t < nf * 9; t += kK23Threads) g.fv[t / 9][t % 9] = G->fv[t / 9][t % 9];
    if (tid == 0) {
        g.ox = G->ox, g.oy = G->oy, g.oz = G->oz;
        g.mode = G->mode;
        g.all = G->all;
    }
    const unsigned epoch = *(volatile unsigned*)&p.ws->epoch;
    unsigned nexact = 0;
    __syncthreads();
    const bool keep_all = g.mode != 0;

    // Deferred look-back (as the 2D kernel): tile k's aggregate is published
    // right after its scan, but its prefix is resolved only after tile k+1 has
    // been classified, when every predecessor has long published its own
    // aggregate — no spinning.  Tile k's survivors wait compacted in shared
    // memory (tile-local index + xyz) and are then written with fully
    // coalesced stores; its total lives in shared memory (double-buffered).
    // L2 prefetch one wave ahead: the tile gridDim.x after the claimed one is
    // about the one some block claims next (no ticket is held early).
    const unsigned full_tiles = p.n / kK23TilePts;
    bool have_prev = false;
    unsigned prev_tile = 0;
    int par = 0;
    // the first tile; every later one is claimed by thread 0 once warp 0 is
    // done classifying its share of the current tile (the barriers that
    // follow make it visible), so the loop needs no barrier of its own at the
    // top
    if (tid == 0) {
        g.done = 0u;
        const unsigned t = atomicAdd(&p.ws->k2_ticket, 1u);
        g.tile[0] = t;
        const unsigned ahead = t + gridDim.x;
        if (VEC && ahead < full_tiles) prefetch_l2(p.pts + 3ull * kK23TilePts * ahead, 12u * kK23TilePts);
    }
    __syncthreads();
    for (;;) {
        const unsigned tile = g.tile[par];
        const bool live = tile < p.num_tiles;
        constexpr int kP = kK23Quads / 2;   // packed scan words: two quad slots each (16-bit halves)
        unsigned bits[kK23Quads], c[kP], incl[kP];
        float v[kK23Quads][12];
#pragma unroll
        for (int h = 0; h < kK23Quads; ++h) bits[h] = 0;
#pragma unroll
        for (int w = 0; w < kP; ++w) c[w] = incl[w] = 0;
        if (live) {
            unsigned nv[kK23Quads];
#pragma unroll
            for (int h = 0; h < kK23Quads; ++h)
                nv[h] = load_quad<VEC>(p.pts, tile * kK23TileQuads + h * kK23Threads + tid, p.n, v[h]);
            if (keep_all) {
#pragma unroll
                for (int h = 0; h < kK23Quads; ++h) bits[h] = (1u << nv[h]) - 1u;
            } else {
                auto classify_quad = [&](const float(&q)[12], unsigned n) -> unsigned {
                    unsigned b = 0;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        unsigned cw = 0;
                        const int st = (unsigned)e < n ? classify_fast(g, q[3 * e], q[3 * e + 1], q[3 * e + 2], cw) : 0;
                        b |= (st == 1 ? 1u : 0u) << e;
                        // slow points of this element, one at a time by the whole warp
                        for (unsigned slow = __ballot_sync(kFull, st == 2); slow; slow &= slow - 1u) {
                            const int src = __ffs(slow) - 1;
                            const float sx = __shfl_sync(kFull, q[3 * e], src);
                            const float sy = __shfl_sync(kFull, q[3 * e + 1], src);
                            const float sz = __shfl_sync(kFull, q[3 * e + 2], src);
                            const unsigned sw = __shfl_sync(kFull, cw, src);
                            const bool k = slow_coop(g, sx, sy, sz, cell_mask(g, G, sw), lane, &nexact);
                            if ((int)lane == src && k) b |= 1u << e;
                        }
                    }
                    return b;
                };
#pragma unroll
                for (int h = 0; h < kK23Quads; ++h) bits[h] = classify_quad(v[h], nv[h]);
            }
            // packed scans: word w = quad slots 2w (low half) and 2w+1 (high half)
#pragma unroll
            for (int w = 0; w < kP; ++w) {
                c[w] = (unsigned)__popc(bits[2 * w]) | ((unsigned)__popc(bits[2 * w + 1]) << 16);
                incl[w] = c[w];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned t = __shfl_up_sync(kFull, incl[w], o);
                    if (lane >= (unsigned)o) incl[w] += t;
                }
                if (lane == 31) g.wsum[w][warp] = incl[w];
            }
        }
        // the first warp done with its share of tile k takes the next ticket and
        // resolves the previous tile, while the other warps still classify
        // (its aggregate went out a tile ago, so predecessors are normally
        // published: no spinning), instead of between the two barriers with
        // every other warp waiting
        unsigned first = 0;
        if (lane == 0) first = atomicAdd(&g.done, 1u) == 0u;
        if (__shfl_sync(kFull, first, 0)) {
            if (live && lane == 0) {   // the next tile (read after the barriers)
                const unsigned t = atomicAdd(&p.ws->k2_ticket, 1u);
                g.tile[par ^ 1] = t;
                const unsigned ahead = t + gridDim.x;
                if (VEC && ahead < full_tiles) prefetch_l2(p.pts + 3ull * kK23TilePts * ahead, 12u * kK23TilePts);
            }
            if (have_prev) {
                unsigned total = 0;
#pragma unroll
                for (int w = 0; w < kP; ++w) {
                    const unsigned tot = g.total[par ^ 1][w];
                    total += (tot & 0xffffu) + (tot >> 16);
                }
                const unsigned long long ex = prev_tile == 0 ? 0ull : resolve(p, prev_tile, epoch, lane);
                if (lane == 0) {
                    if (prev_tile != 0) publish(p, prev_tile, kFlagP, ex + total, epoch);
                    g.ex = ex;
                    if (prev_tile == p.num_tiles - 1) p.ws->count = ex + total;
                }
            }
        }
        __syncthreads();
        if (warp == 0) {
            if (lane == 0) g.done = 0u;   // (next counted after the coming barrier)
            if (live) {
                unsigned total = 0;
#pragma unroll
                for (int w = 0; w < kP; ++w) {
                    const unsigned ws = lane < kWarps ? g.wsum[w][lane] : 0u;
                    unsigned wi = ws;
#pragma unroll
                    for (int o = 1; o < kWarps; o <<= 1) {
                        const unsigned t = __shfl_up_sync(kFull, wi, o);
                        if (lane >= (unsigned)o) wi += t;
                    }
                    const unsigned tot = __shfl_sync(kFull, wi, kWarps - 1);
                    if (lane < kWarps) g.wbase[par][w][lane] = wi - ws;
                    if (lane == 0) g.total[par][w] = tot;
                    total += (tot & 0xffffu) + (tot >> 16);
                }
                if (lane == 0) {
                    publish(p, tile, tile == 0 ? kFlagP : kFlagA, total, epoch);
                    if (tile == 0 && tile == p.num_tiles - 1) p.ws->count = total;
                }
            }
        }
        __syncthreads();
        if (have_prev) {   // the previous tile's survivors: coalesced stores from the staging area
            const unsigned long long ex = g.ex;
            unsigned total = 0;
#pragma unroll
            for (int w = 0; w < kP; ++w) {
                const unsigned tot = g.total[par ^ 1][w];
                total += (tot & 0xffffu) + (tot >> 16);
            }
            const long long gbase = p.base + (long long)prev_tile * kK23TilePts;
            const unsigned long long cap = p.capacity > ex ? p.capacity - ex : 0ull;
            const unsigned lim = (unsigned)(cap < total ? cap : total);
            for (unsigned j = tid; j < lim; j += kK23Threads) p.out_idx[ex + j] = gbase + g.sidx[j];
            if (p.out_pts) {   // xyz: a scalar head up to 16-byte alignment, then float4 stores
                float* o = p.out_pts + 3ull * ex;
                const unsigned nfl = 3u * lim;
                unsigned h = (unsigned)((16u - ((uintptr_t)o & 15u)) & 15u) / 4u;
                if (h > nfl) h = nfl;
                if (tid < h) o[tid] = g.spts[tid];
                const unsigned nb = (nfl - h) / 4u;
                float4* o4 = reinterpret_cast<float4*>(o + h);
                for (unsigned j = tid; j < nb; j += kK23Threads) {
                    const unsigned s0 = h + 4u * j;
                    o4[j] = make_float4(g.spts[s0], g.spts[s0 + 1], g.spts[s0 + 2], g.spts[s0 + 3]);
                }
                const unsigned t0 = h + 4u * nb;
                if (tid < nfl - t0) o[t0 + tid] = g.spts[t0 + tid];
            }
        }
        if (!live) break;
        __syncthreads();   // the staging area is free
        {
            unsigned slot_base = 0;
#pragma unroll
            for (int h = 0; h < kK23Quads; ++h) {
                const int w = h >> 1, sh = 16 * (h & 1);
                const unsigned wb = (g.wbase[par][w][warp] >> sh) & 0xffffu;
                const unsigned ex = ((incl[w] - c[w]) >> sh) & 0xffffu;
                stage(g, v[h], bits[h], h * kK23Threads + tid, slot_base + wb + ex);
                slot_base += (g.total[par][w] >> sh) & 0xffffu;
            }
        }
        have_prev = true;
        prev_tile = tile;
        par ^= 1;
    }
    nexact = __reduce_add_sync(kFull, nexact);
    if (lane == 0 && nexact) atomicAdd(&p.ws->k2_exact, nexact);
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(&p.ws->k2_done, 1u) == gridDim.x - 1u) {   // last block out: reset for the next call
            p.ws->k2_ticket = 0u;
            p.ws->k2_done = 0u;
            p.ws->epoch = (epoch + 1u) & kEpochMask;
            __threadfence();
        }
    }
}

}  // namespace

int launch_filter3(const K23Params& p, void* stream, int* launches) {
    unsigned blocks = (unsigned)device_sm_count() * kK23BlocksPerSM;
    if (blocks > p.num_tiles) blocks = p.num_tiles;
    if (blocks == 0) blocks = 1;
    cudaStream_t s = (cudaStream_t)stream;
    static std::once_flag once[kMaxDevices];
    static int done[kMaxDevices];
    per_device(once, done, [] {   // the staging area takes the block past the 48 KB static limit (per device)
        cudaFuncSetAttribute(k2_filter3<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem3));
        cudaFuncSetAttribute(k2_filter3<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem3));
        return 1;
    });
    if (p.vec)
        k2_filter3<true><<<blocks, kK23Threads, sizeof(Smem3), s>>>(p);
    else
        k2_filter3<false><<<blocks, kK23Threads, sizeof(Smem3), s>>>(p);
    *launches += 1;
    return (int)cudaGetLastError();
}

}  // namespace cudapre
