// k2_filter3.cu — Step 3 of the 3D extension ("Those points
// locating inside the convex polyhedron must be interior points, and can be
// directly discarded"; DESIGN.md §3 B5, §6.5) as ONE streaming pass:
// classify every point against the polyhedron and stream-compact the
// survivors in ascending index order.
//
// Classification (exact semantics): p is DISCARDED iff orient3d(f, p) > 0
// for every facet plane f.  With the centre o strictly inside (checked
// exactly on the host), the ray from o through p leaves the polyhedron
// through a facet whose face contains the ray's direction, and that
// direction lies in p's closed octant around o — an exact float compare per
// axis.  So p is strictly inside iff it is strictly inside every facet whose
// face meets its octant: the host lists those per octant (conservatively,
// DESIGN.md §6.5), and the kernel tests only them:
//   g = fma(A, x, fma(B, y, fma(C, z, D))), |g - orient3d| <= E over the
//   data bounding box:   g < -E on any entry -> keep;  g > E on all -> discard;
//   otherwise the exact orient3d (exact3.cuh) on the undecided entries.
// Compaction: persistent blocks take 2048-point tiles (24 KiB) from an atomic
// ticket; each thread classifies two quads (8 points); a packed two-half
// block scan orders the survivors; warp 0 resolves the tile's exclusive
// prefix by a decoupled look-back over epoch-tagged status words (one per
// 128-byte line); survivors' int64 index (+ xyz) are written in order.
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

struct Smem3 {
    float4 pl[kMax3Entries];
    float pe[kMax3Entries];
    unsigned char pf[kMax3Entries];
    float fv[kMax3Facets][9];
    int beg[8], end[8];
    float ox, oy, oz;
    int mode;
    unsigned wsum[kWarps];
    unsigned wbase[kWarps];
    unsigned tile;
    unsigned total;
    unsigned long long ex;
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
    constexpr int kPer = 8;
    const unsigned long long PF = (unsigned long long)kFlagP << 32;
    const unsigned long long E = (unsigned long long)(epoch & kEpochMask) << 34;
    unsigned long long ex = 0;
    long long pred = (long long)tile - 1;
    while (pred >= 0) {
        unsigned long long w[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const long long t = pred - (long long)(kPer * lane + k);
            w[k] = (t >= 0) ? ld_status(&p.status[(size_t)t * kStatus3Stride]) : (E | PF);
        }
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
            __nanosleep(64);
            continue;
        }
        unsigned long long v = (lane <= lim) ? sum : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        ex += v;
        if (pmask) break;
        pred -= 32 * kPer;
    }
    return ex;
}

// the exact decision over the candidate entries [b, e) (rare path)
__device__ __noinline__ bool keep_exact(const Smem3& g, float x, float y, float z, int b, int e,
                                        unsigned* nexact) {
    if (!(fabsf(x) <= FLT_MAX && fabsf(y) <= FLT_MAX && fabsf(z) <= FLT_MAX)) return true;
    ++*nexact;
    const float q[3] = {x, y, z};
    for (int t = b; t < e; ++t) {
        const float4 P = g.pl[t];
        const float v = __fmaf_rn(P.x, x, __fmaf_rn(P.y, y, __fmaf_rn(P.z, z, P.w)));
        const float E = g.pe[t];
        if (v < -E) return true;
        if (v > E) continue;
        const float* f = g.fv[g.pf[t]];
        if (orient3d_sign_f(f, f + 3, f + 6, q) <= 0) return true;
    }
    return false;
}

__device__ __forceinline__ bool keep_pt(const Smem3& g, float x, float y, float z, unsigned* nexact) {
    const int o = (x < g.ox ? 1 : 0) | (y < g.oy ? 2 : 0) | (z < g.oz ? 4 : 0);
    const int b = g.beg[o], e = g.end[o];
    bool unsure = false;
    for (int t = b; t < e; ++t) {
        const float4 P = g.pl[t];
        const float v = __fmaf_rn(P.x, x, __fmaf_rn(P.y, y, __fmaf_rn(P.z, z, P.w)));
        const float E = g.pe[t];
        if (v < -E) return true;
        unsure |= !(v > E);
    }
    if (!unsure) return false;
    return keep_exact(g, x, y, z, b, e, nexact);
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
        for (int j = 0; j < 12; ++j) v[j] = (unsigned)(j / 3) < valid ? __ldg(pts + 3u * i0 + j) : 0.0f;
    }
    return valid;
}

__device__ __forceinline__ void emit(const K23Params& p, const float (&v)[12], unsigned bits, unsigned i0,
                                     unsigned long long pos) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if ((bits >> e) & 1u) {
            if (pos < p.capacity) {
                p.out_idx[pos] = p.base + (long long)(i0 + e);
                if (p.out_pts) {
                    float* o = p.out_pts + 3ull * pos;
                    o[0] = v[3 * e], o[1] = v[3 * e + 1], o[2] = v[3 * e + 2];
                }
            }
            ++pos;
        }
    }
}

template <bool VEC>
__global__ void __launch_bounds__(kK23Threads, kK23BlocksPerSM) k2_filter3(const __grid_constant__ K23Params p) {
    __shared__ Smem3 g;
    const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const K3Geom* G = p.g;
    const int nent = G->nent;
    for (int t = tid; t < nent; t += kK23Threads) {
        g.pl[t] = G->pl[t];
        g.pe[t] = G->pe[t];
        g.pf[t] = G->pf[t];
    }
    for (int t = tid; t < G->nf * 9; t += kK23Threads) g.fv[t / 9][t % 9] = G->fv[t / 9][t % 9];
    if (tid < 8) {
        g.beg[tid] = G->oct_start[tid];
        g.end[tid] = G->oct_start[tid + 1];
        if (!G->octants) {   // one list for every octant
            g.beg[tid] = 0;
            g.end[tid] = G->oct_start[1];
        }
    }
    if (tid == 0) {
        g.ox = G->ox, g.oy = G->oy, g.oz = G->oz;
        g.mode = G->mode;
    }
    const unsigned epoch = *(volatile unsigned*)&p.ws->epoch;
    unsigned nexact = 0;
    __syncthreads();
    const bool keep_all = g.mode != 0;

    for (;;) {
        if (tid == 0) g.tile = atomicAdd(&p.ws->k2_ticket, 1u);
        __syncthreads();
        const unsigned tile = g.tile;
        if (tile >= p.num_tiles) break;
        const unsigned q0 = tile * kK23TileQuads + tid, q1 = q0 + kK23Threads;
        float v0[12], v1[12];
        const unsigned n0 = load_quad<VEC>(p.pts, q0, p.n, v0);
        const unsigned n1 = load_quad<VEC>(p.pts, q1, p.n, v1);
        unsigned b0 = 0, b1 = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if ((unsigned)e < n0 && (keep_all || keep_pt(g, v0[3 * e], v0[3 * e + 1], v0[3 * e + 2], &nexact)))
                b0 |= 1u << e;
            if ((unsigned)e < n1 && (keep_all || keep_pt(g, v1[3 * e], v1[3 * e + 1], v1[3 * e + 2], &nexact)))
                b1 |= 1u << e;
        }
        // packed scan: low half = first 256 quads, high half = second 256
        const unsigned c = (unsigned)__popc(b0) | ((unsigned)__popc(b1) << 16);
        unsigned incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(kFull, incl, o);
            if (lane >= (unsigned)o) incl += t;
        }
        if (lane == 31) g.wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const unsigned ws = lane < kWarps ? g.wsum[lane] : 0u;
            unsigned wi = ws;
#pragma unroll
            for (int o = 1; o < kWarps; o <<= 1) {
                const unsigned t = __shfl_up_sync(kFull, wi, o);
                if (lane >= (unsigned)o) wi += t;
            }
            const unsigned tot = __shfl_sync(kFull, wi, kWarps - 1);
            if (lane < kWarps) g.wbase[lane] = wi - ws;
            const unsigned total = (tot & 0xffffu) + (tot >> 16);
            if (lane == 0) {
                g.total = tot;
                publish(p, tile, tile == 0 ? kFlagP : kFlagA, total, epoch);
            }
            const unsigned long long ex = tile == 0 ? 0ull : resolve(p, tile, epoch, lane);
            if (lane == 0) {
                if (tile != 0) publish(p, tile, kFlagP, ex + total, epoch);
                g.ex = ex;
                if (tile == p.num_tiles - 1) p.ws->count = ex + total;
            }
        }
        __syncthreads();
        const unsigned long long ex = g.ex;
        const unsigned wb = g.wbase[warp], lo_tot = g.total & 0xffffu;
        const unsigned excl = incl - c;
        emit(p, v0, b0, 4u * q0, ex + (wb & 0xffffu) + (excl & 0xffffu));
        emit(p, v1, b1, 4u * q1, ex + lo_tot + (wb >> 16) + (excl >> 16));
        __syncthreads();   // g.tile / wsum reuse
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
    if (p.vec)
        k2_filter3<true><<<blocks, kK23Threads, 0, s>>>(p);
    else
        k2_filter3<false><<<blocks, kK23Threads, 0, s>>>(p);
    *launches += 1;
    return (int)cudaGetLastError();
}

}  // namespace cudapre
