// k_hull.cu — the final hull of the survivors on the GPU (
// the paper hands the survivors to Qhull on the host).
//
// The survivors of Step 3 still number ~3 % of the input (C5: 68 M points),
// too many for a host hull.  A second, much finer filter removes almost all
// of them without ever removing a hull vertex:
//   H1  every survivor votes, per pseudo-angle bucket around a centre c
//       strictly inside the Step-2 polygon, for the farthest point of its
//       bucket (one 64-bit atomicMax of (RN(|p-c|^2) bits, position));
//       a gather kernel reads those points;
//   (host) P' = exact hull of those <= 4097 points and the Step-2 vertices —
//       all survivors, so P' lies inside conv(S), and P' contains the Step-2
//       polygon, hence c; per bucket the candidate edges of P' (the same
//       guarded-bucket argument as K2's sector tables, DESIGN.md §6.2/§6.4);
//   H2  a survivor is dropped iff it is strictly inside P' (exact orientation
//       against the bucket's candidate edges), the rest compacted (unordered).
// The host's monotone chain on what is left gives the canonical ring.
#include <cuda_runtime.h>

#include "exact.cuh"
#include "internal.h"

namespace cudapre {
namespace {

constexpr int kHullThreads = 256;

__device__ __forceinline__ float hull_rcp(float a) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    return r;
}

// Bucket b = round(1024 pa) of (dx, dy) = p - c, pa = dy/(|dx|+|dy|) + 1
// (dx >= 0) or 3 - dy/(|dx|+|dy|) (dx < 0), in [0, 4].  One approximate
// reciprocal: |bucket error| < 2^-11 buckets, far inside the host's 1/64
// guard band.
__device__ __forceinline__ unsigned hull_bucket(float dx, float dy) {
    const float t = __fmul_rn(dy, hull_rcp(__fadd_rn(fabsf(dx), fabsf(dy))));
    const bool pos = dx >= 0.0f;
    const float v = __fmaf_rn(t, pos ? 1024.0f : -1024.0f, pos ? 8389632.0f : 8391680.0f);   // 2^23 + 1024 pa
    return min(__float_as_uint(v) - 0x4B000000u, (unsigned)kHullBuckets - 1u);
}

__global__ void __launch_bounds__(kHullThreads) k_hull_votes(const float2* __restrict__ pts, unsigned m, float cx,
                                                          float cy, unsigned long long* __restrict__ gmax) {
    __shared__ unsigned long long smax[kHullBuckets];
    for (int b = threadIdx.x; b < kHullBuckets; b += kHullThreads) smax[b] = 0ull;
    __syncthreads();
    for (unsigned i = blockIdx.x * kHullThreads + threadIdx.x; i < m; i += gridDim.x * kHullThreads) {
        const float2 p = __ldcs(pts + i);
        const float dx = __fadd_rn(p.x, -cx), dy = __fadd_rn(p.y, -cy);
        const float d2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
        const unsigned b = hull_bucket(dx, dy);
        atomicMax(&smax[b], ((unsigned long long)__float_as_uint(d2) << 32) | i);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < kHullBuckets; b += kHullThreads)
        if (smax[b]) atomicMax(&gmax[b], smax[b]);
}

__global__ void k_hull_gather(const float2* __restrict__ pts, const long long* __restrict__ ids,
                              const unsigned long long* __restrict__ gmax, float2* __restrict__ cpts,
                              long long* __restrict__ cids) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= kHullBuckets) return;
    const unsigned long long e = gmax[b];
    if (!e) {
        cids[b] = -1;
        return;
    }
    const unsigned i = (unsigned)e;
    cpts[b] = pts[i];
    cids[b] = ids[i];
}

// table[b] = first candidate edge | count << 16 (count 0: every edge)
__global__ void __launch_bounds__(kHullThreads) k_hull_filter(const float2* __restrict__ pts,
                                                           const long long* __restrict__ ids, unsigned m,
                                                           float cx, float cy, const unsigned* __restrict__ table,
                                                           const float* __restrict__ vx,
                                                           const float* __restrict__ vy, int nv,
                                                           float2* __restrict__ opts, long long* __restrict__ oids,
                                                           unsigned long long* __restrict__ count) {
    const unsigned lane = threadIdx.x & 31;
    for (unsigned base = blockIdx.x * kHullThreads; base < m; base += gridDim.x * kHullThreads) {
        const unsigned i = base + threadIdx.x;
        bool keep = false;
        float2 p = make_float2(0.f, 0.f);
        if (i < m) {
            p = __ldcs(pts + i);
            const float dx = __fadd_rn(p.x, -cx), dy = __fadd_rn(p.y, -cy);
            const unsigned t = table[hull_bucket(dx, dy)];
            int e = (int)(t & 0xffffu);
            const int cnt = (t >> 16) ? (int)(t >> 16) : nv;
            for (int k = 0; k < cnt && !keep; ++k) {
                keep = orient_sign_f(vx[e], vy[e], vx[e + 1], vy[e + 1], p.x, p.y) <= 0;
                e = e + 1 == nv ? 0 : e + 1;
            }
        }
        const unsigned kb = __ballot_sync(0xffffffffu, keep);
        if (kb) {   // warp-aggregated append (order is irrelevant for the hull)
            unsigned long long w0 = 0;
            if (lane == 0) w0 = atomicAdd(count, (unsigned long long)__popc(kb));
            w0 = __shfl_sync(0xffffffffu, w0, 0);
            if (keep) {
                const unsigned long long o = w0 + __popc(kb & ((1u << lane) - 1u));
                opts[o] = p;
                oids[o] = ids[i];
            }
        }
    }
}

}  // namespace

int launch_hull_votes(const cudapre_pt* d_pts, const int64_t* d_ids, int64_t m, float cx, float cy,
                      unsigned long long* gmax, cudapre_pt* cand_pts, int64_t* cand_ids, void* stream,
                      int* launches) {
    cudaStream_t s = (cudaStream_t)stream;
    const int blocks = device_sm_count() * 4;
    k_hull_votes<<<blocks, kHullThreads, 0, s>>>(reinterpret_cast<const float2*>(d_pts), (unsigned)m, cx, cy,
                                                 gmax);
    k_hull_gather<<<(kHullBuckets + 255) / 256, 256, 0, s>>>(
        reinterpret_cast<const float2*>(d_pts), reinterpret_cast<const long long*>(d_ids), gmax,
        reinterpret_cast<float2*>(cand_pts), reinterpret_cast<long long*>(cand_ids));
    *launches += 2;
    return (int)cudaGetLastError();
}

int launch_hull_filter(const cudapre_pt* d_pts, const int64_t* d_ids, int64_t m, float cx, float cy,
                       const unsigned* table, const float* vx, const float* vy, int nv, cudapre_pt* out_pts,
                       int64_t* out_ids, unsigned long long* count, void* stream, int* launches) {
    const int blocks = device_sm_count() * 4;
    k_hull_filter<<<blocks, kHullThreads, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const float2*>(d_pts), reinterpret_cast<const long long*>(d_ids), (unsigned)m, cx, cy,
        table, vx, vy, nv, reinterpret_cast<float2*>(out_pts), reinterpret_cast<long long*>(out_ids), count);
    *launches += 1;
    return (int)cudaGetLastError();
}

}  // namespace cudapre
