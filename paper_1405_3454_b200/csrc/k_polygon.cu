// k_polygon.cu — Step 2 on the device: one block builds the
// polygon and the Step-3 geometry from the Step-1 result K1 left in the
// workspace, so Steps 1-3 run back to back on a stream (and inside one CUDA
// graph) with no host round trip.  The arithmetic is geom.cuh, shared with
// the host builder; this file is compiled with -fmad=false so no
// multiply-add is contracted and both builders agree to the bit.
//
// Parallel phases (256 threads): per-edge coefficients, the 4 x nv corner /
// edge tests of each box-search step (__syncthreads_and), per-edge distance
// bounds, the 2052 sample rays of the sector tables, the 1025 buckets.
// Sequential (thread 0): the monotone chain of <= 32 picks, the disk centre
// check and the final scalars.
#include <cuda_runtime.h>

#include "geom.cuh"
#include "internal.h"

namespace cudapre {
namespace {

constexpr int kGeomThreads = 256;
#ifndef CUDAPRE_GEOM_TIMING
#define CUDAPRE_GEOM_TIMING 0
#endif
#define GT(i) do { if (CUDAPRE_GEOM_TIMING && tid == 0) tmark[i] = clock64(); } while (0)

// d_parts[0..nparts): per-shard Step-1 results (nparts > 1: merged here, slot
// by slot, and the merged result written to *d_merged if not null).
__global__ void __launch_bounds__(kGeomThreads) k_build_geom(const cudapre_extremes_t* d_parts, int nparts,
                                                             cudapre_extremes_t* d_merged,
                                                             cudapre_polygon_t* __restrict__ poly,
                                                             K2Geom* __restrict__ g) {
    using namespace geom;
    __shared__ Work w;
    __shared__ double rs[kS];
    __shared__ int exe[kS];
    // bucket radii as the bit patterns of non-negative doubles (their order =
    // the numeric order), so the vertex / normal corrections are atomics
    __shared__ unsigned long long rbu[CUDAPRE_SECTORS + 1], rou[CUDAPRE_SECTORS + 1];
    __shared__ cudapre_extremes_t ext;
    const int tid = threadIdx.x;
    long long tmark[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    GT(0);
    {   // stage the Step-1 result (one coalesced load per thread) ...
        static_assert(sizeof(cudapre_extremes_t) % 4 == 0 && sizeof(cudapre_extremes_t) / 4 <= kGeomThreads, "ext");
        constexpr int kWords = (int)(sizeof(cudapre_extremes_t) / 4);
        const unsigned* src = reinterpret_cast<const unsigned*>(d_parts);
        if (tid < kWords) reinterpret_cast<unsigned*>(&ext)[tid] = src[tid];
        __syncthreads();
        if (nparts > 1) {   // ... or the merge of the shards' results
            if (tid == 0) merge_header(d_parts, nparts, ext);
            if (tid < 4 * ext.nang) merge_slot(d_parts, nparts, tid, ext);
            __syncthreads();
            if (d_merged && tid < kWords)
                reinterpret_cast<unsigned*>(d_merged)[tid] = reinterpret_cast<const unsigned*>(&ext)[tid];
        }
    }
    GT(8);

    // phase A: warp 0 collects the picks, rank-sorts them under the total
    // (x, y, id) order (= the host's insertion sort) and keeps the first of
    // each run of equal coordinates; lane 0 runs the chain
    __shared__ Pick sp[CUDAPRE_MAX_SLOTS], sd[CUDAPRE_MAX_SLOTS], sh[2 * CUDAPRE_MAX_SLOTS + 1];
    __shared__ int su;
    if (tid < 32) {
        const int slots = 4 * ext.nang;
        const bool valid = tid < slots && ext.idx[tid] >= 0;
        const unsigned vb = __ballot_sync(0xffffffffu, valid);
        const int m = __popc(vb);
        Pick me = {0.f, 0.f, 0};
        if (valid) {
            me = Pick{ext.pt[tid].x, ext.pt[tid].y, (long long)ext.idx[tid]};
            sp[__popc(vb & ((1u << tid) - 1u))] = me;
        }
        __syncwarp();
        const int i = valid ? __popc(vb & ((1u << tid) - 1u)) : -1;   // this lane's pick position
        int rank = 0;
        if (i >= 0)
            for (int j = 0; j < m; ++j) {
                const Pick o = sp[j];
                rank += pick_less(o, me) || (!pick_less(me, o) && j < i);
            }
        __syncwarp();
        if (i >= 0) sp[rank] = me;   // (equal picks are identical: any order is the same array)
        __syncwarp();
        const bool first = tid < m && (tid == 0 || sp[tid].x != sp[tid - 1].x || sp[tid].y != sp[tid - 1].y);
        const unsigned fb = __ballot_sync(0xffffffffu, first);
        if (first) sd[__popc(fb & ((1u << tid) - 1u))] = sp[tid];
        __syncwarp();
        if (tid == 0) {
            su = __popc(fb);
            phase_a_chain(sd, su, sh, w);
            phase_a_tail(ext, w);
            // non-finite or empty Step-1 input (the host API rejects both): keep
            // everything; the caller sees the flags in the Step-1 result
            if (ext.nonfinite || ext.n <= 0) w.degenerate = 1;
        }
    }
    GT(9);
    __syncthreads();
    if (tid == 0) defaults(w, poly, g);
    if (tid <= CUDAPRE_MAX_SLOTS) defaults_item(w, poly, g, tid);
    GT(10);
    for (int b = tid; b <= CUDAPRE_SECTORS; b += kGeomThreads) {
        poly->sector_r2[b] = -1.0f;
        poly->sector_out_r2[b] = INFINITY;
        g->sr2[b] = -1.0f;
        g->sro2[b] = INFINITY;
        g->sedge[b] = 0xffff;
    }
    GT(1);
    if (w.degenerate) return;   // (uniform: w is in shared memory)
    const int nv = w.nv;
    if (tid < nv) phase_b_edge(w, tid);

    // inner box: every thread follows the same (lo, hi) sequence
    if (box_searchable(w)) {
        double lo = 0.0, hi = 1.0;
        const int q = tid >> 5, j = tid & 31;   // corner, edge
        for (int it = 0; it < 16; ++it) {
            const double t = box_t(it, lo, hi);
            float c[4];
            box_corners(w, t, c);
            const bool my = (q < 4 && j < nv) ? box_corner_edge_ok(w, c, q, j) : true;
            const bool ok = __syncthreads_and(my) && c[0] <= c[1] && c[2] <= c[3];
            if (ok) {
                if (tid == 0) {
                    w.have_box = 1;
                    for (int k = 0; k < 4; ++k) w.box[k] = c[k];
                }
                lo = t;
                if (it == 0) break;
            } else {
                hi = t;
            }
        }
    }
    __syncthreads();
    GT(2);
    // inner disk
    if (tid == 0) disk_centre(w);
    __syncthreads();
    if (w.centre_ok && tid < nv) phase_d_edge(w, tid);
    __syncthreads();
    if (tid == 0) disk_finish(w);
    __syncthreads();
    GT(3);
    // sector tables + candidate edges
    if (tid < nv) phase_e_edge(w, tid);
    __syncthreads();
    if (tid == 0) sector_prep_finish(w);
    __syncthreads();
    if (w.sok) {
        GT(4);
        for (int i = tid; i < kS; i += kGeomThreads) phase_f_sample(w, i, rs[i], exe[i]);
        __syncthreads();
        GT(5);
        for (int b = tid; b <= CUDAPRE_SECTORS; b += kGeomThreads) {
            double rb, ro;
            phase_g_init(w, b, rs, rb, ro);
            rbu[b] = __double_as_longlong(rb);
            rou[b] = __double_as_longlong(ro);
        }
        __syncthreads();
        if (tid < nv) {
            const unsigned long long vr = __double_as_longlong(vertex_radius(w, tid));
            for_buckets_of(w.pv[tid], [&](int bb) { atomicMax(&rou[bb], vr); });
        } else if (tid >= 128 && tid - 128 < nv) {
            const int j = tid - 128;
            const unsigned long long dj = __double_as_longlong(w.dj[j]);
            for_buckets_of(w.pn[j], [&](int bb) { atomicMin(&rbu[bb], dj); });
        }
        __syncthreads();
        for (int b = tid; b <= CUDAPRE_SECTORS; b += kGeomThreads) {
            float a2, o2;
            unsigned short se;
            phase_g_finish(w, b, __longlong_as_double(rbu[b]), __longlong_as_double(rou[b]), exe, a2, o2, se);
            poly->sector_r2[b] = a2;
            poly->sector_out_r2[b] = o2;
            g->sr2[b] = a2;
            g->sro2[b] = o2;
            g->sedge[b] = se;
        }
    }
    __syncthreads();
    GT(6);
    if (tid < nv) finish_item(w, poly, g, tid);
    if (tid == 0) finish(w, poly, g);
    GT(7);
    if (CUDAPRE_GEOM_TIMING && tid == 0)
        for (int i = 1; i < 8; ++i) reinterpret_cast<long long*>(g)[-64 + i] = tmark[i] - tmark[i - 1];
    if (CUDAPRE_GEOM_TIMING && tid == 0) {
        reinterpret_cast<long long*>(g)[-64 + 8] = tmark[8] - tmark[0];
        reinterpret_cast<long long*>(g)[-64 + 9] = tmark[9] - tmark[8];
        reinterpret_cast<long long*>(g)[-64 + 10] = tmark[10] - tmark[9];
    }
}

}  // namespace

int launch_build_geom(const cudapre_extremes_t* d_parts, int nparts, cudapre_extremes_t* d_merged,
                      cudapre_polygon_t* d_poly, K2Geom* d_g, void* stream, int* launches) {
    k_build_geom<<<1, kGeomThreads, 0, (cudaStream_t)stream>>>(d_parts, nparts, d_merged, d_poly, d_g);
    ++*launches;
    return (int)cudaGetLastError();
}

}  // namespace cudapre
