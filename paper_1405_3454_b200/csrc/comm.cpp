// comm.cpp — the multi-GPU path of the C ABI (SURVEY §8 a3 / e):
// an in-library NCCL communicator, the cross-rank combine of the Step-1
// results, the sharded Steps 1-3 on the stream, and the collection of the
// survivors (or of per-rank partial hulls) on one rank.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": in a PyTorch process the
// copy PyTorch already loaded, otherwise the system one), so the library has no
// link-time NCCL dependency and every single-GPU entry point works without it;
// the comm entry points return CUDAPRE_ERR_NCCL if it cannot be loaded.
//
// Points are sharded into contiguous global index ranges, rank r holding
// [base_r, base_r + n_r) with base increasing in r.  Every rank runs K1 on its
// shard (global indices via index_base); the 912-byte Step-1 results are
// all-gathered (one ncclAllGather, 912 * world bytes, straight from the
// workspace block K1 wrote, on the caller's stream: capturable in a CUDA
// graph); each rank merges them with the lexicographic (key, global index)
// rule — associative and commutative, so every rank gets the single-GPU
// answer — builds the identical polygon and runs Step 3 on its shard.  The
// survivors of rank r are ascending global indices in [base_r, base_r + n_r),
// so rank order = index order: concatenating them in rank order is the
// single-GPU survivor array.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

using namespace cudapre;

namespace {

struct NcclApi {
    bool ok = false;
    std::string err;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclAllGather) AllGather = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            api.err = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return;
        }
#define LOAD(name)                                                                       \
    api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, "nccl" #name));            \
    if (!api.name) {                                                                     \
        api.err = "libnccl.so.2 lacks nccl" #name;                                       \
        return;                                                                          \
    }
        LOAD(GetUniqueId)
        LOAD(CommInitRank)
        LOAD(CommDestroy)
        LOAD(AllGather)
        LOAD(Send)
        LOAD(Recv)
        LOAD(GroupStart)
        LOAD(GroupEnd)
        LOAD(GetErrorString)
#undef LOAD
        api.ok = true;
    });
    return api;
}

cudapre_status cfail(cudapre_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    return api_fail(st, buf);
}

#define CUDA_TRYC(expr)                                                                     \
    do {                                                                                    \
        cudaError_t e_ = (cudaError_t)(expr);                                               \
        if (e_ != cudaSuccess)                                                              \
            return cfail(CUDAPRE_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                         __FILE__, __LINE__);                                               \
    } while (0)
#define NCCL_TRY(expr)                                                                          \
    do {                                                                                        \
        ncclResult_t r_ = (expr);                                                               \
        if (r_ != ncclSuccess)                                                                  \
            return cfail(CUDAPRE_ERR_NCCL, "%s: %s (%s:%d)", #expr, nccl().GetErrorString(r_),  \
                         __FILE__, __LINE__);                                                   \
    } while (0)

cudapre_status need_nccl() {
    if (!nccl().ok) return cfail(CUDAPRE_ERR_NCCL, "%s", nccl().err.c_str());
    return CUDAPRE_OK;
}

}  // namespace

// int64 words every rank contributes to the exchanges below
constexpr int kRec = 4;

struct cudapre_comm {
    ncclComm_t nc = nullptr;
    int rank = 0, world = 1, device = 0;
    long long* d_counts = nullptr;   // kRec * world int64 exchanged per rank (see gather_survivors), device
    long long* h_counts = nullptr;   // pinned host copy
};

// All-gather of kRec int64 words per rank (v[0..kRec)), read back into
// c->h_counts on every rank.
static cudapre_status exchange_words(cudapre_comm_t* c, const long long* v, cudaStream_t s) {
    for (int k = 0; k < kRec; ++k) c->h_counts[kRec * c->rank + k] = v[k];
    CUDA_TRYC(cudaMemcpyAsync(c->d_counts + kRec * c->rank, c->h_counts + kRec * c->rank, kRec * sizeof(long long),
                              cudaMemcpyHostToDevice, s));
    NCCL_TRY(nccl().AllGather(c->d_counts + kRec * c->rank, c->d_counts, kRec, ncclInt64, c->nc, s));
    CUDA_TRYC(cudaMemcpyAsync(c->h_counts, c->d_counts, kRec * sizeof(long long) * (size_t)c->world,
                              cudaMemcpyDeviceToHost, s));
    CUDA_TRYC(cudaStreamSynchronize(s));
    return CUDAPRE_OK;
}

extern "C" {

cudapre_status cudapre_comm_unique_id(void* h_id) {
    api_fail(CUDAPRE_OK, "");
    if (!h_id) return cfail(CUDAPRE_ERR_INVALID_ARGUMENT, "h_id is NULL");
    cudapre_status st = need_nccl();
    if (st) return st;
    ncclUniqueId id;
    NCCL_TRY(nccl().GetUniqueId(&id));
    std::memcpy(h_id, &id, sizeof(id));
    return CUDAPRE_OK;
}

cudapre_status cudapre_comm_create(const void* h_id, int32_t rank, int32_t world, cudapre_comm_t** out) {
    api_fail(CUDAPRE_OK, "");
    if (!h_id || !out || world < 1 || rank < 0 || rank >= world)
        return cfail(CUDAPRE_ERR_INVALID_ARGUMENT, "bad comm arguments (rank %d, world %d)", rank, world);
    *out = nullptr;
    cudapre_status st = need_nccl();
    if (st) return st;
    ncclUniqueId id;
    std::memcpy(&id, h_id, sizeof(id));
    cudapre_comm_t* c = new cudapre_comm_t;
    c->rank = rank;
    c->world = world;
    c->device = current_device();
    ncclResult_t r = nccl().CommInitRank(&c->nc, world, id, rank);
    if (r != ncclSuccess) {
        delete c;
        return cfail(CUDAPRE_ERR_NCCL, "ncclCommInitRank: %s", nccl().GetErrorString(r));
    }
    if (cudaMalloc(&c->d_counts, kRec * sizeof(long long) * (size_t)world) != cudaSuccess ||
        cudaHostAlloc(&c->h_counts, kRec * sizeof(long long) * (size_t)world, cudaHostAllocPortable) != cudaSuccess) {
        cudapre_comm_destroy(c);
        return cfail(CUDAPRE_ERR_CUDA, "comm buffers");
    }
    *out = c;
    return CUDAPRE_OK;
}

cudapre_status cudapre_comm_destroy(cudapre_comm_t* c) {
    if (!c) return CUDAPRE_OK;
    if (c->nc) nccl().CommDestroy(c->nc);
    if (c->d_counts) cudaFree(c->d_counts);
    if (c->h_counts) cudaFreeHost(c->h_counts);
    delete c;
    return CUDAPRE_OK;
}

cudapre_status cudapre_comm_rank(const cudapre_comm_t* c, int32_t* rank, int32_t* world) {
    if (!c) return cfail(CUDAPRE_ERR_INVALID_ARGUMENT, "comm is NULL");
    if (rank) *rank = c->rank;
    if (world) *world = c->world;
    return CUDAPRE_OK;
}

cudapre_status cudapre_comm_allgather_extremes(cudapre_comm_t* c, const void* d_ws, cudapre_extremes_t* d_parts,
                                               void* stream) {
    api_fail(CUDAPRE_OK, "");
    if (!c || !d_ws || !d_parts) return cfail(CUDAPRE_ERR_INVALID_ARGUMENT, "NULL argument");
    const char* res = reinterpret_cast<const char*>(d_ws) + CUDAPRE_WS_RESULT_OFFSET;
    NCCL_TRY(nccl().AllGather(res, d_parts, sizeof(cudapre_extremes_t), ncclUint8, c->nc, (cudaStream_t)stream));
    return CUDAPRE_OK;
}

cudapre_status cudapre_extremes_comm(const cudapre_pt* d_pts, int64_t n_local, int64_t index_base, int32_t nang,
                                     const double* cc, const double* ss, void* d_ws, size_t ws_bytes,
                                     cudapre_comm_t* c, cudapre_extremes_t* d_parts, void* stream,
                                     cudapre_extremes_t* h_out) {
    if (!c || !d_parts || !h_out) return cfail(CUDAPRE_ERR_INVALID_ARGUMENT, "NULL argument");
    // an empty shard contributes an empty part (every idx = -1), written to the
    // workspace's result block like a K1 result
    cudapre_extremes_t* d_res =
        n_local == 0 ? reinterpret_cast<cudapre_extremes_t*>(reinterpret_cast<char*>(d_ws) + CUDAPRE_WS_RESULT_OFFSET)
                     : nullptr;
    cudapre_status st = cudapre_extremes(d_pts, n_local, index_base, nang, cc, ss, d_ws, ws_bytes, stream, d_res,
                                         nullptr, nullptr);
    if (st && st != CUDAPRE_ERR_EMPTY_INPUT && st != CUDAPRE_ERR_NONFINITE_INPUT) return st;
    st = cudapre_comm_allgather_extremes(c, d_ws, d_parts, stream);
    if (st) return st;
    std::vector<cudapre_extremes_t> parts((size_t)c->world);
    CUDA_TRYC(cudaMemcpyAsync(parts.data(), d_parts, sizeof(cudapre_extremes_t) * parts.size(),
                              cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    CUDA_TRYC(cudaStreamSynchronize((cudaStream_t)stream));
    return cudapre_extremes_merge(parts.data(), c->world, h_out);
}

cudapre_status cudapre_pipeline_comm(const cudapre_pt* d_pts, int64_t n_local, int64_t index_base, int32_t nang,
                                     const double* cc, const double* ss, int64_t* d_surv_idx,
                                     cudapre_pt* d_surv_pts, int64_t capacity, void* d_ws, size_t ws_bytes,
                                     cudapre_comm_t* c, cudapre_extremes_t* d_parts, void* stream,
                                     int64_t* d_count) {
    if (!c || !d_parts || n_local < 0) return cfail(CUDAPRE_ERR_INVALID_ARGUMENT, "bad pipeline_comm arguments");
    // an empty shard takes part in the collective with an empty Step-1 block
    // (every idx = -1: never wins the merge) and has no survivors
    cudapre_extremes_t* d_res =
        n_local == 0 ? reinterpret_cast<cudapre_extremes_t*>(reinterpret_cast<char*>(d_ws) + CUDAPRE_WS_RESULT_OFFSET)
                     : nullptr;
    cudapre_status st = cudapre_extremes(d_pts, n_local, index_base, nang, cc, ss, d_ws, ws_bytes, stream, d_res,
                                         nullptr, nullptr);
    if (st && !(n_local == 0 && st == CUDAPRE_ERR_EMPTY_INPUT)) return st;
    st = cudapre_comm_allgather_extremes(c, d_ws, d_parts, stream);
    if (st) return st;
    st = cudapre_polygon_device(d_parts, c->world, d_ws, ws_bytes, stream, nullptr);
    if (st) return st;
    if (n_local == 0) {
        if (d_count) CUDA_TRYC(cudaMemsetAsync(d_count, 0, sizeof(int64_t), (cudaStream_t)stream));
        return CUDAPRE_OK;
    }
    return cudapre_filter_geom(d_pts, n_local, index_base, d_surv_idx, d_surv_pts, capacity, d_ws, ws_bytes, stream,
                               d_count);
}

cudapre_status cudapre_gather_survivors(cudapre_comm_t* c, const int64_t* d_idx, const cudapre_pt* d_pts,
                                        int64_t count, int32_t root, int64_t* d_out_idx, cudapre_pt* d_out_pts,
                                        int64_t out_capacity, void* stream, int64_t* h_total) {
    api_fail(CUDAPRE_OK, "");
    if (!c || !h_total || root < 0 || root >= c->world)   // (a bad root differs per rank only by misuse)
        return cfail(CUDAPRE_ERR_INVALID_ARGUMENT, "bad gather arguments");
    cudaStream_t s = (cudaStream_t)stream;
    const bool me_root = c->rank == root;
    // 1. all-gather of (count, root capacity, root wants points, this rank's
    //    arguments are usable) per rank: every rank sees the same numbers and
    //    takes the same decision, so an error on one rank never leaves another
    //    blocked in a send or receive
    const bool ok = count >= 0 && (count == 0 || d_idx);
    const long long mine[kRec] = {ok ? count : 0, me_root && d_out_idx ? (long long)out_capacity : 0,
                                  me_root && d_out_pts ? 1 : 0, (ok ? 1 : 0) | (d_pts ? 2 : 0)};
    cudapre_status st = exchange_words(c, mine, s);
    if (st) return st;
    const long long* w = c->h_counts;
    std::vector<long long> off((size_t)c->world + 1, 0);
    bool all_ok = true, pts_ok = true;
    for (int r = 0; r < c->world; ++r) {
        off[r + 1] = off[r] + w[kRec * r];
        all_ok &= (w[kRec * r + 3] & 1) != 0;
        pts_ok &= w[kRec * r] == 0 || (w[kRec * r + 3] & 2) != 0;
    }
    const bool with_pts = w[kRec * root + 2] != 0;   // the root decides: it has a place for them
    *h_total = off[c->world];
    if (!all_ok) return cfail(CUDAPRE_ERR_INVALID_ARGUMENT, "bad gather arguments on some rank (count < 0 or NULL d_idx)");
    if (with_pts && !pts_ok)
        return cfail(CUDAPRE_ERR_INVALID_ARGUMENT, "the root takes points: every rank with survivors must pass d_pts");
    if (off[c->world] > w[kRec * root + 1])
        return cfail(CUDAPRE_ERR_CAPACITY, "%lld survivors > root capacity %lld", off[c->world], w[kRec * root + 1]);
    // 2. the root's own part (a device copy), then grouped point-to-point:
    //    rank r's survivors land at off[r] on the root
    if (me_root && count > 0) {
        CUDA_TRYC(cudaMemcpyAsync(d_out_idx + off[root], d_idx, (size_t)count * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
        if (with_pts)
            CUDA_TRYC(cudaMemcpyAsync(d_out_pts + off[root], d_pts, (size_t)count * sizeof(cudapre_pt),
                                      cudaMemcpyDeviceToDevice, s));
    }
    ncclResult_t r0 = nccl().GroupStart();
    if (me_root) {
        for (int r = 0; r < c->world && r0 == ncclSuccess; ++r) {
            const size_t m = (size_t)w[kRec * r];
            if (!m || r == root) continue;
            r0 = nccl().Recv(d_out_idx + off[r], m, ncclInt64, r, c->nc, s);
            if (r0 == ncclSuccess && with_pts) r0 = nccl().Recv(d_out_pts + off[r], 2 * m, ncclFloat32, r, c->nc, s);
        }
    } else if (count > 0) {
        r0 = nccl().Send(d_idx, (size_t)count, ncclInt64, root, c->nc, s);
        if (r0 == ncclSuccess && with_pts) r0 = nccl().Send(d_pts, 2 * (size_t)count, ncclFloat32, root, c->nc, s);
    }
    const ncclResult_t r1 = nccl().GroupEnd();   // always closed, also after an error inside
    if (r0 != ncclSuccess || r1 != ncclSuccess)
        return cfail(CUDAPRE_ERR_NCCL, "survivor gather: %s", nccl().GetErrorString(r0 != ncclSuccess ? r0 : r1));
    return CUDAPRE_OK;
}

// Final hull of the sharded set: each rank computes the hull ring of
// its own survivors on its GPU (cudapre_hull_device), the rings' vertices
// (ids + points) are gathered on the root, and the root's monotone chain over
// them gives the ring of the whole set: hull(U S_r) = hull(U hull(S_r)), and
// the lowest index among duplicate coordinates wins there as everywhere.
cudapre_status cudapre_hull_comm(cudapre_comm_t* c, const cudapre_pt* d_pts, const int64_t* d_ids, int64_t m,
                                 const cudapre_polygon_t* h_poly, void* d_scratch, size_t scratch_bytes,
                                 int32_t root, void* stream, int64_t* h_ring, int64_t ring_capacity,
                                 int64_t* h_ring_len) {
    api_fail(CUDAPRE_OK, "");
    if (!c || !h_ring_len || root < 0 || root >= c->world)
        return cfail(CUDAPRE_ERR_INVALID_ARGUMENT, "bad hull_comm arguments");
    cudaStream_t s = (cudaStream_t)stream;
    // local ring: ids and coordinates on the host
    std::vector<int64_t> ring((size_t)(m > 0 ? m : 1) + 1);
    std::vector<cudapre_pt> rpt((size_t)(m > 0 ? m : 1) + 1);
    int64_t len = 0, rem = 0;
    const cudapre_status st = cudapre_hull_device_ex(d_pts, d_ids, m, h_poly, d_scratch, scratch_bytes, stream,
                                                     ring.data(), rpt.data(), (int64_t)ring.size(), &len, &rem);
    const std::string local_err = st ? cudapre_last_error() : "";
    // gather (len, ids, points) of every rank on the root through the comm's
    // device buffers: a counts all-gather (a rank whose local hull failed still
    // takes part, with len = -1, so every rank returns the error instead of
    // waiting in a collective), then grouped send / recv
    const bool ring_ok = c->rank != root || (h_ring && ring_capacity >= 0);
    const long long mine[kRec] = {st ? -1 : (long long)len, ring_ok ? 1 : 0, 0, 0};
    cudapre_status xs = exchange_words(c, mine, s);
    if (xs) return xs;
    std::vector<long long> off((size_t)c->world + 1, 0);
    int failed = -1;
    bool root_ok = true;
    for (int r = 0; r < c->world; ++r) {
        const long long k = c->h_counts[kRec * r];
        if (k < 0 && failed < 0) failed = r;
        root_ok &= c->h_counts[kRec * r + 1] != 0;
        off[r + 1] = off[r] + (k > 0 ? k : 0);
    }
    if (st) return cfail(st, "%s", local_err.c_str());
    if (failed >= 0) return cfail(CUDAPRE_ERR_CUDA, "the local hull failed on rank %d", failed);
    if (!root_ok) return cfail(CUDAPRE_ERR_INVALID_ARGUMENT, "h_ring is NULL on the root");
    void* d_buf = nullptr;
    const size_t rec = sizeof(int64_t) + sizeof(cudapre_pt);
    const long long tot = off[c->world];
    CUDA_TRYC(cudaMalloc(&d_buf, rec * (size_t)(tot > 0 ? tot : 1)));
    int64_t* d_gid = reinterpret_cast<int64_t*>(d_buf);
    cudapre_pt* d_gpt = reinterpret_cast<cudapre_pt*>(d_gid + (tot > 0 ? tot : 1));
    if (len > 0) {   // own vertices into place (root) / the send buffer (others)
        CUDA_TRYC(cudaMemcpyAsync(d_gid + off[c->rank], ring.data(), sizeof(int64_t) * (size_t)len,
                                  cudaMemcpyHostToDevice, s));
        CUDA_TRYC(cudaMemcpyAsync(d_gpt + off[c->rank], rpt.data(), sizeof(cudapre_pt) * (size_t)len,
                                  cudaMemcpyHostToDevice, s));
    }
    cudapre_status out = CUDAPRE_OK;
    ncclResult_t r0 = nccl().GroupStart();
    for (int r = 0; r < c->world && r0 == ncclSuccess; ++r) {
        const size_t k = (size_t)c->h_counts[kRec * r];
        if (!k) continue;
        if (c->rank == root && r != root) {
            r0 = nccl().Recv(d_gid + off[r], k, ncclInt64, r, c->nc, s);
            if (r0 == ncclSuccess) r0 = nccl().Recv(d_gpt + off[r], 2 * k, ncclFloat32, r, c->nc, s);
        } else if (c->rank != root && r == c->rank) {
            r0 = nccl().Send(d_gid + off[r], k, ncclInt64, root, c->nc, s);
            if (r0 == ncclSuccess) r0 = nccl().Send(d_gpt + off[r], 2 * k, ncclFloat32, root, c->nc, s);
        }
    }
    const ncclResult_t r1 = nccl().GroupEnd();
    if (r0 != ncclSuccess || r1 != ncclSuccess)
        out = cfail(CUDAPRE_ERR_NCCL, "hull gather: %s", nccl().GetErrorString(r0 != ncclSuccess ? r0 : r1));
    *h_ring_len = 0;
    if (!out && c->rank == root && tot > 0) {
        std::vector<int64_t> gid((size_t)tot);
        std::vector<cudapre_pt> gpt((size_t)tot);
        if (cudaMemcpyAsync(gid.data(), d_gid, sizeof(int64_t) * (size_t)tot, cudaMemcpyDeviceToHost, s) ||
            cudaMemcpyAsync(gpt.data(), d_gpt, sizeof(cudapre_pt) * (size_t)tot, cudaMemcpyDeviceToHost, s) ||
            cudaStreamSynchronize(s)) {
            out = cfail(CUDAPRE_ERR_CUDA, "hull gather copy-back");
        } else {
            std::vector<int64_t> rr((size_t)tot + 1);
            const int64_t k = hull_ring_points(gpt.data(), gid.data(), tot, rr.data(), nullptr);
            if (k > ring_capacity) {
                out = cfail(CUDAPRE_ERR_CAPACITY, "hull of %lld vertices > capacity", (long long)k);
            } else {
                std::memcpy(h_ring, rr.data(), sizeof(int64_t) * (size_t)k);
                *h_ring_len = k;
            }
        }
    } else {
        cudaStreamSynchronize(s);
    }
    cudaFree(d_buf);
    return out;
}

}  // extern "C"
