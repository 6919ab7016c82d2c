// api3.cpp — the C ABI of the 3D extension (include/cudapre.h, "The 3D
// extension"): argument checks, workspace, launches, host
// Step 2, transfers.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "exact3.cuh"
#include "internal3.h"

using namespace cudapre;

namespace {

cudapre_status fail3(cudapre_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    return api_fail(st, buf);
}

#define CUDA_TRY3(expr)                                                                      \
    do {                                                                                     \
        cudaError_t e_ = (cudaError_t)(expr);                                                \
        if (e_ != cudaSuccess)                                                               \
            return fail3(CUDAPRE_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                         __FILE__, __LINE__);                                                \
    } while (0)

Ws3Header* ws3_header(void* d_ws) { return reinterpret_cast<Ws3Header*>(d_ws); }
K3Geom* ws3_geom(void* d_ws) { return reinterpret_cast<K3Geom*>(reinterpret_cast<char*>(d_ws) + kWs3HeaderBytes); }
K13Partial* ws3_partials(void* d_ws) {
    return reinterpret_cast<K13Partial*>(reinterpret_cast<char*>(d_ws) + kWs3HeaderBytes + kWs3GeomBytes);
}
unsigned long long* ws3_status(void* d_ws) {
    return reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(d_ws) + kWs3FixedBytes);
}

cudapre_status check_pts3(const float* d_xyz, int64_t n) {
    if (n < 0) return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "n_local < 0");
    if (n >= (int64_t)0xffffffffLL) return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "n_local >= 2^32 (shard the input)");
    if (n > 0 && !d_xyz) return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "d_xyz is NULL");
    if (((uintptr_t)d_xyz & 3u) != 0) return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "d_xyz not 4-byte aligned");
    return CUDAPRE_OK;
}

cudapre_status check_ws3(void* d_ws, size_t ws_bytes, int64_t n) {
    if (!d_ws) return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "d_ws is NULL");
    if (((uintptr_t)d_ws & 255u) != 0) return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "d_ws not 256-byte aligned");
    if (ws_bytes < ws3_bytes_for(n))
        return fail3(CUDAPRE_ERR_WORKSPACE, "workspace %zu bytes < cudapre3_workspace_bytes = %zu", ws_bytes,
                     ws3_bytes_for(n));
    return CUDAPRE_OK;
}

// CUDA events around one launch (per host thread, created on first use)
struct Timer3 {
    static thread_local cudaEvent_t ev[2];
    cudaError_t start(cudaStream_t s) {
        if (!ev[0]) {
            cudaError_t e = cudaEventCreate(&ev[0]);
            if (e == cudaSuccess) e = cudaEventCreate(&ev[1]);
            if (e != cudaSuccess) return e;
        }
        return cudaEventRecord(ev[0], s);
    }
    cudaError_t stop(cudaStream_t s, double* ms) {
        cudaError_t e = cudaEventRecord(ev[1], s);
        if (e == cudaSuccess) e = cudaEventSynchronize(ev[1]);
        float f = 0.f;
        if (e == cudaSuccess) e = cudaEventElapsedTime(&f, ev[0], ev[1]);
        *ms = f;
        return e;
    }
};
thread_local cudaEvent_t Timer3::ev[2] = {nullptr, nullptr};

void empty_result3(cudapre3_extremes_t* r, int nang, const double* c, const double* s) {
    std::memset(r, 0, sizeof(*r));
    r->nang = nang;
    for (int k = 0; k < CUDAPRE3_MAX_SLOTS; ++k) r->idx[k] = -1;
    for (int k = 0; k < nang; ++k) r->c[k] = c[k], r->s[k] = s[k];
}

}  // namespace

extern "C" {

size_t cudapre3_workspace_bytes(int64_t n_local) { return ws3_bytes_for(n_local < 0 ? 0 : n_local); }

int32_t cudapre3_orient(const float* a, const float* b, const float* c, const float* d) {
    return orient3d_sign_f(a, b, c, d);
}

cudapre_status cudapre3_extremes(const float* d_xyz, int64_t n_local, int64_t index_base, int32_t nang,
                                 const double* c, const double* s, void* d_ws, size_t ws_bytes, void* stream,
                                 cudapre3_extremes_t* d_out, cudapre3_extremes_t* h_out, double* h_ms_kernel) {
    api_fail(CUDAPRE_OK, "");
    double c0[CUDAPRE_MAX_ANGLES], s0[CUDAPRE_MAX_ANGLES];
    if (!c || !s) {
        int32_t na = 0;
        cudapre_angles_preset(0, &na, c0, s0);
        nang = na;
        c = c0;
        s = s0;
    }
    if (!(nang == 1 || nang == 2 || nang == 3 || nang == 4 || nang == 8))
        return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "nang=%d not in {1,2,3,4,8}", nang);
    if (c[0] != 1.0 || s[0] != 0.0)
        return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "the first angle must be 0 degrees (c=1, s=0)");
    for (int k = 0; k < nang; ++k)
        if (!(c[k] >= -1.0 && c[k] <= 1.0 && s[k] >= -1.0 && s[k] <= 1.0))
            return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "angle %d: |c|,|s| must be <= 1", k);
    cudapre_status st = check_pts3(d_xyz, n_local);
    if (st) return st;
    cudaStream_t strm = (cudaStream_t)stream;
    if (h_ms_kernel) *h_ms_kernel = 0.0;
    if (n_local == 0) {
        cudapre3_extremes_t r;
        empty_result3(&r, nang, c, s);
        if (h_out) *h_out = r;
        if (d_out) {
            CUDA_TRY3(cudaMemcpyAsync(d_out, &r, sizeof(r), cudaMemcpyHostToDevice, strm));
            CUDA_TRY3(cudaStreamSynchronize(strm));
        }
        return fail3(CUDAPRE_ERR_EMPTY_INPUT, "empty input (n_local == 0)");
    }
    st = check_ws3(d_ws, ws_bytes, n_local);
    if (st) return st;
    K13Params p;
    std::memset(&p, 0, sizeof(p));
    p.pts = d_xyz;
    p.n = (unsigned)n_local;
    p.vec = (((uintptr_t)d_xyz & 15u) == 0);
    p.base = index_base;
    p.ws = ws3_header(d_ws);
    p.partials = ws3_partials(d_ws);
    p.nang = nang;
    for (int k = 0; k < nang; ++k) {
        p.c[k] = c[k];
        p.s[k] = s[k];
        p.cf[k] = (float)c[k];
        p.sf[k] = (float)s[k];
        p.nsf[k] = -(float)s[k];
    }
    int launches = 0;
    Timer3 tm;
    if (h_ms_kernel) CUDA_TRY3(tm.start(strm));
    CUDA_TRY3(launch_extremes3(p, stream, &launches));
    if (h_ms_kernel) CUDA_TRY3(tm.stop(strm, h_ms_kernel));
    if (d_out) CUDA_TRY3(cudaMemcpyAsync(d_out, &p.ws->result, sizeof(cudapre3_extremes_t),
                                         cudaMemcpyDeviceToDevice, strm));
    if (h_out) {
        void* stage = nullptr;
        size_t sb = 0;
        st = api_staging(&stage, &sb);
        if (st) return st;
        CUDA_TRY3(cudaMemcpyAsync(stage, &p.ws->result, sizeof(cudapre3_extremes_t), cudaMemcpyDeviceToHost,
                                  strm));
        CUDA_TRY3(cudaStreamSynchronize(strm));
        std::memcpy(h_out, stage, sizeof(cudapre3_extremes_t));
        if (h_out->nonfinite)
            return fail3(CUDAPRE_ERR_NONFINITE_INPUT, "non-finite coordinate in the input (result flagged)");
    }
    return CUDAPRE_OK;
}

cudapre_status cudapre3_extremes_merge(const cudapre3_extremes_t* h_parts, int32_t count,
                                       cudapre3_extremes_t* h_out) {
    api_fail(CUDAPRE_OK, "");
    if (!h_parts || !h_out || count <= 0) return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "bad merge arguments");
    const int rc = merge_extremes3(h_parts, count, h_out);
    if (rc == CUDAPRE_ERR_EMPTY_INPUT) return fail3(CUDAPRE_ERR_EMPTY_INPUT, "no point in any part");
    if (rc) return fail3((cudapre_status)rc, "parts disagree on the angle count");
    return CUDAPRE_OK;
}

cudapre_status cudapre3_polyhedron(const cudapre3_extremes_t* h_ext, cudapre3_polyhedron_t* h_poly) {
    api_fail(CUDAPRE_OK, "");
    if (!h_ext || !h_poly) return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "NULL argument");
    static thread_local K3Geom g;
    const int rc = build_polyhedron3(*h_ext, h_poly, &g);
    if (rc) return fail3((cudapre_status)rc, "polyhedron build failed");
    return CUDAPRE_OK;
}

cudapre_status cudapre3_cells(const cudapre3_extremes_t* h_ext, uint64_t* h_masks, int32_t n_cells,
                              float* h_centre, int32_t* h_grid, int32_t* h_cells) {
    api_fail(CUDAPRE_OK, "");
    if (!h_ext || !h_grid || !h_cells) return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "NULL argument");
    *h_grid = kCellG;
    if (!h_masks) return CUDAPRE_OK;
    if (n_cells < kCells) return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "n_cells < %d", kCells);
    static thread_local K3Geom g;
    const int rc = build_polyhedron3(*h_ext, nullptr, &g);
    if (rc) return fail3((cudapre_status)rc, "polyhedron build failed");
    *h_cells = (g.mode == 0 && g.cells) ? 1 : 0;
    if (h_centre) h_centre[0] = g.ox, h_centre[1] = g.oy, h_centre[2] = g.oz;
    for (int c = 0; c < kCells; ++c) {
        const unsigned w = g.clist[c];
        unsigned long long m = 0;
        if ((w >> 24) > (unsigned)kCellSlots) {
            const unsigned li = w & 0xffffffu;
            m = li == kNoLong ? g.all : g.lmask[li];
        } else {
            for (int k = 0; k < kCellSlots; ++k) {
                const unsigned t = (w >> (8 * k)) & 0xffu;
                if (t < (unsigned)kMax3Facets) m |= 1ull << t;
            }
        }
        h_masks[c] = m;
    }
    return CUDAPRE_OK;
}

cudapre_status cudapre3_planes(const cudapre3_extremes_t* h_ext, float* h_planes, int32_t capacity,
                               int32_t* h_nf) {
    api_fail(CUDAPRE_OK, "");
    if (!h_ext || !h_nf) return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "NULL argument");
    static thread_local K3Geom g;
    const int rc = build_polyhedron3(*h_ext, nullptr, &g);
    if (rc) return fail3((cudapre_status)rc, "polyhedron build failed");
    *h_nf = g.nf;
    if (!h_planes) return CUDAPRE_OK;
    if (capacity < g.nf) return fail3(CUDAPRE_ERR_CAPACITY, "capacity %d < %d facets", capacity, g.nf);
    for (int f = 0; f < g.nf; ++f) {
        h_planes[5 * f] = g.pl[f].x, h_planes[5 * f + 1] = g.pl[f].y;
        h_planes[5 * f + 2] = g.pl[f].z, h_planes[5 * f + 3] = g.pl[f].w;
        h_planes[5 * f + 4] = g.pe[f];
    }
    return CUDAPRE_OK;
}

cudapre_status cudapre3_filter(const float* d_xyz, int64_t n_local, int64_t index_base,
                               const cudapre3_extremes_t* h_ext, int64_t* d_surv_idx, float* d_surv_xyz,
                               int64_t capacity, void* d_ws, size_t ws_bytes, void* stream, int64_t* h_count,
                               cudapre3_polyhedron_t* h_poly, double* h_ms_kernel) {
    return cudapre3_filter_ex(d_xyz, n_local, index_base, h_ext, d_surv_idx, d_surv_xyz, capacity, d_ws, ws_bytes,
                              stream, h_count, h_poly, h_ms_kernel, 0);
}

cudapre_status cudapre3_filter_ex(const float* d_xyz, int64_t n_local, int64_t index_base,
                                  const cudapre3_extremes_t* h_ext, int64_t* d_surv_idx, float* d_surv_xyz,
                                  int64_t capacity, void* d_ws, size_t ws_bytes, void* stream, int64_t* h_count,
                                  cudapre3_polyhedron_t* h_poly, double* h_ms_kernel, int32_t flags) {
    if (flags & ~CUDAPRE3_FLAG_NO_CELLS) return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "unknown flags");
    api_fail(CUDAPRE_OK, "");
    if (!h_ext || !h_count) return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "h_ext / h_count is NULL");
    if (h_ext->nonfinite) return fail3(CUDAPRE_ERR_NONFINITE_INPUT, "the extremes saw a non-finite coordinate");
    cudapre_status st = check_pts3(d_xyz, n_local);
    if (st) return st;
    if (n_local > 0 && !d_surv_idx) return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "d_surv_idx is NULL");
    if (capacity < 0) return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "capacity < 0");
    st = check_ws3(d_ws, ws_bytes, n_local);
    if (st) return st;
    void* stage = nullptr;
    size_t sb = 0;
    st = api_staging(&stage, &sb);
    if (st) return st;
    if (sb < 4096 + sizeof(K3Geom)) return fail3(CUDAPRE_ERR_INVALID_ARGUMENT, "staging buffer too small");
    K3Geom* g = reinterpret_cast<K3Geom*>(static_cast<char*>(stage) + 4096);
    const int rc = build_polyhedron3(*h_ext, h_poly, g, flags);
    if (rc) return fail3((cudapre_status)rc, "polyhedron build failed");
    cudaStream_t strm = (cudaStream_t)stream;
    *h_count = 0;
    if (h_ms_kernel) *h_ms_kernel = 0.0;
    if (n_local == 0) return CUDAPRE_OK;
    CUDA_TRY3(cudaMemcpyAsync(ws3_geom(d_ws), g, sizeof(K3Geom), cudaMemcpyHostToDevice, strm));
    K23Params p;
    std::memset(&p, 0, sizeof(p));
    p.pts = d_xyz;
    p.n = (unsigned)n_local;
    p.vec = (((uintptr_t)d_xyz & 15u) == 0);
    p.base = index_base;
    p.out_idx = reinterpret_cast<long long*>(d_surv_idx);
    p.out_pts = d_surv_xyz;
    p.capacity = (unsigned long long)capacity;
    p.ws = ws3_header(d_ws);
    p.g = ws3_geom(d_ws);
    p.status = ws3_status(d_ws);
    p.num_tiles = (unsigned)ws3_tiles(n_local);
    int launches = 0;
    Timer3 tm;
    if (h_ms_kernel) CUDA_TRY3(tm.start(strm));
    CUDA_TRY3(launch_filter3(p, stream, &launches));
    if (h_ms_kernel) CUDA_TRY3(tm.stop(strm, h_ms_kernel));
    CUDA_TRY3(cudaMemcpyAsync(stage, &p.ws->count, sizeof(unsigned long long), cudaMemcpyDeviceToHost, strm));
    CUDA_TRY3(cudaStreamSynchronize(strm));
    unsigned long long cnt;
    std::memcpy(&cnt, stage, sizeof(cnt));
    *h_count = (int64_t)cnt;
    if ((int64_t)cnt > capacity)
        return fail3(CUDAPRE_ERR_CAPACITY, "%lld survivors > capacity %lld", (long long)cnt, (long long)capacity);
    return CUDAPRE_OK;
}

}  // extern "C"
