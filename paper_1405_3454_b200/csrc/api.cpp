// api.cpp — the C ABI (include/cudapre.h): argument checking, workspace
// layout, kernel launches, host Step 2, device<->host transfers, errors.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

using namespace cudapre;

namespace {

thread_local std::string g_err;

cudapre_status fail(cudapre_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

#define CUDA_TRY(expr)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (cudaError_t)(expr);                                              \
        if (e_ != cudaSuccess)                                                             \
            return fail(CUDAPRE_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                               \
    } while (0)

// Small pinned staging buffer per host thread for the 8-byte count and the
// result struct (a pageable destination would force a staged synchronous copy).
// per-thread pinned staging: [0, 4 KiB) small D2H results, [4 KiB, ...) the
// host-built Step-3 geometry on its way to the workspace
constexpr size_t kStageGeomOff = 4096;
constexpr size_t kStageBytes = kStageGeomOff + 65536;   // either dimension's geometry page (2D 32 KiB, 3D 64 KiB)
struct Staging {
    void* p = nullptr;
    cudaEvent_t busy = nullptr;   // recorded after an H2D from p that the call did not wait for
    bool pending = false;
    ~Staging() {
        if (p) cudaFreeHost(p);
        if (busy) cudaEventDestroy(busy);
    }
};
thread_local Staging g_stage;

// The calling thread's pinned staging buffer, free to overwrite: a copy out
// of it that an earlier call left in flight (cudapre_pipeline_host returns
// without waiting, and the next call may use another stream) is waited for.
cudapre_status staging(void** out) {
    if (!g_stage.p) CUDA_TRY(cudaHostAlloc(&g_stage.p, kStageBytes, cudaHostAllocPortable));
    if (g_stage.pending) {
        CUDA_TRY(cudaEventSynchronize(g_stage.busy));
        g_stage.pending = false;
    }
    *out = g_stage.p;
    return CUDAPRE_OK;
}
// mark the staging buffer in use by work enqueued on strm
cudapre_status staging_in_flight(cudaStream_t strm) {
    if (!g_stage.busy) CUDA_TRY(cudaEventCreateWithFlags(&g_stage.busy, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(g_stage.busy, strm));
    g_stage.pending = true;
    return CUDAPRE_OK;
}

// Per-thread mapped pinned block the Step-1 result is written to by K1's
// last block directly (cudapre_pipeline_host: no copy call between the kernels).
struct Mapped {
    void* h = nullptr;
    void* d = nullptr;
    ~Mapped() {
        if (h) cudaFreeHost(h);
    }
};
thread_local Mapped g_mapped;

cudapre_status mapped_block(void** h, void** d) {
    if (!g_mapped.h) {
        CUDA_TRY(cudaHostAlloc(&g_mapped.h, 4096, cudaHostAllocMapped | cudaHostAllocPortable));
        CUDA_TRY(cudaHostGetDevicePointer(&g_mapped.d, g_mapped.h, 0));
    }
    *h = g_mapped.h;
    *d = g_mapped.d;
    return CUDAPRE_OK;
}

// Per-thread timing events (created on first use).
struct Events {
    cudaEvent_t e[4] = {nullptr, nullptr, nullptr, nullptr};
    ~Events() {
        for (auto& x : e)
            if (x) cudaEventDestroy(x);
    }
};
thread_local Events g_ev;

cudapre_status events(cudaEvent_t** out) {
    if (!g_ev.e[0])
        for (auto& x : g_ev.e) CUDA_TRY(cudaEventCreate(&x));
    *out = g_ev.e;
    return CUDAPRE_OK;
}

// Correctly rounded coefficients (reading A5): the binary64 nearest to the
// exact cos/sin of each angle.  Typed from the closed forms sqrt(3)/2,
// sqrt(2)/2, sqrt(2 +- sqrt(2))/2, (sqrt(6) +- sqrt(2))/4 (tests/test_abi.py checks them against
// 80-digit decimal evaluations).
struct Coef {
    double deg, c, s;
};
const Coef kCoef[] = {
    {0.0, 1.0, 0.0},
    {15.0, 0x1.ee8dd4748bf15p-1, 0x1.0907dc1930690p-2},   // (sqrt6 +- sqrt2)/4
    {22.5, 0x1.d906bcf328d46p-1, 0x1.87de2a6aea963p-2},
    {30.0, 0x1.bb67ae8584caap-1, 0x1.0p-1},
    {45.0, 0x1.6a09e667f3bcdp-1, 0x1.6a09e667f3bcdp-1},
    {60.0, 0x1.0p-1, 0x1.bb67ae8584caap-1},
    {67.5, 0x1.87de2a6aea963p-2, 0x1.d906bcf328d46p-1},
    {75.0, 0x1.0907dc1930690p-2, 0x1.ee8dd4748bf15p-1},
};

void preset_coef(double deg, double* c, double* s) {
    for (const Coef& k : kCoef)
        if (k.deg == deg) {
            *c = k.c;
            *s = k.s;
            return;
        }
}

WsHeader* ws_header(void* d_ws) { return reinterpret_cast<WsHeader*>(d_ws); }
static_assert(CUDAPRE_WS_GEOM_OFFSET == kWsHeaderBytes && CUDAPRE_WS_POLY_OFFSET == kWsHeaderBytes + kWsPolyOff &&
                  CUDAPRE_WS_RESULT_OFFSET == offsetof(WsHeader, result),
              "workspace page offsets in include/cudapre.h");
K2Geom* ws_geom(void* d_ws) { return reinterpret_cast<K2Geom*>(reinterpret_cast<char*>(d_ws) + kWsHeaderBytes); }
cudapre_polygon_t* ws_poly(void* d_ws) {
    return reinterpret_cast<cudapre_polygon_t*>(reinterpret_cast<char*>(d_ws) + kWsHeaderBytes + kWsPolyOff);
}
K1Partial* ws_partials(void* d_ws) {
    return reinterpret_cast<K1Partial*>(reinterpret_cast<char*>(d_ws) + kWsFixedBytes);
}
unsigned long long* ws_status(void* d_ws) {
    return reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(d_ws) + kWsFixedBytes +
                                                 kWsPartialBytes);
}
// The overflow scratch sits at the END of the caller's workspace: the
// tile-status words start at a fixed offset and are epoch-tagged across calls,
// so a workspace reused for a smaller n must never write scratch data where a
// larger n's status words live (status(n) grows from the front, scratch from
// the back; ws_bytes >= ws_bytes_for(n) keeps them apart).
SurvEntry* ws_scratch(void* d_ws, size_t ws_bytes, int64_t n, unsigned* blocks) {
    const size_t used = kWsFixedBytes + kWsPartialBytes + ws_status_bytes(n);
    size_t nb = ws_bytes > used + 16 ? (ws_bytes - used - 16) / kK2ScratchPerBlock : 0;
    const size_t want = (size_t)kK2BlocksPerSM * (size_t)device_sm_count();
    if (nb > want) nb = want;
    *blocks = (unsigned)nb;
    const size_t off = (ws_bytes - nb * kK2ScratchPerBlock) & ~(size_t)15;
    return reinterpret_cast<SurvEntry*>(reinterpret_cast<char*>(d_ws) + off);
}

cudapre_status check_points(const cudapre_pt* d_pts, int64_t n) {
    if (n < 0 || n > (int64_t)0xffffffffll)
        return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "n_local=%lld out of range [0, 2^32-1]", (long long)n);
    if (n > 0 && !d_pts) return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "d_pts is NULL");
    if (((uintptr_t)d_pts & 7u) != 0)
        return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "d_pts must be 8-byte aligned");
    return CUDAPRE_OK;
}

cudapre_status check_ws(void* d_ws, size_t ws_bytes, int64_t n) {
    if (!d_ws || ((uintptr_t)d_ws & 15u) != 0)
        return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "d_ws must be a 16-byte aligned device pointer");
    if (ws_bytes < ws_bytes_for(n))
        return fail(CUDAPRE_ERR_WORKSPACE, "workspace %zu B < %zu B needed for n=%lld", ws_bytes,
                    ws_bytes_for(n), (long long)n);
    return CUDAPRE_OK;
}

void empty_result(cudapre_extremes_t* r, int nang, const double* c, const double* s) {
    std::memset(r, 0, sizeof(*r));
    r->nang = nang;
    for (int k = 0; k < CUDAPRE_MAX_SLOTS; ++k) r->idx[k] = -1;
    for (int k = 0; k < nang; ++k) {
        r->c[k] = c[k];
        r->s[k] = s[k];
    }
}

// K2 parameters that do not depend on the polygon (the geometry is read from
// the workspace's geometry page, p.g)
void k2_params(K2Params& p, const cudapre_pt* d_pts, int64_t n_local, int64_t index_base, int64_t* d_surv_idx,
               cudapre_pt* d_surv_pts, int64_t capacity, void* d_ws, size_t ws_bytes) {
    p.pts = reinterpret_cast<const float*>(d_pts);
    p.n = (unsigned)n_local;
    p.base = index_base;
    p.out_idx = reinterpret_cast<long long*>(d_surv_idx);
    p.out_pts = reinterpret_cast<float*>(d_surv_pts);
    p.capacity = (unsigned long long)(capacity < 0 ? 0 : capacity);
    p.ws = ws_header(d_ws);
    p.status = ws_status(d_ws);
    p.scratch = ws_scratch(d_ws, ws_bytes, n_local, &p.scratch_blocks);
    p.num_tiles = (unsigned)((n_local + kK2TilePts - 1) / kK2TilePts);
    p.g = ws_geom(d_ws);
    p.edges = 32;
}

}  // namespace

namespace cudapre {   // hooks for api3.cpp (the 3D ABI)
cudapre_status api_fail(cudapre_status st, const char* msg) { return fail(st, "%s", msg); }
cudapre_status api_staging(void** out, size_t* bytes) {
    *bytes = kStageBytes;
    return staging(out);
}
}  // namespace cudapre

extern "C" {

const char* cudapre_version(void) { return "cudapre-b200 0.1.0 (sm_100a)"; }

const char* cudapre_last_error(void) { return g_err.c_str(); }

cudapre_status cudapre_angles_preset(int preset, int32_t* nang, double* c, double* s) {
    static const double lists[5][8] = {{0.0, 30.0, 45.0, 60.0},
                                       {0.0, 30.0, 45.0, 45.0},
                                       {0.0},
                                       {0.0, 22.5, 45.0, 67.5},
                                       {0.0, 15.0, 22.5, 30.0, 45.0, 60.0, 67.5, 75.0}};
    static const int counts[5] = {4, 4, 1, 4, 8};
    if (preset < 0 || preset > 4 || !nang || !c || !s)
        return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "unknown angle preset %d", preset);
    *nang = counts[preset];
    for (int k = 0; k < CUDAPRE_MAX_ANGLES; ++k) c[k] = s[k] = 0.0;
    for (int k = 0; k < counts[preset]; ++k) preset_coef(lists[preset][k], &c[k], &s[k]);
    return CUDAPRE_OK;
}

size_t cudapre_workspace_bytes(int64_t n_local) { return ws_bytes_for(n_local < 0 ? 0 : n_local); }

cudapre_status cudapre_workspace_init(void* d_ws, size_t ws_bytes, void* stream) {
    if (!d_ws) return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "d_ws is NULL");
    CUDA_TRY(cudaMemsetAsync(d_ws, 0, ws_bytes, (cudaStream_t)stream));
    return CUDAPRE_OK;
}

cudapre_status cudapre_extremes(const cudapre_pt* d_pts, int64_t n_local, int64_t index_base,
                                int32_t nang, const double* c, const double* s, void* d_ws,
                                size_t ws_bytes, void* stream, cudapre_extremes_t* d_out,
                                cudapre_extremes_t* h_out, cudapre_report_t* h_rep) {
    g_err.clear();
    double c0[CUDAPRE_MAX_ANGLES], s0[CUDAPRE_MAX_ANGLES];
    if (!c || !s) {
        int32_t na = 0;
        cudapre_angles_preset(0, &na, c0, s0);
        nang = na;
        c = c0;
        s = s0;
    }
    if (!(nang == 1 || nang == 2 || nang == 3 || nang == 4 || nang == 8))
        return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "nang=%d not in {1,2,3,4,8}", nang);
    if (c[0] != 1.0 || s[0] != 0.0)
        return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "the first angle must be 0 degrees (c=1, s=0)");
    for (int k = 0; k < nang; ++k)
        if (!(c[k] >= -1.0 && c[k] <= 1.0 && s[k] >= -1.0 && s[k] <= 1.0))
            return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "angle %d: |c|,|s| must be <= 1", k);
    cudapre_status st = check_points(d_pts, n_local);
    if (st) return st;
    if (h_rep) std::memset(h_rep, 0, sizeof(*h_rep));
    cudaStream_t strm = (cudaStream_t)stream;
    if (n_local == 0) {
        cudapre_extremes_t r;
        empty_result(&r, nang, c, s);
        if (h_out) *h_out = r;
        if (d_out) {
            CUDA_TRY(cudaMemcpyAsync(d_out, &r, sizeof(r), cudaMemcpyHostToDevice, strm));
            CUDA_TRY(cudaStreamSynchronize(strm));
        }
        return fail(CUDAPRE_ERR_EMPTY_INPUT, "empty input (n_local == 0)");
    }
    st = check_ws(d_ws, ws_bytes, n_local);
    if (st) return st;

    K1Params p;
    std::memset(&p, 0, sizeof(p));
    p.pts = reinterpret_cast<const float*>(d_pts);
    p.n = (unsigned)n_local;
    p.nang = nang;
    p.base = index_base;
    for (int k = 0; k < nang; ++k) {
        p.c[k] = c[k];
        p.s[k] = s[k];
        p.cf[k] = (float)c[k];
        p.sf[k] = (float)s[k];
        p.nsf[k] = -(float)s[k];
    }
    p.ws = ws_header(d_ws);
    p.partials = ws_partials(d_ws);
    p.d_out = d_out;
    if (n_local >= 65536) {
        int64_t ch = n_local / 16384;
        p.seed_chunks = (unsigned)(ch < 16 ? 16 : (ch > 4096 ? 4096 : ch));
    }
    // 16-B aligned input: the warp-specialised cp.async.bulk ring; 8-B
    // aligned: register double-buffered loads
    const int vec16 = (((uintptr_t)d_pts & 15u) == 0);
    cudaEvent_t* ev = nullptr;
    if (h_rep) {
        st = events(&ev);
        if (st) return st;
        CUDA_TRY(cudaEventRecord(ev[0], strm));
    }
    int launches = 0;
    CUDA_TRY(launch_extremes(p, vec16, stream, &launches));
    if (h_rep) CUDA_TRY(cudaEventRecord(ev[1], strm));
    if (h_out) {
        void* stage = nullptr;
        st = staging(&stage);
        if (st) return st;
        CUDA_TRY(cudaMemcpyAsync(stage, &p.ws->result, sizeof(cudapre_extremes_t),
                                 cudaMemcpyDeviceToHost, strm));
        CUDA_TRY(cudaStreamSynchronize(strm));
        std::memcpy(h_out, stage, sizeof(cudapre_extremes_t));
    }
    if (h_rep) {
        float ms = 0.f;
        CUDA_TRY(cudaEventSynchronize(ev[1]));
        CUDA_TRY(cudaEventElapsedTime(&ms, ev[0], ev[1]));
        h_rep->n = n_local;
        h_rep->ms_extremes_kernels = ms;
        h_rep->launches = launches;
    }
    if (h_out && h_out->nonfinite)
        return fail(CUDAPRE_ERR_NONFINITE_INPUT, "non-finite coordinate in the input");
    return CUDAPRE_OK;
}

cudapre_status cudapre_extremes_merge(const cudapre_extremes_t* h_parts, int32_t count,
                                      cudapre_extremes_t* h_out) {
    g_err.clear();
    if (!h_parts || count < 1 || !h_out)
        return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "need >= 1 part and an output");
    for (int p = 1; p < count; ++p)
        if (h_parts[p].nang != h_parts[0].nang)
            return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "parts use different angle lists");
    merge_extremes(h_parts, count, h_out);
    if (h_out->n == 0) return fail(CUDAPRE_ERR_EMPTY_INPUT, "empty input (all parts empty)");
    if (h_out->nonfinite) return fail(CUDAPRE_ERR_NONFINITE_INPUT, "non-finite coordinate in the input");
    return CUDAPRE_OK;
}

cudapre_status cudapre_polygon(const cudapre_extremes_t* h_ext, cudapre_polygon_t* h_poly) {
    g_err.clear();
    if (!h_ext || !h_poly) return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "NULL argument");
    if (h_ext->n <= 0) return fail(CUDAPRE_ERR_EMPTY_INPUT, "empty input");
    if (h_ext->nang < 1 || h_ext->nang > CUDAPRE_MAX_ANGLES)
        return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "bad nang in extremes");
    build_polygon(*h_ext, h_poly, nullptr);
    return CUDAPRE_OK;
}

cudapre_status cudapre_filter(const cudapre_pt* d_pts, int64_t n_local, int64_t index_base,
                              const cudapre_extremes_t* h_ext, int64_t* d_surv_idx,
                              cudapre_pt* d_surv_pts, int64_t capacity, void* d_ws, size_t ws_bytes,
                              void* stream, int64_t* h_count, cudapre_polygon_t* h_poly,
                              cudapre_report_t* h_rep) {
    g_err.clear();
    cudapre_status st = check_points(d_pts, n_local);
    if (st) return st;
    if (!h_ext || !h_count) return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "h_ext and h_count are required");
    if (capacity < 0) return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "capacity < 0");
    if (n_local > 0 && !d_surv_idx) return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "d_surv_idx is NULL");
    if (h_ext->nonfinite) return fail(CUDAPRE_ERR_NONFINITE_INPUT, "non-finite coordinate in the input");
    if (h_ext->n <= 0) return fail(CUDAPRE_ERR_EMPTY_INPUT, "empty input");
    if (h_ext->nang < 1 || h_ext->nang > CUDAPRE_MAX_ANGLES)
        return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "bad nang in extremes");
    if (h_rep) std::memset(h_rep, 0, sizeof(*h_rep));

    K2Params p;
    std::memset(&p, 0, sizeof(p));
    cudapre_polygon_t poly;
    void* stage = nullptr;
    st = staging(&stage);
    if (st) return st;
    K2Geom* hg = reinterpret_cast<K2Geom*>(reinterpret_cast<char*>(stage) + kStageGeomOff);
    const auto t0 = std::chrono::steady_clock::now();
    build_polygon(*h_ext, &poly, hg);
    const auto t1 = std::chrono::steady_clock::now();
    if (h_poly) *h_poly = poly;
    if (h_rep) {
        h_rep->n = n_local;
        h_rep->ms_polygon_host = std::chrono::duration<double, std::milli>(t1 - t0).count();
    }
    *h_count = 0;
    if (n_local == 0) return CUDAPRE_OK;
    st = check_ws(d_ws, ws_bytes, n_local);
    if (st) return st;

    cudaStream_t strm = (cudaStream_t)stream;
    k2_params(p, d_pts, n_local, index_base, d_surv_idx, d_surv_pts, capacity, d_ws, ws_bytes);
    p.edges = poly.nv <= 16 ? 16 : 32;
    CUDA_TRY(cudaMemcpyAsync(ws_geom(d_ws), hg, sizeof(K2Geom), cudaMemcpyHostToDevice, strm));
    const int vec16 = (((uintptr_t)d_pts & 15u) == 0);

    cudaEvent_t* ev = nullptr;
    if (h_rep) {
        st = events(&ev);
        if (st) return st;
        CUDA_TRY(cudaEventRecord(ev[2], strm));
    }
    int launches = 0;
    CUDA_TRY(launch_filter(p, vec16, stream, &launches));
    if (h_rep) CUDA_TRY(cudaEventRecord(ev[3], strm));
    CUDA_TRY(cudaMemcpyAsync(stage, &p.ws->count, 16, cudaMemcpyDeviceToHost, strm));   // count + stats
    CUDA_TRY(cudaStreamSynchronize(strm));
    const int64_t count = (int64_t) * reinterpret_cast<unsigned long long*>(stage);
    const unsigned* lb = reinterpret_cast<const unsigned*>(reinterpret_cast<const char*>(stage) + 8);
    if (h_rep) {
        h_rep->lookback_rounds = lb[0];
        h_rep->lookback_spins = lb[1];
    }
    *h_count = count;
    if (h_rep) {
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, ev[2], ev[3]));
        h_rep->ms_filter_kernel = ms;
        h_rep->survivors = count;
        h_rep->launches = launches;
    }
    if (count > capacity)
        return fail(CUDAPRE_ERR_CAPACITY, "%lld survivors > capacity %lld", (long long)count,
                    (long long)capacity);
    return CUDAPRE_OK;
}

cudapre_status cudapre_hull(const cudapre_pt* h_pts, const int64_t* h_ids, int64_t n,
                            int64_t* h_ring, int64_t* h_ring_len) {
    g_err.clear();
    if (n < 0 || !h_ring_len || (n > 0 && (!h_pts || !h_ring)))
        return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "bad hull arguments");
    *h_ring_len = n == 0 ? 0 : hull_ring(h_pts, h_ids, n, h_ring);
    return CUDAPRE_OK;
}

cudapre_status cudapre_run_host(const cudapre_pt* h_pts, int64_t n, int32_t nang, const double* c,
                                const double* s, cudapre_pt* d_pts, void* d_ws, size_t ws_bytes,
                                int64_t* d_surv_idx, int64_t* h_surv_idx, int64_t capacity,
                                void* stream, int64_t* h_count, cudapre_report_t* h_rep) {
    g_err.clear();
    if (n < 0 || (n > 0 && (!h_pts || !d_pts || !h_surv_idx || !d_surv_idx)) || !h_count)
        return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "bad run_host arguments");
    cudaStream_t strm = (cudaStream_t)stream;
    if (n > 0)
        CUDA_TRY(cudaMemcpyAsync(d_pts, h_pts, (size_t)n * sizeof(cudapre_pt), cudaMemcpyHostToDevice,
                                 strm));
    cudapre_extremes_t ext;
    cudapre_report_t r1, r2;
    cudapre_status st = cudapre_extremes(d_pts, n, 0, nang, c, s, d_ws, ws_bytes, stream, nullptr, &ext,
                                         h_rep ? &r1 : nullptr);
    if (st) return st;
    st = cudapre_filter(d_pts, n, 0, &ext, d_surv_idx, nullptr, capacity, d_ws, ws_bytes, stream,
                        h_count, nullptr, h_rep ? &r2 : nullptr);
    if (st && st != CUDAPRE_ERR_CAPACITY) return st;
    const int64_t m = *h_count < capacity ? *h_count : capacity;
    if (m > 0)
        CUDA_TRY(cudaMemcpyAsync(h_surv_idx, d_surv_idx, (size_t)m * sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, strm));
    CUDA_TRY(cudaStreamSynchronize(strm));
    if (h_rep) {
        *h_rep = r2;
        h_rep->ms_extremes_kernels = r1.ms_extremes_kernels;
        h_rep->launches = r1.launches + r2.launches;
    }
    return st;
}

// ------------------------------------------------------------------ device-resident Steps 2-3 (f3)
cudapre_status cudapre_geometry(const cudapre_extremes_t* h_ext, void* h_out, size_t out_bytes, size_t* needed) {
    g_err.clear();
    if (needed) *needed = sizeof(K2Geom);
    if (!h_ext || !h_out) return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "NULL argument");
    if (out_bytes < sizeof(K2Geom))
        return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "out_bytes %zu < %zu", out_bytes, sizeof(K2Geom));
    if (h_ext->n <= 0) return fail(CUDAPRE_ERR_EMPTY_INPUT, "empty input");
    if (h_ext->nang < 1 || h_ext->nang > CUDAPRE_MAX_ANGLES)
        return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "bad nang in extremes");
    cudapre_polygon_t poly;
    build_polygon(*h_ext, &poly, reinterpret_cast<K2Geom*>(h_out));
    return CUDAPRE_OK;
}

cudapre_status cudapre_polygon_device(const cudapre_extremes_t* d_parts, int32_t nparts, void* d_ws,
                                      size_t ws_bytes, void* stream, cudapre_polygon_t* d_poly) {
    g_err.clear();
    if (!d_ws || ((uintptr_t)d_ws & 15u) != 0 || ws_bytes < kWsFixedBytes)
        return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "d_ws must be a 16-byte aligned workspace");
    if (nparts < 0 || (nparts > 1 && !d_parts))
        return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "nparts > 1 needs d_parts");
    cudapre_extremes_t* res = &ws_header(d_ws)->result;
    const cudapre_extremes_t* parts = d_parts ? d_parts : res;
    int launches = 0;
    CUDA_TRY(launch_build_geom(parts, nparts > 1 ? nparts : 1, nparts > 1 ? res : nullptr,
                               d_poly ? d_poly : ws_poly(d_ws), ws_geom(d_ws), stream, &launches));
    return CUDAPRE_OK;
}

cudapre_status cudapre_filter_geom(const cudapre_pt* d_pts, int64_t n_local, int64_t index_base,
                                   int64_t* d_surv_idx, cudapre_pt* d_surv_pts, int64_t capacity, void* d_ws,
                                   size_t ws_bytes, void* stream, int64_t* d_count) {
    g_err.clear();
    cudapre_status st = check_points(d_pts, n_local);
    if (st) return st;
    if (capacity < 0) return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "capacity < 0");
    if (n_local > 0 && !d_surv_idx) return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "d_surv_idx is NULL");
    cudaStream_t strm = (cudaStream_t)stream;
    if (n_local == 0) {
        if (d_count) CUDA_TRY(cudaMemsetAsync(d_count, 0, sizeof(int64_t), strm));
        return CUDAPRE_OK;
    }
    st = check_ws(d_ws, ws_bytes, n_local);
    if (st) return st;
    K2Params p;
    std::memset(&p, 0, sizeof(p));
    k2_params(p, d_pts, n_local, index_base, d_surv_idx, d_surv_pts, capacity, d_ws, ws_bytes);
    const int vec16 = (((uintptr_t)d_pts & 15u) == 0);
    int launches = 0;
    CUDA_TRY(launch_filter(p, vec16, stream, &launches));
    if (d_count)
        CUDA_TRY(cudaMemcpyAsync(d_count, &p.ws->count, sizeof(int64_t), cudaMemcpyDeviceToDevice, strm));
    return CUDAPRE_OK;
}

cudapre_status cudapre_filter_device(const cudapre_pt* d_pts, int64_t n_local, int64_t index_base,
                                     const cudapre_extremes_t* d_ext, int64_t* d_surv_idx,
                                     cudapre_pt* d_surv_pts, int64_t capacity, void* d_ws, size_t ws_bytes,
                                     void* stream, int64_t* d_count, cudapre_polygon_t* d_poly) {
    g_err.clear();
    cudapre_status st = check_points(d_pts, n_local);
    if (st) return st;
    if (n_local > 0) {
        st = check_ws(d_ws, ws_bytes, n_local);
        if (st) return st;
        st = cudapre_polygon_device(d_ext, d_ext ? 1 : 0, d_ws, ws_bytes, stream, d_poly);
        if (st) return st;
    }
    return cudapre_filter_geom(d_pts, n_local, index_base, d_surv_idx, d_surv_pts, capacity, d_ws, ws_bytes,
                               stream, d_count);
}

cudapre_status cudapre_pipeline_device(const cudapre_pt* d_pts, int64_t n_local, int64_t index_base,
                                       int32_t nang, const double* c, const double* s, int64_t* d_surv_idx,
                                       cudapre_pt* d_surv_pts, int64_t capacity, void* d_ws, size_t ws_bytes,
                                       void* stream, int64_t* d_count) {
    cudapre_status st = cudapre_extremes(d_pts, n_local, index_base, nang, c, s, d_ws, ws_bytes, stream,
                                         nullptr, nullptr, nullptr);
    if (st) return st;
    return cudapre_filter_device(d_pts, n_local, index_base, nullptr, d_surv_idx, d_surv_pts, capacity, d_ws,
                                 ws_bytes, stream, d_count, nullptr);
}

cudapre_status cudapre_pipeline_host(const cudapre_pt* d_pts, int64_t n_local, int64_t index_base, int32_t nang,
                                     const double* c, const double* s, int64_t* d_surv_idx, cudapre_pt* d_surv_pts,
                                     int64_t capacity, void* d_ws, size_t ws_bytes, void* stream, int64_t* d_count,
                                     cudapre_polygon_t* h_poly, double* h_ms_polygon) {
    g_err.clear();
    if (capacity < 0 || (n_local > 0 && !d_surv_idx)) return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "bad survivor buffers");
    void *hm = nullptr, *dm = nullptr;
    cudapre_status st = mapped_block(&hm, &dm);
    if (st) return st;
    cudaStream_t strm = (cudaStream_t)stream;
    // Step 1; K1's last block writes the result straight into the mapped block
    st = cudapre_extremes(d_pts, n_local, index_base, nang, c, s, d_ws, ws_bytes, stream,
                          reinterpret_cast<cudapre_extremes_t*>(dm), nullptr, nullptr);
    if (st) return st;
    CUDA_TRY(cudaStreamSynchronize(strm));   // (the one host wait of the step: the picks)
    cudapre_extremes_t ext;
    std::memcpy(&ext, hm, sizeof(ext));
    if (ext.nonfinite) return fail(CUDAPRE_ERR_NONFINITE_INPUT, "non-finite coordinate in the input");
    // Step 2 on the host, straight into pinned staging
    void* stage = nullptr;
    st = staging(&stage);
    if (st) return st;
    K2Geom* hg = reinterpret_cast<K2Geom*>(reinterpret_cast<char*>(stage) + kStageGeomOff);
    cudapre_polygon_t poly;
    const auto t0 = std::chrono::steady_clock::now();
    build_polygon(ext, &poly, hg);
    const auto t1 = std::chrono::steady_clock::now();
    if (h_poly) *h_poly = poly;
    if (h_ms_polygon) *h_ms_polygon = std::chrono::duration<double, std::milli>(t1 - t0).count();
    // Step 3, enqueued: one H2D of the geometry, K2, the count stays on the device
    K2Params p;
    std::memset(&p, 0, sizeof(p));
    k2_params(p, d_pts, n_local, index_base, d_surv_idx, d_surv_pts, capacity, d_ws, ws_bytes);
    p.edges = poly.nv <= 16 ? 16 : 32;
    CUDA_TRY(cudaMemcpyAsync(ws_geom(d_ws), hg, sizeof(K2Geom), cudaMemcpyHostToDevice, strm));
    st = staging_in_flight(strm);   // the next call waits for this copy before reusing the buffer
    if (st) return st;
    int launches = 0;
    CUDA_TRY(launch_filter(p, (((uintptr_t)d_pts & 15u) == 0), stream, &launches));
    if (d_count)
        CUDA_TRY(cudaMemcpyAsync(d_count, &p.ws->count, sizeof(int64_t), cudaMemcpyDeviceToDevice, strm));
    return CUDAPRE_OK;
}

struct cudapre_graph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
};

cudapre_status cudapre_graph_destroy(cudapre_graph_t* g) {
    if (!g) return CUDAPRE_OK;
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
    return CUDAPRE_OK;
}

cudapre_status cudapre_graph_create(const cudapre_pt* d_pts, int64_t n_local, int64_t index_base, int32_t nang,
                                    const double* c, const double* s, int64_t* d_surv_idx,
                                    cudapre_pt* d_surv_pts, int64_t capacity, void* d_ws, size_t ws_bytes,
                                    void* stream, int64_t* d_count, cudapre_graph_t** out) {
    g_err.clear();
    if (!out) return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    cudaStream_t strm = (cudaStream_t)stream;
    // one uncaptured run: argument checks and the launchers' lazy set-up
    cudapre_status st = cudapre_pipeline_device(d_pts, n_local, index_base, nang, c, s, d_surv_idx, d_surv_pts,
                                                capacity, d_ws, ws_bytes, stream, d_count);
    if (st) return st;
    CUDA_TRY(cudaStreamSynchronize(strm));
    cudaStream_t cs = nullptr;
    CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudapre_graph_t* g = new cudapre_graph_t;
    cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        st = cudapre_pipeline_device(d_pts, n_local, index_base, nang, c, s, d_surv_idx, d_surv_pts, capacity,
                                     d_ws, ws_bytes, cs, d_count);
        const cudaError_t e2 = cudaStreamEndCapture(cs, &g->graph);
        if (!st && e2 != cudaSuccess) e = e2;
    }
    if (!st && e == cudaSuccess) e = cudaGraphInstantiate(&g->exec, g->graph, 0);
    cudaStreamDestroy(cs);
    if (st || e != cudaSuccess) {
        cudapre_graph_destroy(g);
        if (st) return st;
        return fail(CUDAPRE_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
    }
    *out = g;
    return CUDAPRE_OK;
}

cudapre_status cudapre_graph_launch(cudapre_graph_t* g, void* stream) {
    g_err.clear();
    if (!g || !g->exec) return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "graph is NULL");
    CUDA_TRY(cudaGraphLaunch(g->exec, (cudaStream_t)stream));
    return CUDAPRE_OK;
}

// ------------------------------------------------------------------ final hull on the GPU (f1)
namespace {
struct HullScratch {
    unsigned long long* gmax;
    cudapre_pt* cand_pts;
    int64_t* cand_ids;
    unsigned* table;
    float* vx;
    float* vy;
    unsigned long long* count;
    cudapre_pt* out_pts;
    int64_t* out_ids;
    size_t bytes;
};
HullScratch hull_scratch(void* base, int64_t m) {
    HullScratch h;
    size_t off = 0;
    auto take = [&](size_t n) {
        const size_t o = off;
        off = (off + n + 255) & ~(size_t)255;
        return reinterpret_cast<char*>(base) + o;
    };
    h.gmax = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * kHullBuckets));
    h.cand_pts = reinterpret_cast<cudapre_pt*>(take(sizeof(cudapre_pt) * kHullBuckets));
    h.cand_ids = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * kHullBuckets));
    h.table = reinterpret_cast<unsigned*>(take(sizeof(unsigned) * kHullBuckets));
    h.vx = reinterpret_cast<float*>(take(sizeof(float) * (kHullMaxVerts + 1)));
    h.vy = reinterpret_cast<float*>(take(sizeof(float) * (kHullMaxVerts + 1)));
    h.count = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long)));
    h.out_pts = reinterpret_cast<cudapre_pt*>(take(sizeof(cudapre_pt) * (size_t)(m > 0 ? m : 1)));
    h.out_ids = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * (size_t)(m > 0 ? m : 1)));
    h.bytes = off;
    return h;
}
bool inside_ring(const cudapre_pt* v, int nv, float px, float py) {
    if (nv < 3) return false;
    for (int j = 0; j < nv; ++j) {
        const cudapre_pt a = v[j], b = v[(j + 1) % nv];
        if (orient_exact(a.x, a.y, b.x, b.y, px, py) <= 0) return false;
    }
    return true;
}
}  // namespace

size_t cudapre_hull_device_bytes(int64_t m) { return hull_scratch(nullptr, m < 0 ? 0 : m).bytes; }

cudapre_status cudapre_hull_device(const cudapre_pt* d_pts, const int64_t* d_ids, int64_t m,
                                   const cudapre_polygon_t* h_poly, void* d_scratch, size_t scratch_bytes,
                                   void* stream, int64_t* h_ring, int64_t ring_capacity, int64_t* h_ring_len,
                                   int64_t* h_remaining) {
    return cudapre_hull_device_ex(d_pts, d_ids, m, h_poly, d_scratch, scratch_bytes, stream, h_ring, nullptr,
                                  ring_capacity, h_ring_len, h_remaining);
}

cudapre_status cudapre_hull_device_ex(const cudapre_pt* d_pts, const int64_t* d_ids, int64_t m,
                                      const cudapre_polygon_t* h_poly, void* d_scratch, size_t scratch_bytes,
                                      void* stream, int64_t* h_ring, cudapre_pt* h_ring_pts, int64_t ring_capacity,
                                      int64_t* h_ring_len, int64_t* h_remaining) {
    g_err.clear();
    if (m < 0 || !h_ring_len || (m > 0 && (!d_pts || !d_ids || !h_poly || !d_scratch)))
        return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "bad hull_device arguments");
    if (m > (int64_t)0xffffffffll) return fail(CUDAPRE_ERR_INVALID_ARGUMENT, "m out of range");
    *h_ring_len = 0;
    if (h_remaining) *h_remaining = m;
    if (m == 0) return CUDAPRE_OK;
    const HullScratch S = hull_scratch(d_scratch, m);
    if (scratch_bytes < S.bytes)
        return fail(CUDAPRE_ERR_WORKSPACE, "scratch %zu B < %zu B needed", scratch_bytes, S.bytes);
    cudaStream_t strm = (cudaStream_t)stream;
    std::vector<cudapre_pt> keep_pts;
    std::vector<int64_t> keep_ids;
    const float cx = h_poly->circle[0], cy = h_poly->circle[1];
    bool filtered = false;
    if (!h_poly->degenerate && inside_ring(h_poly->v, h_poly->nv, cx, cy)) {
        // H1: sector maxima around c -> candidates
        int launches = 0;
        CUDA_TRY(cudaMemsetAsync(S.gmax, 0, sizeof(unsigned long long) * kHullBuckets, strm));
        CUDA_TRY(launch_hull_votes(d_pts, d_ids, m, cx, cy, S.gmax, S.cand_pts, S.cand_ids, stream, &launches));
        std::vector<cudapre_pt> cp_((size_t)kHullBuckets + CUDAPRE_MAX_SLOTS);
        std::vector<int64_t> ci((size_t)kHullBuckets + CUDAPRE_MAX_SLOTS);
        CUDA_TRY(cudaMemcpyAsync(cp_.data(), S.cand_pts, sizeof(cudapre_pt) * kHullBuckets, cudaMemcpyDeviceToHost,
                                 strm));
        CUDA_TRY(cudaMemcpyAsync(ci.data(), S.cand_ids, sizeof(int64_t) * kHullBuckets, cudaMemcpyDeviceToHost,
                                 strm));
        CUDA_TRY(cudaStreamSynchronize(strm));
        int64_t nc = 0;
        for (int b = 0; b < kHullBuckets; ++b)
            if (ci[b] >= 0) {
                cp_[nc] = cp_[b];
                ci[nc++] = ci[b];
            }
        for (int j = 0; j < h_poly->nv; ++j) {   // the Step-2 ring (survivors too): P' contains c
            cp_[nc] = h_poly->v[j];
            ci[nc++] = h_poly->vidx[j];
        }
        std::vector<int64_t> rid((size_t)nc);
        std::vector<cudapre_pt> rpt((size_t)nc + 1);
        const int nv = (int)hull_ring_points(cp_.data(), ci.data(), nc, rid.data(), rpt.data());
        if (nv >= 3 && nv <= kHullMaxVerts && inside_ring(rpt.data(), nv, cx, cy)) {
            // H2: drop the survivors strictly inside P'
            std::vector<unsigned> table((size_t)kHullBuckets);
            hull_bucket_table(rpt.data(), nv, cx, cy, table.data());
            std::vector<float> vx((size_t)nv + 1), vy((size_t)nv + 1);
            for (int j = 0; j <= nv; ++j) {
                vx[j] = rpt[j % nv].x;
                vy[j] = rpt[j % nv].y;
            }
            CUDA_TRY(cudaMemcpyAsync(S.table, table.data(), sizeof(unsigned) * kHullBuckets,
                                     cudaMemcpyHostToDevice, strm));
            CUDA_TRY(cudaMemcpyAsync(S.vx, vx.data(), sizeof(float) * (nv + 1), cudaMemcpyHostToDevice, strm));
            CUDA_TRY(cudaMemcpyAsync(S.vy, vy.data(), sizeof(float) * (nv + 1), cudaMemcpyHostToDevice, strm));
            CUDA_TRY(cudaMemsetAsync(S.count, 0, sizeof(unsigned long long), strm));
            CUDA_TRY(launch_hull_filter(d_pts, d_ids, m, cx, cy, S.table, S.vx, S.vy, nv, S.out_pts, S.out_ids,
                                        S.count, stream, &launches));
            unsigned long long k = 0;
            CUDA_TRY(cudaMemcpyAsync(&k, S.count, sizeof(k), cudaMemcpyDeviceToHost, strm));
            CUDA_TRY(cudaStreamSynchronize(strm));
            keep_pts.resize((size_t)k);
            keep_ids.resize((size_t)k);
            if (k) {
                CUDA_TRY(cudaMemcpyAsync(keep_pts.data(), S.out_pts, sizeof(cudapre_pt) * k, cudaMemcpyDeviceToHost,
                                         strm));
                CUDA_TRY(cudaMemcpyAsync(keep_ids.data(), S.out_ids, sizeof(int64_t) * k, cudaMemcpyDeviceToHost,
                                         strm));
                CUDA_TRY(cudaStreamSynchronize(strm));
            }
            filtered = true;
        }
    }
    if (!filtered) {   // no certified centre: the host chain on every survivor
        keep_pts.resize((size_t)m);
        keep_ids.resize((size_t)m);
        CUDA_TRY(cudaMemcpyAsync(keep_pts.data(), d_pts, sizeof(cudapre_pt) * m, cudaMemcpyDeviceToHost, strm));
        CUDA_TRY(cudaMemcpyAsync(keep_ids.data(), d_ids, sizeof(int64_t) * m, cudaMemcpyDeviceToHost, strm));
        CUDA_TRY(cudaStreamSynchronize(strm));
    }
    if (h_remaining) *h_remaining = (int64_t)keep_ids.size();
    std::vector<int64_t> ring(keep_ids.size() + 1);
    std::vector<cudapre_pt> rpts(keep_ids.size() + 1);
    const int64_t len =
        keep_ids.empty() ? 0 : hull_ring_points(keep_pts.data(), keep_ids.data(), (int64_t)keep_ids.size(),
                                                ring.data(), rpts.data());
    if (len > ring_capacity) return fail(CUDAPRE_ERR_CAPACITY, "hull of %lld vertices > capacity", (long long)len);
    if (len > 0) std::memcpy(h_ring, ring.data(), sizeof(int64_t) * len);
    if (len > 0 && h_ring_pts) std::memcpy(h_ring_pts, rpts.data(), sizeof(cudapre_pt) * len);
    *h_ring_len = len;
    return CUDAPRE_OK;
}

}  // extern "C"
