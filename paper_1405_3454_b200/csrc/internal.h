// internal.h — shared declarations of the CudaPre B200 library (not part of the ABI).
#pragma once

#include <cstddef>
#include <cstdint>

#include "../../include/cudapre.h"
#include "device.h"

namespace cudapre {

// ---------------------------------------------------------------- launch shape
constexpr int kK1Threads = 256;        // K1 block
constexpr int kK1Unroll = 4;           // float4 (= 2 points) per thread per iteration
constexpr int kSeedThreads = 128;      // seed block; one chunk = 128 float4 = 256 points
constexpr int kK1StagePairs = kK1Threads * kK1Unroll;   // 1024 pairs = 16 KiB per TMA stage
constexpr int kK1Stages = 4;           // TMA ring depth per block
constexpr int kK1Queue = 32 + 2 * kK1Unroll * 32;   // per-warp pre-screen queue: 31 carried + one iteration (256)
constexpr int kK2Threads = 256;        // K2 block
constexpr int kK2Items = 4;            // float4 per thread per sub-tile
constexpr int kK2SubPairs = kK2Threads * kK2Items;    // 1024 pairs = 2048 points per sub-tile
constexpr int kK2Sub = 8;              // sub-tiles per super-tile (one look-back each)
constexpr int kK2TilePairs = kK2Sub * kK2SubPairs;    // 8192 pairs
constexpr int kK2TilePts = 2 * kK2TilePairs;          // 16384 points = 128 KiB per super-tile
constexpr int kMaxK1Blocks = 148 * 16;

// ---------------------------------------------------------------- workspace
// Device workspace layout (caller-owned, zero-filled once):
//   [WsHeader, padded to 4 KiB][geometry page 32 KiB][K1Partial x kMaxK1Blocks x 32][tile status x ntiles]
//   ... [TMA K2 list-overflow scratch, at the END of the buffer]
// Every kernel leaves the counters it uses back at their reset values, so the
// workspace stays valid from call to call.
struct alignas(16) WsHeader {
    unsigned int k1_ticket;      // K1 blocks finished (last-block finalize)
    unsigned int k1_nonfinite;   // set by K1's exact path on NaN/Inf input
    unsigned int k1_exact;       // points that took K1's exact path (diagnostic)
    unsigned int k2_ticket;      // K2 dynamic tile counter
    unsigned int k2_done;        // K2 blocks finished
    unsigned int epoch;          // K2 tile-status epoch (never 0 after the first call)
    unsigned int pad0[2];
    unsigned long long count;    // K2 survivors (written by the last tile)
    unsigned int lb_rounds;      // K2 look-back rounds (diagnostic; copied with count)
    unsigned int lb_spins;       // K2 look-back rounds that waited
    unsigned int seed[CUDAPRE_MAX_SLOTS];   // seed thresholds, order-preserving encoding, 0 = none
    cudapre_extremes_t result;   // K1 final result
};
static_assert(sizeof(WsHeader) <= 2048, "header too large");

struct K1Partial {
    double key;
    unsigned int idx;   // local index, 0xffffffff = none
    unsigned int pad;
};

constexpr size_t kWsHeaderBytes = 4096;
// geometry page after the header: K2Geom at +0, the device copy of the
// polygon (cudapre_polygon_t) at +kWsPolyOff
constexpr size_t kWsGeomBytes = 32768;
constexpr size_t kWsPolyOff = 16384;
constexpr size_t kWsFixedBytes = kWsHeaderBytes + kWsGeomBytes;   // header + geometry page
constexpr size_t kWsPartialBytes = sizeof(K1Partial) * kMaxK1Blocks * CUDAPRE_MAX_SLOTS;

// One tile-status word per super-tile, each on its own 128-byte line: packed
// words put up to 16 publishing SMs and every look-back reader on one L2 line
// and cost ~0.6 ms per 2e9 points (profiles/r01_experiments.md, "status
// false sharing"); padded, the 256-wide look-back costs ~0.1 ms.
constexpr int kStatusTilePts = kK2TilePts;
constexpr int kStatusStride = 16;   // u64 words per status line (128 B)
inline size_t ws_tiles(int64_t n) { return (size_t)((n + kStatusTilePts - 1) / kStatusTilePts); }
inline size_t ws_status_bytes(int64_t n) { return 8 * kStatusStride * (ws_tiles(n) + 1); }

// TMA K2 survivor-list overflow: a warp's list entries beyond its shared-memory
// capacity go to global scratch, per (resident block, list buffer, warp), sized
// for the worst case (every point of the warp's 2048-point share survives).
struct SurvEntry {
    float x, y;
    unsigned meta;   // (sub-tile << 8) | offset in the warp's 256-point chunk
};
constexpr int kK2Bufs = 3;                          // survivor-list buffers per block
constexpr int kK2WarpPts = kK2Sub * 256;            // 2048 points per warp per super-tile
constexpr int kK2MaxWarps = 10;                    // compute warps per TMA K2 block, at most
constexpr size_t kK2ScratchPerBlock = (size_t)kK2Bufs * kK2MaxWarps * kK2WarpPts * sizeof(SurvEntry);
constexpr int kK2BlocksPerSM = 2;
inline size_t ws_scratch_blocks(int64_t n) {
    const size_t cap = (size_t)kK2BlocksPerSM * (size_t)device_sm_count();
    const size_t t = ws_tiles(n);
    return t < cap ? t : cap;
}
inline size_t ws_bytes_for(int64_t n) {   // (+16: alignment slack of the scratch at the end)
    return kWsFixedBytes + kWsPartialBytes + ws_status_bytes(n) + kK2ScratchPerBlock * ws_scratch_blocks(n) + 16;
}

// ---------------------------------------------------------------- kernel params
struct K1Params {
    const float* pts;         // n points, x y interleaved
    unsigned int n;
    int nang;
    long long base;           // global index of pts[0]
    float cf[CUDAPRE_MAX_ANGLES], sf[CUDAPRE_MAX_ANGLES], nsf[CUDAPRE_MAX_ANGLES];
    double c[CUDAPRE_MAX_ANGLES], s[CUDAPRE_MAX_ANGLES];
    WsHeader* ws;
    K1Partial* partials;
    cudapre_extremes_t* d_out;   // nullable extra copy of the result
    unsigned int seed_chunks;    // number of 256-point sample chunks (0 = no seed)
    int pad_;
};

// Step-3 geometry (built from the polygon on the host or on the device,
// geom.cuh; lives in the workspace, read by the K2 kernels).
struct K2Geom {
    int nv;                   // ring length
    int mode;                 // 0 = filter, 1 = keep everything (degenerate), 2 = exact only
    int fast;                 // TMA K2 pass-A test: 0 = inner disk, 1 = inner box, 2 = none
    int pad;
    float bx0, bx1, by0, by1; // inner box (closed), strictly inside the ring
    float ox, oy, r2;         // inner disk: RN(RN(dx^2)+RN(dy^2)) < r2 => strictly inside (r2 < 0: off)
    float e2max;              // 2 * max_j E_j
    float A[CUDAPRE_MAX_SLOTS], B[CUDAPRE_MAX_SLOTS], C[CUDAPRE_MAX_SLOTS];   // C already lowered by E_j
    float vx[CUDAPRE_MAX_SLOTS + 1], vy[CUDAPRE_MAX_SLOTS + 1];               // ring, v[nv] = v[0]
    float sr2[CUDAPRE_SECTORS + 1];    // sector inner radii^2 around (ox, oy) (-1 = off)
    float sro2[CUDAPRE_SECTORS + 1];   // sector outer radii^2 (+inf = off)
    // edges a ray of bucket b can exit through: lo | hi << 8 (hi = lo or lo+1
    // cyclically); 0xffff = more than two (or no table): test every edge
    unsigned short sedge[CUDAPRE_SECTORS + 1];
};
static_assert(sizeof(K2Geom) <= kWsPolyOff && sizeof(cudapre_polygon_t) <= kWsGeomBytes - kWsPolyOff,
              "geometry page");

struct K2Params {
    const float* pts;
    unsigned int n;
    int edges;                // 16 or 32: unrolled edge-loop length (>= nv; 32 when nv is not known on the host)
    long long base;
    long long* out_idx;
    float* out_pts;           // nullable, float2 per survivor
    unsigned long long capacity;
    WsHeader* ws;
    unsigned long long* status;   // ntiles tile-status words, kStatusStride apart
    unsigned int num_tiles;
    int pad_;
    const K2Geom* g;          // device geometry (workspace)
    SurvEntry* scratch;       // TMA K2 list overflow, kK2ScratchPerBlock per block
    unsigned int scratch_blocks;   // blocks the scratch region covers (caps the TMA K2 grid)
};

// ---------------------------------------------------------------- launchers (.cu)
// All return a cudaError_t as int (0 = success).
int launch_extremes(const K1Params& p, int vec16, void* stream, int* launches);
int launch_filter(const K2Params& p, int vec16, void* stream, int* launches);
int launch_filter_tma(const K2Params& p, void* stream, int* launches);     // 16-B aligned input

// ---------------------------------------------------------------- final hull on the GPU (k_hull.cu, f1)
constexpr int kHullBuckets = 4097;   // b = round(1024 pa), pa in [0, 4]
constexpr int kHullMaxVerts = kHullBuckets + CUDAPRE_MAX_SLOTS;
int launch_hull_votes(const cudapre_pt* d_pts, const int64_t* d_ids, int64_t m, float cx, float cy,
                      unsigned long long* gmax, cudapre_pt* cand_pts, int64_t* cand_ids, void* stream,
                      int* launches);
int launch_hull_filter(const cudapre_pt* d_pts, const int64_t* d_ids, int64_t m, float cx, float cy,
                       const unsigned* table, const float* vx, const float* vy, int nv, cudapre_pt* out_pts,
                       int64_t* out_ids, unsigned long long* count, void* stream, int* launches);
// Canonical ring (monotone chain) of the points (pts[j], ids[j]), ids
// distinct: ring ids (and coordinates if ring_pts), CCW from the
// lexicographically smallest vertex; returns its length.
int64_t hull_ring_points(const cudapre_pt* pts, const int64_t* ids, int64_t n, int64_t* ring_ids,
                         cudapre_pt* ring_pts);
// Candidate-edge table of ring v[0..nv) around c for the hull filter
// (kHullBuckets entries: first edge | count << 16, count 0 = all edges).
void hull_bucket_table(const cudapre_pt* v, int nv, float cx, float cy, unsigned* table);

// error message for the calling thread (api.cpp; used by api3.cpp, comm.cpp)
cudapre_status api_fail(cudapre_status st, const char* msg);

// ---------------------------------------------------------------- host geometry (host_geom.cpp)
int orient_exact(float ax, float ay, float bx, float by, float cx, float cy);
// Step 2 from global extremes (geom.cuh): the polygon (poly) and, if g is
// not null, the Step-3 geometry.  Sequential host build.
void build_polygon(const cudapre_extremes_t& ext, cudapre_polygon_t* poly, K2Geom* g);
// The same on the device: one block reads d_parts[0..nparts) (merged first
// if nparts > 1, the merge written to *d_merged if not null) and writes
// *d_poly, *d_g (byte-identical to the host build).
int launch_build_geom(const cudapre_extremes_t* d_parts, int nparts, cudapre_extremes_t* d_merged,
                      cudapre_polygon_t* d_poly, K2Geom* d_g, void* stream, int* launches);
// Canonical monotone-chain ring of pts[ids[j]] (ids nullptr = identity).
int64_t hull_ring(const cudapre_pt* pts, const int64_t* ids, int64_t n, int64_t* ring);
void merge_extremes(const cudapre_extremes_t* parts, int count, cudapre_extremes_t* out);

}  // namespace cudapre
