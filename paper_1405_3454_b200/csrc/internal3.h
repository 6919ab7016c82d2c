// internal3.h — declarations of the 3D extension (SURVEY §8
// f4).  Not part of the ABI.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/cudapre.h"
#include "device.h"

namespace cudapre {

constexpr int kMax3Slots = CUDAPRE3_MAX_SLOTS;     // 6 per angle
constexpr int kMax3Facets = CUDAPRE3_MAX_FACETS;   // facet planes of conv(<= 34 points)

// ---------------------------------------------------------------- launch shape
constexpr int kK13Threads = 256;              // K1-3D block
constexpr int kK13Quads = 2;                  // quads (4 points, 48 B) per thread per iteration
constexpr int kMaxK13Blocks = 148 * 8;
constexpr int kK23Threads = 256;              // K2-3D block
#ifndef K23_QUADS
#define K23_QUADS 2
#endif
constexpr int kK23Quads = K23_QUADS;                         // quads per thread per tile (2 or 4)
constexpr int kK23TileQuads = kK23Quads * kK23Threads;
constexpr int kK23TilePts = 4 * kK23TileQuads;              // 2048 points (24 KiB) per tile
constexpr int kK23BlocksPerSM = kK23Quads == 2 ? 3 : 2;     // shared memory: cell lists + staging
constexpr int kStatus3Stride = 16;            // one 8-byte status word per 128-byte line

// ---------------------------------------------------------------- workspace
// [Ws3Header, 4 KiB][K3Geom page, 32 KiB][K13Partial x kMaxK13Blocks x 48][status x ntiles]
struct alignas(16) Ws3Header {
    unsigned int k1_ticket;     // K1-3D blocks finished (last block finalizes, resets)
    unsigned int k1_nonfinite;  // NaN / Inf seen by K1-3D
    unsigned int k1_exact;      // points that took the exact path (diagnostic)
    unsigned int k2_ticket;     // K2-3D dynamic tile counter
    unsigned int k2_done;       // K2-3D blocks finished
    unsigned int epoch;         // K2-3D tile-status epoch
    unsigned int k2_exact;      // points that took the exact orient3d path (diagnostic)
    unsigned int pad0;
    unsigned long long count;   // K2-3D survivors
    unsigned long long pad1;
    cudapre3_extremes_t result; // K1-3D final result
};
static_assert(sizeof(Ws3Header) <= 4096, "3D header too large");
constexpr size_t kWs3HeaderBytes = 4096;
constexpr size_t kWs3GeomBytes = 65536;

struct K13Partial {
    double key;
    unsigned int idx;   // local index, 0xffffffff = none
    unsigned int pad;
};
constexpr size_t kWs3PartialBytes = sizeof(K13Partial) * (size_t)kMaxK13Blocks * kMax3Slots;
constexpr size_t kWs3FixedBytes = kWs3HeaderBytes + kWs3GeomBytes + kWs3PartialBytes;

inline size_t ws3_tiles(int64_t n) { return (size_t)((n + kK23TilePts - 1) / kK23TilePts); }
inline size_t ws3_bytes_for(int64_t n) {
    return kWs3FixedBytes + ws3_tiles(n) * kStatus3Stride * sizeof(unsigned long long) + 128;
}

// Step-3 geometry (host-built, copied to the geometry page; K2-3D stages it
// in shared memory).  Direction cells around the centre o (strictly inside):
// d = RN(p - o); the major axis a of |d| (ties: x before y before z) and its
// sign give the cube face f = 2a + (d_a < 0); with (u, v) the two other
// components in the order (y, z), (z, x), (x, y) for a = x, y, z, the cell is
// (f, iu, iv), iu = clamp(floor((u / |d_a| + 1) G / 2), 0, G - 1) (same for
// v), computed with one approximate reciprocal.  The candidates of a cell are
// the facets whose face meets the cell's direction pyramid widened by
// kCellGuard; clist[cell] holds up to kCellSlots of them as
// bytes (unused: kDummyFacet, whose plane test always says "inside") and the
// count in the top byte; a longer list (count > kCellSlots) keeps in its low
// bits an index into lmask[] (the candidate mask), or kNoLong = every facet.  Facet
// j: plane test g = fma(A, x, fma(B, y, fma(C, z, D))) with |g -
// orient3d(facet, p)| <= E over the data bounding box; fv[j] its supporting
// triple for the exact decision.
constexpr int kCellG = 32;                      // cells per cube-face side
constexpr int kCells = 6 * kCellG * kCellG;     // 6144
constexpr int kMaxLong = 1024;                  // long lists with their own mask
constexpr unsigned kNoLong = 0xffffffu;
constexpr int kCellSlots = 3;
constexpr int kDummyFacet = kMax3Facets;        // plane (0, 0, 0, 1), E = 0
constexpr double kCellGuard = 0x1p-12;          // widening of every cell, in (u, v) units

struct alignas(16) K3Geom {
    int nf;          // facet planes
    int mode;        // 0 = filter, 1 = keep everything (degenerate polyhedron)
    int cells;       // 1 if the centre is strictly inside (cell lists), 0 = every cell = all facets
    int pad0;
    float ox, oy, oz, pad1;
    unsigned long long all;                // mask of every facet
    unsigned long long pad2;
    unsigned clist[kCells];                // candidate lists (bytes) + count
    unsigned long long lmask[kMaxLong];    // candidate masks of long lists
    float4 pl[kMax3Facets + 1];            // (A, B, C, D); [kDummyFacet] = (0, 0, 0, 1)
    float pe[kMax3Facets + 1];             // E; [kDummyFacet] = 0
    float fv[kMax3Facets][9];              // facet triple coordinates (a, b, c)
};
static_assert(sizeof(K3Geom) <= kWs3GeomBytes, "3D geometry page");

struct K13Params {
    const float* pts;     // xyz AoS
    unsigned int n;
    int vec;              // 16-B aligned base
    long long base;
    Ws3Header* ws;
    K13Partial* partials;
    double c[CUDAPRE_MAX_ANGLES], s[CUDAPRE_MAX_ANGLES];
    float cf[CUDAPRE_MAX_ANGLES], sf[CUDAPRE_MAX_ANGLES], nsf[CUDAPRE_MAX_ANGLES];
    int nang;
};

struct K23Params {
    const float* pts;
    unsigned int n;
    int vec;
    long long base;
    long long* out_idx;
    float* out_pts;       // xyz, nullable
    unsigned long long capacity;
    Ws3Header* ws;
    const K3Geom* g;
    unsigned long long* status;
    unsigned int num_tiles;
};

int launch_extremes3(const K13Params& p, void* stream, int* launches);
int launch_filter3(const K23Params& p, void* stream, int* launches);

// host Step 2 (host_geom3.cpp): polyhedron + K3Geom from the merged extremes
// (bbox = exact data bounding box from the angle-0 slots).  Returns 0 or a
// cudapre_status.
int build_polyhedron3(const cudapre3_extremes_t& ext, cudapre3_polyhedron_t* poly, K3Geom* g, int flags = 0);
int merge_extremes3(const cudapre3_extremes_t* parts, int count, cudapre3_extremes_t* out);

// api.cpp hooks shared with api3.cpp
cudapre_status api_fail(cudapre_status st, const char* msg);
cudapre_status api_staging(void** out, size_t* bytes);
int device_sm_count();

}  // namespace cudapre
