/*
 * cudapre.h — C ABI of the B200-native CudaPre interior-point filter
 * (G. Mei, arXiv 1405.3454).  Library: paper_1405_3454_b200/libcudapre.so
 *
 * The method (§2):
 *   Step 1  locate the extreme points: for the original point set and the
 *           point set rotated by each further angle, the points with min/max
 *           x and y.                        -> cudapre_extremes
 *   Step 2  Andrew's monotone chain on those <= 16 points, on the CPU
 *           (correction P:71).               -> cudapre_polygon
 *   Step 3  discard every point inside that convex polygon and
 *           keep the rest, in ascending index order.  -> cudapre_filter
 *   Then    the convex hull of the remaining points -> cudapre_hull
 *   3D      the extension outlined in P:115 (six extremes per rotation about
 *           z, a convex polyhedron, discard what is strictly inside) ->
 *           cudapre3_extremes / cudapre3_polyhedron / cudapre3_filter
 *           (float3 AoS points; section "The 3D extension" at the end)
 *
 * Citations: "P:nn" = PAPER.md line nn, "S:nn" = SPEC.md line nn, "A#" =
 * the reading numbered # in DESIGN.md §3 (where the paper is silent).
 *
 * Conventions for every entry point:
 *   - Nothing throws across the ABI; every function returns cudapre_status and,
 *     on a non-OK status, cudapre_last_error() returns a thread-local message.
 *   - Ownership: the CALLER allocates and frees every buffer (device buffers
 *     are plain device pointers, e.g. from torch; host structs are plain
 *     memory).  The library keeps no device state between calls; everything
 *     persistent lives in the caller's workspace (d_ws).
 *   - Device pointers marked d_*, host pointers h_*.  Streams are passed as
 *     `void*` holding a cudaStream_t (NULL = legacy default stream).
 *   - Points are float2 AoS ("cudapre_pt": x then y, 8 bytes), at least 8-byte
 *     aligned; 16-byte alignment enables the 128-bit vector path (any 8-byte
 *     aligned pointer works).
 *   - Indices are int64 and GLOBAL: index_base + local position, so a caller
 *     that shards one point set over several GPUs gets the same indices as a
 *     single GPU would.
 *   - A workspace is bound to one stream at a time: do not run two calls that
 *     share a workspace concurrently.  It must be zero-filled once before
 *     first use (cudapre_workspace_init); every call leaves it re-usable.
 *   - Limits: n_local <= 4294967295 points per call; at most
 *     CUDAPRE_MAX_ANGLES angles; the first angle must be 0 degrees (the
 *     original, unrotated set, "together with the group of extreme
 *     points of the original point set").
 */
#ifndef CUDAPRE_H
#define CUDAPRE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CUDAPRE_MAX_ANGLES 8
#define CUDAPRE_MAX_SLOTS (4 * CUDAPRE_MAX_ANGLES)
#define CUDAPRE_SECTORS 1024   /* Step-3 sector buckets: pseudo-angle [0,4] x 256 */

typedef enum {
    CUDAPRE_OK = 0,
    CUDAPRE_ERR_EMPTY_INPUT = 1,      /* no points at all where extremes are required */
    CUDAPRE_ERR_INVALID_ARGUMENT = 2, /* NULL / misaligned pointer, bad size, bad angle list */
    CUDAPRE_ERR_NONFINITE_INPUT = 3,  /* a NaN / Inf coordinate was seen (precondition S:32, A16) */
    CUDAPRE_ERR_CUDA = 4,             /* a CUDA runtime call failed (message has the CUDA error) */
    CUDAPRE_ERR_CAPACITY = 5,         /* survivor buffer too small; *h_count holds the needed size */
    CUDAPRE_ERR_WORKSPACE = 6,        /* workspace smaller than cudapre_workspace_bytes(n) */
    CUDAPRE_ERR_NCCL = 7              /* NCCL could not be loaded or a NCCL call failed */
} cudapre_status;

typedef struct { float x, y; } cudapre_pt; /* == float2 */

/* Step 1 result.  Slot 4k+{0,1,2,3} = {argmin X_k, argmax X_k, argmin Y_k,
 * argmax Y_k} for angle k in list order (A8), where
 *   X_k = RN(RN(x*c_k) + RN(y*s_k)),  Y_k = RN(RN(y*c_k) - RN(x*s_k))
 * in IEEE binary64 without FMA (A3, A6), lowest index on equal keys
 * (A7).  A slot of an empty shard has idx = -1 and never wins a merge.      */
typedef struct {
    int32_t nang;                        /* number of angles (slots = 4*nang) */
    int32_t nonfinite;                   /* 1 if a non-finite coordinate was seen */
    int64_t n;                           /* points reduced (summed over merged parts) */
    int64_t idx[CUDAPRE_MAX_SLOTS];      /* global index of each pick, -1 if none */
    double key[CUDAPRE_MAX_SLOTS];       /* the binary64 key value of each pick */
    cudapre_pt pt[CUDAPRE_MAX_SLOTS];    /* coordinates of each pick */
    double c[CUDAPRE_MAX_ANGLES];        /* cos of each angle used (correctly rounded, A5) */
    double s[CUDAPRE_MAX_ANGLES];        /* sin of each angle used */
    int64_t exact_points;                /* diagnostic: points that took the exact binary64 path
                                          * (passed the float screen), summed over merged parts */
} cudapre_extremes_t;

/* Step 2 result: the filter polygon and the parameters the Step-3 kernel
 * uses.  ring = Andrew's monotone chain of the distinct picks: CCW, starting
 * at the lexicographically smallest vertex, collinear points excluded (A10,
 * A17).  nv < 3 means degenerate: nothing is discarded (A13). */
typedef struct {
    int32_t nv;                          /* ring length, 0..CUDAPRE_MAX_SLOTS */
    int32_t degenerate;                  /* 1 if nv < 3 */
    int32_t n_distinct;                  /* distinct pick coordinates ("less than 16") */
    int32_t exact_only;                  /* 1 if the float fast path was disabled (extreme ranges) */
    int64_t vidx[CUDAPRE_MAX_SLOTS];     /* global index of each ring vertex */
    cudapre_pt v[CUDAPRE_MAX_SLOTS];     /* ring vertex coordinates */
    float box[4];                        /* inner box x0,x1,y0,y1 strictly inside the ring (x0>x1: none) */
    float circle[4];                     /* inner disk: centre x, y; r2 with RN32(RN32(dx^2)+RN32(dy^2)), d = RN32(p - c),
                                          * < r2 => strictly inside (r2 < 0: none); pad */
    float err_max;                       /* largest per-edge float error bound E_j */
    int32_t pad;
    /* Step-3 kernel line tests, edge j = v[j] -> v[j+1]:  g_j(p) = fma(A_j, p.x,
     * fma(B_j, p.y, C_j)) with C_j already lowered by E_j, where E_j bounds
     * |float evaluation - exact orient(v_j, v_j+1, p)| over the exact data
     * bounding box.                                        */
    float A[CUDAPRE_MAX_SLOTS], B[CUDAPRE_MAX_SLOTS], C[CUDAPRE_MAX_SLOTS], E[CUDAPRE_MAX_SLOTS];
    /* Step-3 sector test around the centre (circle[0], circle[1]): with
     * (dx, dy) = RN32(p - c), t = dy / (|dx| + |dy|) and the pseudo-angle
     * pa = t + 1 (dx >= 0) or 3 - t (dx < 0) in [0, 4], bucket
     * b = round(256 pa); RN32(RN32(dx^2) + RN32(dy^2)) < sector_r2[b] implies p
     * strictly inside the ring.  -1 = bucket disabled.
     * sector_out_r2[b]: RN32(...) > sector_out_r2[b] implies p strictly
     * outside the ring (+inf = disabled).                                  */
    float sector_r2[CUDAPRE_SECTORS + 1];
    float sector_out_r2[CUDAPRE_SECTORS + 1];
} cudapre_polygon_t;

/* Per-call report (S:118-123 FilterReport; per-phase timings S:189). */
typedef struct {
    int64_t n;                           /* points filtered by this call */
    int64_t survivors;                   /* points kept (== *h_count) */
    double ms_extremes_kernels;          /* device time of the Step-1 kernels (CUDA events) */
    double ms_filter_kernel;             /* device time of the Step-3 kernel (CUDA events) */
    double ms_polygon_host;              /* host time of Step 2 */
    int32_t launches;                    /* kernels launched by the call */
    int32_t pad;
    int64_t lookback_rounds;             /* Step-3 look-back rounds (256 status words each),
                                          * counted since the last Step-1 call on the workspace */
    int64_t lookback_spins;              /* of which had to wait for a predecessor */
} cudapre_report_t;

/* ---------------------------------------------------------------- helpers */

/* Library version string. */
const char* cudapre_version(void);

/* Message for the last non-OK status returned on this thread ("" if none). */
const char* cudapre_last_error(void);

/* Angle presets (A1).  preset 0 = {0, 30, 45, 60} degrees (default);
 * preset 1 = {0, 30, 45, 45} (P:25, P:35 literal text); preset 2 = {0}
 * (Akl-Toussaint quadrilateral); preset 3 = {0, 22.5, 45, 67.5}
 * (even spacing); preset 4 = {0, 15, 22.5, 30, 45, 60, 67.5, 75} ("more
 * angles": 32 extremes, rings of up to 32 vertices).
 * Writes *nang and the correctly rounded c[k] = cos, s[k] = sin (A5) into
 * caller arrays of CUDAPRE_MAX_ANGLES doubles.  INVALID_ARGUMENT for an
 * unknown preset.                                                          */
cudapre_status cudapre_angles_preset(int preset, int32_t* nang, double* c, double* s);

/* Bytes of device workspace needed for shards of up to n_local points. */
size_t cudapre_workspace_bytes(int64_t n_local);

/* Zero-fill a workspace on `stream` (required once before first use). */
cudapre_status cudapre_workspace_init(void* d_ws, size_t ws_bytes, void* stream);

/* --------------------------------------------------------------- Step 1 */

/* Step 1 over the local shard d_pts[0, n_local):
 * one streaming pass (HBM read of 8 bytes/point) reduces all 4*nang keys.
 *   d_pts       device, n_local points (may be NULL iff n_local == 0)
 *   index_base  global index of d_pts[0]
 *   nang, c, s  angle list (host arrays of nang doubles; c[0]=1, s[0]=0
 *               required); NULL c/s = preset 0
 *   d_ws        workspace of ws_bytes >= cudapre_workspace_bytes(n_local)
 *   stream      cudaStream_t as void*
 *   d_out       nullable DEVICE cudapre_extremes_t receiving the result
 *               (e.g. for an NCCL all-gather across ranks)
 *   h_out       nullable HOST cudapre_extremes_t; if given the call blocks
 *               until it is valid
 *   h_rep       nullable report (ms_extremes_kernels, launches)
 * Errors: EMPTY_INPUT if n_local == 0 — the empty part (n = 0, every idx
 * = -1) is still written to d_out / h_out, so a caller that shards one point
 * set may treat EMPTY_INPUT from one shard as benign and merge it;
 * NONFINITE_INPUT (result still written, flagged); INVALID_ARGUMENT;
 * WORKSPACE; CUDA.                                                         */
cudapre_status cudapre_extremes(const cudapre_pt* d_pts, int64_t n_local, int64_t index_base,
                                int32_t nang, const double* c, const double* s,
                                void* d_ws, size_t ws_bytes, void* stream,
                                cudapre_extremes_t* d_out, cudapre_extremes_t* h_out,
                                cudapre_report_t* h_rep);

/* Combine per-shard Step-1 results (host): for every slot the lexicographic
 * (key, global index) extreme — the same rule as inside one GPU, so the
 * result is independent of how the points were sharded.
 * EMPTY_INPUT if the parts hold no point at all.                           */
cudapre_status cudapre_extremes_merge(const cudapre_extremes_t* h_parts, int32_t count,
                                      cudapre_extremes_t* h_out);

/* --------------------------------------------------------------- Step 2 */

/* Step 2 on the host: distinct picks -> Andrew's
 * monotone chain with the EXACT orientation predicate (A11) -> ring, plus
 * the Step-3 kernel parameters (per-edge float coefficients with rigorous
 * error bounds over the exact data bounding box, inner box).               */
cudapre_status cudapre_polygon(const cudapre_extremes_t* h_ext, cudapre_polygon_t* h_poly);

/* --------------------------------------------------------------- Step 3 */

/* Steps 2+3: builds the polygon from h_ext (the GLOBAL
 * extremes, merged if sharded), then one streaming pass over the local shard
 * classifies every point and stream-compacts the survivors.
 * Point i is DISCARDED iff orient(v_j, v_j+1, p_i) > 0 exactly for every
 * ring edge j (strictly inside, A12); everything else survives.  Survivors
 * are written in ascending global index order (A15):
 *   d_surv_idx  device int64[capacity]   global indices (required)
 *   d_surv_pts  device cudapre_pt[capacity] their coordinates (nullable)
 *   h_count     host: number of survivors (always written on OK/CAPACITY)
 *   h_poly      nullable host copy of the polygon used
 *   h_rep       nullable report
 * The call blocks until *h_count is valid.  Degenerate polygon: every point
 * survives — not an error.  CAPACITY if *h_count > capacity (the
 * first `capacity` survivors are written).                                 */
cudapre_status cudapre_filter(const cudapre_pt* d_pts, int64_t n_local, int64_t index_base,
                              const cudapre_extremes_t* h_ext,
                              int64_t* d_surv_idx, cudapre_pt* d_surv_pts, int64_t capacity,
                              void* d_ws, size_t ws_bytes, void* stream,
                              int64_t* h_count, cudapre_polygon_t* h_poly,
                              cudapre_report_t* h_rep);

/* ----------------------------------------------------------- final hull */

/* Convex hull on the host by Andrew's monotone chain with
 * the exact orientation predicate, over h_pts[h_ids[j]] (h_ids NULL =
 * identity over 0..n-1).  h_ring (capacity n) receives the canonical ring
 * of point ids: CCW, starting at the lexicographically smallest (x, y)
 * vertex, collinear points excluded, duplicate coordinates represented by
 * their lowest id (A17).  *h_ring_len = 1 or 2 means a degenerate
 * point / segment; 0 for n == 0.                                           */
cudapre_status cudapre_hull(const cudapre_pt* h_pts, const int64_t* h_ids, int64_t n,
                            int64_t* h_ring, int64_t* h_ring_len);

/* ------------------------------------------------------- end to end */

/* The whole Steps 1-3 starting from HOST points (pinned memory recommended):
 * copies h_pts into the caller's device buffer d_pts (n points) on `stream`,
 * runs Step 1, Step 2 and Step 3 there, and copies the survivors' global
 * indices back into h_surv_idx (host int64[capacity]).  index_base = 0.
 * Same errors as cudapre_extremes / cudapre_filter.                        */
cudapre_status cudapre_run_host(const cudapre_pt* h_pts, int64_t n, int32_t nang,
                                const double* c, const double* s, cudapre_pt* d_pts,
                                void* d_ws, size_t ws_bytes, int64_t* d_surv_idx,
                                int64_t* h_surv_idx, int64_t capacity, void* stream,
                                int64_t* h_count, cudapre_report_t* h_rep);

/* ---------------------------------------------------------------- device-resident Steps 2-3
 * Step 2 (§2 Step 2, P:39 — the host chain in the
 * paper) can also run on the device, so Steps 1-3 are enqueued back to back
 * with no host round trip and can be captured in one CUDA graph.  The device
 * builder executes the same arithmetic as the host one (shared code, no FMA
 * contraction): the polygon and the Step-3 geometry are byte-identical.
 *
 * Workspace pages written by the device path (readable by the caller): the
 * Step-3 geometry at byte CUDAPRE_WS_GEOM_OFFSET and the polygon
 * (cudapre_polygon_t) at CUDAPRE_WS_POLY_OFFSET; the Step-1 result that
 * cudapre_extremes leaves on the device at CUDAPRE_WS_RESULT_OFFSET.     */
#define CUDAPRE_WS_GEOM_OFFSET 4096
#define CUDAPRE_WS_POLY_OFFSET (4096 + 16384)
#define CUDAPRE_WS_RESULT_OFFSET 176   /* the Step-1 result K1 leaves (cudapre_extremes_t) */

/* Host build of the Step-3 geometry block for h_ext (the block the device
 * path writes at CUDAPRE_WS_GEOM_OFFSET), for tests and inspection.
 * *needed (nullable) receives its size.  INVALID_ARGUMENT if out_bytes is
 * too small; EMPTY_INPUT if h_ext->n == 0.                                 */
cudapre_status cudapre_geometry(const cudapre_extremes_t* h_ext, void* h_out, size_t out_bytes,
                                size_t* needed);

/* Step 2 on the device: builds the polygon and the Step-3 geometry into the
 * workspace pages (and into d_poly if not NULL) from
 *   d_parts, nparts  device Step-1 results of nparts shards (e.g. an NCCL
 *                    all-gather of every rank's CUDAPRE_WS_RESULT_OFFSET
 *                    block), merged here with the rule of
 *                    cudapre_extremes_merge and the merge written to
 *                    this workspace's result block; d_parts NULL / nparts
 *                    <= 1: the result cudapre_extremes left in d_ws.
 * One block, one launch; byte-identical to cudapre_extremes_merge +
 * cudapre_polygon / cudapre_geometry.                                      */
cudapre_status cudapre_polygon_device(const cudapre_extremes_t* d_parts, int32_t nparts, void* d_ws,
                                      size_t ws_bytes, void* stream, cudapre_polygon_t* d_poly);

/* Step 3 alone, with the geometry already in the workspace (from
 * cudapre_polygon_device): the K2 launch + the device count copy.        */
cudapre_status cudapre_filter_geom(const cudapre_pt* d_pts, int64_t n_local, int64_t index_base,
                                   int64_t* d_surv_idx, cudapre_pt* d_surv_pts, int64_t capacity,
                                   void* d_ws, size_t ws_bytes, void* stream, int64_t* d_count);

/* Steps 2 + 3 on the stream (cudapre_polygon_device + cudapre_filter_geom),
 * nothing waits for the host.
 *   d_ext      device Step-1 result; NULL = the one cudapre_extremes left in d_ws
 *   d_count    device int64 (nullable): the survivor count (may exceed capacity;
 *              only the first `capacity` survivors are written)
 *   d_poly     device polygon struct, nullable (default: the workspace page)
 * Other arguments as cudapre_filter.  A degenerate ring keeps every point;
 * non-finite input (flagged in the Step-1 result) keeps every point too —
 * check d_ext->nonfinite before trusting the survivors.  Capture-safe.    */
cudapre_status cudapre_filter_device(const cudapre_pt* d_pts, int64_t n_local, int64_t index_base,
                                     const cudapre_extremes_t* d_ext, int64_t* d_surv_idx,
                                     cudapre_pt* d_surv_pts, int64_t capacity, void* d_ws,
                                     size_t ws_bytes, void* stream, int64_t* d_count,
                                     cudapre_polygon_t* d_poly);

/* Steps 1-3 on the stream (single GPU or one shard without the cross-rank
 * combine): cudapre_extremes without host outputs + cudapre_filter_device.
 * Capture-safe after one uncaptured call (launcher set-up).               */
cudapre_status cudapre_pipeline_device(const cudapre_pt* d_pts, int64_t n_local, int64_t index_base,
                                       int32_t nang, const double* c, const double* s,
                                       int64_t* d_surv_idx, cudapre_pt* d_surv_pts, int64_t capacity,
                                       void* d_ws, size_t ws_bytes, void* stream, int64_t* d_count);

/* Steps 1-3 with the paper's host Step 2 between the kernels, one
 * call, one host wait per step: K1's last block writes the Step-1 result into
 * a mapped pinned host block, the host waits for it, builds the polygon and
 * the Step-3 geometry, enqueues one H2D copy of the geometry and K2, and
 * returns; the survivor count stays on the device (*d_count, nullable).
 *   h_poly         nullable host copy of the polygon
 *   h_ms_polygon   nullable: host time of Step 2 (ms)
 * Other arguments as cudapre_pipeline_device.  EMPTY_INPUT / NONFINITE_INPUT
 * as cudapre_extremes (nothing enqueued after Step 1 then).               */
cudapre_status cudapre_pipeline_host(const cudapre_pt* d_pts, int64_t n_local, int64_t index_base,
                                     int32_t nang, const double* c, const double* s,
                                     int64_t* d_surv_idx, cudapre_pt* d_surv_pts, int64_t capacity,
                                     void* d_ws, size_t ws_bytes, void* stream, int64_t* d_count,
                                     cudapre_polygon_t* h_poly, double* h_ms_polygon);

/* One CUDA graph of cudapre_pipeline_device on fixed buffers: create runs
 * the pipeline once on `stream` (synchronised), then captures it; launch
 * replays it (one graph launch per step); destroy frees it.  The buffers
 * must outlive the graph.                                                 */
typedef struct cudapre_graph cudapre_graph_t;
cudapre_status cudapre_graph_create(const cudapre_pt* d_pts, int64_t n_local, int64_t index_base,
                                    int32_t nang, const double* c, const double* s,
                                    int64_t* d_surv_idx, cudapre_pt* d_surv_pts, int64_t capacity,
                                    void* d_ws, size_t ws_bytes, void* stream, int64_t* d_count,
                                    cudapre_graph_t** out);
cudapre_status cudapre_graph_launch(cudapre_graph_t* g, void* stream);
cudapre_status cudapre_graph_destroy(cudapre_graph_t* g);

/* ---------------------------------------------------------------- final hull on the GPU
 * SURVEY §8 f1 (the paper runs Qhull on the survivors).
 * The canonical ring of the survivors (identical to cudapre_hull on them)
 * from device buffers:
 *   d_pts, d_ids, m   the survivors: points and their global ids (e.g. the
 *                     outputs of cudapre_filter / cudapre_filter_device)
 *   h_poly            the Step-2 polygon they were filtered with (its disk
 *                     centre anchors the second filter)
 *   d_scratch         >= cudapre_hull_device_bytes(m) bytes of device memory
 *   h_ring            host int64[ring_capacity]: the ring's global ids, CCW
 *                     from the lexicographically smallest vertex
 *   h_remaining       (nullable) points left for the host chain (diagnostic)
 * Two kernels filter the survivors again with an inner polygon P' of up to
 * 4097 survivors (farthest point per pseudo-angle sector, exact hull) —
 * discarding only points strictly inside P' (exact predicate) — and the
 * host's monotone chain finishes on the rest.  Without a certified centre
 * (degenerate polygon) the chain runs on every survivor.  Synchronises the
 * stream.  CAPACITY if the ring exceeds ring_capacity.                   */
size_t cudapre_hull_device_bytes(int64_t m);
/* cudapre_hull_device that also returns the ring's coordinates
 * (h_ring_pts: host cudapre_pt[ring_capacity], nullable).                  */
cudapre_status cudapre_hull_device_ex(const cudapre_pt* d_pts, const int64_t* d_ids, int64_t m,
                                      const cudapre_polygon_t* h_poly, void* d_scratch, size_t scratch_bytes,
                                      void* stream, int64_t* h_ring, cudapre_pt* h_ring_pts,
                                      int64_t ring_capacity, int64_t* h_ring_len, int64_t* h_remaining);
cudapre_status cudapre_hull_device(const cudapre_pt* d_pts, const int64_t* d_ids, int64_t m,
                                   const cudapre_polygon_t* h_poly, void* d_scratch, size_t scratch_bytes,
                                   void* stream, int64_t* h_ring, int64_t ring_capacity,
                                   int64_t* h_ring_len, int64_t* h_remaining);

/* ---------------------------------------------------------------- multi-GPU (e)
 * One process per GPU.  The points are sharded into contiguous global index
 * ranges, rank r holding [base_r, base_r + n_r) with base_r increasing in r
 * (pass base_r as index_base everywhere).  The communicator wraps NCCL, which
 * is loaded at run time (libnccl.so.2; CUDAPRE_ERR_NCCL if it is missing); it
 * is bound to the CUDA device current at cudapre_comm_create.
 *
 * cudapre_comm_unique_id   rank 0 makes the 128-byte NCCL id (h_id) and the
 *                          caller distributes it (e.g. a torch broadcast)
 * cudapre_comm_create      collective over the `world` ranks; *out owned by
 *                          the caller, freed with cudapre_comm_destroy      */
typedef struct cudapre_comm cudapre_comm_t;
cudapre_status cudapre_comm_unique_id(void* h_id);
cudapre_status cudapre_comm_create(const void* h_id, int32_t rank, int32_t world, cudapre_comm_t** out);
cudapre_status cudapre_comm_destroy(cudapre_comm_t* comm);
cudapre_status cudapre_comm_rank(const cudapre_comm_t* comm, int32_t* rank, int32_t* world);

/* Cross-rank combine input: all-gather of every rank's Step-1 result block
 * (the one cudapre_extremes left at CUDAPRE_WS_RESULT_OFFSET of d_ws) into
 * d_parts (device, world entries, rank order), enqueued on `stream` (no host
 * synchronisation; capturable).  Merge with cudapre_polygon_device(d_parts,
 * world, ...) on the device or cudapre_extremes_merge on the host.        */
cudapre_status cudapre_comm_allgather_extremes(cudapre_comm_t* comm, const void* d_ws,
                                               cudapre_extremes_t* d_parts, void* stream);

/* Step 1 of a sharded set with the paper's host Step 2 in mind: K1 on the
 * local shard (may be empty), the all-gather, and the host merge: h_out =
 * the single-GPU result of the whole set on every rank (then call
 * cudapre_filter with it).  Blocks.  EMPTY_INPUT if every shard is empty.   */
cudapre_status cudapre_extremes_comm(const cudapre_pt* d_pts, int64_t n_local, int64_t index_base,
                                     int32_t nang, const double* c, const double* s, void* d_ws,
                                     size_t ws_bytes, cudapre_comm_t* comm, cudapre_extremes_t* d_parts,
                                     void* stream, cudapre_extremes_t* h_out);

/* Steps 1-3 of a sharded set on the stream, no host synchronisation: K1 on
 * the local shard, the all-gather into d_parts, the merge and Step 2 on the
 * device (every rank builds the same polygon), Step 3 on the local shard.
 * Survivors (ascending global indices of this shard) in d_surv_idx /
 * d_surv_pts, their number in *d_count (device int64).  An empty shard
 * (n_local == 0, d_pts may be NULL) takes part in the collective with an
 * empty Step-1 block and gets *d_count = 0.                                 */
cudapre_status cudapre_pipeline_comm(const cudapre_pt* d_pts, int64_t n_local, int64_t index_base,
                                     int32_t nang, const double* c, const double* s, int64_t* d_surv_idx,
                                     cudapre_pt* d_surv_pts, int64_t capacity, void* d_ws, size_t ws_bytes,
                                     cudapre_comm_t* comm, cudapre_extremes_t* d_parts, void* stream,
                                     int64_t* d_count);

/* Survivor collection: every rank passes its `count` survivors (d_idx and,
 * nullable, d_pts); the root receives all of them in rank order = ascending
 * global index order (the single-GPU survivor array) in d_out_idx /
 * d_out_pts (root only; capacity out_capacity, ignored on other ranks).
 * *h_total = the number of survivors, on every rank.  An all-gather of
 * (count, the root's capacity, whether the root takes points, whether this
 * rank's arguments are usable) — 32 bytes per rank — then one grouped
 * ncclSend / ncclRecv; blocks.  Every rank takes the same decision from the
 * gathered words, so errors are collective (no rank is left waiting):
 * CAPACITY on every rank if the total exceeds the root's out_capacity (or
 * the root passed no d_out_idx; nothing is sent, *h_total says how much is
 * needed); INVALID_ARGUMENT on every rank if some rank passed count < 0, a
 * NULL d_idx with count > 0, or no d_pts while the root takes points
 * (d_out_pts != NULL).                                                      */
cudapre_status cudapre_gather_survivors(cudapre_comm_t* comm, const int64_t* d_idx, const cudapre_pt* d_pts,
                                        int64_t count, int32_t root, int64_t* d_out_idx, cudapre_pt* d_out_pts,
                                        int64_t out_capacity, void* stream, int64_t* h_total);

/* Final hull of the sharded set: each rank's GPU hull of its own
 * survivors (cudapre_hull_device with its polygon), the rings' vertices
 * gathered on the root, the root's monotone chain over them: hull(U S_r) =
 * hull(U hull(S_r)).  The root gets the canonical ring of the whole set (as
 * cudapre_hull on all survivors) in h_ring; other ranks get *h_ring_len = 0.
 * Blocks.  Errors are collective: a rank whose local hull fails still takes
 * part in the counts exchange, and every rank then returns an error.       */
cudapre_status cudapre_hull_comm(cudapre_comm_t* comm, const cudapre_pt* d_pts, const int64_t* d_ids, int64_t m,
                                 const cudapre_polygon_t* h_poly, void* d_scratch, size_t scratch_bytes,
                                 int32_t root, void* stream, int64_t* h_ring, int64_t ring_capacity,
                                 int64_t* h_ring_len);

/* ====================================================================
 * The 3D extension (DESIGN.md §3 B1-B6, §6.5).
 * "In 3D, typically six extreme points can be obtained by finding those
 * points with the min or max x, y, or z coordinates.  More groups of six
 * extreme points can also be found after rotating the set of points along a
 * specific axis.  These extreme points can be then used to form a convex
 * polyhedron.  Those points locating inside the convex polyhedron must be
 * interior points, and can be directly discarded."
 * Points are float32 xyz AoS (12 bytes each), caller-owned device memory,
 * 4-byte aligned (16-byte aligned: vector path).  The workspace is its own
 * (cudapre3_workspace_bytes), zero-filled once with cudapre_workspace_init.
 * ==================================================================== */
#define CUDAPRE3_MAX_SLOTS (6 * CUDAPRE_MAX_ANGLES)   /* 48 */
#define CUDAPRE3_MAX_FACETS 64                       /* >= 2 * (4 * 8 + 2) - 4 */

typedef struct { float x, y, z; } cudapre_pt3;

/* Step 1 in 3D (B1, B2): rotation about the z axis.  Slot 6k+{0..5} =
 * {argmin X_k, argmax X_k, argmin Y_k, argmax Y_k, argmin Z, argmax Z} with
 * X_k, Y_k as in 2D (binary64, no FMA) and Z = z; lowest index on equal
 * keys.  The Z slots repeat for every k (a rotation about z leaves z as is). */
typedef struct {
    int32_t nang;                          /* angles (slots = 6*nang); angle 0 first */
    int32_t nonfinite;                     /* 1 if a non-finite coordinate was seen */
    int64_t n;                             /* points reduced (summed over merged parts) */
    int64_t idx[CUDAPRE3_MAX_SLOTS];       /* global index of each pick, -1 if none */
    double key[CUDAPRE3_MAX_SLOTS];        /* binary64 key of each pick */
    cudapre_pt3 pt[CUDAPRE3_MAX_SLOTS];    /* coordinates of each pick */
    double c[CUDAPRE_MAX_ANGLES];          /* cos / sin of each angle (correctly rounded, A5) */
    double s[CUDAPRE_MAX_ANGLES];
    int64_t exact_points;                  /* diagnostic: points through the exact binary64 path */
} cudapre3_extremes_t;

/* Step 2 in 3D (B3, B4): the polyhedron conv(E), E = the distinct picks
 * (equal coordinates -> lowest index), ascending index.  Facet f is the
 * first supporting triple (a < b < c in E's order) of each facet plane,
 * stored so that E lies on its positive side: a point p is strictly inside
 * iff orient3d(fv[f], p) > 0 for every f (B5, B6).  nf = 0: degenerate
 * (|E| < 4 or E coplanar): nothing is inside.                              */
typedef struct {
    int32_t nf;                                 /* facet planes, 0 = degenerate */
    int32_t n_distinct;                         /* |E| */
    int32_t cells;                              /* 1: per-direction-cell candidate lists around centre */
    int32_t n_entries;                          /* candidate facets summed over the 384 cells */
    int64_t eidx[CUDAPRE3_MAX_SLOTS];           /* E (global ids, ascending) */
    int64_t fidx[CUDAPRE3_MAX_FACETS][3];       /* supporting triple of each facet plane */
    cudapre_pt3 fv[CUDAPRE3_MAX_FACETS][3];     /* its coordinates */
    float centre[3];                            /* strictly inside (cells == 1) */
    float err_max;                              /* largest plane-test error bound */
    int32_t max_candidates;                     /* largest candidate list of a cell */
    int32_t long_cells;                         /* cells whose list exceeds the kernel's 3 slots */
    int32_t n_cells;                            /* direction cells (6 * 32 * 32) */
    int32_t empty_cells;                        /* cells with no candidate facet (set to every facet
                                                 * as a fail-safe; 0 by construction) */
    int32_t pad[4];
} cudapre3_polyhedron_t;

/* Workspace bytes for a shard of n_local points (3D). */
size_t cudapre3_workspace_bytes(int64_t n_local);

/* Step 1 in 3D over d_xyz[0, n_local) (one streaming pass, 12 bytes/point):
 *   d_xyz       device float[3*n_local] (NULL iff n_local == 0), 4-B aligned
 *   index_base  global index of the first point
 *   nang, c, s  angle list (host, c[0] = 1, s[0] = 0 required; NULL = preset 0)
 *   d_out       nullable DEVICE cudapre3_extremes_t receiving the result
 *   h_out       nullable HOST result; if given the call blocks until valid
 *   h_ms_kernel nullable: device time of the K1-3D launch (CUDA events on
 *               `stream`; the call then blocks)
 * Errors: EMPTY_INPUT (n_local == 0; the empty part, every idx = -1, is still
 * written), NONFINITE_INPUT (result written, flagged), INVALID_ARGUMENT,
 * WORKSPACE, CUDA.  n_local < 2^32.                                        */
cudapre_status cudapre3_extremes(const float* d_xyz, int64_t n_local, int64_t index_base, int32_t nang,
                                 const double* c, const double* s, void* d_ws, size_t ws_bytes,
                                 void* stream, cudapre3_extremes_t* d_out, cudapre3_extremes_t* h_out,
                                 double* h_ms_kernel);

/* Shard merge (host): per slot the lexicographic (key, global index) extreme. */
cudapre_status cudapre3_extremes_merge(const cudapre3_extremes_t* h_parts, int32_t count,
                                       cudapre3_extremes_t* h_out);

/* Step 2 in 3D on the host: the polyhedron of h_ext (global extremes). */
cudapre_status cudapre3_polyhedron(const cudapre3_extremes_t* h_ext, cudapre3_polyhedron_t* h_poly);

/* Steps 2+3 in 3D: builds the polyhedron from h_ext, then one streaming pass
 * classifies every local point and stream-compacts the survivors in
 * ascending global index order.  Point i is DISCARDED iff orient3d(f, p_i)
 * > 0 exactly for every facet f; degenerate polyhedron: all survive.
 *   d_surv_idx  device int64[capacity] global indices (required)
 *   d_surv_xyz  device float[3*capacity] their coordinates (nullable)
 *   h_count     host: number of survivors (always written on OK / CAPACITY)
 *   h_poly      nullable host copy of the polyhedron used
 *   h_ms_kernel nullable: device time of the K2-3D launch (CUDA events)
 * Blocks until *h_count is valid.  NONFINITE_INPUT if h_ext is flagged.
 * CAPACITY if *h_count > capacity (the first `capacity` are written).      */
cudapre_status cudapre3_filter(const float* d_xyz, int64_t n_local, int64_t index_base,
                               const cudapre3_extremes_t* h_ext, int64_t* d_surv_idx, float* d_surv_xyz,
                               int64_t capacity, void* d_ws, size_t ws_bytes, void* stream,
                               int64_t* h_count, cudapre3_polyhedron_t* h_poly, double* h_ms_kernel);

/* cudapre3_filter with explicit options: flags = 0 is cudapre3_filter;
 * CUDAPRE3_FLAG_NO_CELLS forces the every-facet path (no direction cells:
 * every point goes through the warp-cooperative all-facet test, the path the
 * library takes by itself when the centre is not certified).  Same result.
 * INVALID_ARGUMENT for unknown flag bits.                                   */
#define CUDAPRE3_FLAG_NO_CELLS 1
cudapre_status cudapre3_filter_ex(const float* d_xyz, int64_t n_local, int64_t index_base,
                                  const cudapre3_extremes_t* h_ext, int64_t* d_surv_idx, float* d_surv_xyz,
                                  int64_t capacity, void* d_ws, size_t ws_bytes, void* stream,
                                  int64_t* h_count, cudapre3_polyhedron_t* h_poly, double* h_ms_kernel,
                                  int32_t flags);

/* Test hook (host): the direction cells K2-3D would use for h_ext — for
 * every cell the mask of candidate facets (bit j = facet j in
 * cudapre3_polyhedron's order), the centre, and the grid G (6 * G * G
 * cells; cell = (face * G + iu) * G + iv with face = 2 * axis + (d_axis < 0)
 * and (u, v) = the other two components in the order (y, z), (z, x),
 * (x, y)).  n_cells must be >= 6 * G * G (query with h_masks = NULL).
 * *h_cells = 0 when the centre is not strictly inside (every cell = every
 * facet) or the polyhedron is degenerate.                                  */
cudapre_status cudapre3_cells(const cudapre3_extremes_t* h_ext, uint64_t* h_masks, int32_t n_cells,
                              float* h_centre, int32_t* h_grid, int32_t* h_cells);

/* Test hook (host): K2-3D's float plane test of each facet, 5 floats per
 * facet (A, B, C, D, E): g = fma(A, x, fma(B, y, fma(C, z, D))) (float32)
 * is within E of orient3d(facet, p) for every p in the data bounding box
 * (E = +inf: the facet always takes the exact predicate).                  */
cudapre_status cudapre3_planes(const cudapre3_extremes_t* h_ext, float* h_planes, int32_t capacity,
                               int32_t* h_nf);

/* Exact orient3d sign of float triples (host; tests and callers): sign of
 * det[b-a; c-a; d-a].                                                       */
int32_t cudapre3_orient(const float* a, const float* b, const float* c, const float* d);

#ifdef __cplusplus
}
#endif

#endif /* CUDAPRE_H */
