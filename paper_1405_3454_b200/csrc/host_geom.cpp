// host_geom.cpp — host side of the CudaPre pipeline:
//   * Step 2: Andrew's monotone chain of the <= 16 extreme
//     points with the exact orientation predicate (A10, A11), and the
//     parameters the Step-3 kernel needs (per-edge float line coefficients with
//     rigorous error bounds, an inner box) — DESIGN.md §6.2.
//   * the final hull of the survivors, canonical ring (A17).
//   * the cross-shard merge of Step-1 results.
// Compiled with -ffp-contract=off (no FMA contraction anywhere in this file).
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>
#include <vector>

#include "exact.cuh"
#include "geom.cuh"
#include "internal.h"

namespace cudapre {

int orient_exact(float ax, float ay, float bx, float by, float cx, float cy) {
    return orient_sign_f(ax, ay, bx, by, cx, cy);
}

namespace {

struct CP {
    float x, y;
    int64_t id;
};

bool lex_less(const CP& a, const CP& b) {
    if (a.x < b.x) return true;
    if (a.x > b.x) return false;
    if (a.y < b.y) return true;
    if (a.y > b.y) return false;
    return a.id < b.id;
}

int turn(const CP& a, const CP& b, const CP& c) { return orient_exact(a.x, a.y, b.x, b.y, c.x, c.y); }

// Andrew's monotone chain over P (sorted in place).  Writes ring ids, returns length.
int64_t chain(std::vector<CP>& P, int64_t* ring) {
    const int64_t m = (int64_t)P.size();
    if (m == 0) return 0;
    std::sort(P.begin(), P.end(), lex_less);
    // distinct coordinates: first of each run has the lowest id (-0 == +0)
    int64_t u = 1;
    for (int64_t j = 1; j < m; ++j)
        if (P[j].x != P[u - 1].x || P[j].y != P[u - 1].y) P[u++] = P[j];
    if (u == 1) {
        ring[0] = P[0].id;
        return 1;
    }
    std::vector<CP> H((size_t)(2 * u + 1));
    int64_t k = 0;
    for (int64_t j = 0; j < u; ++j) {   // lower chain, pop while not a strict left turn
        while (k >= 2 && turn(H[k - 2], H[k - 1], P[j]) <= 0) --k;
        H[k++] = P[j];
    }
    const int64_t lower = k;
    for (int64_t j = u - 2; j >= 0; --j) {   // upper chain
        while (k > lower && turn(H[k - 2], H[k - 1], P[j]) <= 0) --k;
        H[k++] = P[j];
    }
    --k;   // the last point repeats the first
    for (int64_t j = 0; j < k; ++j) ring[j] = H[j].id;
    return k;
}

}  // namespace

int64_t hull_ring(const cudapre_pt* pts, const int64_t* ids, int64_t n, int64_t* ring) {
    std::vector<CP> P((size_t)n);
    for (int64_t j = 0; j < n; ++j) {
        const int64_t id = ids ? ids[j] : j;
        P[j] = CP{pts[id].x, pts[id].y, id};
    }
    return chain(P, ring);
}

int64_t hull_ring_points(const cudapre_pt* pts, const int64_t* ids, int64_t n, int64_t* ring_ids,
                         cudapre_pt* ring_pts) {
    std::vector<CP> P((size_t)n);
    for (int64_t j = 0; j < n; ++j) P[j] = CP{pts[j].x, pts[j].y, ids[j]};
    const int64_t k = chain(P, ring_ids);
    if (ring_pts) {   // chain() sorted P; look the ring ids up by binary search over ids
        std::vector<CP> byid(P);
        std::sort(byid.begin(), byid.end(), [](const CP& a, const CP& b) { return a.id < b.id; });
        for (int64_t j = 0; j < k; ++j) {
            const auto it = std::lower_bound(byid.begin(), byid.end(), ring_ids[j],
                                             [](const CP& a, int64_t id) { return a.id < id; });
            ring_pts[j] = cudapre_pt{it->x, it->y};
        }
    }
    return k;
}

void hull_bucket_table(const cudapre_pt* v, int nv, float cx, float cy, unsigned* table) {
    // exit edge of the ray of pseudo-angle pa around c: the first edge counted
    // from cs (first max of the vertex pseudo-angles) whose closed range holds
    // pa (geom.cuh phase F); candidates of bucket b: exit edge of its lower
    // guarded boundary ray to that of its upper one (a rounding slip near a
    // vertex only widens the range; points of the bucket lie >= 2^-16 in pa
    // from the boundary rays)
    std::vector<double> pv((size_t)nv), U((size_t)nv);
    for (int j = 0; j < nv; ++j) pv[j] = geom::pa_of((double)v[j].x - cx, (double)v[j].y - cy);
    int cs = 0;
    for (int j = 0; j < nv; ++j)
        if (pv[j] > pv[cs]) cs = j;
    for (int k = 0; k < nv; ++k) U[k] = pv[(cs + k + 1) % nv] + 4.0;
    auto exit_edge = [&](double pa) {
        if (pa < 0.0) pa += 4.0;
        if (pa >= 4.0) pa -= 4.0;
        const double q = pa < pv[cs] ? pa + 4.0 : pa;
        int lo = 0, hi = nv - 1;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (q <= U[mid]) hi = mid;
            else lo = mid + 1;
        }
        return (cs + lo) % nv;
    };
    const double g = geom::kGuard;
    for (int b = 0; b < kHullBuckets; ++b) {
        const int e0 = exit_edge((b - 0.5 - g) / 1024.0), e1 = exit_edge((b + 0.5 + g) / 1024.0);
        const int cnt = (e1 - e0 + nv) % nv + 1;
        table[b] = (unsigned)e0 | ((unsigned)cnt << 16);
    }
}

void merge_extremes(const cudapre_extremes_t* parts, int count, cudapre_extremes_t* out) {
    cudapre_extremes_t r = parts[0];   // (padding and unused slots as part 0)
    geom::merge_header(parts, count, r);
    for (int s = 0; s < 4 * r.nang; ++s) geom::merge_slot(parts, count, s, r);
    *out = r;
}

void build_polygon(const cudapre_extremes_t& ext, cudapre_polygon_t* poly, K2Geom* g) {
    using namespace geom;
    static thread_local Work w;
    static thread_local double rs[kS];
    static thread_local int exe[kS];
    static thread_local double rb[CUDAPRE_SECTORS + 1], ro[CUDAPRE_SECTORS + 1];
    std::memset(poly, 0, sizeof(*poly));
    phase_a(ext, w);
    defaults(w, poly, g);
    for (int j = 0; j <= CUDAPRE_MAX_SLOTS; ++j) defaults_item(w, poly, g, j);
    for (int b = 0; b <= CUDAPRE_SECTORS; ++b) {
        poly->sector_r2[b] = -1.0f;
        poly->sector_out_r2[b] = INFINITY;
        if (g) {
            g->sr2[b] = -1.0f;
            g->sro2[b] = INFINITY;
            g->sedge[b] = 0xffff;
        }
    }
    if (w.degenerate) return;
    for (int j = 0; j < w.nv; ++j) phase_b_edge(w, j);
    // inner box: 16-step binary search (it 0: the full extent)
    w.have_box = 0;
    if (box_searchable(w)) {
        double lo = 0.0, hi = 1.0;
        for (int it = 0; it < 16; ++it) {
            const double t = box_t(it, lo, hi);
            float c[4];
            box_corners(w, t, c);
            bool ok = c[0] <= c[1] && c[2] <= c[3];
            for (int q = 0; q < 4 && ok; ++q)
                for (int j = 0; j < w.nv && ok; ++j) ok = box_corner_edge_ok(w, c, q, j);
            if (ok) {
                w.have_box = 1;
                for (int q = 0; q < 4; ++q) w.box[q] = c[q];
                lo = t;
                if (it == 0) break;
            } else {
                hi = t;
            }
        }
    }
    // inner disk
    disk_centre(w);
    if (w.centre_ok)
        for (int j = 0; j < w.nv; ++j) phase_d_edge(w, j);
    disk_finish(w);
    // sector tables + candidate edges
    for (int j = 0; j < w.nv; ++j) phase_e_edge(w, j);
    sector_prep_finish(w);
    if (w.sok) {
        for (int i = 0; i < kS; ++i) phase_f_sample(w, i, rs[i], exe[i]);
        for (int b = 0; b <= CUDAPRE_SECTORS; ++b) phase_g_init(w, b, rs, rb[b], ro[b]);
        for (int j = 0; j < w.nv; ++j) {
            const double vr = vertex_radius(w, j);
            for_buckets_of(w.pv[j], [&](int bb) { ro[bb] = dmax(ro[bb], vr); });
            const double dj = w.dj[j];
            for_buckets_of(w.pn[j], [&](int bb) { rb[bb] = dmin(rb[bb], dj); });
        }
        for (int b = 0; b <= CUDAPRE_SECTORS; ++b) {
            float a2, o2;
            unsigned short se;
            phase_g_finish(w, b, rb[b], ro[b], exe, a2, o2, se);
            poly->sector_r2[b] = a2;
            poly->sector_out_r2[b] = o2;
            if (g) {
                g->sr2[b] = a2;
                g->sro2[b] = o2;
                g->sedge[b] = se;
            }
        }
    }
    for (int j = 0; j < w.nv; ++j) finish_item(w, poly, g, j);
    finish(w, poly, g);
}

}  // namespace cudapre
