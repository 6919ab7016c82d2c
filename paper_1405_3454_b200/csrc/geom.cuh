// geom.cuh — Step 2 of CudaPre (§2 Step 2; SPEC.md
// S:146-154) and the Step-3 parameters derived from the polygon, written ONCE
// as __host__ __device__ code shared by the host builder (host_geom.cpp,
// sequential) and the device builder (k_polygon.cu, one block, parallel over
// edges / corners / sample rays / buckets).  Every parallel phase computes
// per-item values with the same arithmetic and combines them with exact,
// order-independent reductions (min, max, and, or), and every sum is taken
// by one thread in a fixed order, so both builders produce byte-identical
// parameters (tests/test_gpu_parity.py checks it).  Both translation units
// are compiled without FMA contraction (host: -ffp-contract=off, device:
// -fmad=false).  The rigour arguments are in DESIGN.md §6.2.
#pragma once

#include <cmath>
#include <cstdint>

#include "exact.cuh"
#include "internal.h"

#if defined(__CUDACC__)
#define GEOM_HD __host__ __device__ __forceinline__
#else
#define GEOM_HD inline
#endif

namespace cudapre {
namespace geom {

constexpr int kS = 2 * (CUDAPRE_SECTORS + 2);   // sample rays: pseudo-angles (k - 0.5 -+ 1/64)/256, k = 0..1025
constexpr double kGuard = 1.0 / 64.0;

struct Pick {
    float x, y;
    long long id;
};

// Everything the phases exchange (lives in shared memory on the device).
struct Work {
    // phase A
    int nv, n_distinct, degenerate;
    long long vid[CUDAPRE_MAX_SLOTS];
    float vx[CUDAPRE_MAX_SLOTS], vy[CUDAPRE_MAX_SLOTS];
    double Mx, My;                       // exact data bbox (angle-0 picks)
    double ox, oy, hw, hh;               // vertex mean, half extents
    // phase B (per edge)
    float A[CUDAPRE_MAX_SLOTS], B[CUDAPRE_MAX_SLOTS], C[CUDAPRE_MAX_SLOTS], E[CUDAPRE_MAX_SLOTS];
    int bad[CUDAPRE_MAX_SLOTS];
    // phase C (box)
    float box[4];
    int have_box;
    // phase D (disk)
    float cx, cy, r2;
    double rmin_e[CUDAPRE_MAX_SLOTS];
    int dok_e[CUDAPRE_MAX_SLOTS];
    int centre_ok;
    // phase E (sector prep)
    double dj[CUDAPRE_MAX_SLOTS], rsu[CUDAPRE_MAX_SLOTS], nx[CUDAPRE_MAX_SLOTS], ny[CUDAPRE_MAX_SLOTS],
        pn[CUDAPRE_MAX_SLOTS], pv[CUDAPRE_MAX_SLOTS], U[CUDAPRE_MAX_SLOTS];
    int sok_e[CUDAPRE_MAX_SLOTS];
    int sok, cs;
    double rs_up;
};

// ------------------------------------------------------------------ helpers
GEOM_HD bool gfinite(double x) {
#if defined(__CUDA_ARCH__)
    return isfinite(x);
#else
    return std::isfinite(x);
#endif
}
GEOM_HD float gnextafter(float x, float to) {
#if defined(__CUDA_ARCH__)
    return nextafterf(x, to);
#else
    return std::nextafter(x, to);
#endif
}
// std::min / std::max semantics (the first argument on ties / NaN)
GEOM_HD double dmin(double a, double b) { return (b < a) ? b : a; }
GEOM_HD double dmax(double a, double b) { return (a < b) ? b : a; }
GEOM_HD float smax(float a, float b) { return (a < b) ? b : a; }
GEOM_HD bool pick_less(const Pick& a, const Pick& b) {
    if (a.x < b.x) return true;
    if (a.x > b.x) return false;
    if (a.y < b.y) return true;
    if (a.y > b.y) return false;
    return a.id < b.id;
}
// float nearest-below / nearest-above of a double (directed conversion)
GEOM_HD float f_down(double d) {
    float f = (float)d;
    if ((double)f > d) f = gnextafter(f, -INFINITY);
    return f;
}
GEOM_HD float f_up(double d) {
    float f = (float)d;
    if ((double)f < d) f = gnextafter(f, INFINITY);
    return f;
}
GEOM_HD double pa_of(double ux, double uy) {
    const double t = uy / (fabs(ux) + fabs(uy));
    return ux >= 0.0 ? t + 1.0 : 3.0 - t;
}
// unnormalised direction of pseudo-angle pa (wrapped into [0, 4)):
// pa in [0,2]: t = pa-1, (1-|t|, t);  pa in [2,4]: t = 3-pa, (-(1-|t|), t)
GEOM_HD void pa_dir(double pa, double& ux, double& uy) {
    if (pa < 0.0) pa += 4.0;
    if (pa >= 4.0) pa -= 4.0;
    if (pa <= 2.0) {
        const double t = pa - 1.0;
        ux = 1.0 - fabs(t);
        uy = t;
    } else {
        const double t = 3.0 - pa;
        ux = -(1.0 - fabs(t));
        uy = t;
    }
}
GEOM_HD double sample_pa(int i) {
    double pw = ((double)(i >> 1) - 0.5 + ((i & 1) ? kGuard : -kGuard)) / 256.0;
    if (pw < 0.0) pw += 4.0;
    if (pw >= 4.0) pw -= 4.0;
    return pw;
}
GEOM_HD bool strictly_inside_ring(const float* vx, const float* vy, int nv, float px, float py) {
    for (int j = 0; j < nv; ++j) {
        const int k = j + 1 == nv ? 0 : j + 1;
        if (orient_sign_filtered(vx[j], vy[j], vx[k], vy[k], px, py) <= 0) return false;
    }
    return true;
}

// ------------------------------------------------------------------ cross-shard merge
// Slot s of the merge of `count` per-shard Step-1 results: the lexicographic
// (key, global index) best (lowest index on equal keys, A7); per slot, so
// slots can be merged in parallel.
GEOM_HD void merge_slot(const cudapre_extremes_t* parts, int count, int s, cudapre_extremes_t& r) {
    const bool is_max = (s & 1) != 0;
    long long idx = -1;
    double key = 0.0;
    cudapre_pt pt = {0.f, 0.f};
    for (int p = 0; p < count; ++p) {
        const cudapre_extremes_t& q = parts[p];
        if (q.idx[s] < 0) continue;
        bool better;
        if (idx < 0) better = true;
        else if (q.key[s] == key) better = q.idx[s] < idx;
        else better = is_max ? (q.key[s] > key) : (q.key[s] < key);
        if (better) {
            idx = q.idx[s];
            key = q.key[s];
            pt = q.pt[s];
        }
    }
    r.idx[s] = idx;
    r.key[s] = idx < 0 ? parts[0].key[s] : key;
    r.pt[s] = idx < 0 ? parts[0].pt[s] : pt;
}
// Everything but the slots (one thread): counts and flags summed / or-ed,
// angles and unused slots from part 0.
GEOM_HD void merge_header(const cudapre_extremes_t* parts, int count, cudapre_extremes_t& r) {
    r.nang = parts[0].nang;
    long long n = 0, ex = 0;
    int nf = 0;
    for (int p = 0; p < count; ++p) {
        n += parts[p].n;
        nf |= parts[p].nonfinite;
        ex += parts[p].exact_points;
    }
    r.n = n;
    r.nonfinite = nf;
    r.exact_points = ex;
    for (int k = 0; k < CUDAPRE_MAX_ANGLES; ++k) {
        r.c[k] = parts[0].c[k];
        r.s[k] = parts[0].s[k];
    }
}

// ------------------------------------------------------------------ phase A (one thread)
// Picks -> Andrew's monotone chain (A9, A10): lexicographic (x, y, id)
// order, distinct coordinates keep the lowest id (-0 == +0), pop while not a
// strict left turn.  Plus the exact bbox and the vertex mean.
// (a) the chain over the sorted distinct picks P[0..u) (H: scratch of
//     2*CUDAPRE_MAX_SLOTS+1 entries); (b) bbox / mean.  phase_a() runs the
//     whole phase on one thread; the device builder sorts and dedups with a
//     warp first (a rank sort under the same total order gives the same array).
GEOM_HD void phase_a_chain(const Pick* P, int u, Pick* H, Work& w) {
    w.n_distinct = u;
    int nv = 0;
    if (u == 1) {
        w.vid[0] = P[0].id;
        w.vx[0] = P[0].x;
        w.vy[0] = P[0].y;
        nv = 1;
    } else if (u > 1) {
        int k = 0;
        for (int j = 0; j < u; ++j) {
            while (k >= 2 && orient_sign_filtered(H[k - 2].x, H[k - 2].y, H[k - 1].x, H[k - 1].y, P[j].x, P[j].y) <= 0) --k;
            H[k++] = P[j];
        }
        const int lower = k;
        for (int j = u - 2; j >= 0; --j) {
            while (k > lower && orient_sign_filtered(H[k - 2].x, H[k - 2].y, H[k - 1].x, H[k - 1].y, P[j].x, P[j].y) <= 0)
                --k;
            H[k++] = P[j];
        }
        nv = k - 1;   // the last point repeats the first
        for (int j = 0; j < nv; ++j) {
            w.vid[j] = H[j].id;
            w.vx[j] = H[j].x;
            w.vy[j] = H[j].y;
        }
    }
    w.nv = nv;
    w.degenerate = nv < 3;
    w.have_box = 0;
    w.centre_ok = 0;
    w.sok = 0;
    w.cs = 0;
    w.r2 = -1.0f;
    w.cx = w.cy = 0.0f;
    w.rs_up = 1.0;
}
GEOM_HD void phase_a_tail(const cudapre_extremes_t& ext, Work& w) {
    const int nv = w.nv;
    // exact data bounding box: the angle-0 picks (c0 = 1, s0 = 0)
    const double xmin = ext.pt[0].x, xmax = ext.pt[1].x, ymin = ext.pt[2].y, ymax = ext.pt[3].y;
    w.Mx = dmax(fabs(xmin), fabs(xmax));
    w.My = dmax(fabs(ymin), fabs(ymax));
    double ox = 0, oy = 0, pxmin = 0, pxmax = 0, pymin = 0, pymax = 0;
    if (nv > 0) {
        pxmin = pxmax = w.vx[0];
        pymin = pymax = w.vy[0];
    }
    for (int j = 0; j < nv; ++j) {
        ox += w.vx[j];
        oy += w.vy[j];
        pxmin = dmin(pxmin, (double)w.vx[j]);
        pxmax = dmax(pxmax, (double)w.vx[j]);
        pymin = dmin(pymin, (double)w.vy[j]);
        pymax = dmax(pymax, (double)w.vy[j]);
    }
    if (nv > 0) {
        ox /= nv;
        oy /= nv;
    }
    w.ox = ox;
    w.oy = oy;
    w.hw = 0.5 * (pxmax - pxmin);
    w.hh = 0.5 * (pymax - pymin);
}
// Picks -> Andrew's monotone chain (A9, A10): lexicographic (x, y, id)
// order, distinct coordinates keep the lowest id (-0 == +0), pop while not a
// strict left turn.  Plus the exact bbox and the vertex mean.
GEOM_HD void phase_a(const cudapre_extremes_t& ext, Work& w) {
    Pick P[CUDAPRE_MAX_SLOTS];
    int m = 0;
    const int slots = 4 * ext.nang;
    for (int s = 0; s < slots; ++s)
        if (ext.idx[s] >= 0) P[m++] = Pick{ext.pt[s].x, ext.pt[s].y, (long long)ext.idx[s]};
    for (int i = 1; i < m; ++i) {   // insertion sort (total order: ids are distinct or equal picks)
        const Pick t = P[i];
        int j = i - 1;
        while (j >= 0 && pick_less(t, P[j])) {
            P[j + 1] = P[j];
            --j;
        }
        P[j + 1] = t;
    }
    int u = m ? 1 : 0;
    for (int j = 1; j < m; ++j)
        if (P[j].x != P[u - 1].x || P[j].y != P[u - 1].y) P[u++] = P[j];
    Pick H[2 * CUDAPRE_MAX_SLOTS + 1];
    phase_a_chain(P, u, H, w);
    phase_a_tail(ext, w);
}

// ------------------------------------------------------------------ phase B (per edge)
// g_j(p) = A px + B py + C' with C' = RD(C - E_j); E_j bounds |float eval -
// exact orient| over the bbox with a factor >= 2.6 of slack.
GEOM_HD void phase_b_edge(Work& w, int j) {
    const int nv = w.nv, k = j + 1 == nv ? 0 : j + 1;
    const double ax = w.vx[j], ay = w.vy[j], bx = w.vx[k], by = w.vy[k];
    const double A = ay - by, B = bx - ax, C = ax * by - ay * bx;
    const double S = fabs(A) * w.Mx + fabs(B) * w.My + fabs(C);
    const double Ed = S * 0x1p-20 + (w.Mx + w.My + 1.0) * 0x1p-140 + 0x1p-126;
    const float E = f_up(Ed);
    const float Cl = f_down(C - (double)E);
    const float Af = (float)A, Bf = (float)B;
    w.bad[j] = (!(S < 1e36) || !gfinite(E) || !gfinite(Cl) || !gfinite(Af) || !gfinite(Bf)) ? 1 : 0;
    w.A[j] = Af;
    w.B[j] = Bf;
    w.C[j] = Cl;
    w.E[j] = E;
}

// ------------------------------------------------------------------ phase C (box)
// Binary search step t of the largest vertex-mean-centred box whose 4 float
// corners are strictly inside every edge (exact predicate); convexity => the
// closed box is strictly inside.
GEOM_HD double box_t(int it, double lo, double hi) { return it == 0 ? 1.0 : 0.5 * (lo + hi); }
GEOM_HD void box_corners(const Work& w, double t, float c[4]) {
    c[0] = f_up(w.ox - t * w.hw);
    c[1] = f_down(w.ox + t * w.hw);
    c[2] = f_up(w.oy - t * w.hh);
    c[3] = f_down(w.oy + t * w.hh);
}
GEOM_HD bool box_searchable(const Work& w) {
    return gfinite(w.ox) && gfinite(w.oy) && gfinite(w.hw) && gfinite(w.hh);
}
// corner q (0..3: (x0,y0) (x1,y0) (x1,y1) (x0,y1)) strictly inside edge j
GEOM_HD bool box_corner_edge_ok(const Work& w, const float c[4], int q, int j) {
    const float px = (q == 0 || q == 3) ? c[0] : c[1];
    const float py = (q <= 1) ? c[2] : c[3];
    const int k = j + 1 == w.nv ? 0 : j + 1;
    return orient_sign_filtered(w.vx[j], w.vy[j], w.vx[k], w.vy[k], px, py) > 0;
}

// ------------------------------------------------------------------ phase D (disk)
// Centre (box centre, else vertex mean) and, per edge, a rigorous lower bound
// of the distance from the centre to the edge line.
GEOM_HD void disk_centre(Work& w) {
    w.cx = w.have_box ? 0.5f * (w.box[0] + w.box[1]) : (float)w.ox;
    w.cy = w.have_box ? 0.5f * (w.box[2] + w.box[3]) : (float)w.oy;
    w.centre_ok = (gfinite(w.cx) && gfinite(w.cy) && strictly_inside_ring(w.vx, w.vy, w.nv, w.cx, w.cy)) ? 1 : 0;
}
GEOM_HD void phase_d_edge(Work& w, int j) {
    const int k = j + 1 == w.nv ? 0 : j + 1;
    const double ax = w.vx[j], ay = w.vy[j], bx = w.vx[k], by = w.vy[k];
    const double ex = bx - ax, ey = by - ay, px = w.cx - ax, py = w.cy - ay;
    const double t1 = ex * py, t2 = ey * px;
    const double num = t1 - t2;
    // each of ex, ey, px, py, t1, t2, num carries <= 1 rounding (2^-53 rel.)
    const double err = (fabs(t1) + fabs(t2)) * 0x1p-49;
    const double len = sqrt(ex * ex + ey * ey) * (1.0 + 0x1p-48);
    w.dok_e[j] = (num - err > 0.0) && (len > 0.0) && gfinite(len);
    w.rmin_e[j] = w.dok_e[j] ? (num - err) / len * (1.0 - 0x1p-50) : INFINITY;
}
// after the per-edge pass: r2 = RD32((1 - 2^-16) rmin^2), disabled outside [2^-100, 2^100]
// The sector phase centres on (cx, cy) when the centre passed its check, and
// on (0, 0) otherwise (then the sector tables check (0, 0) themselves).
GEOM_HD void disk_finish(Work& w) {
    w.r2 = -1.0f;
    if (w.centre_ok) {
        bool ok = true;
        double rmin = INFINITY;
        for (int j = 0; j < w.nv && ok; ++j) {
            ok = w.dok_e[j] != 0;
            if (ok) rmin = dmin(rmin, w.rmin_e[j]);
        }
        const double r2 = rmin * rmin * (1.0 - 0x1p-16);
        if (ok && r2 >= 0x1p-100 && r2 <= 0x1p100) w.r2 = f_down(r2);
    } else {
        w.cx = 0.0f;
        w.cy = 0.0f;
    }
}

// ------------------------------------------------------------------ phase E (sector prep)
GEOM_HD bool sector_centre_ok(const Work& w) {
    return w.r2 > 0.0f ||
           (gfinite(w.cx) && gfinite(w.cy) && strictly_inside_ring(w.vx, w.vy, w.nv, w.cx, w.cy));
}
GEOM_HD void phase_e_edge(Work& w, int j) {
    const int k = j + 1 == w.nv ? 0 : j + 1;
    const double ax = w.vx[j], ay = w.vy[j], bx = w.vx[k], by = w.vy[k];
    const double ex = bx - ax, ey = by - ay, px = w.cx - ax, py = w.cy - ay;
    const double t1 = ex * py, t2 = ey * px;
    const double num = t1 - t2, err = (fabs(t1) + fabs(t2)) * 0x1p-49;
    const double len = sqrt(ex * ex + ey * ey);
    w.sok_e[j] = (num - err > 0.0) && (len > 0.0) && gfinite(len);
    w.dj[j] = (num - err) / (len * (1.0 + 0x1p-48));
    w.rsu[j] = ((num + err) * (1.0 + 0x1p-48)) / (num - err);
    w.nx[j] = ey / len;   // outward unit normal of a CCW ring
    w.ny[j] = -ex / len;
    w.pn[j] = pa_of(w.nx[j], w.ny[j]);
    w.pv[j] = pa_of((double)w.vx[j] - w.cx, (double)w.vy[j] - w.cy);
}
// after the per-edge pass: ok, rs_up, the start edge cs (first max of pv) and
// the unwrapped end pseudo-angles U[k] of edge (cs + k) mod nv
GEOM_HD void sector_prep_finish(Work& w) {
    bool ok = sector_centre_ok(w);
    double rs_up = 1.0;
    for (int j = 0; j < w.nv && ok; ++j) {
        ok = w.sok_e[j] != 0;
        if (ok) rs_up = dmax(rs_up, w.rsu[j]);
    }
    w.sok = ok;
    w.rs_up = rs_up;
    int cs = 0;
    for (int k = 0; k < w.nv; ++k)
        if (w.pv[k] > w.pv[cs]) cs = k;
    w.cs = cs;
    for (int k = 0; k < w.nv; ++k) {
        int e = cs + k + 1;
        if (e >= w.nv) e -= w.nv;
        w.U[k] = w.pv[e] + 4.0;
    }
}

// ------------------------------------------------------------------ phase F (per sample ray)
// Exit edge of the ray of pseudo-angle pw: the first edge, counted from cs,
// whose closed pseudo-angle range holds pw (binary search over U; the same
// edge a forward two-pointer walk over increasing pw finds), and the exit
// distance: min over that edge and its neighbours of d_j / cos(th - phi_j),
// by cross-multiplication, times |u|.
GEOM_HD void phase_f_sample(const Work& w, int i, double& rs, int& exe) {
    const double pw = sample_pa(i);
    double ux, uy;
    pa_dir(pw, ux, uy);
    const double ul = sqrt(ux * ux + uy * uy);
    const double q = pw < w.pv[w.cs] ? pw + 4.0 : pw;
    int lo = 0, hi = w.nv - 1;   // first k with q <= U[k] (U[nv-1] = pv[cs] + 4 > q always)
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (q <= w.U[mid]) hi = mid;
        else lo = mid + 1;
    }
    int cur = w.cs + lo;
    if (cur >= w.nv) cur -= w.nv;
    double bn = INFINITY, bd = 1.0;
    const int nb[3] = {cur == 0 ? w.nv - 1 : cur - 1, cur, cur + 1 == w.nv ? 0 : cur + 1};
    for (int dd = 0; dd < 3; ++dd) {
        const int j = nb[dd];
        const double c = w.nx[j] * ux + w.ny[j] * uy;
        if (c > 0.0 && w.dj[j] * bd < bn * c) {
            bn = w.dj[j];
            bd = c;
        }
    }
    rs = bn / bd * ul;
    exe = cur;
}

// ------------------------------------------------------------------ phase G (buckets)
// Bucket b spans pseudo-angles [(b-0.5-g), (b+0.5+g)]/256.  Inner radius:
// min(ray distances at both ends, d_j of every edge normal inside); outer:
// max(ends, with the upper-bound factor rs_up) and the radius of every vertex
// inside (min / max are exact: any evaluation order gives the same bits).
GEOM_HD bool pa_in_bucket(double pa, int b) {
    const double lo = (b - 0.5 - kGuard) / 256.0, hi = (b + 0.5 + kGuard) / 256.0;
    for (int w2 = -1; w2 <= 1; ++w2) {
        const double q = pa + 4.0 * w2;
        if (q >= lo && q <= hi) return true;
    }
    return false;
}
// Bucket b's radii before the vertex / normal corrections: the ray distances
// at both (guarded) ends; the outer one raised by the rs_up factor.
GEOM_HD void phase_g_init(const Work& w, int b, const double* rs, double& rb, double& ro) {
    rb = dmin(rs[2 * b], rs[2 * (b + 1) + 1]);
    ro = dmax(rs[2 * b], rs[2 * (b + 1) + 1]) * w.rs_up;
}
// The buckets whose guarded range holds pseudo-angle pa (<= 4 of them, with
// wrap-around): visits each such bucket once.
template <typename F>
GEOM_HD void for_buckets_of(double pa, F&& f) {
    const double c = pa * 256.0;
    for (int b = (int)floor(c - 0.5 - kGuard) - 1; b <= (int)ceil(c + 0.5 + kGuard) + 1; ++b)
        for (int wv = -1; wv <= 1; ++wv) {
            const int bb = b + 1024 * wv;
            if (bb >= 0 && bb <= CUDAPRE_SECTORS && pa_in_bucket(pa, bb)) f(bb);
        }
}
// Vertex j inside a bucket raises its outer radius to the vertex's radius;
// the normal of edge j inside a bucket lowers its inner radius to d_j.
GEOM_HD double vertex_radius(const Work& w, int j) {
    const double vx = (double)w.vx[j] - w.cx, vy = (double)w.vy[j] - w.cy;
    return sqrt(vx * vx + vy * vy) * (1.0 + 0x1p-40);
}
// Final conversion of bucket b: squared radii with directed rounding and a
// 2^-16 margin; candidate edges: exit edge of the lower sample to that of the
// upper one (<= 2, else all edges).
GEOM_HD void phase_g_finish(const Work& w, int b, double rb, double ro, const int* exe, float& sr2, float& sro2,
                            unsigned short& sedge) {
    sro2 = INFINITY;
    {
        const double r = ro * (1.0 + 0x1p-30);
        const double r2 = r * r * (1.0 + 0x1p-16);
        if (r2 >= 0x1p-100 && r2 <= 0x1p100) sro2 = f_up(r2);
    }
    sr2 = -1.0f;
    {
        const double r = rb * (1.0 - 0x1p-30);
        const double r2 = r * r * (1.0 - 0x1p-16);
        if (r2 >= 0x1p-100 && r2 <= 0x1p100) sr2 = f_down(r2);
    }
    const int lo = exe[2 * b], hi = exe[2 * (b + 1) + 1];
    const int cnt = (hi - lo + w.nv) % w.nv + 1;
    sedge = cnt <= 2 ? (unsigned short)(lo | (hi << 8)) : (unsigned short)0xffff;
}

// ------------------------------------------------------------------ outputs
// Defaults of the outputs (degenerate / no tables): the scalars (one
// thread) and the per-index entries j = 0..CUDAPRE_MAX_SLOTS (any thread).
GEOM_HD void defaults(const Work& w, cudapre_polygon_t* poly, K2Geom* g) {
    if (poly) {
        poly->nv = w.nv;
        poly->degenerate = w.degenerate;
        poly->n_distinct = w.n_distinct;
        poly->exact_only = 0;
        poly->box[0] = 1.0f;
        poly->box[1] = 0.0f;
        poly->box[2] = 1.0f;
        poly->box[3] = 0.0f;
        poly->circle[0] = poly->circle[1] = poly->circle[3] = 0.0f;
        poly->circle[2] = -1.0f;
        poly->err_max = 0.0f;
        poly->pad = 0;
    }
    if (g) {
        g->nv = w.nv;
        g->mode = w.degenerate ? 1 : 0;
        g->fast = 2;
        g->pad = 0;
        g->bx0 = 1.0f;
        g->bx1 = 0.0f;
        g->by0 = 1.0f;
        g->by1 = 0.0f;
        g->ox = g->oy = 0.0f;
        g->r2 = -1.0f;
        g->e2max = 0.0f;
    }
}
GEOM_HD void defaults_item(const Work& w, cudapre_polygon_t* poly, K2Geom* g, int j) {
    if (poly && j < CUDAPRE_MAX_SLOTS) {
        poly->vidx[j] = j < w.nv ? (int64_t)w.vid[j] : 0;
        poly->v[j] = j < w.nv ? cudapre_pt{w.vx[j], w.vy[j]} : cudapre_pt{0.f, 0.f};
        poly->A[j] = poly->B[j] = poly->C[j] = poly->E[j] = 0.0f;
    }
    if (g) {
        if (j < CUDAPRE_MAX_SLOTS) {
            g->A[j] = 0.0f;
            g->B[j] = 0.0f;
            g->C[j] = INFINITY;   // padding edges: g = +inf, never the minimum
        }
        const int m = w.nv ? w.nv : 1;
        g->vx[j] = w.nv ? w.vx[j % m] : 0.0f;
        g->vy[j] = w.nv ? w.vy[j % m] : 0.0f;
    }
}
// Per-edge outputs once the phases ran (any thread, j < nv).
GEOM_HD void finish_item(const Work& w, cudapre_polygon_t* poly, K2Geom* g, int j) {
    if (poly) {
        poly->A[j] = w.A[j];
        poly->B[j] = w.B[j];
        poly->C[j] = w.C[j];
        poly->E[j] = w.E[j];
    }
    if (g) {
        g->A[j] = w.A[j];
        g->B[j] = w.B[j];
        g->C[j] = w.C[j];
    }
}
// Scalar outputs once the phases ran (one thread; plus finish_item per edge).
GEOM_HD void finish(const Work& w, cudapre_polygon_t* poly, K2Geom* g) {
    bool exact_only = false;
    float emax = 0.0f;
    for (int j = 0; j < w.nv; ++j) {
        exact_only = exact_only || w.bad[j];
        emax = smax(emax, w.E[j]);
    }
    if (!(emax < 1e37f)) exact_only = true;
    if (poly) {
        poly->exact_only = exact_only;
        poly->err_max = emax;
        if (w.have_box)
            for (int q = 0; q < 4; ++q) poly->box[q] = w.box[q];
        poly->circle[0] = w.centre_ok ? w.cx : 0.0f;
        poly->circle[1] = w.centre_ok ? w.cy : 0.0f;
        poly->circle[2] = w.r2;
    }
    if (g) {
        g->ox = w.centre_ok ? w.cx : 0.0f;
        g->oy = w.centre_ok ? w.cy : 0.0f;
        g->r2 = w.r2;
        g->mode = exact_only ? 2 : 0;
        g->e2max = 2.0f * emax;
        if (w.have_box) {
            g->bx0 = w.box[0];
            g->bx1 = w.box[1];
            g->by0 = w.box[2];
            g->by1 = w.box[3];
        }
        // the TMA kernel runs one fast test in pass A: the one covering more area
        const double disk = g->r2 > 0.0f ? 3.141592653589793 * (double)g->r2 : 0.0;
        const double box = (g->bx0 <= g->bx1 && g->by0 <= g->by1)
                               ? ((double)g->bx1 - g->bx0) * ((double)g->by1 - g->by0)
                               : 0.0;
        g->fast = exact_only ? 2 : (box > disk ? 1 : 0);
    }
}

}  // namespace geom
}  // namespace cudapre
