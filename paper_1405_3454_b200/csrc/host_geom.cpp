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

// float nearest-below / nearest-above of a double (directed conversion)
float f_down(double d) {
    float f = (float)d;
    if ((double)f > d) f = std::nextafter(f, -INFINITY);
    return f;
}
float f_up(double d) {
    float f = (float)d;
    if ((double)f < d) f = std::nextafter(f, INFINITY);
    return f;
}

bool strictly_inside_ring(const cudapre_pt* v, int nv, float px, float py) {
    for (int j = 0; j < nv; ++j) {
        const cudapre_pt& a = v[j];
        const cudapre_pt& b = v[(j + 1) % nv];
        if (orient_exact(a.x, a.y, b.x, b.y, px, py) <= 0) return false;
    }
    return true;
}

// direction (unnormalised) of pseudo-angle pa (wrapped into [0, 4)):
// pa in [0,2]: t = pa-1, (1-|t|, t);  pa in [2,4]: t = 3-pa, (-(1-|t|), t)
void pa_dir(double pa, double& ux, double& uy) {   // pa in [-4, 8)
    if (pa < 0.0) pa += 4.0;
    if (pa >= 4.0) pa -= 4.0;
    if (pa <= 2.0) {
        const double t = pa - 1.0;
        ux = 1.0 - std::fabs(t);
        uy = t;
    } else {
        const double t = 3.0 - pa;
        ux = -(1.0 - std::fabs(t));
        uy = t;
    }
}
double pa_of(double ux, double uy) {
    const double t = uy / (std::fabs(ux) + std::fabs(uy));
    return ux >= 0.0 ? t + 1.0 : 3.0 - t;
}

// The sector sample rays are fixed: pseudo-angles (k - 0.5 -+ 1/64)/256,
// k = 0..1025 (wrapped into [0, 4)), with their unnormalised directions and
// lengths; built once per process.
struct SectorSamples {
    static constexpr int kS = 2 * (CUDAPRE_SECTORS + 2);
    double pa[kS], ux[kS], uy[kS], ul[kS];
    SectorSamples() {
        const double g = 1.0 / 64.0;
        for (int i = 0; i < kS; ++i) {
            double pw = ((double)(i >> 1) - 0.5 + ((i & 1) ? g : -g)) / 256.0;
            if (pw < 0.0) pw += 4.0;
            if (pw >= 4.0) pw -= 4.0;
            pa[i] = pw;
            pa_dir(pw, ux[i], uy[i]);
            ul[i] = std::sqrt(ux[i] * ux[i] + uy[i] * uy[i]);
        }
    }
};
const SectorSamples& sector_samples() {
    static const SectorSamples s;
    return s;
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

void merge_extremes(const cudapre_extremes_t* parts, int count, cudapre_extremes_t* out) {
    cudapre_extremes_t r = parts[0];
    r.n = 0;
    r.nonfinite = 0;
    r.exact_points = 0;
    const int slots = 4 * r.nang;
    for (int s = 0; s < slots; ++s) r.idx[s] = -1;
    for (int p = 0; p < count; ++p) {
        const cudapre_extremes_t& q = parts[p];
        r.n += q.n;
        r.nonfinite |= q.nonfinite;
        r.exact_points += q.exact_points;
        for (int s = 0; s < slots; ++s) {
            if (q.idx[s] < 0) continue;
            const bool is_max = (s & 1) != 0;
            bool better;
            if (r.idx[s] < 0) {
                better = true;
            } else if (q.key[s] == r.key[s]) {
                better = q.idx[s] < r.idx[s];   // lowest global index on equal keys (A7)
            } else {
                better = is_max ? (q.key[s] > r.key[s]) : (q.key[s] < r.key[s]);
            }
            if (better) {
                r.idx[s] = q.idx[s];
                r.key[s] = q.key[s];
                r.pt[s] = q.pt[s];
            }
        }
    }
    *out = r;
}

void build_polygon(const cudapre_extremes_t& ext, cudapre_polygon_t* poly, K2Params* kp) {
    std::memset(poly, 0, sizeof(*poly));
    const int slots = 4 * ext.nang;
    // ---- Step 2: distinct picks -> monotone chain (A9, A10)
    std::vector<CP> P;
    std::vector<cudapre_pt> byid;
    for (int s = 0; s < slots; ++s)
        if (ext.idx[s] >= 0) P.push_back(CP{ext.pt[s].x, ext.pt[s].y, ext.idx[s]});
    {
        std::vector<CP> Q = P;
        std::sort(Q.begin(), Q.end(), lex_less);
        int d = Q.empty() ? 0 : 1;
        for (size_t j = 1; j < Q.size(); ++j)
            if (Q[j].x != Q[j - 1].x || Q[j].y != Q[j - 1].y) ++d;
        poly->n_distinct = d;
    }
    int64_t ring[CUDAPRE_MAX_SLOTS];
    std::vector<CP> Pc = P;
    const int nv = (int)chain(Pc, ring);
    poly->nv = nv;
    for (int j = 0; j < nv; ++j) {
        poly->vidx[j] = ring[j];
        for (const CP& c : P)
            if (c.id == ring[j]) { poly->v[j] = cudapre_pt{c.x, c.y}; break; }
    }
    poly->degenerate = nv < 3;
    poly->box[0] = 1.0f;
    poly->box[1] = 0.0f;   // empty box
    poly->box[2] = 1.0f;
    poly->box[3] = 0.0f;
    poly->circle[2] = -1.0f;
    for (int b = 0; b <= CUDAPRE_SECTORS; ++b) {
        poly->sector_r2[b] = -1.0f;
        poly->sector_out_r2[b] = INFINITY;
    }
    if (kp) {
        kp->nv = nv;
        kp->mode = poly->degenerate ? 1 : 0;
        kp->bx0 = 1.0f; kp->bx1 = 0.0f; kp->by0 = 1.0f; kp->by1 = 0.0f;
        kp->e2max = 0.0f;
        kp->ox = kp->oy = 0.0f;
        kp->r2 = -1.0f;
        for (int b = 0; b <= CUDAPRE_SECTORS; ++b) {
            kp->sr2[b] = -1.0f;
            kp->sro2[b] = INFINITY;
            kp->sedge[b] = 0xffff;
        }
        kp->fast = 0;
        for (int j = 0; j <= nv && j <= CUDAPRE_MAX_SLOTS; ++j) {
            kp->vx[j] = poly->v[j % (nv ? nv : 1)].x;
            kp->vy[j] = poly->v[j % (nv ? nv : 1)].y;
        }
    }
    if (poly->degenerate) return;

    // ---- exact data bounding box: the angle-0 picks (slots 0..3 = min x, max x,
    //      min y, max y of the whole point set; c0 = 1, s0 = 0).
    const double xmin = ext.pt[0].x, xmax = ext.pt[1].x, ymin = ext.pt[2].y, ymax = ext.pt[3].y;
    const double Mx = std::max(std::fabs(xmin), std::fabs(xmax));
    const double My = std::max(std::fabs(ymin), std::fabs(ymax));

    // ---- per-edge float line g_j(p) = A px + B py + C'.
    // orient(a, b, p) = A p.x + B p.y + C with A = ay-by, B = bx-ax, C = ax*by-ay*bx.
    // E_j bounds |float evaluation - exact orient| over the bbox with a factor
    // >= 2.6 of slack: coefficient rounding <= 2^-23 S, the two fma roundings
    // <= 2^-23 S', subnormal / absolute terms <= 2^-140 (Mx+My+1) + 2^-126.
    bool exact_only = false;
    float emax = 0.0f;
    for (int j = 0; j < nv; ++j) {
        const double ax = poly->v[j].x, ay = poly->v[j].y;
        const double bx = poly->v[(j + 1) % nv].x, by = poly->v[(j + 1) % nv].y;
        const double A = ay - by, B = bx - ax, C = ax * by - ay * bx;
        const double S = std::fabs(A) * Mx + std::fabs(B) * My + std::fabs(C);
        const double Ed = S * 0x1p-20 + (Mx + My + 1.0) * 0x1p-140 + 0x1p-126;
        const float E = f_up(Ed);
        const float Cl = f_down(C - (double)E);
        const float Af = (float)A, Bf = (float)B;
        if (!(S < 1e36) || !std::isfinite(E) || !std::isfinite(Cl) || !std::isfinite(Af) ||
            !std::isfinite(Bf))
            exact_only = true;
        emax = std::max(emax, E);
        poly->A[j] = Af;
        poly->B[j] = Bf;
        poly->C[j] = Cl;
        poly->E[j] = E;
        if (kp) {
            kp->A[j] = Af;
            kp->B[j] = Bf;
            kp->C[j] = Cl;
        }
    }
    if (kp)   // padding edges for the kernel's fixed-length loop: g = +inf, never the minimum
        for (int j = nv; j < CUDAPRE_MAX_SLOTS; ++j) {
            kp->A[j] = 0.0f;
            kp->B[j] = 0.0f;
            kp->C[j] = INFINITY;
        }
    if (!(emax < 1e37f)) exact_only = true;
    poly->err_max = emax;
    poly->exact_only = exact_only;

    // ---- inner box: centred at the vertex mean, the largest scale (binary
    //      search) whose 4 float corners are strictly inside every edge,
    //      checked with the exact predicate.  Convexity => the closed box is
    //      strictly inside.
    double ox = 0, oy = 0, pxmin = poly->v[0].x, pxmax = pxmin, pymin = poly->v[0].y, pymax = pymin;
    for (int j = 0; j < nv; ++j) {
        ox += poly->v[j].x;
        oy += poly->v[j].y;
        pxmin = std::min(pxmin, (double)poly->v[j].x);
        pxmax = std::max(pxmax, (double)poly->v[j].x);
        pymin = std::min(pymin, (double)poly->v[j].y);
        pymax = std::max(pymax, (double)poly->v[j].y);
    }
    ox /= nv;
    oy /= nv;
    const double hw = 0.5 * (pxmax - pxmin), hh = 0.5 * (pymax - pymin);
    double lo = 0.0, hi = 1.0;
    bool have = false;
    float best[4] = {1.0f, 0.0f, 1.0f, 0.0f};
    if (std::isfinite(ox) && std::isfinite(oy) && std::isfinite(hw) && std::isfinite(hh)) {
        for (int it = 0; it < 16; ++it) {
            const double t = (it == 0) ? 1.0 : 0.5 * (lo + hi);
            const float x0 = f_up(ox - t * hw), x1 = f_down(ox + t * hw);
            const float y0 = f_up(oy - t * hh), y1 = f_down(oy + t * hh);
            bool ok = x0 <= x1 && y0 <= y1 && strictly_inside_ring(poly->v, nv, x0, y0) &&
                      strictly_inside_ring(poly->v, nv, x1, y0) &&
                      strictly_inside_ring(poly->v, nv, x1, y1) &&
                      strictly_inside_ring(poly->v, nv, x0, y1);
            if (ok) {
                have = true;
                best[0] = x0; best[1] = x1; best[2] = y0; best[3] = y1;
                lo = t;
                if (it == 0) break;
            } else {
                hi = t;
            }
        }
    }
    if (have) std::memcpy(poly->box, best, sizeof(best));

    // ---- inner disk: centre O (box centre, else vertex mean,
    //      rounded to float and checked strictly inside exactly), radius^2 =
    //      (1 - 2^-16) * (a rigorous LOWER bound of min_j dist(O, edge line j))^2.
    //      Kernel test RN32(RN32(dx*dx) + RN32(dy*dy)) < r2 with dx = RN32(x - ox):
    //      the float value is >= true d^2 (1 - 4u), so acceptance implies true
    //      d^2 < R^2 (1 - 2^-16) / (1 - 4u) < R^2.  Disabled outside [2^-100, 2^100].
    poly->circle[0] = 0.0f;
    poly->circle[1] = 0.0f;
    poly->circle[2] = -1.0f;
    {
        const float cx = have ? 0.5f * (best[0] + best[1]) : (float)ox;
        const float cy = have ? 0.5f * (best[2] + best[3]) : (float)oy;
        if (std::isfinite(cx) && std::isfinite(cy) && strictly_inside_ring(poly->v, nv, cx, cy)) {
            double rmin = INFINITY;
            bool ok = true;
            for (int j = 0; j < nv && ok; ++j) {
                const double ax = poly->v[j].x, ay = poly->v[j].y;
                const double bx = poly->v[(j + 1) % nv].x, by = poly->v[(j + 1) % nv].y;
                const double ex = bx - ax, ey = by - ay, px = cx - ax, py = cy - ay;
                const double t1 = ex * py, t2 = ey * px;
                const double num = t1 - t2;
                // each of ex, ey, px, py, t1, t2, num carries <= 1 rounding (2^-53 rel.)
                const double err = (std::fabs(t1) + std::fabs(t2)) * 0x1p-49;
                const double len = std::sqrt(ex * ex + ey * ey) * (1.0 + 0x1p-48);
                if (!(num - err > 0.0) || !(len > 0.0) || !std::isfinite(len)) {
                    ok = false;
                    break;
                }
                rmin = std::min(rmin, (num - err) / len * (1.0 - 0x1p-50));
            }
            const double r2 = rmin * rmin * (1.0 - 0x1p-16);
            poly->circle[0] = cx;   // centre kept for the sector test even if the disk is off
            poly->circle[1] = cy;
            if (ok && r2 >= 0x1p-100 && r2 <= 0x1p100) poly->circle[2] = f_down(r2);
        }
    }
    // ---- sector table: for bucket b = round(256 pa) the
    //      radius^2 below which every point whose pseudo-angle lies in
    //      [(b - 0.5 - g)/256, (b + 0.5 + g)/256] (guard g = 1/64 bucket) is
    //      strictly inside.  Along one edge j the exit distance of the ray at
    //      angle th is d_j / cos(th - phi_j) (d_j: rigorous lower bound of the
    //      distance from the centre to the edge line, phi_j: outward normal),
    //      convex in th with its minimum d_j at phi_j, so over a bucket
    //      r_min = min(r(lower end), r(upper end), d_j for normals inside).
    for (int b = 0; b <= CUDAPRE_SECTORS; ++b) {
        poly->sector_r2[b] = -1.0f;
        poly->sector_out_r2[b] = INFINITY;
    }
    {
        const float cx = poly->circle[0], cy = poly->circle[1];
        bool ok = poly->circle[2] > 0.0f || (std::isfinite(cx) && std::isfinite(cy) &&
                                              strictly_inside_ring(poly->v, nv, cx, cy));
        double nx[CUDAPRE_MAX_SLOTS], ny[CUDAPRE_MAX_SLOTS], dj[CUDAPRE_MAX_SLOTS], pn[CUDAPRE_MAX_SLOTS];
        double rs_up = 1.0;   // max over edges of (upper bound of dj) / (lower bound of dj)
        for (int j = 0; j < nv && ok; ++j) {
            const double ax = poly->v[j].x, ay = poly->v[j].y;
            const double bx = poly->v[(j + 1) % nv].x, by = poly->v[(j + 1) % nv].y;
            const double ex = bx - ax, ey = by - ay, px = cx - ax, py = cy - ay;
            const double t1 = ex * py, t2 = ey * px;
            const double num = t1 - t2, err = (std::fabs(t1) + std::fabs(t2)) * 0x1p-49;
            const double len = std::sqrt(ex * ex + ey * ey);
            if (!(num - err > 0.0) || !(len > 0.0) || !std::isfinite(len)) {
                ok = false;
                break;
            }
            dj[j] = (num - err) / (len * (1.0 + 0x1p-48));
            rs_up = std::max(rs_up, ((num + err) * (1.0 + 0x1p-48)) / (num - err));
            nx[j] = ey / len;   // outward unit normal of a CCW ring
            ny[j] = -ex / len;
            pn[j] = pa_of(nx[j], ny[j]);
        }
        // Vertex pseudo-angles around the centre: the ray of pseudo-angle pa
        // exits through edge j iff pa lies in [pv_j, pv_j+1] (cyclically).
        // Rays are visited in increasing pa, so the exit edge only moves forward.
        double pv[CUDAPRE_MAX_SLOTS + 1];
        if (ok)
            for (int j = 0; j < nv; ++j) pv[j] = pa_of((double)poly->v[j].x - cx, (double)poly->v[j].y - cy);
        if (ok) {
            const double g = 1.0 / 64.0;
            double rb[CUDAPRE_SECTORS + 1];
            // Exit distances of the rays at pseudo-angles (k - 0.5 -+ g)/256,
            // k = 0..1025, visited in increasing order so the exit edge only
            // moves forward; the exit edge and both neighbours are evaluated
            // (robust at vertex directions).  Bucket b spans
            // [(b-0.5-g), (b+0.5+g)]/256 -> min(rm[b], rp[b+1]).
            const SectorSamples& SS = sector_samples();
            constexpr int kS = SectorSamples::kS;
            double rs[kS];
            int exe[kS];   // exit edge of each sample ray
            int cur = 0;
            for (int k = 0; k < nv; ++k)   // start at the edge whose range holds pa = 4 - eps
                if (pv[k] > pv[cur]) cur = k;
            for (int i = 0; i < kS; ++i) {
                const double pw = SS.pa[i];
                for (int steps = 0; steps < nv; ++steps) {   // advance to the edge holding pw
                    const int cn = cur + 1 == nv ? 0 : cur + 1;
                    double e0 = pv[cur], e1 = pv[cn], q = pw;
                    if (e1 < e0) e1 += 4.0;
                    if (q < e0) q += 4.0;
                    if (q <= e1) break;
                    cur = cn;
                }
                // min over the exit edge and its neighbours of dj / c (c > 0), by
                // cross-multiplication; one division at the end
                double bn = INFINITY, bd = 1.0;
                const int nb[3] = {cur == 0 ? nv - 1 : cur - 1, cur, cur + 1 == nv ? 0 : cur + 1};
                for (int dd = 0; dd < 3; ++dd) {
                    const int j = nb[dd];
                    const double c = nx[j] * SS.ux[i] + ny[j] * SS.uy[i];
                    if (c > 0.0 && dj[j] * bd < bn * c) {
                        bn = dj[j];
                        bd = c;
                    }
                }
                rs[i] = bn / bd * SS.ul[i];
                exe[i] = cur;
            }
            // Candidate edges of bucket b: every ray with pseudo-angle strictly
            // inside the guarded range exits through an edge from exe[2b] to
            // exe[2b+3] (CCW; the ring is convex around the centre).  A rounding
            // slip in the walk can only pick the other edge of a vertex lying
            // within ~1e-15 of a sample ray, which widens the range; points of
            // the bucket lie >= 2^-15 in pa from the samples (guard 2^-14, bucket
            // error < 2^-20), so they never need an edge outside it.
            if (kp)
                for (int b = 0; b <= CUDAPRE_SECTORS; ++b) {
                    const int lo = exe[2 * b], hi = exe[2 * (b + 1) + 1];
                    const int cnt = (hi - lo + nv) % nv + 1;
                    kp->sedge[b] = cnt <= 2 ? (unsigned short)(lo | (hi << 8)) : (unsigned short)0xffff;
                }
            for (int b = 0; b <= CUDAPRE_SECTORS; ++b) rb[b] = std::min(rs[2 * b], rs[2 * (b + 1) + 1]);
            // outer bound: r(th) is maximal at the interval ends or at a vertex
            // inside it; dj is a LOWER bound of the line distance, so the ray
            // distances are recomputed from an upper bound of dj
            double ro[CUDAPRE_SECTORS + 1];
            for (int b = 0; b <= CUDAPRE_SECTORS; ++b)
                ro[b] = std::max(rs[2 * b], rs[2 * (b + 1) + 1]) * rs_up;
            for (int j = 0; j < nv; ++j) {   // vertices inside a bucket
                const double vx = (double)poly->v[j].x - cx, vy = (double)poly->v[j].y - cy;
                const double vr = std::sqrt(vx * vx + vy * vy) * (1.0 + 0x1p-40);
                const double c = pv[j] * 256.0;
                for (int b = (int)std::floor(c - 0.5 - g) - 1; b <= (int)std::ceil(c + 0.5 + g) + 1; ++b)
                    for (int w = -1; w <= 1; ++w) {
                        const int bb = b + w * 1024;
                        if (bb < 0 || bb > CUDAPRE_SECTORS) continue;
                        const double lo = (bb - 0.5 - g) / 256.0, hi = (bb + 0.5 + g) / 256.0;
                        for (int w2 = -1; w2 <= 1; ++w2) {
                            const double q = pv[j] + 4.0 * w2;
                            if (q >= lo && q <= hi) ro[bb] = std::max(ro[bb], vr);
                        }
                    }
            }
            for (int b = 0; b <= CUDAPRE_SECTORS; ++b) {
                const double r = ro[b] * (1.0 + 0x1p-30);
                const double r2 = r * r * (1.0 + 0x1p-16);
                if (r2 >= 0x1p-100 && r2 <= 0x1p100) poly->sector_out_r2[b] = f_up(r2);
            }
            // edge normals: the minimum d_j of edge j is attained at its normal
            for (int j = 0; j < nv; ++j) {
                const double c = pn[j] * 256.0;   // bucket coordinate of the normal
                for (int b = (int)std::floor(c - 0.5 - g) - 1; b <= (int)std::ceil(c + 0.5 + g) + 1; ++b) {
                    for (int w = -1; w <= 1; ++w) {   // wrap: buckets 0 and 1024 overlap at pa = 0 / 4
                        const int bb = b + w * 1024;
                        if (bb < 0 || bb > CUDAPRE_SECTORS) continue;
                        const double lo = (bb - 0.5 - g) / 256.0, hi = (bb + 0.5 + g) / 256.0;
                        for (int w2 = -1; w2 <= 1; ++w2) {
                            const double q = pn[j] + 4.0 * w2;
                            if (q >= lo && q <= hi) rb[bb] = std::min(rb[bb], dj[j]);
                        }
                    }
                }
            }
            for (int b = 0; b <= CUDAPRE_SECTORS; ++b) {
                const double r = rb[b] * (1.0 - 0x1p-30);
                const double r2 = r * r * (1.0 - 0x1p-16);
                if (r2 >= 0x1p-100 && r2 <= 0x1p100) poly->sector_r2[b] = f_down(r2);
            }
        }
    }
    if (kp) {
        for (int b = 0; b <= CUDAPRE_SECTORS; ++b) {
            kp->sr2[b] = poly->sector_r2[b];
            kp->sro2[b] = poly->sector_out_r2[b];
        }
        kp->ox = poly->circle[0];
        kp->oy = poly->circle[1];
        kp->r2 = poly->circle[2];
        kp->mode = exact_only ? 2 : 0;
        kp->e2max = 2.0f * emax;
        kp->bx0 = poly->box[0];
        kp->bx1 = poly->box[1];
        kp->by0 = poly->box[2];
        kp->by1 = poly->box[3];
        // the TMA kernel runs one fast test in pass A: the one covering more area
        const double disk = kp->r2 > 0.0f ? 3.141592653589793 * (double)kp->r2 : 0.0;
        const double box = (kp->bx0 <= kp->bx1 && kp->by0 <= kp->by1)
                               ? ((double)kp->bx1 - kp->bx0) * ((double)kp->by1 - kp->by0)
                               : 0.0;
        kp->fast = box > disk ? 1 : 0;
    }
}

}  // namespace cudapre
