// host_geom3.cpp — Step 2 of the 3D extension on the host (PAPER.md P:115:
// "These extreme points can be then used to form a convex polyhedron";
// DESIGN.md §3 B3-B4, §6.5), plus the Step-3 geometry K2-3D reads.
// Compiled with -ffp-contract=off.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "exact3.cuh"
#include "internal3.h"

namespace cudapre {
namespace {

float f_up(double v) {   // smallest float >= v (v finite)
    float f = (float)v;
    if ((double)f < v) f = std::nextafter(f, INFINITY);
    return f;
}

struct P3 {
    float v[3];
    int64_t id;
};

// Clip the convex polygon poly[0..n) (in place) by the half-space
// h[0] x + h[1] y + h[2] z + h[3] >= 0.  Returns the new vertex count.
int clip(double (*poly)[3], int n, const double* h) {
    double out[24][3];
    int m = 0;
    for (int i = 0; i < n && m < 22; ++i) {
        const double* P = poly[i];
        const double* Q = poly[(i + 1) % n];
        const double dp = h[0] * P[0] + h[1] * P[1] + h[2] * P[2] + h[3];
        const double dq = h[0] * Q[0] + h[1] * Q[1] + h[2] * Q[2] + h[3];
        if (dp >= 0) {
            for (int k = 0; k < 3; ++k) out[m][k] = P[k];
            ++m;
        }
        if ((dp >= 0) != (dq >= 0)) {
            const double t = dp / (dp - dq);
            for (int k = 0; k < 3; ++k) out[m][k] = P[k] + t * (Q[k] - P[k]);
            ++m;
        }
    }
    for (int i = 0; i < m; ++i)
        for (int k = 0; k < 3; ++k) poly[i][k] = out[i][k];
    return m;
}

// Mark in cmask every direction cell that the triangle (A, B, C) (relative to
// the centre) may be seen through: per cube face (axis a, sign s) clip it to
// the face's pyramid widened by the guard, project the rest centrally to
// (u, v) = (d_b, d_c) / (s d_a) — the projection of a convex polygon in
// front of the centre is convex — and mark every cell whose rectangle,
// widened by the guard (the border cells unbounded outwards: the kernel
// clamps), meets it.  The guard covers the kernel's rounding of the cell
// index; clipping is done in binary64, far below the guard.
void mark_cells(const double* A, const double* B, const double* C, double tau, int bit, unsigned long long* cmask) {
    static const int U[3] = {1, 2, 0}, V[3] = {2, 0, 1};
    const double w = 1.0 + 4 * kCellGuard;
    for (int a = 0; a < 3; ++a)
        for (int sg = 0; sg < 2; ++sg) {
            const double s = sg ? -1.0 : 1.0;
            {   // trivial reject: all three vertices outside one of the pyramid's half-spaces
                const double* T3[3] = {A, B, C};
                bool o0 = true, o1 = true, o2 = true, o3 = true, o4 = true;
                for (int k = 0; k < 3; ++k) {
                    const double mk = s * T3[k][a];
                    o0 &= mk + tau < 0;
                    o1 &= w * mk - T3[k][U[a]] + tau < 0;
                    o2 &= w * mk + T3[k][U[a]] + tau < 0;
                    o3 &= w * mk - T3[k][V[a]] + tau < 0;
                    o4 &= w * mk + T3[k][V[a]] + tau < 0;
                }
                if (o0 || o1 || o2 || o3 || o4) continue;
            }
            double poly[24][3];
            for (int k = 0; k < 3; ++k) poly[0][k] = A[k], poly[1][k] = B[k], poly[2][k] = C[k];
            int n = 3;
            double h[4];
            // s d_a >= 0;  w s d_a -+ d_u >= 0;  w s d_a -+ d_v >= 0   (each relaxed by tau)
            h[0] = h[1] = h[2] = 0;
            h[a] = s;
            h[3] = tau;
            n = clip(poly, n, h);
            for (int t = 0; t < 4 && n > 0; ++t) {
                const int c = (t < 2) ? U[a] : V[a];
                h[0] = h[1] = h[2] = 0;
                h[a] = w * s;
                h[c] = (t & 1) ? 1.0 : -1.0;
                h[3] = tau;
                n = clip(poly, n, h);
            }
            if (n == 0) continue;
            double ulo = 1e300, uhi = -1e300, vlo = 1e300, vhi = -1e300;
            double uv[24][2];
            bool far = false;
            for (int i = 0; i < n; ++i) {
                const double m = s * poly[i][a];
                if (!(m > tau)) {   // at the apex: the polygon reaches the centre's neighbourhood
                    far = true;
                    break;
                }
                uv[i][0] = poly[i][U[a]] / m, uv[i][1] = poly[i][V[a]] / m;
                ulo = std::min(ulo, uv[i][0]), uhi = std::max(uhi, uv[i][0]);
                vlo = std::min(vlo, uv[i][1]), vhi = std::max(vhi, uv[i][1]);
            }
            const int face = 2 * a + sg;
            auto cell_of = [](double x) {
                const double f = std::floor((x + 1.0) * (kCellG / 2.0));
                return (int)std::min<double>(kCellG - 1, std::max<double>(0.0, f));
            };
            if (far) {
                for (int c = 0; c < kCellG * kCellG; ++c) cmask[face * kCellG * kCellG + c] |= 1ull << bit;
                continue;
            }
            const int iu0 = cell_of(ulo - kCellGuard), iu1 = cell_of(uhi + kCellGuard);
            for (int iu = iu0; iu <= iu1; ++iu) {
                // the polygon within this row's u-strip (widened by the guard; the
                // border rows unbounded outwards: the kernel clamps) is convex, so
                // its v-extent is exactly the v-range of the row's cells it meets
                const double cu0 = iu == 0 ? -1e300 : -1.0 + 2.0 * iu / kCellG - kCellGuard;
                const double cu1 = iu == kCellG - 1 ? 1e300 : -1.0 + 2.0 * (iu + 1) / kCellG + kCellGuard;
                double q[24][3];
                for (int i = 0; i < n; ++i) q[i][0] = uv[i][0], q[i][1] = uv[i][1], q[i][2] = 0.0;
                int k = n;
                const double h0[4] = {1, 0, 0, -cu0}, h1[4] = {-1, 0, 0, cu1};
                if (iu != 0) k = clip(q, k, h0);
                if (k > 0 && iu != kCellG - 1) k = clip(q, k, h1);
                if (k == 0) continue;
                double v0 = 1e300, v1 = -1e300;
                for (int i = 0; i < k; ++i) v0 = std::min(v0, q[i][1]), v1 = std::max(v1, q[i][1]);
                const int iv0 = cell_of(v0 - kCellGuard), iv1 = cell_of(v1 + kCellGuard);
                for (int iv = iv0; iv <= iv1; ++iv) cmask[(face * kCellG + iu) * kCellG + iv] |= 1ull << bit;
            }
    }
}

}  // namespace

int build_polyhedron3(const cudapre3_extremes_t& ext, cudapre3_polyhedron_t* poly, K3Geom* g, int flags) {
    cudapre3_polyhedron_t P;
    std::memset(&P, 0, sizeof(P));
    std::memset(g, 0, sizeof(*g));
    const int nslots = 6 * ext.nang;
    // E: distinct picks, ascending id, equal coordinates -> lowest id (B3)
    std::vector<P3> cand;
    for (int s = 0; s < nslots; ++s)
        if (ext.idx[s] >= 0) cand.push_back(P3{{ext.pt[s].x, ext.pt[s].y, ext.pt[s].z}, ext.idx[s]});
    std::sort(cand.begin(), cand.end(), [](const P3& a, const P3& b) { return a.id < b.id; });
    std::vector<P3> E;
    for (size_t j = 0; j < cand.size(); ++j) {
        if (j > 0 && cand[j].id == cand[j - 1].id) continue;
        bool dup = false;
        for (const P3& e : E)
            if (e.v[0] == cand[j].v[0] && e.v[1] == cand[j].v[1] && e.v[2] == cand[j].v[2]) dup = true;
        if (!dup) E.push_back(cand[j]);
    }
    const int m = (int)E.size();
    P.n_distinct = m;
    for (int j = 0; j < m; ++j) P.eidx[j] = E[j].id;

    // facets: first supporting triple of each plane, E on the positive side (B4).
    // The support test yields the triple's on-plane points (sign 0); a later
    // supporting triple lies on a kept facet's plane iff its three points are
    // all in that facet's on-plane set (a supporting plane is determined by
    // any three non-collinear points on it), so duplicates cost no predicate.
    int nf = 0;
    int F[kMax3Facets][3];
    unsigned long long onp[kMax3Facets];   // points of E on each kept facet's plane
    for (int a = 0; a < m; ++a)
        for (int b = a + 1; b < m; ++b)
            for (int c = b + 1; c < m; ++c) {
                const unsigned long long abc = (1ull << a) | (1ull << b) | (1ull << c);
                bool dup = false;
                for (int f = 0; f < nf && !dup; ++f) dup = (onp[f] & abc) == abc;
                if (dup) continue;   // on an earlier facet's plane: never kept (supporting or not)
                bool pos = false, neg = false;
                unsigned long long on = abc;
                for (int d = 0; d < m && !(pos && neg); ++d) {
                    if (d == a || d == b || d == c) continue;
                    const int o = orient3d_sign_f(E[a].v, E[b].v, E[c].v, E[d].v);
                    pos |= o > 0;
                    neg |= o < 0;
                    if (o == 0) on |= 1ull << d;
                }
                if (pos == neg) continue;   // not supporting, or everything on the plane
                if (nf >= kMax3Facets) return CUDAPRE_ERR_INVALID_ARGUMENT;   // cannot happen for <= 34 points
                F[nf][0] = a;
                F[nf][1] = pos ? b : c;
                F[nf][2] = pos ? c : b;
                onp[nf] = on;
                ++nf;
            }
    P.nf = nf;
    for (int f = 0; f < nf; ++f)
        for (int k = 0; k < 3; ++k) {
            const P3& q = E[F[f][k]];
            P.fidx[f][k] = q.id;
            P.fv[f][k] = cudapre_pt3{q.v[0], q.v[1], q.v[2]};
        }
    g->nf = nf;
    if (nf == 0) {   // degenerate: nothing is inside
        g->mode = 1;
        if (poly) *poly = P;
        return 0;
    }
    for (int f = 0; f < nf; ++f)
        for (int k = 0; k < 3; ++k)
            for (int c = 0; c < 3; ++c) g->fv[f][3 * k + c] = E[F[f][k]].v[c];

    // data bounding box: the angle-0 slots hold the exact min / max of x, y, z
    const double Mx = std::max(std::fabs((double)ext.pt[0].x), std::fabs((double)ext.pt[1].x));
    const double My = std::max(std::fabs((double)ext.pt[2].y), std::fabs((double)ext.pt[3].y));
    const double Mz = std::max(std::fabs((double)ext.pt[4].z), std::fabs((double)ext.pt[5].z));

    // plane tests: g = A x + B y + C z + D ~ orient3d(a, b, c, p) = N . (p - a),
    // N = (b - a) x (c - a).  S bounds sum |term| of the exact and the float
    // evaluation over the box; the float evaluation (4 coefficient roundings,
    // 3 fma roundings) and the binary64 coefficient errors stay below
    // 2^-20 S; the absolute terms cover underflow.
    float4 pl[kMax3Facets];
    float pe[kMax3Facets];
    float emax = 0.f;
    for (int f = 0; f < nf; ++f) {
        const float* a = E[F[f][0]].v;
        const float* b = E[F[f][1]].v;
        const float* c = E[F[f][2]].v;
        const double ux = (double)b[0] - a[0], uy = (double)b[1] - a[1], uz = (double)b[2] - a[2];
        const double vx = (double)c[0] - a[0], vy = (double)c[1] - a[1], vz = (double)c[2] - a[2];
        const double Nx = uy * vz - uz * vy, Ny = uz * vx - ux * vz, Nz = ux * vy - uy * vx;
        const double Px = std::fabs(uy * vz) + std::fabs(uz * vy);
        const double Py = std::fabs(uz * vx) + std::fabs(ux * vz);
        const double Pz = std::fabs(ux * vy) + std::fabs(uy * vx);
        const double D = -(Nx * a[0] + Ny * a[1] + Nz * a[2]);
        const double S = Px * (Mx + std::fabs((double)a[0])) + Py * (My + std::fabs((double)a[1])) +
                         Pz * (Mz + std::fabs((double)a[2]));
        const double Ed = S * 0x1p-20 + (Mx + My + Mz + 1.0) * 0x1p-140 + 0x1p-126;
        const bool ok = S < 1e36 && std::isfinite(Ed);
        pl[f] = ok ? make_float4((float)Nx, (float)Ny, (float)Nz, (float)D) : make_float4(0.f, 0.f, 0.f, 0.f);
        pe[f] = ok ? f_up(Ed) : INFINITY;   // INFINITY: always undecided -> exact
        if (ok) emax = std::max(emax, pe[f]);
    }
    P.err_max = emax;

    // centre: mean of E, rounded to float; direction cells only if it is
    // strictly inside every facet (exact check)
    double cx = 0, cy = 0, cz = 0;
    for (const P3& e : E) cx += e.v[0], cy += e.v[1], cz += e.v[2];
    const float o[3] = {(float)(cx / m), (float)(cy / m), (float)(cz / m)};
    bool inside = std::isfinite(o[0]) && std::isfinite(o[1]) && std::isfinite(o[2]);
    for (int f = 0; f < nf && inside; ++f)
        inside = orient3d_sign_f(E[F[f][0]].v, E[F[f][1]].v, E[F[f][2]].v, o) > 0;
    if (flags & CUDAPRE3_FLAG_NO_CELLS) inside = false;   // caller: force the every-facet path
    g->ox = o[0], g->oy = o[1], g->oz = o[2];
    g->cells = inside ? 1 : 0;
    P.cells = g->cells;
    P.centre[0] = o[0], P.centre[1] = o[1], P.centre[2] = o[2];
    g->all = nf == 64 ? ~0ull : ((1ull << nf) - 1ull);
    std::vector<unsigned long long> cmask(kCells, 0ull);
    for (int f = 0; f < nf; ++f) {
        g->pl[f] = pl[f];
        g->pe[f] = pe[f];
    }
    if (!inside) {
        for (int c = 0; c < kCells; ++c) cmask[c] = g->all;
    } else {
        // face of facet f = conv(points of E on its plane) = the union of the
        // triangles of those points; relative to the centre, in binary64
        double ext_max = 0;
        for (const P3& e : E)
            for (int k = 0; k < 3; ++k) ext_max = std::max(ext_max, std::fabs((double)e.v[k] - o[k]));
        const double tau = ext_max * 0x1p-30 + 0x1p-140;
        for (int f = 0; f < nf; ++f) {
            std::vector<int> on;
            for (int j = 0; j < m; ++j)
                if ((onp[f] >> j) & 1ull) on.push_back(j);
            for (size_t i = 0; i < on.size(); ++i)
                for (size_t j = i + 1; j < on.size(); ++j)
                    for (size_t k = j + 1; k < on.size(); ++k) {
                        double A[3], B[3], C[3];
                        for (int c = 0; c < 3; ++c) {
                            A[c] = (double)E[on[i]].v[c] - o[c];
                            B[c] = (double)E[on[j]].v[c] - o[c];
                            C[c] = (double)E[on[k]].v[c] - o[c];
                        }
                        mark_cells(A, B, C, tau, f, cmask.data());
                    }
        }
    }
    g->pl[kDummyFacet] = make_float4(0.f, 0.f, 0.f, 1.f);
    g->pe[kDummyFacet] = 0.f;
    int nent = 0, mx = 0, nlong = 0, nempty = 0;
    for (int c = 0; c < kCells; ++c) {
        // fail-safe: a cell with no candidate facet would discard its points
        // untested (the dummy slots say "inside"); the exit-facet argument
        // says it cannot happen, so such a cell tests every facet instead and
        // is counted (tests assert the count is 0)
        if (cmask[c] == 0ull) {
            cmask[c] = g->all;
            ++nempty;
        }
        const int k = __builtin_popcountll(cmask[c]);
        nent += k;
        mx = std::max(mx, k);
        unsigned w = (unsigned)std::min(k, 255) << 24;
        if (k > kCellSlots) {   // long list: its mask (or every facet once lmask is full)
            ++P.long_cells;
            if (nlong < kMaxLong) {
                g->lmask[nlong] = cmask[c];
                w |= (unsigned)nlong++;
            } else {
                w |= kNoLong;
            }
        } else {
            int slot = 0;
            for (unsigned long long b = cmask[c]; b; b &= b - 1, ++slot)
                w |= (unsigned)__builtin_ctzll(b) << (8 * slot);
            for (; slot < kCellSlots; ++slot) w |= (unsigned)kDummyFacet << (8 * slot);
        }
        g->clist[c] = w;
    }
    P.n_entries = nent;
    P.max_candidates = mx;
    P.n_cells = kCells;
    P.empty_cells = nempty;
    if (poly) *poly = P;
    return 0;
}

int merge_extremes3(const cudapre3_extremes_t* parts, int count, cudapre3_extremes_t* out) {
    cudapre3_extremes_t r = parts[0];
    r.n = 0;
    r.nonfinite = 0;
    r.exact_points = 0;
    const int nslots = 6 * r.nang;
    for (int s = 0; s < nslots; ++s) r.idx[s] = -1;
    for (int q = 0; q < count; ++q) {
        const cudapre3_extremes_t& P = parts[q];
        if (P.nang != r.nang) return CUDAPRE_ERR_INVALID_ARGUMENT;
        r.n += P.n;
        r.nonfinite |= P.nonfinite;
        r.exact_points += P.exact_points;
        for (int s = 0; s < nslots; ++s) {
            if (P.idx[s] < 0) continue;
            const bool mx = (s & 1) != 0;
            bool better = r.idx[s] < 0;
            if (!better) {
                const double k = P.key[s], K = r.key[s];
                better = mx ? (k > K || (k == K && P.idx[s] < r.idx[s])) : (k < K || (k == K && P.idx[s] < r.idx[s]));
            }
            if (better) {
                r.idx[s] = P.idx[s];
                r.key[s] = P.key[s];
                r.pt[s] = P.pt[s];
            }
        }
    }
    *out = r;
    return r.n == 0 ? CUDAPRE_ERR_EMPTY_INPUT : 0;
}

}  // namespace cudapre
