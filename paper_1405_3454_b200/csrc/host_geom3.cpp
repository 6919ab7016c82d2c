// host_geom3.cpp — Step 2 of the 3D extension on the host (PAPER.md P:115:
// "These extreme points can be then used to form a convex polyhedron";
// DESIGN.md §3 B3-B4, §6.5), plus the Step-3 geometry K2-3D reads.
// Compiled with -ffp-contract=off.
#include <algorithm>
#include <cmath>
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

// Does the triangle (a, b, c) (coordinates relative to the centre) meet the
// closed octant {sigma_i x_i >= -tau}?  Sutherland-Hodgman clip by the three
// half-spaces; conservative by tau (never misses a true intersection).
bool tri_meets_octant(const double* a, const double* b, const double* c, int oct, double tau) {
    double poly[16][3], tmp[16][3];
    int n = 3;
    for (int k = 0; k < 3; ++k) poly[0][k] = a[k], poly[1][k] = b[k], poly[2][k] = c[k];
    for (int ax = 0; ax < 3 && n > 0; ++ax) {
        const double sg = ((oct >> ax) & 1) ? -1.0 : 1.0;   // bit set: x_ax < centre
        int m = 0;
        for (int i = 0; i < n; ++i) {
            const double* P = poly[i];
            const double* Q = poly[(i + 1) % n];
            const double dp = sg * P[ax] + tau, dq = sg * Q[ax] + tau;
            if (dp >= 0) {
                for (int k = 0; k < 3; ++k) tmp[m][k] = P[k];
                ++m;
            }
            if ((dp >= 0) != (dq >= 0)) {
                const double t = dp / (dp - dq);
                for (int k = 0; k < 3; ++k) tmp[m][k] = P[k] + t * (Q[k] - P[k]);
                ++m;
            }
        }
        n = m;
        for (int i = 0; i < n; ++i)
            for (int k = 0; k < 3; ++k) poly[i][k] = tmp[i][k];
    }
    return n > 0;
}

}  // namespace

int build_polyhedron3(const cudapre3_extremes_t& ext, cudapre3_polyhedron_t* poly, K3Geom* g) {
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

    // facets: first supporting triple of each plane, E on the positive side (B4)
    int nf = 0;
    int F[kMax3Facets][3];
    for (int a = 0; a < m; ++a)
        for (int b = a + 1; b < m; ++b)
            for (int c = b + 1; c < m; ++c) {
                bool pos = false, neg = false;
                for (int d = 0; d < m && !(pos && neg); ++d) {
                    if (d == a || d == b || d == c) continue;
                    const int o = orient3d_sign_f(E[a].v, E[b].v, E[c].v, E[d].v);
                    pos |= o > 0;
                    neg |= o < 0;
                }
                if (pos == neg) continue;   // not supporting, or everything on the plane
                bool same = false;
                for (int f = 0; f < nf && !same; ++f) {
                    const float* A = E[F[f][0]].v;
                    const float* B = E[F[f][1]].v;
                    const float* C = E[F[f][2]].v;
                    same = orient3d_sign_f(A, B, C, E[a].v) == 0 && orient3d_sign_f(A, B, C, E[b].v) == 0 &&
                           orient3d_sign_f(A, B, C, E[c].v) == 0;
                }
                if (same) continue;
                if (nf >= kMax3Facets) return CUDAPRE_ERR_INVALID_ARGUMENT;   // cannot happen for <= 34 points
                F[nf][0] = a;
                F[nf][1] = pos ? b : c;
                F[nf][2] = pos ? c : b;
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

    // centre: mean of E, rounded to float; octant lists only if it is
    // strictly inside every facet (exact check)
    double cx = 0, cy = 0, cz = 0;
    for (const P3& e : E) cx += e.v[0], cy += e.v[1], cz += e.v[2];
    const float o[3] = {(float)(cx / m), (float)(cy / m), (float)(cz / m)};
    bool inside = std::isfinite(o[0]) && std::isfinite(o[1]) && std::isfinite(o[2]);
    for (int f = 0; f < nf && inside; ++f)
        inside = orient3d_sign_f(E[F[f][0]].v, E[F[f][1]].v, E[F[f][2]].v, o) > 0;
    g->ox = o[0], g->oy = o[1], g->oz = o[2];
    g->octants = inside ? 1 : 0;
    P.octants = g->octants;
    P.centre[0] = o[0], P.centre[1] = o[1], P.centre[2] = o[2];

    int nent = 0;
    if (!inside) {
        for (int f = 0; f < nf; ++f) {
            g->pl[nent] = pl[f];
            g->pe[nent] = pe[f];
            g->pf[nent] = (unsigned char)f;
            ++nent;
        }
        g->oct_start[0] = 0;
        for (int k = 1; k <= 8; ++k) g->oct_start[k] = nent;
        for (int k = 0; k < 8; ++k) P.oct_count[k] = nf;
    } else {
        // face of facet f = conv(points of E on its plane) = union of the
        // triangles of those points; relative to the centre, in binary64
        std::vector<std::vector<int>> on(nf);
        double ext_max = 0;
        for (const P3& e : E)
            for (int k = 0; k < 3; ++k) ext_max = std::max(ext_max, std::fabs((double)e.v[k] - o[k]));
        const double tau = ext_max * 0x1p-30 + 0x1p-140;
        for (int f = 0; f < nf; ++f)
            for (int j = 0; j < m; ++j)
                if (j == F[f][0] || j == F[f][1] || j == F[f][2] ||
                    orient3d_sign_f(E[F[f][0]].v, E[F[f][1]].v, E[F[f][2]].v, E[j].v) == 0)
                    on[f].push_back(j);
        for (int oct = 0; oct < 8; ++oct) {
            g->oct_start[oct] = nent;
            for (int f = 0; f < nf; ++f) {
                bool meets = false;
                const std::vector<int>& V = on[f];
                for (size_t i = 0; i < V.size() && !meets; ++i)
                    for (size_t j = i + 1; j < V.size() && !meets; ++j)
                        for (size_t k = j + 1; k < V.size() && !meets; ++k) {
                            double A[3], B[3], C[3];
                            for (int c = 0; c < 3; ++c) {
                                A[c] = (double)E[V[i]].v[c] - o[c];
                                B[c] = (double)E[V[j]].v[c] - o[c];
                                C[c] = (double)E[V[k]].v[c] - o[c];
                            }
                            meets = tri_meets_octant(A, B, C, oct, tau);
                        }
                if (!meets) continue;
                g->pl[nent] = pl[f];
                g->pe[nent] = pe[f];
                g->pf[nent] = (unsigned char)f;
                ++nent;
            }
            P.oct_count[oct] = nent - g->oct_start[oct];
        }
        g->oct_start[8] = nent;
    }
    g->nent = nent;
    P.n_entries = nent;
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
