/*
 * cudapre3_oracle.c — CPU ORACLE for the 3D extension of CudaPre (G. Mei,
 * arXiv 1405.3454, §5 "Conclusion and Outlook").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path in
 * paper_1405_3454_b200/ and never includes anything from it.
 *
 * "In 3D, typically six extreme points can be obtained by finding those
 * points with the min or max x, y, or z coordinates.  More groups of six
 * extreme points can also be found after rotating the set of points along a
 * specific axis.  These extreme points can be then used to form a convex
 * polyhedron.  Those points locating inside the convex polyhedron must be
 * interior points, and can be directly discarded."  Readings (DESIGN.md §3,
 * B1-B6):
 *
 *   Step 1 (B1, B2): the rotation axis is z.  For every angle k of the same
 *          angle sets as the 2D method and every point i (ascending i):
 *              X = RN(RN(x c_k) + RN(y s_k)),  Y = RN(RN(y c_k) - RN(x s_k)),
 *              Z = z
 *          in binary64 without FMA; argmin/argmax of each key, strict
 *          improvement only (lowest index on ties).  Slot order
 *          6k + {minX, maxX, minY, maxY, minZ, maxZ} (the Z slots repeat for
 *          every k: a rotation about z leaves z unchanged).
 *   Step 2 (B3, B4): the polyhedron is conv(E), E = the distinct picks (equal
 *          coordinates collapse to the lowest index), sorted by index.  Its
 *          facet planes are found by brute force: a triple (a, b, c) of E
 *          (a < b < c in that order) SUPPORTS a facet iff orient3d(a, b, c, d)
 *          has the same weak sign for every d in E and is nonzero for at least
 *          one d; it is stored oriented so that E lies on the positive side,
 *          and only the first triple of each plane is kept.  No supporting
 *          triple (|E| < 4 or E coplanar) = degenerate: nothing is inside.
 *   Step 3 (B5): p is discarded iff orient3d(f, p) > 0 for EVERY facet f
 *          (strictly inside the interior of conv(E)); survivors ascend.
 *
 * orient3d(a,b,c,d) is the EXACT sign of det[b-a; c-a; d-a] (rows), i.e.
 * ((b-a) x (c-a)) . (d-a): positive when d lies on the side the right-handed
 * normal of (a, b, c) points to (B6).  Technique (deliberately different from
 * the CUDA path, which uses a floating-point filter and expansions): by
 * multilinearity det(b-a, c-a, d-a) = det(b,c,d) - det(a,c,d) - det(b,a,d) -
 * det(b,c,a) (every term with two rows equal to a vanishes), i.e. 24 signed
 * products x*y*z of input floats.  Each float is an integer mantissa
 * (< 2^24) times a power of two, so each product is an integer (< 2^72)
 * times a power of two; all are added into a wide two's-complement
 * fixed-point accumulator of 32-bit limbs whose sign is the exact sign.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define O3_MAX_ANGLES 8
#define O3_MAX_SLOTS (6 * O3_MAX_ANGLES)

/* ------------------------------------------------------------------------ */
/* Exact orient3d (B6).                                                     */

/* A nonzero float is m * 2^e with 2^23 <= m < 2^24 and e in [-172, 104]
 * (split_float's normalisation); a product of three is M * 2^E with
 * M < 2^72, E in [-516, 312]; |sum of 24| < 2^389.                          */
#define L3 34             /* 34 * 32 = 1088 bits */
#define L3_OFFSET (-544)  /* weight of limb 0 is 2^-544 */

static void split_float(float f, uint64_t* m, int* e, int* neg) {
    int E;
    double d = (double)f;
    *neg = d < 0;
    if (*neg) d = -d;
    if (d == 0.0) { *m = 0; *e = 0; return; }
    d = frexp(d, &E);                        /* d in [0.5, 1) */
    *m = (uint64_t)ldexp(d, 24);             /* exact: a float has <= 24 significant bits */
    *e = E - 24;
}

/* acc += sign * x*y*z (exactly) */
static void acc3_add(int64_t* acc, float x, float y, float z, int sign) {
    uint64_t mx, my, mz;
    int ex, ey, ez, nx, ny, nz, shift, q, r, t;
    unsigned __int128 M;
    split_float(x, &mx, &ex, &nx);
    split_float(y, &my, &ey, &ny);
    split_float(z, &mz, &ez, &nz);
    if (mx == 0 || my == 0 || mz == 0) return;
    if (nx ^ ny ^ nz) sign = -sign;
    M = (unsigned __int128)(mx * my) * mz;   /* mx*my < 2^48, M < 2^72 */
    shift = ex + ey + ez - L3_OFFSET;        /* >= 28 */
    q = shift / 32;
    r = shift % 32;
    for (t = 0; t < 4; ++t) {                /* (M << r) < 2^104: four 32-bit chunks */
        unsigned __int128 v = (M << r) >> (32 * t);
        acc[q + t] += sign * (int64_t)(uint32_t)v;
    }
}

/* acc += sign * det(P; Q; R) (rows), six products */
static void acc3_det(int64_t* acc, const float* P, const float* Q, const float* R, int sign) {
    acc3_add(acc, P[0], Q[1], R[2], +sign);
    acc3_add(acc, P[0], Q[2], R[1], -sign);
    acc3_add(acc, P[1], Q[0], R[2], -sign);
    acc3_add(acc, P[1], Q[2], R[0], +sign);
    acc3_add(acc, P[2], Q[0], R[1], +sign);
    acc3_add(acc, P[2], Q[1], R[0], -sign);
}

/* exact sign of det[b-a; c-a; d-a]; a, b, c, d are xyz triples */
int oracle3_orient(const float* a, const float* b, const float* c, const float* d) {
    int64_t acc[L3 + 1];
    int k;
    memset(acc, 0, sizeof(acc));
    acc3_det(acc, b, c, d, +1);
    acc3_det(acc, a, c, d, -1);
    acc3_det(acc, b, a, d, -1);
    acc3_det(acc, b, c, a, -1);
    for (k = 0; k < L3; ++k) {               /* carry-propagate; top limb signed */
        int64_t carry = acc[k] >> 32;
        acc[k] -= carry * ((int64_t)1 << 32);
        acc[k + 1] += carry;
    }
    if (acc[L3] < 0) return -1;
    for (k = L3; k >= 0; --k)
        if (acc[k] != 0) return 1;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Step 1: the 6 * nang extreme points (P:115 + P:33-35; B1, B2).           */

typedef struct {
    const float* xyz;
    int64_t lo, hi;
    const double* c;
    const double* s;
    int nang;
    int64_t idx[O3_MAX_SLOTS];
    double key[O3_MAX_SLOTS];
} ext3_job;

static void ext3_range(ext3_job* J) {
    int k, r;
    for (k = 0; k < J->nang; ++k) {
        const double c = J->c[k], s = J->s[k];
        int64_t i;
        int64_t* idx = &J->idx[6 * k];
        double* key = &J->key[6 * k];
        for (i = J->lo; i < J->hi; ++i) {
            const double x = (double)J->xyz[3 * i + 0];
            const double y = (double)J->xyz[3 * i + 1];
            const double z = (double)J->xyz[3 * i + 2];
            const double X = x * c + y * s;   /* RN(RN(x c) + RN(y s)), no FMA */
            const double Y = y * c - x * s;   /* RN(RN(y c) - RN(x s)), no FMA */
            const double v[6] = {X, X, Y, Y, z, z};
            if (i == J->lo) {
                for (r = 0; r < 6; ++r) { key[r] = v[r]; idx[r] = i; }
                continue;
            }
            for (r = 0; r < 6; r += 2) {
                if (v[r] < key[r]) { key[r] = v[r]; idx[r] = i; }                 /* min */
                if (v[r + 1] > key[r + 1]) { key[r + 1] = v[r + 1]; idx[r + 1] = i; } /* max */
            }
        }
    }
}

static void* ext3_thread(void* arg) {
    ext3_range((ext3_job*)arg);
    return NULL;
}

/* idx_out[6*nang] (and key_out, nullable).  threads > 1 splits [0, n) into
 * contiguous chunks merged in chunk order with the same strict rule.
 * Returns 0, or -1 on empty input / bad arguments.                          */
int oracle3_extremes(const float* xyz, int64_t n, const double* c, const double* s, int nang,
                     int threads, int64_t* idx_out, double* key_out) {
    ext3_job jobs[64];
    pthread_t tid[64];
    int t, k, T;
    if (n <= 0 || nang <= 0 || nang > O3_MAX_ANGLES) return -1;
    T = threads < 1 ? 1 : (threads > 64 ? 64 : threads);
    if ((int64_t)T > n) T = (int)n;
    for (t = 0; t < T; ++t) {
        jobs[t].xyz = xyz;
        jobs[t].lo = n * t / T;
        jobs[t].hi = n * (t + 1) / T;
        jobs[t].c = c;
        jobs[t].s = s;
        jobs[t].nang = nang;
    }
    if (T == 1) {
        ext3_range(&jobs[0]);
    } else {
        for (t = 0; t < T; ++t) pthread_create(&tid[t], NULL, ext3_thread, &jobs[t]);
        for (t = 0; t < T; ++t) pthread_join(tid[t], NULL);
    }
    for (k = 0; k < 6 * nang; ++k) {
        int64_t bi = jobs[0].idx[k];
        double bk = jobs[0].key[k];
        int is_max = (k % 2) == 1;
        for (t = 1; t < T; ++t) {
            double v = jobs[t].key[k];
            if (is_max ? (v > bk) : (v < bk)) { bk = v; bi = jobs[t].idx[k]; }
        }
        idx_out[k] = bi;
        if (key_out) key_out[k] = bk;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Step 2: the polyhedron conv(E) as its facet planes (B3, B4).             */

static int cmp_i64(const void* pa, const void* pb) {
    const int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
    return (a > b) - (a < b);
}

/* E: the distinct picks, ascending index, equal coordinates -> lowest index.
 * Returns |E|.                                                              */
int64_t oracle3_distinct(const float* xyz, const int64_t* picks, int64_t npicks, int64_t* E) {
    int64_t ids[O3_MAX_SLOTS];
    int64_t j, m = 0;
    if (npicks > O3_MAX_SLOTS) return -1;
    memcpy(ids, picks, sizeof(int64_t) * (size_t)npicks);
    qsort(ids, (size_t)npicks, sizeof(int64_t), cmp_i64);
    for (j = 0; j < npicks; ++j) {
        int64_t i, dup = 0;
        if (j > 0 && ids[j] == ids[j - 1]) continue;
        for (i = 0; i < m; ++i) {
            const float* p = &xyz[3 * E[i]];
            const float* q = &xyz[3 * ids[j]];
            if (p[0] == q[0] && p[1] == q[1] && p[2] == q[2]) { dup = 1; break; }
        }
        if (!dup) E[m++] = ids[j];
    }
    return m;
}

/* Facets of conv(E) (E as returned by oracle3_distinct): facet_out[3*f..]
 * holds point ids (a, b, c) with orient3d(a, b, c, e) >= 0 for every e in E.
 * Returns the number of facets (0 = degenerate), -1 on overflow.            */
int64_t oracle3_facets(const float* xyz, const int64_t* E, int64_t m, int64_t* facet_out,
                       int64_t max_facets) {
    int64_t a, b, c, d, nf = 0;
    for (a = 0; a < m; ++a)
        for (b = a + 1; b < m; ++b)
            for (c = b + 1; c < m; ++c) {
                const float* A = &xyz[3 * E[a]];
                const float* B = &xyz[3 * E[b]];
                const float* C = &xyz[3 * E[c]];
                int pos = 0, neg = 0, f, same = 0;
                for (d = 0; d < m; ++d) {
                    int o;
                    if (d == a || d == b || d == c) continue;
                    o = oracle3_orient(A, B, C, &xyz[3 * E[d]]);
                    pos |= o > 0;
                    neg |= o < 0;
                }
                if ((pos && neg) || (!pos && !neg)) continue;   /* not supporting / all on the plane */
                for (f = 0; f < nf && !same; ++f) {              /* first triple of each plane only */
                    const float* F0 = &xyz[3 * facet_out[3 * f]];
                    const float* F1 = &xyz[3 * facet_out[3 * f + 1]];
                    const float* F2 = &xyz[3 * facet_out[3 * f + 2]];
                    same = oracle3_orient(F0, F1, F2, A) == 0 && oracle3_orient(F0, F1, F2, B) == 0 &&
                           oracle3_orient(F0, F1, F2, C) == 0;
                }
                if (same) continue;
                if (nf >= max_facets) return -1;
                facet_out[3 * nf] = E[a];
                facet_out[3 * nf + 1] = pos ? E[b] : E[c];       /* E on the positive side */
                facet_out[3 * nf + 2] = pos ? E[c] : E[b];
                ++nf;
            }
    return nf;
}

/* ------------------------------------------------------------------------ */
/* Step 3: discard points strictly inside the polyhedron (B5).              */

/* 1 iff orient3d(f, p) > 0 for every facet (coordinates, 9 floats per facet) */
int oracle3_strictly_inside(const float* fxyz, int64_t nf, const float* p) {
    int64_t f;
    if (nf <= 0) return 0;   /* degenerate polyhedron: nothing is inside */
    for (f = 0; f < nf; ++f)
        if (oracle3_orient(&fxyz[9 * f], &fxyz[9 * f + 3], &fxyz[9 * f + 6], p) <= 0) return 0;
    return 1;
}

typedef struct {
    const float* xyz;
    int64_t lo, hi;
    const float* fxyz;
    int64_t nf;
    uint8_t* keep;
} filt3_job;

static void* filt3_thread(void* arg) {
    filt3_job* J = (filt3_job*)arg;
    int64_t i;
    for (i = J->lo; i < J->hi; ++i) J->keep[i] = !oracle3_strictly_inside(J->fxyz, J->nf, &J->xyz[3 * i]);
    return NULL;
}

void oracle3_filter_mask(const float* xyz, int64_t n, const float* fxyz, int64_t nf, int threads,
                         uint8_t* keep) {
    filt3_job jobs[64];
    pthread_t tid[64];
    int t, T = threads < 1 ? 1 : (threads > 64 ? 64 : threads);
    if (n <= 0) return;
    if ((int64_t)T > n) T = (int)n;
    for (t = 0; t < T; ++t) {
        jobs[t].xyz = xyz;
        jobs[t].lo = n * t / T;
        jobs[t].hi = n * (t + 1) / T;
        jobs[t].fxyz = fxyz;
        jobs[t].nf = nf;
        jobs[t].keep = keep;
    }
    if (T == 1) {
        filt3_thread(&jobs[0]);
    } else {
        for (t = 0; t < T; ++t) pthread_create(&tid[t], NULL, filt3_thread, &jobs[t]);
        for (t = 0; t < T; ++t) pthread_join(tid[t], NULL);
    }
}

/* ------------------------------------------------------------------------ */
/* The whole 3D method in order: Step 1, Step 2, Step 3.                    */

/* Outputs: ext_idx[6*nang]; facets[3*max_facets] and *nf (0 = degenerate);
 * keep[n].  Returns 0, or -1 for empty input / bad arguments / overflow.    */
int oracle3_cudapre(const float* xyz, int64_t n, const double* c, const double* s, int nang,
                    int threads, int64_t* ext_idx, int64_t* facets, int64_t max_facets, int64_t* nf,
                    uint8_t* keep) {
    int64_t E[O3_MAX_SLOTS];
    float* fxyz;
    int64_t m, f, k;
    if (oracle3_extremes(xyz, n, c, s, nang, threads, ext_idx, NULL) != 0) return -1;
    m = oracle3_distinct(xyz, ext_idx, 6 * nang, E);
    if (m < 0) return -1;
    *nf = oracle3_facets(xyz, E, m, facets, max_facets);
    if (*nf < 0) return -1;
    fxyz = (float*)malloc(sizeof(float) * 9 * (size_t)(*nf > 0 ? *nf : 1));
    if (!fxyz) return -1;
    for (f = 0; f < *nf; ++f)
        for (k = 0; k < 3; ++k) memcpy(&fxyz[9 * f + 3 * k], &xyz[3 * facets[3 * f + k]], 3 * sizeof(float));
    oracle3_filter_mask(xyz, n, fxyz, *nf, threads, keep);
    free(fxyz);
    return 0;
}
