/*
 * cudapre_oracle.c — CPU ORACLE for the CudaPre interior-point filter
 * (G. Mei, arXiv 1405.3454, "A Straightforward Preprocessing Approach for
 * Accelerating Convex Hull Computations on the GPU").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path in
 * paper_1405_3454_b200/ and never includes anything from it.
 *
 * Plain, slow, obviously correct: every step below follows PAPER.md §2 in the
 * paper's order.  Citations: "P:nn" = /root/reference/PAPER.md line nn,
 * "S:nn" = /root/reference/SPEC.md line nn, "A#" = reading
 *
 *   Step 1: for every angle k and every point i (in
 *          ascending i) compute the rotated-frame keys
 *              X = RN(RN(x*c_k) + RN(y*s_k)),  Y = RN(RN(y*c_k) - RN(x*s_k))
 *          in IEEE binary64 (inputs are float, widened exactly; this file is
 *          compiled with -ffp-contract=off so no FMA is formed, A6) and keep
 *          argmin/argmax of each key, replacing only on STRICT improvement so
 *          the lowest index wins ties (A7).  Slot order 4k+{minX,maxX,minY,maxY}
 *          (A8).
 *   Step 2: Andrew's monotone chain on the distinct
 *          candidate points: lexicographic (x, y, index) sort, lower and upper
 *          chains, pop while orient <= 0 (collinear excluded, A10); a ring of
 *          fewer than 3 vertices is degenerate (A13).
 *   Step 3: point i is discarded iff
 *          orient(v_j, v_j+1, p_i) > 0 for EVERY edge j (strictly inside, A12);
 *          survivors are reported in ascending index order (A15).
 *   Final hull: the same monotone chain on the survivors.
 *
 * orient(a,b,c) is the EXACT sign of (bx-ax)(cy-ay) - (by-ay)(cx-ax) (A11).
 * Technique (deliberately different from the CUDA path, which uses floating
 * point expansions): the six float*float products of the expanded form are
 * each exact in binary64; each is split into an integer mantissa and a power
 * of two and added into a wide two's-complement fixed-point accumulator of
 * 32-bit limbs; the sign of the accumulator is the exact sign.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_MAX_ANGLES 8
#define ORACLE_MAX_SLOTS (4 * ORACLE_MAX_ANGLES)

/* ------------------------------------------------------------------------ */
/* Coefficients (A5): correctly rounded cos/sin of the exact angle.  Each
 * value is the binary64 nearest to the closed form written beside it; they
 * are pinned in tests/test_oracle_pins.py against 80-digit decimal
 * evaluations of those closed forms.  (libm's cos(30*pi/180) is NOT used:
 * it is off by one ulp at 30, 45, 60 and 67.5 degrees.)                     */
typedef struct { double deg, c, s; } oracle_angle;
static const oracle_angle ORACLE_ANGLES[] = {
    {0.0, 1.0, 0.0},
    {15.0, 0x1.ee8dd4748bf15p-1, 0x1.0907dc1930690p-2},  /* (sqrt6+sqrt2)/4, (sqrt6-sqrt2)/4 */
    {22.5, 0x1.d906bcf328d46p-1, 0x1.87de2a6aea963p-2},  /* sqrt(2+sqrt2)/2, sqrt(2-sqrt2)/2 */
    {30.0, 0x1.bb67ae8584caap-1, 0x1.0000000000000p-1},  /* sqrt3/2, 1/2 */
    {45.0, 0x1.6a09e667f3bcdp-1, 0x1.6a09e667f3bcdp-1},  /* sqrt2/2, sqrt2/2 */
    {60.0, 0x1.0000000000000p-1, 0x1.bb67ae8584caap-1},  /* 1/2, sqrt3/2 */
    {67.5, 0x1.87de2a6aea963p-2, 0x1.d906bcf328d46p-1},  /* sqrt(2-sqrt2)/2, sqrt(2+sqrt2)/2 */
    {75.0, 0x1.0907dc1930690p-2, 0x1.ee8dd4748bf15p-1},  /* (sqrt6-sqrt2)/4, (sqrt6+sqrt2)/4 */
    {90.0, 0.0, 1.0},
};

/* Look up (c, s) for an angle in degrees.  Returns 0 on success, -1 if the
 * angle is not one whose correctly rounded coefficients this oracle knows.  */
int oracle_coeffs(double deg, double* c, double* s) {
    size_t k;
    for (k = 0; k < sizeof(ORACLE_ANGLES) / sizeof(ORACLE_ANGLES[0]); ++k) {
        if (ORACLE_ANGLES[k].deg == deg) {
            *c = ORACLE_ANGLES[k].c;
            *s = ORACLE_ANGLES[k].s;
            return 0;
        }
    }
    return -1;
}

/* ------------------------------------------------------------------------ */
/* Exact orientation sign (A11).                                            */

#define LIMBS 26          /* 26 * 32 = 832 bits of accumulator */
#define LIMB_OFFSET (-416) /* weight of limb 0 is 2^-416 */

/* add sign * (m * 2^e) to the accumulator; m < 2^53 */
static void acc_add(int64_t* acc, uint64_t m, int e, int sign) {
    int shift = e - LIMB_OFFSET; /* >= 0 for every float*float product */
    int q = shift / 32, r = shift % 32;
    unsigned __int128 v = (unsigned __int128)m << r; /* < 2^85 */
    int t;
    for (t = 0; t < 3; ++t) {
        int64_t chunk = (int64_t)(uint32_t)(v >> (32 * t));
        acc[q + t] += sign * chunk;
    }
}

/* add sign * p, p = an exactly representable double (a float*float product) */
static void acc_add_double(int64_t* acc, double p, int sign) {
    int E;
    double f;
    if (p == 0.0) return;
    if (p < 0) { p = -p; sign = -sign; }
    f = frexp(p, &E);                       /* p = f * 2^E, f in [0.5, 1) */
    acc_add(acc, (uint64_t)ldexp(f, 53), E - 53, sign); /* f*2^53 is an integer */
}

int oracle_orient(float ax, float ay, float bx, float by, float cx, float cy) {
    int64_t acc[LIMBS + 1];
    int k;
    memset(acc, 0, sizeof(acc));
    /* (bx-ax)(cy-ay) - (by-ay)(cx-ax)
     *   = bx*cy - bx*ay - ax*cy - by*cx + by*ax + ay*cx   (ax*ay cancels)     */
    acc_add_double(acc, (double)bx * (double)cy, +1);
    acc_add_double(acc, (double)bx * (double)ay, -1);
    acc_add_double(acc, (double)ax * (double)cy, -1);
    acc_add_double(acc, (double)by * (double)cx, -1);
    acc_add_double(acc, (double)by * (double)ax, +1);
    acc_add_double(acc, (double)ay * (double)cx, +1);
    /* carry-propagate: limbs 0..LIMBS-1 end in [0, 2^32), top limb signed */
    for (k = 0; k < LIMBS; ++k) {
        int64_t carry = acc[k] >> 32; /* arithmetic shift = floor division */
        acc[k] -= carry * ((int64_t)1 << 32);
        acc[k + 1] += carry;
    }
    if (acc[LIMBS] < 0) return -1;
    for (k = LIMBS; k >= 0; --k)
        if (acc[k] != 0) return 1;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Step 1: extreme points.                             */

typedef struct {
    const float* xy;
    int64_t lo, hi;
    const double* c;
    const double* s;
    int nang;
    int64_t idx[ORACLE_MAX_SLOTS];
    double key[ORACLE_MAX_SLOTS];
} extremes_job;

static void extremes_range(extremes_job* J) {
    int k;
    for (k = 0; k < J->nang; ++k) {
        const double c = J->c[k], s = J->s[k];
        int64_t i;
        int64_t* idx = &J->idx[4 * k];
        double* key = &J->key[4 * k];
        for (i = J->lo; i < J->hi; ++i) {
            const double x = (double)J->xy[2 * i + 0];
            const double y = (double)J->xy[2 * i + 1];
            const double X = x * c + y * s; /* RN(RN(x c) + RN(y s)), no FMA */
            const double Y = y * c - x * s; /* RN(RN(y c) - RN(x s)), no FMA */
            if (i == J->lo) {
                key[0] = key[1] = X;
                key[2] = key[3] = Y;
                idx[0] = idx[1] = idx[2] = idx[3] = i;
                continue;
            }
            if (X < key[0]) { key[0] = X; idx[0] = i; } /* min X */
            if (X > key[1]) { key[1] = X; idx[1] = i; } /* max X */
            if (Y < key[2]) { key[2] = Y; idx[2] = i; } /* min Y */
            if (Y > key[3]) { key[3] = Y; idx[3] = i; } /* max Y */
        }
    }
}

static void* extremes_thread(void* arg) {
    extremes_range((extremes_job*)arg);
    return NULL;
}

/* idx_out[4*nang]: 4k+{argmin X, argmax X, argmin Y, argmax Y}.
 * threads > 1 splits [0,n) into contiguous chunks and merges them in chunk
 * order with the same rule (strict improvement only), so every thread count
 * gives the same answer.  Returns 0, or -1 on empty input
 * / bad arguments.                                                  */
int oracle_extremes(const float* xy, int64_t n, const double* c, const double* s,
                    int nang, int threads, int64_t* idx_out, double* key_out) {
    extremes_job jobs[64];
    pthread_t tid[64];
    int t, k, T;
    if (n <= 0 || nang <= 0 || nang > ORACLE_MAX_ANGLES) return -1;
    T = threads < 1 ? 1 : (threads > 64 ? 64 : threads);
    if ((int64_t)T > n) T = (int)n;
    for (t = 0; t < T; ++t) {
        jobs[t].xy = xy;
        jobs[t].lo = n * t / T;
        jobs[t].hi = n * (t + 1) / T;
        jobs[t].c = c;
        jobs[t].s = s;
        jobs[t].nang = nang;
    }
    if (T == 1) {
        extremes_range(&jobs[0]);
    } else {
        for (t = 0; t < T; ++t) pthread_create(&tid[t], NULL, extremes_thread, &jobs[t]);
        for (t = 0; t < T; ++t) pthread_join(tid[t], NULL);
    }
    for (k = 0; k < 4 * nang; ++k) {
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
/* Step 2 / final hull: Andrew's monotone chain.    */

typedef struct { float x, y; int64_t id; } chain_pt;

static int chain_cmp(const void* pa, const void* pb) {
    const chain_pt* a = (const chain_pt*)pa;
    const chain_pt* b = (const chain_pt*)pb;
    if (a->x < b->x) return -1;
    if (a->x > b->x) return 1;
    if (a->y < b->y) return -1;
    if (a->y > b->y) return 1;
    return (a->id < b->id) ? -1 : (a->id > b->id);
}

static int turn(const chain_pt* a, const chain_pt* b, const chain_pt* c) {
    return oracle_orient(a->x, a->y, b->x, b->y, c->x, c->y);
}

/* Hull of the points xy[ids[j]] (ids == NULL: identity 0..m-1).
 * ring_out (capacity m) receives the vertex ids of the canonical ring: CCW,
 * starting at the lexicographically smallest (x, y) vertex, collinear points
 * excluded, duplicate coordinates represented by their lowest id (S:214,
 * S:221, A17).  Returns the ring length (0 for m == 0; 1 or 2 = degenerate
 * point / segment).  -1 on allocation failure.                              */
int64_t oracle_hull(const float* xy, const int64_t* ids, int64_t m, int64_t* ring_out) {
    chain_pt* P;
    chain_pt* H;
    int64_t j, u, k = 0, lower_len;
    if (m <= 0) return 0;
    P = (chain_pt*)malloc(sizeof(chain_pt) * (size_t)m);
    H = (chain_pt*)malloc(sizeof(chain_pt) * (size_t)(2 * m + 1));
    if (!P || !H) { free(P); free(H); return -1; }
    for (j = 0; j < m; ++j) {
        int64_t id = ids ? ids[j] : j;
        P[j].x = xy[2 * id];
        P[j].y = xy[2 * id + 1];
        P[j].id = id;
    }
    qsort(P, (size_t)m, sizeof(chain_pt), chain_cmp);
    /* drop duplicate coordinates; the first of each run has the lowest id */
    u = 1;
    for (j = 1; j < m; ++j)
        if (P[j].x != P[u - 1].x || P[j].y != P[u - 1].y) P[u++] = P[j];
    if (u == 1) {
        ring_out[0] = P[0].id;
        free(P); free(H);
        return 1;
    }
    /* lower chain */
    for (j = 0; j < u; ++j) {
        while (k >= 2 && turn(&H[k - 2], &H[k - 1], &P[j]) <= 0) --k;
        H[k++] = P[j];
    }
    lower_len = k;
    /* upper chain */
    for (j = u - 2; j >= 0; --j) {
        while (k > lower_len && turn(&H[k - 2], &H[k - 1], &P[j]) <= 0) --k;
        H[k++] = P[j];
    }
    --k; /* last point repeats the first */
    for (j = 0; j < k; ++j) ring_out[j] = H[j].id;
    free(P); free(H);
    return k;
}

/* ------------------------------------------------------------------------ */
/* Step 3: discard interior points.           */

/* 1 if p is strictly inside the CCW ring (every edge orientation > 0). */
int oracle_strictly_inside(const float* ring_xy, int64_t nv, float px, float py) {
    int64_t j;
    if (nv < 3) return 0; /* degenerate polygon: nothing is inside */
    for (j = 0; j < nv; ++j) {
        int64_t j1 = (j + 1 == nv) ? 0 : j + 1;
        if (oracle_orient(ring_xy[2 * j], ring_xy[2 * j + 1], ring_xy[2 * j1],
                          ring_xy[2 * j1 + 1], px, py) <= 0)
            return 0;
    }
    return 1;
}

typedef struct {
    const float* xy;
    int64_t lo, hi;
    const float* ring_xy;
    int64_t nv;
    uint8_t* keep;
} filter_job;

static void* filter_thread(void* arg) {
    filter_job* J = (filter_job*)arg;
    int64_t i;
    for (i = J->lo; i < J->hi; ++i)
        J->keep[i] = !oracle_strictly_inside(J->ring_xy, J->nv, J->xy[2 * i], J->xy[2 * i + 1]);
    return NULL;
}

/* keep[i] = 1 unless point i is strictly inside the polygon ring (ring given
 * as vertex coordinates, CCW).  nv < 3 keeps everything (A13).              */
void oracle_filter_mask(const float* xy, int64_t n, const float* ring_xy, int64_t nv,
                        int threads, uint8_t* keep) {
    filter_job jobs[64];
    pthread_t tid[64];
    int t, T = threads < 1 ? 1 : (threads > 64 ? 64 : threads);
    if (n <= 0) return;
    if ((int64_t)T > n) T = (int)n;
    for (t = 0; t < T; ++t) {
        jobs[t].xy = xy;
        jobs[t].lo = n * t / T;
        jobs[t].hi = n * (t + 1) / T;
        jobs[t].ring_xy = ring_xy;
        jobs[t].nv = nv;
        jobs[t].keep = keep;
    }
    if (T == 1) {
        filter_thread(&jobs[0]);
    } else {
        for (t = 0; t < T; ++t) pthread_create(&tid[t], NULL, filter_thread, &jobs[t]);
        for (t = 0; t < T; ++t) pthread_join(tid[t], NULL);
    }
}

/* ------------------------------------------------------------------------ */
/* The whole method, Steps 1-3 in the paper's order.              */

/* Outputs:
 *   ext_idx[4*nang]      Step 1 picks (slot order 4k+{minX,maxX,minY,maxY})
 *   ring_idx[<=4*nang]   Step 2 polygon ring (vertex ids, canonical CCW)
 *   *nv                  ring length; < 3 means degenerate (no filtering)
 *   keep[n]              Step 3 mask (1 = survivor)
 * Returns 0, or -1 for empty input / bad arguments.                         */
int oracle_cudapre(const float* xy, int64_t n, const double* c, const double* s, int nang,
                   int threads, int64_t* ext_idx, int64_t* ring_idx, int64_t* nv,
                   uint8_t* keep) {
    int64_t cand[ORACLE_MAX_SLOTS];
    float ring_xy[2 * ORACLE_MAX_SLOTS];
    int64_t k, ncand = 0, m;
    if (oracle_extremes(xy, n, c, s, nang, threads, ext_idx, NULL) != 0) return -1;
    /* candidates: the picks (duplicates collapse inside the chain, A9) */
    for (k = 0; k < 4 * nang; ++k) cand[ncand++] = ext_idx[k];
    m = oracle_hull(xy, cand, ncand, ring_idx);
    if (m < 0) return -1;
    *nv = m;
    for (k = 0; k < m; ++k) {
        ring_xy[2 * k] = xy[2 * ring_idx[k]];
        ring_xy[2 * k + 1] = xy[2 * ring_idx[k] + 1];
    }
    oracle_filter_mask(xy, n, ring_xy, m, threads, keep);
    return 0;
}
