/* TEST INFRASTRUCTURE ONLY -- CPU oracle for the quantized SFC 3x3 path.
 * See sfc_oracle.h for the contract.  Line references are to /root/reference.
 *
 * Parity status: pinned.  tests/test_oracle.py checks this restatement
 * bitwise against the compiled reference (oracle/_ref) on seeded inputs and
 * against the committed fixtures in tests/golden/ (generated from the
 * reference by tests/golden/make_golden.py).
 */
#define _GNU_SOURCE
#include "sfc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];
const char* sfo_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* The three 3x3 SFC specs of the reference catalog (catalog.cpp:246-248,    */
/* derived by derive_correction_spec, catalog.cpp:132-215).  Entries are the */
/* integer numerators; every denominator is 1.  Pinned against the reference */
/* export in tests/golden/catalog_3x3.json.                                  */
/* ------------------------------------------------------------------------ */
/* buffer bounds over every catalogued SFC size */
#define SFO_KMAX 14
#define SFO_NMAX 10
#define SFO_MMAX 7
#define SFO_RMAX 7
#define SFO_FMAX (SFO_KMAX * SFO_KMAX)

typedef struct {
    const char* name;
    int K, n, M, R, N, offset, a_denom, ncorr, triples;
    const signed char* bt; /* K x n */
    const signed char* g;  /* K x R */
    const signed char* a;  /* K x M */
} spec_t;

/* Core channel rows for N=6 over the 6-sample window (DC, a1, b1, a1+b1, a2, b2,
 * a2+b2, Nyquist); the window starts at column `offset` = 1. */
static const signed char BT6x6[10 * 8] = {
    0, 1, 1, 1, 1, 1, 1, 0,    0, 1, 1, 0, -1, -1, 0, 0,  0, 0, -1, -1, 0, 1, 1, 0,
    0, 1, 0, -1, -1, 0, 1, 0,  0, 1, 0, -1, 1, 0, -1, 0,  0, 0, -1, 1, 0, -1, 1, 0,
    0, 1, -1, 0, 1, -1, 0, 0,  0, 1, -1, 1, -1, 1, -1, 0, 1, 0, 0, 0, 0, 0, -1, 0,
    0, -1, 0, 0, 0, 0, 0, 1};
static const signed char G6[12 * 3] = {1, 1, 1,  0, 1, 1,  -1, -1, 0, -1, 0, 1,
                                       -1, 0, 1, 1, -1, 0, 0, -1, 1, 1, -1, 1,
                                       1, 0, 0,  0, 1, 0,  0, 0, 1,   0, 0, 1};
static const signed char G6x6[10 * 3] = {1, 1, 1,  0, 1, 1,  -1, -1, 0, -1, 0, 1, -1, 0, 1,
                                         1, -1, 0, 0, -1, 1, 1, -1, 1,  1, 0, 0,  0, 0, 1};
static const signed char A6x6[10 * 6] = {
    1, 1, 1, 1, 1, 1,    2, 1, -1, -2, -1, 1,  -1, 1, 2, 1, -1, -2, -1, -2, -1, 1, 2, 1,
    1, -2, 1, 1, -2, 1,  1, 1, -2, 1, 1, -2,   -2, 1, 1, -2, 1, 1,  -1, 1, -1, 1, -1, 1,
    6, 0, 0, 0, 0, 0,    0, 0, 0, 0, 0, 6};
static const signed char BT7x7[12 * 9] = {
    0, 1, 1, 1, 1, 1, 1, 0, 0,    0, 1, 1, 0, -1, -1, 0, 0, 0,  0, 0, -1, -1, 0, 1, 1, 0, 0,
    0, 1, 0, -1, -1, 0, 1, 0, 0,  0, 1, 0, -1, 1, 0, -1, 0, 0,  0, 0, -1, 1, 0, -1, 1, 0, 0,
    0, 1, -1, 0, 1, -1, 0, 0, 0,  0, 1, -1, 1, -1, 1, -1, 0, 0, 1, 0, 0, 0, 0, 0, -1, 0, 0,
    0, -1, 0, 0, 0, 0, 0, 1, 0,   0, -1, 0, 0, 0, 0, 0, 1, 0,   0, 0, -1, 0, 0, 0, 0, 0, 1};
static const signed char A7x7[12 * 7] = {
    1, 1, 1, 1, 1, 1, 1,     2, 1, -1, -2, -1, 1, 2,  -1, 1, 2, 1, -1, -2, -1,
    -1, -2, -1, 1, 2, 1, -1, 1, -2, 1, 1, -2, 1, 1,   1, 1, -2, 1, 1, -2, 1,
    -2, 1, 1, -2, 1, 1, -2,  -1, 1, -1, 1, -1, 1, -1, 6, 0, 0, 0, 0, 0, 0,
    0, 0, 0, 0, 0, 0, 6,     0, 0, 0, 0, 0, 6, 0,     0, 0, 0, 0, 0, 0, 6};
static const signed char BT4x4[7 * 6] = {0, 1, 1, 1, 1, 0,   0, -1, 1, -1, 1, 0, 0, 1, -1, -1, 1, 0,
                                         0, 0, -1, 0, 1, 0,  0, 1, 0, -1, 0, 0,  1, 0, 0, 0, -1, 0,
                                         0, -1, 0, 0, 0, 1};
static const signed char G4x4[7 * 3] = {1, 1, 1, 1, -1, 1, 1, -1, -1, 1, 0, -1,
                                        0, -1, 0, 1, 0, 0, 0, 0, 1};
static const signed char A4x4[7 * 4] = {1, 1, 1, 1,   1, -1, 1, -1, 0, 2, 0, -2, 2, -2, -2, 2,
                                        -2, -2, 2, 2, 4, 0, 0, 0,   0, 0, 0, 4};

/* The 5x5 / 7x7 SFC specs (catalog.cpp:249-250), dumped from the compiled reference
 * (oracle/_ref: derive_correction_spec(6, 6, 5) and (6, 4, 7)) and pinned against it in
 * tests/test_oracle.py. */
static const signed char BT6x6r5[140] = {
    0, 0, 1, 1, 1, 1, 1, 1, 0, 0,
    0, 0, 1, 1, 0, -1, -1, 0, 0, 0,
    0, 0, 0, -1, -1, 0, 1, 1, 0, 0,
    0, 0, 1, 0, -1, -1, 0, 1, 0, 0,
    0, 0, 1, 0, -1, 1, 0, -1, 0, 0,
    0, 0, 0, -1, 1, 0, -1, 1, 0, 0,
    0, 0, 1, -1, 0, 1, -1, 0, 0, 0,
    0, 0, 1, -1, 1, -1, 1, -1, 0, 0,
    1, 0, 0, 0, 0, 0, -1, 0, 0, 0,
    0, 1, 0, 0, 0, 0, 0, -1, 0, 0,
    0, 1, 0, 0, 0, 0, 0, -1, 0, 0,
    0, 0, -1, 0, 0, 0, 0, 0, 1, 0,
    0, 0, -1, 0, 0, 0, 0, 0, 1, 0,
    0, 0, 0, -1, 0, 0, 0, 0, 0, 1};
static const signed char G6x6r5[70] = {
    1, 1, 1, 1, 1,
    0, 1, 1, 0, -1,
    -1, -1, 0, 1, 1,
    -1, 0, 1, 1, 0,
    -1, 0, 1, -1, 0,
    1, -1, 0, 1, -1,
    0, -1, 1, 0, -1,
    1, -1, 1, -1, 1,
    1, 0, 0, 0, 0,
    1, 0, 0, 0, 0,
    0, 1, 0, 0, 0,
    0, 0, 0, 1, 0,
    0, 0, 0, 0, 1,
    0, 0, 0, 0, 1};
static const signed char A6x6r5[84] = {
    1, 1, 1, 1, 1, 1,
    1, 2, 1, -1, -2, -1,
    -2, -1, 1, 2, 1, -1,
    1, -1, -2, -1, 1, 2,
    1, 1, -2, 1, 1, -2,
    -2, 1, 1, -2, 1, 1,
    1, -2, 1, 1, -2, 1,
    1, -1, 1, -1, 1, -1,
    6, 0, 0, 0, 0, 0,
    0, 6, 0, 0, 0, 0,
    6, 0, 0, 0, 0, 0,
    0, 0, 0, 0, 0, 6,
    0, 0, 0, 0, 6, 0,
    0, 0, 0, 0, 0, 6};
static const signed char BT4x4r7[140] = {
    0, 0, 1, 1, 1, 1, 1, 1, 0, 0,
    0, 0, 1, 1, 0, -1, -1, 0, 0, 0,
    0, 0, 0, -1, -1, 0, 1, 1, 0, 0,
    0, 0, 1, 0, -1, -1, 0, 1, 0, 0,
    0, 0, 1, 0, -1, 1, 0, -1, 0, 0,
    0, 0, 0, -1, 1, 0, -1, 1, 0, 0,
    0, 0, 1, -1, 0, 1, -1, 0, 0, 0,
    0, 0, 1, -1, 1, -1, 1, -1, 0, 0,
    1, 0, 0, 0, 0, 0, -1, 0, 0, 0,
    0, 1, 0, 0, 0, 0, 0, -1, 0, 0,
    0, 1, 0, 0, 0, 0, 0, -1, 0, 0,
    0, 0, -1, 0, 0, 0, 0, 0, 1, 0,
    0, 0, -1, 0, 0, 0, 0, 0, 1, 0,
    0, 0, 0, -1, 0, 0, 0, 0, 0, 1};
static const signed char G4x4r7[98] = {
    1, 1, 1, 1, 1, 1, 1,
    0, 1, 1, 0, -1, -1, 0,
    -1, -1, 0, 1, 1, 0, -1,
    -1, 0, 1, 1, 0, -1, -1,
    -1, 0, 1, -1, 0, 1, -1,
    1, -1, 0, 1, -1, 0, 1,
    0, -1, 1, 0, -1, 1, 0,
    1, -1, 1, -1, 1, -1, 1,
    1, 0, 0, 0, 0, 0, 0,
    1, 0, 0, 0, 0, 0, 0,
    0, 1, 0, 0, 0, 0, 0,
    0, 0, 0, 0, 0, 1, 0,
    0, 0, 0, 0, 0, 0, 1,
    0, 0, 0, 0, 0, 0, 1};
static const signed char A4x4r7[56] = {
    1, 1, 1, 1,
    1, 2, 1, -1,
    -2, -1, 1, 2,
    1, -1, -2, -1,
    1, 1, -2, 1,
    -2, 1, 1, -2,
    1, -2, 1, 1,
    1, -1, 1, -1,
    6, 0, 0, 0,
    0, 6, 0, 0,
    6, 0, 0, 0,
    0, 0, 0, 6,
    0, 0, 6, 0,
    0, 0, 0, 6};

static const spec_t SPECS[5] = {
    {"sfc4-4x4-3x3", 7, 6, 4, 3, 4, 1, 4, 2, 1, BT4x4, G4x4, A4x4},
    {"sfc6-6x6-3x3", 10, 8, 6, 3, 6, 1, 6, 2, 2, BT6x6, G6x6, A6x6},
    {"sfc6-7x7-3x3", 12, 9, 7, 3, 6, 1, 6, 4, 2, BT7x7, G6, A7x7},
    {"sfc6-6x6-5x5", 14, 10, 6, 5, 6, 2, 6, 6, 2, BT6x6r5, G6x6r5, A6x6r5},
    {"sfc6-4x4-7x7", 14, 10, 4, 7, 6, 2, 6, 6, 2, BT4x4r7, G4x4r7, A4x4r7},
};

static const spec_t* find_spec(const char* name) {
    for (int i = 0; i < 5; ++i)
        if (strcmp(SPECS[i].name, name) == 0) return &SPECS[i];
    snprintf(g_err, sizeof g_err, "unknown algorithm: %s", name);
    return NULL;
}

int sfo_spec(const char* name, int64_t* dims, int64_t* bt, int64_t* g, int64_t* a) {
    const spec_t* s = find_spec(name);
    if (!s) return -1;
    dims[0] = s->K; dims[1] = s->n; dims[2] = s->M; dims[3] = s->R; dims[4] = s->N;
    dims[5] = s->offset; dims[6] = s->a_denom; dims[7] = s->ncorr;
    dims[8] = (int64_t)s->K * s->K;
    dims[9] = dims[8] - 3 * (int64_t)s->triples * s->triples; /* spec.hpp:54-57 */
    if (bt) for (int i = 0; i < s->K * s->n; ++i) bt[i] = s->bt[i];
    if (g) for (int i = 0; i < s->K * s->R; ++i) g[i] = s->g[i];
    if (a) for (int i = 0; i < s->K * s->M; ++i) a[i] = s->a[i];
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Scalar quantization helpers (quant.cpp:13-30, 102-134).                   */
/* ------------------------------------------------------------------------ */
static const double kScaleFloor = 1e-8;

int64_t sfo_quantize_value(double v, double scale, int bits, int64_t* saturated) {
    const int64_t qmax = ((int64_t)1 << (bits - 1)) - 1;
    const int64_t qmin = -((int64_t)1 << (bits - 1));
    double q = nearbyint(v / scale);
    int64_t qi = (int64_t)q;
    if (qi > qmax) {
        qi = qmax;
        if (saturated) ++*saturated;
    } else if (qi < qmin) {
        qi = qmin;
        if (saturated) ++*saturated;
    }
    return qi;
}

static double absmax_of(const double* v, int64_t n) {
    double m = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double a = fabs(v[i]);
        if (a > m) m = a; /* std::max(m, |v|) keeps m on ties; same value */
    }
    return m;
}

double sfo_scale_minmax(const double* v, int64_t n, int bits) {
    const double qmax = (double)(((int64_t)1 << (bits - 1)) - 1);
    double s = absmax_of(v, n) / qmax;
    return s > kScaleFloor ? s : kScaleFloor;
}

static double group_mse(const double* v, int64_t n, double scale, int bits) {
    const double qmax = (double)(((int64_t)1 << (bits - 1)) - 1);
    const double qmin = -(double)((int64_t)1 << (bits - 1));
    double err = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double q = nearbyint(v[i] / scale);
        q = fmin(qmax, fmax(qmin, q));
        const double d = v[i] - q * scale;
        err += d * d;
    }
    return err;
}

double sfo_scale_mse_grid(const double* v, int64_t n, int bits) {
    const double base = sfo_scale_minmax(v, n, bits);
    double best = base, best_err = group_mse(v, n, base, bits);
    for (int i = 0; i < 100; ++i) {
        double s = base * (0.3 + 0.7 * (double)i / 99.0);
        if (s < kScaleFloor) s = kScaleFloor;
        const double err = group_mse(v, n, s, bits);
        if (err < best_err) {
            best_err = err;
            best = s;
        }
    }
    return best;
}

static double pick_scale(const double* v, int64_t n, int bits, int search) {
    return search == SFO_SEARCH_MINMAX ? sfo_scale_minmax(v, n, bits) : sfo_scale_mse_grid(v, n, bits);
}

/* ------------------------------------------------------------------------ */
/* Tile transform (quant.cpp:44-93): V = BT * window * BT^T in fp64, window  */
/* origin (ti*M - pad, tj*M - pad), zero outside the image.                  */
/* ------------------------------------------------------------------------ */
typedef struct {
    const spec_t* s;
    double bt[SFO_KMAX * SFO_NMAX], gm[SFO_KMAX * SFO_RMAX], a[SFO_KMAX * SFO_MMAX]; /* a already divided by a_denom */
    int B, C, H, W, OC, pad, HO, WO, th, tw, K, F;
    const int8_t* x;
    const int8_t* w;
} plan_t;

static void tile_transform(const plan_t* p, int b, int ti, int tj, int c, double* V) {
    const int n = p->s->n, K = p->K, M = p->s->M;
    double window[SFO_NMAX * SFO_NMAX], tmp[SFO_KMAX * SFO_NMAX];
    const int ih0 = ti * M - p->pad, iw0 = tj * M - p->pad;
    for (int r = 0; r < n; ++r) {
        const int ih = ih0 + r;
        for (int s = 0; s < n; ++s) {
            const int iw = iw0 + s;
            window[r * n + s] = (ih >= 0 && ih < p->H && iw >= 0 && iw < p->W)
                                    ? (double)p->x[(((size_t)b * p->C + c) * p->H + ih) * p->W + iw]
                                    : 0.0;
        }
    }
    for (int i = 0; i < K; ++i)
        for (int j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int k = 0; k < n; ++k) acc += p->bt[i * n + k] * window[k * n + j];
            tmp[i * n + j] = acc;
        }
    for (int i = 0; i < K; ++i)
        for (int j = 0; j < K; ++j) {
            double acc = 0.0;
            for (int k = 0; k < n; ++k) acc += tmp[i * n + k] * p->bt[j * n + k];
            V[i * K + j] = acc;
        }
}

/* transform_filters (conv.cpp:352-382) for one (oc, ic). */
static void filter_transform(const plan_t* p, int oc, int ic, double* U) {
    const int R = p->s->R, K = p->K;
    double tmp[SFO_KMAX * SFO_RMAX];
    const int8_t* f = p->w + ((size_t)oc * p->C + ic) * R * R;
    for (int i = 0; i < K; ++i)
        for (int j = 0; j < R; ++j) {
            double acc = 0.0;
            for (int k = 0; k < R; ++k) acc += p->gm[i * R + k] * (double)f[k * R + j];
            tmp[i * R + j] = acc;
        }
    for (int i = 0; i < K; ++i)
        for (int j = 0; j < K; ++j) {
            double acc = 0.0;
            for (int k = 0; k < R; ++k) acc += tmp[i * R + k] * p->gm[j * R + k];
            U[i * K + j] = acc;
        }
}

/* ------------------------------------------------------------------------ */
/* Threaded passes.  Each worker owns a contiguous tile range; all outputs   */
/* are per-tile so the results do not depend on the thread count.           */
/* ------------------------------------------------------------------------ */
typedef struct {
    const plan_t* p;
    const sfo_config* cfg;
    int64_t t0, t1;
    /* pass 1 */
    double* absmax; /* [F] per-frequency absmax of V */
    /* pass 2 */
    const double* act_scale;
    const double* fil_scale;
    const int64_t* uq64; /* [OC][C][F] */
    double* out;
    int64_t* y_int;
    int64_t* pacc_out;
    int32_t* vq_out;
    int64_t saturations;
} work_t;

static void* pass_absmax(void* arg) {
    work_t* wk = (work_t*)arg;
    const plan_t* p = wk->p;
    double V[SFO_FMAX];
    for (int64_t t = wk->t0; t < wk->t1; ++t) {
        const int b = (int)(t / ((int64_t)p->th * p->tw));
        const int rem = (int)(t % ((int64_t)p->th * p->tw));
        const int ti = rem / p->tw, tj = rem % p->tw;
        for (int c = 0; c < p->C; ++c) {
            tile_transform(p, b, ti, tj, c, V);
            for (int f = 0; f < p->F; ++f) {
                const double a = fabs(V[f]);
                if (a > wk->absmax[f]) wk->absmax[f] = a;
            }
        }
    }
    return NULL;
}

static void* pass_main(void* arg) {
    work_t* wk = (work_t*)arg;
    const plan_t* p = wk->p;
    const sfo_config* cfg = wk->cfg;
    const int K = p->K, F = p->F, M = p->s->M, C = p->C;
    const int per_tensor = cfg->act_scope == SFO_ACT_PER_TENSOR;
    int64_t* vq = (int64_t*)malloc(sizeof(int64_t) * (size_t)C * F);
    int64_t pacc[SFO_FMAX];
    double pd[SFO_FMAX], q[SFO_MMAX * SFO_KMAX], V[SFO_FMAX];
    const signed char* A = p->s->a;
    for (int64_t t = wk->t0; t < wk->t1; ++t) {
        const int b = (int)(t / ((int64_t)p->th * p->tw));
        const int rem = (int)(t % ((int64_t)p->th * p->tw));
        const int ti = rem / p->tw, tj = rem % p->tw;
        for (int c = 0; c < C; ++c) {
            tile_transform(p, b, ti, tj, c, V);
            for (int f = 0; f < F; ++f) {
                const double s = wk->act_scale[per_tensor ? 0 : f];
                vq[(size_t)c * F + f] = sfo_quantize_value(V[f], s, cfg->bits, &wk->saturations);
                if (wk->vq_out) wk->vq_out[((size_t)t * C + c) * F + f] = (int32_t)vq[(size_t)c * F + f];
            }
        }
        for (int oc = 0; oc < p->OC; ++oc) {
            for (int f = 0; f < F; ++f) pacc[f] = 0;
            for (int ic = 0; ic < C; ++ic) {
                const int64_t* uf = wk->uq64 + ((size_t)oc * C + ic) * F;
                const int64_t* vf = vq + (size_t)ic * F;
                for (int f = 0; f < F; ++f) pacc[f] += uf[f] * vf[f];
            }
            if (wk->pacc_out)
                memcpy(wk->pacc_out + ((size_t)t * p->OC + oc) * F, pacc, sizeof(int64_t) * F);
            const int oh0 = ti * M, ow0 = tj * M;
            if (wk->out) {
                for (int f = 0; f < F; ++f) {
                    const double sa = wk->act_scale[per_tensor ? 0 : f];
                    double sf;
                    switch (cfg->filter_scope) {
                        case SFO_FIL_PER_CHANNEL: sf = wk->fil_scale[oc]; break;
                        case SFO_FIL_PER_FREQUENCY: sf = wk->fil_scale[f]; break;
                        default: sf = wk->fil_scale[(size_t)oc * F + f]; break;
                    }
                    pd[f] = (double)pacc[f] * sa * sf;
                }
                for (int tt = 0; tt < M; ++tt)
                    for (int j = 0; j < K; ++j) {
                        double acc = 0.0;
                        for (int k = 0; k < K; ++k) acc += p->a[k * M + tt] * pd[k * K + j];
                        q[tt * K + j] = acc;
                    }
                for (int t1 = 0; t1 < M && oh0 + t1 < p->HO; ++t1)
                    for (int t2 = 0; t2 < M && ow0 + t2 < p->WO; ++t2) {
                        double acc = 0.0;
                        for (int k = 0; k < K; ++k) acc += q[t1 * K + k] * p->a[k * M + t2];
                        wk->out[(((size_t)b * p->OC + oc) * p->HO + oh0 + t1) * p->WO + ow0 + t2] = acc;
                    }
            }
            if (wk->y_int) {
                int64_t Q[7 * 12];
                for (int t1 = 0; t1 < M; ++t1)
                    for (int l = 0; l < K; ++l) {
                        int64_t acc = 0;
                        for (int k = 0; k < K; ++k) acc += (int64_t)A[k * M + t1] * pacc[k * K + l];
                        Q[t1 * K + l] = acc;
                    }
                for (int t1 = 0; t1 < M && oh0 + t1 < p->HO; ++t1)
                    for (int t2 = 0; t2 < M && ow0 + t2 < p->WO; ++t2) {
                        int64_t acc = 0;
                        for (int l = 0; l < K; ++l) acc += Q[t1 * K + l] * (int64_t)A[l * M + t2];
                        wk->y_int[(((size_t)b * p->OC + oc) * p->HO + oh0 + t1) * p->WO + ow0 + t2] = acc;
                    }
            }
        }
    }
    free(vq);
    return NULL;
}

static int run_threads(void* (*fn)(void*), work_t* wk, int nthreads) {
    if (nthreads <= 1) {
        fn(&wk[0]);
        return 0;
    }
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, fn, &wk[i]);
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
    free(th);
    return 0;
}

/* Gather every V in the reference's [B][th][tw][C][K][K] order (MseGrid only,
 * where the summation order of quant_group_mse matters). */
static double* gather_all(const plan_t* p) {
    const int64_t T = (int64_t)p->B * p->th * p->tw;
    double* g = (double*)malloc(sizeof(double) * (size_t)T * p->C * p->F);
    if (!g) return NULL;
    for (int64_t t = 0; t < T; ++t) {
        const int b = (int)(t / ((int64_t)p->th * p->tw));
        const int rem = (int)(t % ((int64_t)p->th * p->tw));
        for (int c = 0; c < p->C; ++c)
            tile_transform(p, b, rem / p->tw, rem % p->tw, c, g + ((size_t)t * p->C + c) * p->F);
    }
    return g;
}

int sfo_direct_conv(const int8_t* x, int B, int C, int H, int W, const int8_t* w, int OC, int R,
                    int pad, int threads, double* out) {
    (void)threads;
    const int HO = H + 2 * pad - R + 1, WO = W + 2 * pad - R + 1;
    for (int b = 0; b < B; ++b)
        for (int oc = 0; oc < OC; ++oc)
            for (int oh = 0; oh < HO; ++oh)
                for (int ow = 0; ow < WO; ++ow) {
                    double acc = 0.0;
                    for (int ic = 0; ic < C; ++ic)
                        for (int fr = 0; fr < R; ++fr) {
                            const int ih = oh - pad + fr;
                            if (ih < 0 || ih >= H) continue;
                            for (int fc = 0; fc < R; ++fc) {
                                const int iw = ow - pad + fc;
                                if (iw < 0 || iw >= W) continue;
                                acc += (double)x[(((size_t)b * C + ic) * H + ih) * W + iw] *
                                       (double)w[(((size_t)oc * C + ic) * R + fr) * R + fc];
                            }
                        }
                    out[(((size_t)b * OC + oc) * HO + oh) * WO + ow] = acc;
                }
    return 0;
}

int sfo_quantized_conv(const int8_t* x, int B, int C, int H, int W, const int8_t* w, int OC,
                       const char* spec, int pad, const sfo_config* cfg, double* out,
                       int64_t* y_int, int64_t* pacc, int32_t* vq, int32_t* uq,
                       double* act_scale_out, double* fil_scale_out, sfo_report* rep) {
    if (cfg->bits < 2 || cfg->bits > 16) {
        snprintf(g_err, sizeof g_err, "quantization width must be between 2 and 16 bits");
        return -1;
    }
    const spec_t* s = find_spec(spec);
    if (!s) return -1;
    plan_t p;
    memset(&p, 0, sizeof p);
    p.s = s;
    p.K = s->K;
    p.F = s->K * s->K;
    p.B = B; p.C = C; p.H = H; p.W = W; p.OC = OC; p.pad = pad;
    p.HO = H + 2 * pad - s->R + 1;
    p.WO = W + 2 * pad - s->R + 1;
    if (p.HO <= 0 || p.WO <= 0) {
        snprintf(g_err, sizeof g_err, "filter larger than padded input");
        return -1;
    }
    p.th = (p.HO + s->M - 1) / s->M;
    p.tw = (p.WO + s->M - 1) / s->M;
    p.x = x;
    p.w = w;
    for (int i = 0; i < s->K * s->n; ++i) p.bt[i] = (double)s->bt[i];
    for (int i = 0; i < s->K * s->R; ++i) p.gm[i] = (double)s->g[i];
    for (int i = 0; i < s->K * s->M; ++i) p.a[i] = (double)s->a[i] / (double)s->a_denom; /* quant.cpp:232-233 */
    const int F = p.F;
    const int64_t T = (int64_t)B * p.th * p.tw;
    int nthreads = cfg->threads < 1 ? 1 : cfg->threads;
    if (nthreads > T) nthreads = (int)(T > 0 ? T : 1);
    int64_t saturations = 0;

    /* --- activation scales (quant.cpp:168-181) --- */
    double act_scale[SFO_FMAX];
    const int n_act = cfg->act_scope == SFO_ACT_PER_TENSOR ? 1 : F;
    double* gall = NULL;
    int64_t vmax = 0;
    if (cfg->search == SFO_SEARCH_MINMAX) {
        work_t* wk = (work_t*)calloc((size_t)nthreads, sizeof(work_t));
        double* am = (double*)calloc((size_t)nthreads * F, sizeof(double));
        for (int i = 0; i < nthreads; ++i) {
            wk[i].p = &p;
            wk[i].t0 = T * i / nthreads;
            wk[i].t1 = T * (i + 1) / nthreads;
            wk[i].absmax = am + (size_t)i * F;
        }
        run_threads(pass_absmax, wk, nthreads);
        double fmaxv[SFO_FMAX];
        for (int f = 0; f < F; ++f) {
            fmaxv[f] = 0.0;
            for (int i = 0; i < nthreads; ++i)
                if (am[(size_t)i * F + f] > fmaxv[f]) fmaxv[f] = am[(size_t)i * F + f];
        }
        const double qmax = (double)(((int64_t)1 << (cfg->bits - 1)) - 1);
        double all = 0.0;
        for (int f = 0; f < F; ++f) all = fmaxv[f] > all ? fmaxv[f] : all;
        vmax = (int64_t)all;
        if (cfg->vmax_override >= 0) all = (double)cfg->vmax_override;
        if (n_act == 1) {
            double sc = all / qmax;
            act_scale[0] = sc > kScaleFloor ? sc : kScaleFloor;
        } else {
            for (int f = 0; f < F; ++f) {
                double sc = fmaxv[f] / qmax;
                act_scale[f] = sc > kScaleFloor ? sc : kScaleFloor;
            }
        }
        free(am);
        free(wk);
    } else {
        gall = gather_all(&p);
        if (!gall) {
            snprintf(g_err, sizeof g_err, "out of host memory");
            return -1;
        }
        const int64_t nv = T * C * F;
        vmax = (int64_t)absmax_of(gall, nv);
        if (n_act == 1) {
            act_scale[0] = pick_scale(gall, nv, cfg->bits, cfg->search);
        } else {
            const int64_t groups = nv / F;
            double* vals = (double*)malloc(sizeof(double) * (size_t)groups);
            for (int f = 0; f < F; ++f) {
                for (int64_t g = 0; g < groups; ++g) vals[g] = gall[g * F + f];
                act_scale[f] = pick_scale(vals, groups, cfg->bits, cfg->search);
            }
            free(vals);
        }
        free(gall);
    }

    if (cfg->act_scale_override)
        for (int i = 0; i < n_act; ++i) act_scale[i] = cfg->act_scale_override[i];

    /* --- filter transform, scales and quantization (quant.cpp:183-229) --- */
    double* u = (double*)malloc(sizeof(double) * (size_t)OC * C * F);
    for (int oc = 0; oc < OC; ++oc)
        for (int ic = 0; ic < C; ++ic) filter_transform(&p, oc, ic, u + ((size_t)oc * C + ic) * F);
    int n_fil;
    double* fil_scale;
    if (cfg->filter_scope == SFO_FIL_PER_CHANNEL) {
        n_fil = OC;
        fil_scale = (double*)malloc(sizeof(double) * (size_t)n_fil);
        for (int oc = 0; oc < OC; ++oc)
            fil_scale[oc] = pick_scale(u + (size_t)oc * C * F, (int64_t)C * F, cfg->bits, cfg->search);
    } else if (cfg->filter_scope == SFO_FIL_PER_FREQUENCY) {
        n_fil = F;
        fil_scale = (double*)malloc(sizeof(double) * (size_t)n_fil);
        double* vals = (double*)malloc(sizeof(double) * (size_t)OC * C);
        for (int f = 0; f < F; ++f) {
            for (int oc = 0; oc < OC; ++oc)
                for (int ic = 0; ic < C; ++ic) vals[(size_t)oc * C + ic] = u[((size_t)oc * C + ic) * F + f];
            fil_scale[f] = pick_scale(vals, (int64_t)OC * C, cfg->bits, cfg->search);
        }
        free(vals);
    } else {
        n_fil = OC * F;
        fil_scale = (double*)malloc(sizeof(double) * (size_t)n_fil);
        double* vals = (double*)malloc(sizeof(double) * (size_t)C);
        for (int oc = 0; oc < OC; ++oc)
            for (int f = 0; f < F; ++f) {
                for (int ic = 0; ic < C; ++ic) vals[ic] = u[((size_t)oc * C + ic) * F + f];
                fil_scale[(size_t)oc * F + f] = pick_scale(vals, C, cfg->bits, cfg->search);
            }
        free(vals);
    }
    int64_t* uq64 = (int64_t*)malloc(sizeof(int64_t) * (size_t)OC * C * F);
    for (int oc = 0; oc < OC; ++oc)
        for (int ic = 0; ic < C; ++ic)
            for (int f = 0; f < F; ++f) {
                double sf;
                switch (cfg->filter_scope) {
                    case SFO_FIL_PER_CHANNEL: sf = fil_scale[oc]; break;
                    case SFO_FIL_PER_FREQUENCY: sf = fil_scale[f]; break;
                    default: sf = fil_scale[(size_t)oc * F + f]; break;
                }
                const size_t idx = ((size_t)oc * C + ic) * F + f;
                uq64[idx] = sfo_quantize_value(u[idx], sf, cfg->bits, &saturations);
                if (uq) uq[idx] = (int32_t)uq64[idx];
            }
    free(u);

    /* --- main loop (quant.cpp:239-279) --- */
    work_t* wk = (work_t*)calloc((size_t)nthreads, sizeof(work_t));
    for (int i = 0; i < nthreads; ++i) {
        wk[i].p = &p;
        wk[i].cfg = cfg;
        wk[i].t0 = T * i / nthreads;
        wk[i].t1 = T * (i + 1) / nthreads;
        wk[i].act_scale = act_scale;
        wk[i].fil_scale = fil_scale;
        wk[i].uq64 = uq64;
        wk[i].out = out;
        wk[i].y_int = y_int;
        wk[i].pacc_out = pacc;
        wk[i].vq_out = vq;
    }
    /* Nothing requested from the tile loop: the call only wanted scales / vmax. */
    if (out || y_int || pacc || vq) run_threads(pass_main, wk, nthreads);
    for (int i = 0; i < nthreads; ++i) saturations += wk[i].saturations;
    free(wk);

    if (act_scale_out) memcpy(act_scale_out, act_scale, sizeof(double) * (size_t)n_act);
    if (fil_scale_out) memcpy(fil_scale_out, fil_scale, sizeof(double) * (size_t)n_fil);
    if (rep) {
        memset(rep, 0, sizeof *rep);
        rep->saturations = saturations;
        rep->values_quantized = (int64_t)OC * C * F + T * C * F;
        rep->vmax = vmax;
        rep->tiles = T;
        rep->th = p.th;
        rep->tw = p.tw;
        rep->HO = p.HO;
        rep->WO = p.WO;
        if (cfg->want_report && out) {
            /* quant.cpp:282-291: error against the fp64 direct conv, summed in order. */
            const size_t n = (size_t)B * OC * p.HO * p.WO;
            double* ref = (double*)malloc(sizeof(double) * n);
            sfo_direct_conv(x, B, C, H, W, w, OC, s->R, pad, 1, ref);
            double err = 0.0, sig = 0.0;
            for (size_t i = 0; i < n; ++i) {
                const double d = out[i] - ref[i];
                err += d * d;
                sig += ref[i] * ref[i];
            }
            rep->mse = err / (double)n;
            rep->signal_energy = sig / (double)n;
            rep->snr_db = 10.0 * log10(sig / (err > 1e-300 ? err : 1e-300));
            free(ref);
        }
    }
    free(fil_scale);
    free(uq64);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Exact single-tile execution (catalog.cpp:324-381) and the exhaustive     */
/* per-axis identity that makes every 2-D tile exact.                        */
/* ------------------------------------------------------------------------ */
int sfo_execute_tile(const char* spec, const int64_t* x, const int64_t* f, int64_t* y) {
    const spec_t* s = find_spec(spec);
    if (!s) return -1;
    const int K = s->K, n = s->n, R = s->R, M = s->M;
    int64_t tmp[SFO_KMAX * SFO_NMAX], V[SFO_FMAX], tf[SFO_KMAX * SFO_RMAX], U[SFO_FMAX], ta[SFO_MMAX * SFO_KMAX];
    for (int i = 0; i < K; ++i)
        for (int j = 0; j < n; ++j) {
            int64_t acc = 0;
            for (int t = 0; t < n; ++t) acc += s->bt[i * n + t] * x[t * n + j];
            tmp[i * n + j] = acc;
        }
    for (int i = 0; i < K; ++i)
        for (int j = 0; j < K; ++j) {
            int64_t acc = 0;
            for (int t = 0; t < n; ++t) acc += tmp[i * n + t] * s->bt[j * n + t];
            V[i * K + j] = acc;
        }
    for (int i = 0; i < K; ++i)
        for (int j = 0; j < R; ++j) {
            int64_t acc = 0;
            for (int t = 0; t < R; ++t) acc += s->g[i * R + t] * f[t * R + j];
            tf[i * R + j] = acc;
        }
    for (int i = 0; i < K; ++i)
        for (int j = 0; j < K; ++j) {
            int64_t acc = 0;
            for (int t = 0; t < R; ++t) acc += tf[i * R + t] * s->g[j * R + t];
            U[i * K + j] = acc;
        }
    for (int i = 0; i < K * K; ++i) V[i] *= U[i];
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < K; ++j) {
            int64_t acc = 0;
            for (int t = 0; t < K; ++t) acc += s->a[t * M + i] * V[t * K + j];
            ta[i * K + j] = acc;
        }
    const int64_t d2 = (int64_t)s->a_denom * s->a_denom;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < M; ++j) {
            int64_t acc = 0;
            for (int t = 0; t < K; ++t) acc += ta[i * K + t] * s->a[t * M + j];
            if (acc % d2 != 0) {
                snprintf(g_err, sizeof g_err, "%s: output not divisible by denominator fold", s->name);
                return -2;
            }
            y[i * M + j] = acc / d2;
        }
    return 0;
}

int sfo_check_identity(const char* spec) {
    const spec_t* s = find_spec(spec);
    if (!s) return -1;
    int bad = 0;
    for (int t = 0; t < s->M; ++t)
        for (int i = 0; i < s->n; ++i)
            for (int j = 0; j < s->R; ++j) {
                int64_t acc = 0;
                for (int k = 0; k < s->K; ++k)
                    acc += (int64_t)s->a[k * s->M + t] * s->bt[k * s->n + i] * s->g[k * s->R + j];
                if (acc != (i == t + j ? s->a_denom : 0)) ++bad;
            }
    return bad;
}
