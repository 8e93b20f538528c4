/*
 * ktune_oracle.c -- CPU restatement of the reference's hot-path arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * evaluation path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.  The product (libktc.so and the
 * paper_1703_06503_b200 package) never links, imports or executes it.
 *
 * Every function restates one reference routine; the citation is given on
 * each.  Paths are relative to the reference checkout (proj/include/ktune/).
 *
 * Build: see oracle/Makefile.  The file MUST be compiled without -march and
 * with -ffp-contract=off: the reference is built with plain x86-64 flags
 * (proj/CMakeLists.txt:7-9,20), so its `acc += a * b` is a rounded multiply
 * followed by a rounded add.  Contracting into an FMA changes the digests
 * (SURVEY.md 8(c) "Build-flag hazard").
 *
 * Parity pin: tests/test_oracle.py checks this file against the reference's
 * own known-answer tests (test_landscapes.cpp:41-170, test_tuner.cpp:209-297)
 * and against the golden digests in tests/golden/oracle_golden.json, which
 * were produced by the reference headers compiled under oracle/_ref/
 * (tests/golden/make_golden.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* std::mt19937_64 (rng.hpp:12).  The output sequence is fixed by the C++    */
/* standard ([rand.predef]: 10000th output 9981545732273789042).             */
/* ------------------------------------------------------------------------ */
#define MT_N 312
#define MT_M 156

typedef struct {
    uint64_t s[MT_N];
    int i;
} ko_mt64;

void ko_mt64_seed(ko_mt64 *g, uint64_t seed) {
    g->s[0] = seed;
    for (int k = 1; k < MT_N; ++k) {
        uint64_t p = g->s[k - 1];
        g->s[k] = 6364136223846793005ull * (p ^ (p >> 62)) + (uint64_t)k;
    }
    g->i = MT_N;
}

static void mt64_twist(ko_mt64 *g) {
    const uint64_t upper = 0xFFFFFFFF80000000ull, lower = 0x7FFFFFFFull;
    for (int k = 0; k < MT_N; ++k) {
        uint64_t y = (g->s[k] & upper) | (g->s[(k + 1) % MT_N] & lower);
        uint64_t v = g->s[(k + MT_M) % MT_N] ^ (y >> 1);
        if (y & 1u) v ^= 0xB5026F5AA96619E9ull;
        g->s[k] = v;
    }
    g->i = 0;
}

uint64_t ko_mt64_next(ko_mt64 *g) {
    if (g->i >= MT_N) mt64_twist(g);
    uint64_t y = g->s[g->i++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

/* uniform01: 53-bit construction, rng.hpp:17-19 */
double ko_uniform01(ko_mt64 *g) { return (double)(ko_mt64_next(g) >> 11) * 0x1.0p-53; }

/* uniform_index: rejection sampling, rng.hpp:22-32 */
uint64_t ko_uniform_index(ko_mt64 *g, uint64_t n) {
    if (n <= 1) return 0;
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t d = ko_mt64_next(g);
    while (d >= limit) d = ko_mt64_next(g);
    return d % n;
}

/* ------------------------------------------------------------------------ */
/* materialize_argument (arguments.hpp:126-180).  kind: 0 none, 1 constant,  */
/* 2 ramp, 3 uniform.                                                        */
/* ------------------------------------------------------------------------ */
void ko_materialize_f32(int kind, double constant, uint64_t seed, size_t n, float *out) {
    switch (kind) {
    case 1:
        for (size_t i = 0; i < n; ++i) out[i] = (float)constant;
        break;
    case 2:
        for (size_t i = 0; i < n; ++i) out[i] = (float)i;
        break;
    case 3: {
        ko_mt64 g;
        ko_mt64_seed(&g, seed);
        for (size_t i = 0; i < n; ++i) out[i] = (float)ko_uniform01(&g);
        break;
    }
    default:
        memset(out, 0, n * sizeof(float));
    }
}

void ko_materialize_i32(int kind, double constant, uint64_t seed, size_t n, int32_t *out) {
    switch (kind) {
    case 1:
        for (size_t i = 0; i < n; ++i) out[i] = (int32_t)constant;
        break;
    case 2:
        for (size_t i = 0; i < n; ++i) out[i] = (int32_t)i;
        break;
    case 3: {
        ko_mt64 g;
        ko_mt64_seed(&g, seed);
        for (size_t i = 0; i < n; ++i) out[i] = (int32_t)ko_uniform_index(&g, 1000);
        break;
    }
    default:
        memset(out, 0, n * sizeof(int32_t));
    }
}

/* ------------------------------------------------------------------------ */
/* FNV-1a-64 digest over little-endian 4-byte words (arguments.hpp:184-205,  */
/* rng.hpp:35-44).                                                           */
/* ------------------------------------------------------------------------ */
uint64_t ko_digest_words(const void *data, size_t n_words) {
    const unsigned char *b = (const unsigned char *)data;
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < n_words * 4; ++i) { /* x86-64 is little-endian */
        h ^= (uint64_t)b[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

/* ------------------------------------------------------------------------ */
/* Row-parallel driver.  Each worker owns whole output rows, so the per-    */
/* element operation sequence is exactly the reference's (bit-identical).    */
/* ------------------------------------------------------------------------ */
typedef void (*row_fn)(void *ctx, size_t row);

typedef struct {
    row_fn fn;
    void *ctx;
    size_t rows;
    size_t next; /* guarded by lock */
    pthread_mutex_t lock;
} row_pool;

static void *row_worker(void *arg) {
    row_pool *p = (row_pool *)arg;
    for (;;) {
        pthread_mutex_lock(&p->lock);
        size_t r = p->next;
        size_t end = r + 8 < p->rows ? r + 8 : p->rows;
        p->next = end;
        pthread_mutex_unlock(&p->lock);
        if (r >= p->rows) break;
        for (; r < end; ++r) p->fn(p->ctx, r);
    }
    return NULL;
}

static void run_rows(row_fn fn, void *ctx, size_t rows, int threads) {
    if (threads <= 1 || rows < 16) {
        for (size_t r = 0; r < rows; ++r) fn(ctx, r);
        return;
    }
    if (threads > 256) threads = 256;
    row_pool p = {fn, ctx, rows, 0, PTHREAD_MUTEX_INITIALIZER};
    pthread_t tid[256];
    for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, row_worker, &p);
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* ------------------------------------------------------------------------ */
/* conv_apply (landscapes.hpp:120-143):                                      */
/*   out[r*x+c] = w * sum_{j<f} sum_{i<f} taps[j*f+i] * image[(r+j)*W+c+i]    */
/* fp32 accumulator, j outer, i inner, rounded multiply then rounded add.    */
/* ------------------------------------------------------------------------ */
typedef struct {
    const float *image, *taps;
    float *out;
    size_t x;
    int f;
    float w;
} conv_ctx;

static void conv_row(void *vctx, size_t row) {
    const conv_ctx *c = (const conv_ctx *)vctx;
    const size_t width = c->x + (size_t)c->f - 1;
    for (size_t col = 0; col < c->x; ++col) {
        float acc = 0.0f;
        for (int j = 0; j < c->f; ++j) {
            const float *line = c->image + (row + (size_t)j) * width + col;
            const float *tap = c->taps + (size_t)j * (size_t)c->f;
            for (int i = 0; i < c->f; ++i) acc += tap[i] * line[i];
        }
        c->out[row * c->x + col] = c->w * acc;
    }
}

void ko_conv_apply(const float *image, const float *taps, size_t x, size_t y, int f, float w,
                   float *out, int threads) {
    conv_ctx c = {image, taps, out, x, f, w};
    run_rows(conv_row, &c, y, threads);
}

/* ------------------------------------------------------------------------ */
/* gemm_apply (landscapes.hpp:293-312):                                      */
/*   out[r*n+c] = alpha * sum_{kk<k} a[kk*m+r]*b[kk*n+c] + beta * c[r*n+c]   */
/* Restated row-at-a-time (kk outer, c inner) over a row accumulator: each   */
/* element still sees 0, then + a*b in ascending kk, so results are          */
/* bit-identical while the inner loop is contiguous.           */
/* ------------------------------------------------------------------------ */
typedef struct {
    const float *a, *b, *c;
    float *out;
    size_t m, n, k;
    float alpha, beta;
} gemm_ctx;

static void gemm_row(void *vctx, size_t row) {
    const gemm_ctx *g = (const gemm_ctx *)vctx;
    float *acc = (float *)calloc(g->n, sizeof(float));
    for (size_t kk = 0; kk < g->k; ++kk) {
        const float av = g->a[kk * g->m + row];
        const float *brow = g->b + kk * g->n;
        for (size_t col = 0; col < g->n; ++col) acc[col] += av * brow[col];
    }
    for (size_t col = 0; col < g->n; ++col)
        g->out[row * g->n + col] = g->alpha * acc[col] + g->beta * g->c[row * g->n + col];
    free(acc);
}

void ko_gemm_apply(const float *a, const float *b, const float *c, size_t m, size_t n, size_t k,
                   float alpha, float beta, float *out, int threads) {
    gemm_ctx g = {a, b, c, out, m, n, k, alpha, beta};
    run_rows(gemm_row, &g, m, threads);
}

/* ------------------------------------------------------------------------ */
/* verify_outputs (tuner.hpp:39-106) for one buffer; the report continues    */
/* across buffers exactly as the reference's record() lambda does.           */
/* ------------------------------------------------------------------------ */
typedef struct {
    int pass;
    double max_abs_error;
    double max_rel_error;
    size_t buffer_index;
    size_t element_index;
    size_t elements_compared;
} ko_verify_report;

void ko_verify_init(ko_verify_report *r) { memset(r, 0, sizeof(*r)); r->pass = 1; }

static void record(ko_verify_report *rep, size_t buffer, size_t element, double abs_err,
                   double rel_err, int ok) {
    if (!(abs_err <= rep->max_abs_error)) {
        rep->max_abs_error = abs_err;
        if (rep->pass) {
            rep->buffer_index = buffer;
            rep->element_index = element;
        }
    }
    if (!(rel_err <= rep->max_rel_error)) rep->max_rel_error = rel_err;
    if (!ok && rep->pass) {
        rep->pass = 0;
        rep->buffer_index = buffer;
        rep->element_index = element;
    }
    ++rep->elements_compared;
}

void ko_verify_f32(ko_verify_report *rep, size_t buffer, const float *cand, const float *ref,
                   size_t n, double rel_tol, double abs_tol) {
    for (size_t i = 0; i < n; ++i) {
        double abs_err = fabs((double)cand[i] - (double)ref[i]);
        double mag = fabs((double)ref[i]);
        double rel_err = mag > 0.0 ? abs_err / mag : 0.0;
        int ok = abs_err <= abs_tol + rel_tol * mag;
        record(rep, buffer, i, abs_err, rel_err, ok);
    }
}

void ko_verify_i32(ko_verify_report *rep, size_t buffer, const int32_t *cand, const int32_t *ref,
                   size_t n) {
    for (size_t i = 0; i < n; ++i) {
        double abs_err = fabs((double)cand[i] - (double)ref[i]);
        record(rep, buffer, i, abs_err, abs_err, cand[i] == ref[i]);
    }
}
