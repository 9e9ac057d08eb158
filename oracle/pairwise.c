/*
 * ORACLE / TEST INFRASTRUCTURE ONLY.  Never linked into the product path.
 *
 * Plain-C restatement of the fixed-order float64 arithmetic the reference
 * hot path is built on:
 *
 *   csvd._linalg.gemv_rows  (/root/reference/pkg/src/csvd/_linalg.py:25-37)
 *       out[r] = (rows[r] * h).sum()   -- f64 products, each rounded, then
 *                numpy's pairwise add-reduce along the row
 *   csvd._linalg.l2_norm    (_linalg.py:40-43)  sqrt((v*v).sum())
 *
 * numpy's add-reduce over a contiguous axis is  0.0 + pairwise(a, n)  where
 * pairwise is numpy's `pairwise_sum_DOUBLE` (numpy/_core/src/umath/
 * loops_utils.h.src, third-party dependency numpy>=1.24 per
 * pkg/pyproject.toml:11; verified bit-for-bit here against numpy 2.3.5 by
 * tests/test_oracle_pairwise.py for d in {1..16385}).  Restated:
 *
 *   pw(a, n):  n <  8   : res = 0.0; res += a[i] sequentially
 *              n <= 128 : r[j] = a[j] (j<8); r[j] += a[i+j] for i=8,16,..
 *                         < n - n%8; res = ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7));
 *                         then the n%8 tail added sequentially
 *              else     : n2 = n/2; n2 -= n2%8; pw(a,n2) + pw(a+n2, n-n2)
 *
 * Must be compiled with -ffp-contract=off (no FMA contraction) and without
 * -ffast-math; the Makefile does so.  Rows may be float32 (widened exactly,
 * the reference holds f32-exact values in f64: tensor_io.py:156,214-215),
 * bf16 bit patterns (the bf16-weight variant), or float64 (centroids).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

static double pw(const double *a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pw(a, n2) + pw(a + n2, n - n2);
    }
}

/* numpy add-reduce of a contiguous 1-d f64 array */
double oracle_sum(const double *a, int64_t n) { return 0.0 + pw(a, n); }

static inline double bf16_to_f64(uint16_t b) {
    uint32_t u = ((uint32_t)b) << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

/* dtype: 0 = float32, 1 = bf16 bits (uint16), 2 = float64 */
static inline double load_elem(const void *rows, int dtype, int64_t idx) {
    if (dtype == 0) return (double)((const float *)rows)[idx];
    if (dtype == 1) return bf16_to_f64(((const uint16_t *)rows)[idx]);
    return ((const double *)rows)[idx];
}

typedef struct {
    const void *rows; int dtype; int64_t lo, hi, d;
    const int64_t *sel; const double *h; const void *bias; int bias_dtype; double *out;
} gemv_job;

static void *gemv_worker(void *arg) {
    gemv_job *j = (gemv_job *)arg;
    double *prod = (double *)malloc(sizeof(double) * (size_t)(j->d > 0 ? j->d : 1));
    for (int64_t i = j->lo; i < j->hi; i++) {
        int64_t r = j->sel ? j->sel[i] : i;
        int64_t base = r * j->d;
        for (int64_t e = 0; e < j->d; e++) prod[e] = load_elem(j->rows, j->dtype, base + e) * j->h[e];
        double v = 0.0 + pw(prod, j->d);
        if (j->bias) v = v + load_elem(j->bias, j->bias_dtype, r);
        j->out[i] = v;
    }
    free(prod);
    return NULL;
}

/*
 * out[i] = 0.0 + pw(row(sel[i]) * h)   (+ bias[sel[i]] if bias != NULL, as
 * the separately rounded `+ table.bias[members]` of decode.py:171)
 * sel == NULL means rows 0..n-1.  Threads: nthreads (<=0 -> all online CPUs).
 */
void oracle_gemv_rows(const void *rows, int dtype, int64_t n, int64_t d,
                      const int64_t *sel, const double *h,
                      const void *bias, int bias_dtype, double *out, int nthreads) {
    if (nthreads <= 0) nthreads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (nthreads < 1) nthreads = 1;
    if ((int64_t)nthreads > n) nthreads = (int)(n > 0 ? n : 1);
    if (n * d < 65536) nthreads = 1;
    gemv_job jobs[256];
    pthread_t tids[256];
    if (nthreads > 256) nthreads = 256;
    for (int t = 0; t < nthreads; t++) {
        jobs[t] = (gemv_job){rows, dtype, n * t / nthreads, n * (t + 1) / nthreads, d,
                             sel, h, bias, bias_dtype, out};
    }
    for (int t = 1; t < nthreads; t++) pthread_create(&tids[t], NULL, gemv_worker, &jobs[t]);
    gemv_worker(&jobs[0]);
    for (int t = 1; t < nthreads; t++) pthread_join(tids[t], NULL);
}

/* l2_norm(v) = sqrt(0.0 + pw(v*v)) */
double oracle_l2_norm(const double *v, int64_t n) {
    double *prod = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int64_t j = 0; j < n; j++) prod[j] = v[j] * v[j];
    double s = 0.0 + pw(prod, n);
    free(prod);
    return sqrt(s);
}
