/* Reference-style specialised ladders: the CPU stand-in for pafft at radix
 * 3 and 5 (and 2/4 for calibration).  TEST / BASELINE INFRASTRUCTURE ONLY --
 * used by bench.py's reference arm (radix 3/5, which pafft's Radix enum cannot
 * express, core.hpp:14-19) and checked against the oracle restatement in
 * tests/test_oracle_pins.py.  Never part of the product path.
 *
 * Same algorithm and memory behaviour as pafft's hand-expanded r2/r4/r8
 * kernels (butterfly.cpp:39-75 loop nest: stages k = n..r descending for
 * A^T with output twiddles, k = r..n ascending for A-bar with conjugated
 * input twiddles; one full sweep per stage; table read at e * (n/k),
 * core.hpp:71-88), with the radix-r combine written out per radix instead of
 * the oracle's generic F_r loop.  tools/port_calibration.py compares the
 * radix-2 instance of this file with pafft's own radix-2 kernel. */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "pafft_oracle.h"

#define S60 0.86602540378443864676 /* sin(pi/3) */

/* radix-r combine, y_m = sum_d w_r^{dm} z_d (conj: conjugated roots) */
static inline void comb2(double* zr, double* zi) {
    const double ar = zr[0] + zr[1], ai = zi[0] + zi[1];
    zr[1] = zr[0] - zr[1];
    zi[1] = zi[0] - zi[1];
    zr[0] = ar;
    zi[0] = ai;
}
static inline void comb3(double* zr, double* zi, double s) {
    const double tr = zr[1] + zr[2], ti = zi[1] + zi[2];
    const double dr = zr[1] - zr[2], di = zi[1] - zi[2];
    const double mr = zr[0] - 0.5 * tr, mi = zi[0] - 0.5 * ti;
    zr[0] += tr;
    zi[0] += ti;
    zr[1] = mr + s * di;
    zi[1] = mi - s * dr;
    zr[2] = mr - s * di;
    zi[2] = mi + s * dr;
}
static inline void comb4(double* zr, double* zi, int cj) {
    const double t0r = zr[0] + zr[2], t0i = zi[0] + zi[2], t1r = zr[0] - zr[2], t1i = zi[0] - zi[2];
    const double t2r = zr[1] + zr[3], t2i = zi[1] + zi[3];
    double t3r = zi[1] - zi[3], t3i = zr[3] - zr[1]; /* -i (z1 - z3) */
    if (cj) { t3r = -t3r; t3i = -t3i; }
    zr[0] = t0r + t2r; zi[0] = t0i + t2i;
    zr[2] = t0r - t2r; zi[2] = t0i - t2i;
    zr[1] = t1r + t3r; zi[1] = t1i + t3i;
    zr[3] = t1r - t3r; zi[3] = t1i - t3i;
}
static const double C51 = 0.30901699437494742410, C52 = -0.80901699437494742410;
static const double S51 = 0.95105651629515357212, S52 = 0.58778525229247312917;
static inline void comb5(double* zr, double* zi, double sg) {
    const double s1 = sg * S51, s2 = sg * S52;
    const double t1r = zr[1] + zr[4], t1i = zi[1] + zi[4], t2r = zr[2] + zr[3], t2i = zi[2] + zi[3];
    const double t3r = zr[1] - zr[4], t3i = zi[1] - zi[4], t4r = zr[2] - zr[3], t4i = zi[2] - zi[3];
    const double m1r = zr[0] + C51 * t1r + C52 * t2r, m1i = zi[0] + C51 * t1i + C52 * t2i;
    const double m2r = zr[0] + C52 * t1r + C51 * t2r, m2i = zi[0] + C52 * t1i + C51 * t2i;
    const double n1r = s1 * t3r + s2 * t4r, n1i = s1 * t3i + s2 * t4i;
    const double n2r = s2 * t3r - s1 * t4r, n2i = s2 * t3i - s1 * t4i;
    zr[0] += t1r + t2r;
    zi[0] += t1i + t2i;
    zr[1] = m1r + n1i; zi[1] = m1i - n1r;
    zr[4] = m1r - n1i; zi[4] = m1i + n1r;
    zr[2] = m2r + n2i; zi[2] = m2i - n2r;
    zr[3] = m2r - n2i; zi[3] = m2i + n2r;
}

#define COMBINE(R, zr, zi, cj)                                          \
    do {                                                                \
        if (R == 2) comb2(zr, zi);                                      \
        else if (R == 3) comb3(zr, zi, (cj) ? -S60 : S60);              \
        else if (R == 4) comb4(zr, zi, cj);                             \
        else comb5(zr, zi, (cj) ? -1.0 : 1.0);                          \
    } while (0)

/* A^T (transposed) and A-bar (conjugate) ladders for one radix, generated
 * per R so the combine and the m-loops are compile-time. */
#define DEFINE_LADDERS(R)                                                                              \
    static void transposed_r##R(double* xr, double* xi, size_t n, const double* twr, const double* twi) { \
        double zr[R], zi[R];                                                                           \
        for (size_t k = n; k >= R; k /= R) {                                                           \
            const size_t l = k / R, stride = n / k;                                                    \
            for (size_t b = 0; b < n; b += k)                                                          \
                for (size_t j = 0; j < l; ++j) {                                                       \
                    const size_t i0 = b + j;                                                           \
                    for (int m = 0; m < R; ++m) { zr[m] = xr[i0 + m * l]; zi[m] = xi[i0 + m * l]; }    \
                    COMBINE(R, zr, zi, 0);                                                             \
                    xr[i0] = zr[0];                                                                    \
                    xi[i0] = zi[0];                                                                    \
                    for (int m = 1; m < R; ++m) {                                                      \
                        const size_t e = (size_t)m * j * stride;                                       \
                        const double wr = twr[e], wi = twi[e];                                         \
                        xr[i0 + m * l] = wr * zr[m] - wi * zi[m];                                      \
                        xi[i0 + m * l] = wr * zi[m] + wi * zr[m];                                      \
                    }                                                                                  \
                }                                                                                      \
            if (k == R) break;                                                                         \
        }                                                                                              \
    }                                                                                                  \
    static void conjugate_r##R(double* xr, double* xi, size_t n, const double* twr, const double* twi) {  \
        double zr[R], zi[R];                                                                           \
        for (size_t k = R; k <= n; k *= R) {                                                           \
            const size_t l = k / R, stride = n / k;                                                    \
            for (size_t b = 0; b < n; b += k)                                                          \
                for (size_t j = 0; j < l; ++j) {                                                       \
                    const size_t i0 = b + j;                                                           \
                    zr[0] = xr[i0];                                                                    \
                    zi[0] = xi[i0];                                                                    \
                    for (int m = 1; m < R; ++m) {                                                      \
                        const size_t e = (size_t)m * j * stride;                                       \
                        const double wr = twr[e], wi = -twi[e];                                        \
                        const double ur = xr[i0 + m * l], ui = xi[i0 + m * l];                         \
                        zr[m] = wr * ur - wi * ui;                                                     \
                        zi[m] = wr * ui + wi * ur;                                                     \
                    }                                                                                  \
                    COMBINE(R, zr, zi, 1);                                                             \
                    for (int m = 0; m < R; ++m) { xr[i0 + m * l] = zr[m]; xi[i0 + m * l] = zi[m]; }    \
                }                                                                                      \
            if (k == n) break;                                                                         \
        }                                                                                              \
    }

DEFINE_LADDERS(2)
DEFINE_LADDERS(3)
DEFINE_LADDERS(4)
DEFINE_LADDERS(5)

typedef void (*ladder_fn)(double*, double*, size_t, const double*, const double*);

static int pick(unsigned r, ladder_fn* t, ladder_fn* c) {
    switch (r) {
        case 2: *t = transposed_r2; *c = conjugate_r2; return 1;
        case 3: *t = transposed_r3; *c = conjugate_r3; return 1;
        case 4: *t = transposed_r4; *c = conjugate_r4; return 1;
        case 5: *t = transposed_r5; *c = conjugate_r5; return 1;
        default: return 0;
    }
}

/* convolve_permfree (convolution.cpp:45-52) for one 1-D signal. */
int orc_convolve_permfree_fast(const orc_plan* p, const double* ghat_re, const double* ghat_im, double* re,
                               double* im) {
    ladder_fn tr, cj;
    if (p->rank != 1 || !pick(p->radices[0], &tr, &cj)) return ORC_INVALID_ARGUMENT;
    const size_t n = p->total;
    if (n > 1) tr(re, im, n, p->tw_re[0], p->tw_im[0]);
    orc_hadamard(n, re, im, ghat_re, ghat_im);
    if (n > 1) cj(re, im, n, p->tw_re[0], p->tw_im[0]);
    orc_scale(n, re, im, 1.0 / (double)n);
    return ORC_OK;
}

typedef struct {
    const orc_plan* p;
    const double *gr, *gi;
    double *re, *im;
    size_t first, count;
} fast_job;

static void* fast_worker(void* arg) {
    fast_job* j = (fast_job*)arg;
    for (size_t b = j->first; b < j->first + j->count; ++b)
        orc_convolve_permfree_fast(j->p, j->gr, j->gi, j->re + b * j->p->total, j->im + b * j->p->total);
    return NULL;
}

/* Batch over host threads sharing one plan and prepared filter. */
int orc_convolve_permfree_fast_batch(const orc_plan* p, const double* ghat_re, const double* ghat_im, double* re,
                                     double* im, size_t batch, int threads) {
    ladder_fn tr, cj;
    if (p->rank != 1 || !pick(p->radices[0], &tr, &cj)) return ORC_INVALID_ARGUMENT;
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    if ((size_t)threads > batch) threads = (int)(batch ? batch : 1);
    pthread_t tid[256];
    fast_job jobs[256];
    size_t start = 0;
    for (int t = 0; t < threads; ++t) {
        const size_t cnt = batch / threads + ((size_t)t < batch % threads ? 1 : 0);
        jobs[t] = (fast_job){p, ghat_re, ghat_im, re, im, start, cnt};
        start += cnt;
        pthread_create(&tid[t], NULL, fast_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    return ORC_OK;
}
