/*
 * pafft_oracle.c -- CPU restatement of the reference's permutation-avoiding
 * convolution path at general radix.  TEST INFRASTRUCTURE ONLY (see header).
 *
 * Every function cites the reference file:line it restates; paths are
 * relative to the reference's proj/ directory.  The ladders follow
 * butterfly.cpp's loop nest exactly (stage order, block/butterfly loops,
 * table stride rule, twiddle placement) with the radix-r combine written as
 * the generic F_r of Eq. 25 (ladders PAPER.md:1481-1514),
 * so radix 3 and 5, which pafft's Radix enum cannot express
 * (core.hpp:14-19), run through the same code as 2/4/8.
 */
#include "pafft_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static const double ORC_PI = 3.14159265358979323846264338327950288;

/* ------------------------------------------------------------ plan -- */

/* core.cpp:17-31 */
static int is_power_of(size_t n, unsigned r) {
    if (n == 0) return 0;
    while (n % r == 0) n /= r;
    return n == 1;
}

static unsigned power_depth(size_t n, unsigned r) {
    unsigned t = 0;
    while (n > 1) { n /= r; ++t; }
    return t;
}

static int radix_supported(unsigned r) {
    return r == 2 || r == 3 || r == 4 || r == 5 || r == 8;
}

/* Plan::Plan, core.cpp:93-127; TwiddleTable, core.cpp:84-91. */
int orc_plan_create(unsigned radix, const size_t* dims, int rank, orc_plan** out) {
    unsigned radices[ORC_MAX_RANK];
    for (int q = 0; q < ORC_MAX_RANK; ++q) radices[q] = radix;
    *out = NULL;
    if (rank > ORC_MAX_RANK) return ORC_INVALID_ARGUMENT;
    return orc_plan_create_mixed(radices, dims, rank, out);
}

/* Per-axis radix r_q: axis q is
 * its own radix-r_q ladder with its own digit reversal P_{r_q, n_q}; the
 * tensor structure (butterfly.cpp:423-466 mode loop) is unchanged. */
int orc_plan_create_mixed(const unsigned* radices, const size_t* dims, int rank, orc_plan** out) {
    *out = NULL;
    if (rank <= 0) return ORC_EMPTY_SHAPE;
    if (rank > ORC_MAX_RANK) return ORC_INVALID_ARGUMENT;
    for (int q = 0; q < rank; ++q) {
        if (!radix_supported(radices[q])) return ORC_INVALID_ARGUMENT;
        if (!is_power_of(dims[q], radices[q])) return ORC_NOT_A_POWER_OF_RADIX;
        if (dims[q] > 0xffffffffull) return ORC_INVALID_ARGUMENT;
    }
    orc_plan* p = (orc_plan*)calloc(1, sizeof(orc_plan));
    p->radix = radices[0];
    p->rank = rank;
    p->total = 1;
    for (int q = 0; q < rank; ++q) {
        const unsigned radix = radices[q];
        p->radices[q] = radix;
        const size_t n = dims[q];
        p->dims[q] = n;
        p->total *= n;
        p->depth[q] = power_depth(n, radix);
        p->tw_re[q] = (double*)malloc(n * sizeof(double));
        p->tw_im[q] = (double*)malloc(n * sizeof(double));
        const double step = -2.0 * ORC_PI / (double)n;
        for (size_t j = 0; j < n; ++j) {
            const double ang = step * (double)j;
            p->tw_re[q][j] = cos(ang);
            p->tw_im[q][j] = sin(ang);
        }
        p->rev[q] = (uint32_t*)malloc(n * sizeof(uint32_t));
        for (size_t j = 0; j < n; ++j) {
            size_t v = j, o = 0;
            for (unsigned s = 0; s < p->depth[q]; ++s) { o = o * radix + v % radix; v /= radix; }
            p->rev[q][j] = (uint32_t)o;
        }
    }
    *out = p;
    return ORC_OK;
}

void orc_plan_destroy(orc_plan* p) {
    if (!p) return;
    for (int q = 0; q < p->rank; ++q) {
        free(p->tw_re[q]);
        free(p->tw_im[q]);
        free(p->rev[q]);
    }
    free(p);
}

/* ---------------------------------------------------- permutation -- */

static _Thread_local uint64_t g_pass_count = 0;

/* permutation.cpp:27-37 */
int orc_digit_reverse(uint64_t j, unsigned radix, unsigned digits, uint64_t* out) {
    uint64_t bound = 1;
    for (unsigned s = 0; s < digits; ++s) bound *= radix;
    if (j >= bound) return ORC_INDEX_OUT_OF_RANGE;
    uint64_t o = 0;
    for (unsigned s = 0; s < digits; ++s) { o = o * radix + j % radix; j /= radix; }
    *out = o;
    return ORC_OK;
}

/* permutation.cpp:46-90: one pass over linear offsets; partner is the
 * offset of the per-mode reversed multi-index; swap when it lies ahead. */
int orc_permute_tensor(const orc_plan* p, double* re, double* im) {
    size_t idx[ORC_MAX_RANK] = {0};
    size_t weight[ORC_MAX_RANK];
    size_t w = 1;
    for (int q = 0; q < p->rank; ++q) { weight[q] = w; w *= p->dims[q]; }
    for (size_t j = 0; j < p->total; ++j) {
        size_t partner = 0;
        for (int q = 0; q < p->rank; ++q) partner += weight[q] * p->rev[q][idx[q]];
        if (partner > j) {
            double t = re[j]; re[j] = re[partner]; re[partner] = t;
            t = im[j]; im[j] = im[partner]; im[partner] = t;
        }
        for (int q = 0; q < p->rank; ++q) {
            if (++idx[q] < p->dims[q]) break;
            idx[q] = 0;
        }
    }
    ++g_pass_count;
    return ORC_OK;
}

uint64_t orc_permutation_pass_count(void) { return g_pass_count; }
void orc_reset_permutation_pass_count(void) { g_pass_count = 0; }

/* ------------------------------------------------------- ladders -- */

/* omega_r^e = exp(-2 pi i e / r), exact where the value is exact. */
static void root_table(unsigned r, double* c, double* s) {
    for (unsigned e = 0; e < r; ++e) {
        const long double a = -2.0L * 3.141592653589793238462643383279502884L * (long double)e / (long double)r;
        c[e] = (double)cosl(a);
        s[e] = (double)sinl(a);
    }
    /* Exact quarter-turns (r = 2, 4, 8) so the 2/4/8 combines add and
     * subtract exactly as the reference's hand-expanded kernels do. */
    for (unsigned e = 0; e < r; ++e) {
        if ((4 * e) % r == 0) {
            const unsigned quarter = (4 * e) / r; /* 0..3 */
            const double cc[4] = {1.0, 0.0, -1.0, 0.0};
            const double ss[4] = {0.0, -1.0, 0.0, 1.0};
            c[e] = cc[quarter];
            s[e] = ss[quarter];
        }
    }
    if (r == 8) { /* butterfly.hpp:19-25: a = (1 - i)/sqrt(2) */
        const double h = 0.70710678118654752440;
        c[1] = h;  s[1] = -h;
        c[3] = -h; s[3] = -h;
        c[5] = -h; s[5] = h;
        c[7] = h;  s[7] = h;
    }
}

/* y_m = sum_d omega_r^{(d m) mod r} z_d  (conj = 1: conjugated roots).
 * Unit and zero factors contribute exact terms, so r = 2 and 4 reproduce
 * the reference's add/subtract combines exactly. */
static void combine(unsigned r, const double* c, const double* s, int conj,
                    const double* zr, const double* zi, double* yr, double* yi) {
    for (unsigned m = 0; m < r; ++m) {
        double ar = zr[0], ai = zi[0];
        for (unsigned d = 1; d < r; ++d) {
            const unsigned e = (d * m) % r;
            const double wr = c[e], wi = conj ? -s[e] : s[e];
            if (wi == 0.0) {
                if (wr == 1.0) { ar += zr[d]; ai += zi[d]; }
                else { ar -= zr[d]; ai -= zi[d]; } /* wr == -1 */
            } else if (wr == 0.0) {
                if (wi == 1.0) { ar -= zi[d]; ai += zr[d]; } /* +i */
                else { ar += zi[d]; ai -= zr[d]; }           /* -i */
            } else {
                ar += wr * zr[d] - wi * zi[d];
                ai += wr * zi[d] + wi * zr[d];
            }
        }
        yr[m] = ar;
        yi[m] = ai;
    }
}

/* butterfly.cpp:20-75 (+ :79-193, :197-379 for r = 4, 8) at general r.
 * forward   (A):  k = r..n ascending, twiddle inputs by w_k^{mj}, combine.
 * conjugate (A-bar): same with conjugated twiddles and conj(F_r).
 * transposed (A^T): k = n..r descending, combine, twiddle outputs by w_k^{mj}.
 * The table is read at e * (n/k) (core.hpp:71-88); e < k never wraps. */
static void ladder(unsigned r, int variant, double* xr, double* xi, size_t n,
                   const double* twr, const double* twi) {
    double c[8], s[8], zr[8], zi[8], yr[8], yi[8];
    root_table(r, c, s);
    if (n < 2) return;
    const int ascending = variant != ORC_TRANSPOSED;
    size_t k = ascending ? r : n;
    for (;;) {
        const size_t l = k / r;
        const size_t stride = n / k;
        for (size_t b = 0; b < n; b += k) {
            for (size_t j = 0; j < l; ++j) {
                const size_t i0 = b + j;
                if (variant == ORC_TRANSPOSED) {
                    for (unsigned m = 0; m < r; ++m) { zr[m] = xr[i0 + m * l]; zi[m] = xi[i0 + m * l]; }
                    combine(r, c, s, 0, zr, zi, yr, yi);
                    xr[i0] = yr[0];
                    xi[i0] = yi[0];
                    for (unsigned m = 1; m < r; ++m) {
                        const size_t e = (size_t)m * j * stride;
                        const double wr = twr[e], wi = twi[e];
                        xr[i0 + m * l] = wr * yr[m] - wi * yi[m];
                        xi[i0 + m * l] = wr * yi[m] + wi * yr[m];
                    }
                } else {
                    const int cj = variant == ORC_CONJUGATE;
                    zr[0] = xr[i0];
                    zi[0] = xi[i0];
                    for (unsigned m = 1; m < r; ++m) {
                        const size_t e = (size_t)m * j * stride;
                        const double wr = twr[e], wi = cj ? -twi[e] : twi[e];
                        const double ur = xr[i0 + m * l], ui = xi[i0 + m * l];
                        zr[m] = wr * ur - wi * ui;
                        zi[m] = wr * ui + wi * ur;
                    }
                    combine(r, c, s, cj, zr, zi, yr, yi);
                    for (unsigned m = 0; m < r; ++m) { xr[i0 + m * l] = yr[m]; xi[i0 + m * l] = yi[m]; }
                }
            }
        }
        if (ascending) { if (k == n) break; k *= r; }
        else { if (k == r) break; k /= r; }
    }
}

/* butterfly_line, butterfly.cpp:401-407 */
int orc_butterfly_line(const orc_plan* p, size_t dim, int variant, double* re, double* im, size_t len) {
    if ((int)dim >= p->rank) return ORC_INVALID_ARGUMENT;
    if (len != p->dims[dim]) return ORC_SHAPE_MISMATCH;
    if (len == 1) return ORC_OK;
    ladder(p->radices[dim], variant, re, im, len, p->tw_re[dim], p->tw_im[dim]);
    return ORC_OK;
}

/* butterfly_tensor, butterfly.cpp:423-466: modes ascending; the contiguous
 * mode runs in place per line, strided modes gather into scratch. */
int orc_butterfly_tensor(const orc_plan* p, int variant, double* xr, double* xi) {
    size_t maxd = 0;
    for (int q = 0; q < p->rank; ++q) if (p->dims[q] > maxd) maxd = p->dims[q];
    double* sr = (double*)malloc(maxd * sizeof(double));
    double* si = (double*)malloc(maxd * sizeof(double));
    size_t stride = 1;
    for (int q = 0; q < p->rank; ++q) {
        const size_t nq = p->dims[q];
        if (nq > 1) {
            if (stride == 1) {
                for (size_t base = 0; base < p->total; base += nq)
                    ladder(p->radices[q], variant, xr + base, xi + base, nq, p->tw_re[q], p->tw_im[q]);
            } else {
                const size_t block = stride * nq;
                for (size_t base = 0; base < p->total; base += block) {
                    for (size_t inner = 0; inner < stride; ++inner) {
                        const size_t start = base + inner;
                        for (size_t m = 0; m < nq; ++m) { sr[m] = xr[start + m * stride]; si[m] = xi[start + m * stride]; }
                        ladder(p->radices[q], variant, sr, si, nq, p->tw_re[q], p->tw_im[q]);
                        for (size_t m = 0; m < nq; ++m) { xr[start + m * stride] = sr[m]; xi[start + m * stride] = si[m]; }
                    }
                }
            }
        }
        stride *= nq;
    }
    free(sr);
    free(si);
    return ORC_OK;
}

/* --------------------------------------------------- convolution -- */

/* convolution.cpp:23-35 */
void orc_hadamard(size_t n, double* xr, double* xi, const double* yr, const double* yi) {
    for (size_t i = 0; i < n; ++i) {
        const double r = xr[i] * yr[i] - xi[i] * yi[i];
        const double m = xr[i] * yi[i] + xi[i] * yr[i];
        xr[i] = r;
        xi[i] = m;
    }
}

/* core.cpp:79-82 */
void orc_scale(size_t n, double* xr, double* xi, double s) {
    for (size_t i = 0; i < n; ++i) { xr[i] *= s; xi[i] *= s; }
}

/* transform.cpp:8-26 */
int orc_fft_forward(const orc_plan* p, double* re, double* im) {
    orc_permute_tensor(p, re, im);
    return orc_butterfly_tensor(p, ORC_FORWARD, re, im);
}

int orc_fft_backward(const orc_plan* p, double* re, double* im) {
    orc_permute_tensor(p, re, im);
    orc_butterfly_tensor(p, ORC_CONJUGATE, re, im);
    orc_scale(p->total, re, im, 1.0 / (double)p->total);
    return ORC_OK;
}

/* convolution.cpp:9-14 */
int orc_prepare_filter(const orc_plan* p, const double* g_re, const double* g_im,
                       double* ghat_re, double* ghat_im) {
    memcpy(ghat_re, g_re, p->total * sizeof(double));
    memcpy(ghat_im, g_im, p->total * sizeof(double));
    return orc_permute_tensor(p, ghat_re, ghat_im);
}

/* convolution.cpp:16-21 */
int orc_filter_from_impulse(const orc_plan* p, const double* h_re, const double* h_im,
                            double* g_re, double* g_im) {
    memcpy(g_re, h_re, p->total * sizeof(double));
    memcpy(g_im, h_im, p->total * sizeof(double));
    return orc_fft_forward(p, g_re, g_im);
}

/* convolution.cpp:45-52 */
int orc_convolve_permfree(const orc_plan* p, const double* ghat_re, const double* ghat_im,
                          double* re, double* im) {
    orc_butterfly_tensor(p, ORC_TRANSPOSED, re, im);
    orc_hadamard(p->total, re, im, ghat_re, ghat_im);
    orc_butterfly_tensor(p, ORC_CONJUGATE, re, im);
    orc_scale(p->total, re, im, 1.0 / (double)p->total);
    return ORC_OK;
}

/* convolution.cpp:37-43 */
int orc_convolve_standard(const orc_plan* p, const double* g_re, const double* g_im,
                          double* re, double* im) {
    orc_fft_forward(p, re, im);
    orc_hadamard(p->total, re, im, g_re, g_im);
    return orc_fft_backward(p, re, im);
}

typedef struct {
    const orc_plan* p;
    const double *gr, *gi;
    double *re, *im;
    size_t first, count;
} batch_job;

static void* batch_worker(void* arg) {
    batch_job* j = (batch_job*)arg;
    for (size_t b = j->first; b < j->first + j->count; ++b)
        orc_convolve_permfree(j->p, j->gr, j->gi, j->re + b * j->p->total, j->im + b * j->p->total);
    return NULL;
}

int orc_convolve_permfree_batch(const orc_plan* p, const double* ghat_re, const double* ghat_im,
                                double* re, double* im, size_t batch, int threads) {
    if (threads < 1) threads = 1;
    if ((size_t)threads > batch) threads = (int)(batch ? batch : 1);
    pthread_t tid[256];
    batch_job jobs[256];
    if (threads > 256) threads = 256;
    size_t first = 0;
    for (int t = 0; t < threads; ++t) {
        const size_t cnt = batch / threads + ((size_t)t < batch % threads ? 1 : 0);
        jobs[t] = (batch_job){p, ghat_re, ghat_im, re, im, first, cnt};
        first += cnt;
        pthread_create(&tid[t], NULL, batch_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    return ORC_OK;
}

/* ------------------------------------------------- direct oracles -- */

/* oracle.cpp:14-34: exponent reduced mod n, direct cos/sin, index order. */
static void dft_line(size_t n, int backward, const double* xr, const double* xi, double* yr, double* yi) {
    const double sign = backward ? 1.0 : -1.0;
    for (size_t j = 0; j < n; ++j) {
        double ar = 0.0, ai = 0.0;
        for (size_t k = 0; k < n; ++k) {
            const uint64_t m = ((uint64_t)j * (uint64_t)k) % n;
            const double ang = sign * 2.0 * ORC_PI * (double)m / (double)n;
            const double c = cos(ang), s = sin(ang);
            ar += c * xr[k] - s * xi[k];
            ai += c * xi[k] + s * xr[k];
        }
        yr[j] = ar;
        yi[j] = ai;
    }
}

/* oracle.cpp:50-85 */
int orc_naive_dft_tensor(const size_t* dims, int rank, int backward,
                         const double* xr, const double* xi, double* yr, double* yi) {
    if (rank <= 0) return ORC_EMPTY_SHAPE;
    size_t total = 1, maxd = 0;
    for (int q = 0; q < rank; ++q) { total *= dims[q]; if (dims[q] > maxd) maxd = dims[q]; }
    memcpy(yr, xr, total * sizeof(double));
    memcpy(yi, xi, total * sizeof(double));
    double* lr = (double*)malloc(4 * maxd * sizeof(double));
    double *li = lr + maxd, *or_ = li + maxd, *oi = or_ + maxd;
    size_t stride = 1;
    for (int q = 0; q < rank; ++q) {
        const size_t nq = dims[q], block = stride * nq;
        for (size_t base = 0; base < total; base += block) {
            for (size_t inner = 0; inner < stride; ++inner) {
                const size_t start = base + inner;
                for (size_t m = 0; m < nq; ++m) { lr[m] = yr[start + m * stride]; li[m] = yi[start + m * stride]; }
                dft_line(nq, backward, lr, li, or_, oi);
                for (size_t m = 0; m < nq; ++m) { yr[start + m * stride] = or_[m]; yi[start + m * stride] = oi[m]; }
            }
        }
        stride = block;
    }
    if (backward) {
        const double inv = 1.0 / (double)total;
        for (size_t i = 0; i < total; ++i) { yr[i] *= inv; yi[i] *= inv; }
    }
    free(lr);
    return ORC_OK;
}

/* oracle.cpp:87-123: y[i] = sum_j h[j] x[(i - j) mod shape]. */
int orc_naive_circular_convolution(const size_t* dims, int rank,
                                   const double* xr, const double* xi,
                                   const double* hr, const double* hi,
                                   double* yr, double* yi) {
    if (rank <= 0) return ORC_EMPTY_SHAPE;
    size_t total = 1;
    for (int q = 0; q < rank; ++q) total *= dims[q];
    size_t iidx[ORC_MAX_RANK] = {0};
    for (size_t i = 0; i < total; ++i) {
        double ar = 0.0, ai = 0.0;
        size_t jidx[ORC_MAX_RANK] = {0};
        for (size_t j = 0; j < total; ++j) {
            size_t src = 0, w = 1;
            for (int q = 0; q < rank; ++q) {
                const size_t nq = dims[q];
                src += ((iidx[q] + nq - jidx[q]) % nq) * w;
                w *= nq;
            }
            ar += hr[j] * xr[src] - hi[j] * xi[src];
            ai += hr[j] * xi[src] + hi[j] * xr[src];
            for (int q = 0; q < rank; ++q) { if (++jidx[q] < dims[q]) break; jidx[q] = 0; }
        }
        yr[i] = ar;
        yi[i] = ai;
        for (int q = 0; q < rank; ++q) { if (++iidx[q] < dims[q]) break; iidx[q] = 0; }
    }
    return ORC_OK;
}

/* ---------------------------------------------------- generators -- */

/* bench.cpp:22-42 (SplitMix64, Steele/Lea/Flood). */
uint64_t orc_splitmix64_next(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* bench.cpp:36-49: re then im per element, 2*u - 1 with u = top53/(2^53-1). */
void orc_fill_uniform(uint64_t seed, size_t n, double* re, double* im) {
    uint64_t st = seed;
    for (size_t i = 0; i < n; ++i) {
        re[i] = 2.0 * ((double)(orc_splitmix64_next(&st) >> 11) / 9007199254740991.0) - 1.0;
        im[i] = 2.0 * ((double)(orc_splitmix64_next(&st) >> 11) / 9007199254740991.0) - 1.0;
    }
}

/* Box-Muller on two 53-bit draws per element: u1 in (0, 1], u2 in [0, 1);
 * re = rho cos(2 pi u2), im = rho sin(2 pi u2), rho = sqrt(-2 ln u1). */
void orc_fill_normal(uint64_t seed, size_t n, double* re, double* im) {
    uint64_t st = seed;
    const double inv53 = 1.0 / 9007199254740992.0;
    for (size_t i = 0; i < n; ++i) {
        const double u1 = (double)((orc_splitmix64_next(&st) >> 11) + 1) * inv53;
        const double u2 = (double)(orc_splitmix64_next(&st) >> 11) * inv53;
        const double rho = sqrt(-2.0 * log(u1));
        re[i] = rho * cos(2.0 * ORC_PI * u2);
        im[i] = rho * sin(2.0 * ORC_PI * u2);
    }
}
