/*
 * pafft_oracle.h -- CPU restatement of pafft's permutation-avoiding
 * convolution path, at general radix r in {2,3,4,5,8}.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2506_12718_b200/,
 * include/, csrc/) may include, link or call this.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * use it, and only as the checker (or the timed CPU comparator), never as
 * the thing measured or shipped.
 *
 * Parity status: PINNED.  tests/test_oracle_pins.py checks this restatement
 * against (a) the known-answer values of the reference's own unit tests
 * (test_butterfly.cpp:28-45, test_convolution.cpp:32-61, test_core.cpp:44-70,
 * test_permutation.cpp:15-77), (b) golden vectors produced by the reference
 * itself (oracle/_ref, built from /root/reference/proj/src by
 * oracle/Makefile; fixtures in tests/golden/, script tests/golden/make_golden.py)
 * at r in {2,4,8}, and (c) the radix-agnostic O(N^2) direct sums
 * (oracle.cpp:50-123 restated below) at r in {3,5}.
 *
 * Layout follows the reference: split complex (re[], im[]) in vec order,
 * first index fastest (core.hpp:26-27, 47-63).
 */
#ifndef PAFFT_ORACLE_H
#define PAFFT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (one per pafft exception class, errors.hpp:10-44) ---- */
enum {
    ORC_OK = 0,
    ORC_NOT_A_POWER_OF_RADIX = 1,
    ORC_EMPTY_SHAPE = 2,
    ORC_LENGTH_MISMATCH = 3,
    ORC_SHAPE_MISMATCH = 4,
    ORC_FILTER_PLAN_MISMATCH = 5,
    ORC_INDEX_OUT_OF_RANGE = 6,
    ORC_INVALID_ARGUMENT = 7
};

enum { ORC_FORWARD = 0, ORC_CONJUGATE = 1, ORC_TRANSPOSED = 2 };

#define ORC_MAX_RANK 8

/* Plan (core.cpp:93-127): per-dimension depth, master twiddle table
 * w[j] = exp(-2 pi i j / n_q) and digit-reversal map. */
typedef struct {
    unsigned radix;
    int rank;
    size_t dims[ORC_MAX_RANK];
    unsigned depth[ORC_MAX_RANK];
    size_t total;
    double* tw_re[ORC_MAX_RANK];
    double* tw_im[ORC_MAX_RANK];
    uint32_t* rev[ORC_MAX_RANK];
    unsigned radices[ORC_MAX_RANK]; /* per-axis radix (all equal to radix for pafft plans) */
} orc_plan;

int orc_plan_create(unsigned radix, const size_t* dims, int rank, orc_plan** out);
/* Mixed per-axis radices: n_q = radices[q]^t_q. */
int orc_plan_create_mixed(const unsigned* radices, const size_t* dims, int rank, orc_plan** out);
void orc_plan_destroy(orc_plan* p);

/* digit_reverse (permutation.cpp:27-37). Returns ORC_INDEX_OUT_OF_RANGE for j >= r^t. */
int orc_digit_reverse(uint64_t j, unsigned radix, unsigned digits, uint64_t* out);

/* permute_tensor (permutation.cpp:46-90), in place; bumps the pass counter. */
int orc_permute_tensor(const orc_plan* p, double* re, double* im);
uint64_t orc_permutation_pass_count(void);
void orc_reset_permutation_pass_count(void);

/* One-line ladders (butterfly.cpp:20-75 generalised to any radix) and the
 * tensor driver (butterfly.cpp:423-466). */
int orc_butterfly_line(const orc_plan* p, size_t dim, int variant, double* re, double* im, size_t len);
int orc_butterfly_tensor(const orc_plan* p, int variant, double* re, double* im);

/* convolution.cpp:9-52 */
int orc_prepare_filter(const orc_plan* p, const double* g_re, const double* g_im,
                       double* ghat_re, double* ghat_im);
int orc_filter_from_impulse(const orc_plan* p, const double* h_re, const double* h_im,
                            double* g_re, double* g_im);
void orc_hadamard(size_t n, double* xr, double* xi, const double* yr, const double* yi);
void orc_scale(size_t n, double* xr, double* xi, double s);
int orc_convolve_permfree(const orc_plan* p, const double* ghat_re, const double* ghat_im,
                          double* re, double* im);
int orc_convolve_standard(const orc_plan* p, const double* g_re, const double* g_im,
                          double* re, double* im);
int orc_fft_forward(const orc_plan* p, double* re, double* im);
int orc_fft_backward(const orc_plan* p, double* re, double* im);

/* Batched permfree convolution over `batch` consecutive signals with
 * `threads` POSIX threads sharing the immutable plan and filter.
 * This is the CPU comparator timed by bench.py. */
int orc_convolve_permfree_batch(const orc_plan* p, const double* ghat_re, const double* ghat_im,
                                double* re, double* im, size_t batch, int threads);

/* oracle.cpp:14-123: O(n^2) references, independent of plan and tables. */
int orc_naive_dft_tensor(const size_t* dims, int rank, int backward,
                         const double* xr, const double* xi, double* yr, double* yi);
int orc_naive_circular_convolution(const size_t* dims, int rank,
                                   const double* xr, const double* xi,
                                   const double* hr, const double* hi,
                                   double* yr, double* yi);

/* Workload generators (bench.cpp:22-50 SplitMix64; Box-Muller is new). */
uint64_t orc_splitmix64_next(uint64_t* state);
void orc_fill_uniform(uint64_t seed, size_t n, double* re, double* im);
void orc_fill_normal(uint64_t seed, size_t n, double* re, double* im);

/* Reference-style specialised ladders (fast_ladders.c): pafft's loop nest
 * with a hand-expanded radix-r combine, r in {2,3,4,5}, 1-D plans.  The CPU
 * stand-in for pafft at radix 3/5 in bench.py's reference arm. */
int orc_convolve_permfree_fast(const orc_plan* p, const double* ghat_re, const double* ghat_im, double* re,
                               double* im);
int orc_convolve_permfree_fast_batch(const orc_plan* p, const double* ghat_re, const double* ghat_im, double* re,
                                     double* im, size_t batch, int threads);

#ifdef __cplusplus
}
#endif
#endif
