/*
 * pafft_b200.h -- C ABI of the B200-native permutation-avoiding convolution
 * library (libpafft_b200.so).  Plain pointers and sizes only; no C++ or torch
 * types.  Every entry point names the reference interface it replaces
 * (paths relative to the reference's proj/ directory).  The reference's own
 * foreign-function layer is its pybind11 module (python/src/module.cpp:73-149);
 * INTEGRATION.md shows the ctypes / C++ bindings a maintainer would add.
 *
 * Layout: complex values are interleaved (re, im) pairs in vec order, first
 * index fastest (core.hpp:26-27).  The *_split entry points take the
 * reference's split layout (ComplexBuffer{re, im}, core.hpp:47-63) on the host.
 * Batches are consecutive signals of plan->total elements each.
 *
 * Errors: every function returns a pafft_status; the message of the last
 * failure on the calling thread is pafft_last_error().  Status codes map 1:1
 * onto the reference's exception classes (errors.hpp:10-44).
 */
#ifndef PAFFT_B200_H
#define PAFFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PAFFT_OK = 0,
    PAFFT_NOT_A_POWER_OF_RADIX = 1, /* NotAPowerOfRadix (errors.hpp:15-19) */
    PAFFT_EMPTY_SHAPE = 2,          /* EmptyShape (errors.hpp:22-24) */
    PAFFT_LENGTH_MISMATCH = 3,      /* LengthMismatch (errors.hpp:27-29) */
    PAFFT_SHAPE_MISMATCH = 4,       /* ShapeMismatch (errors.hpp:32-34) */
    PAFFT_FILTER_PLAN_MISMATCH = 5, /* FilterPlanMismatch (errors.hpp:37-39) */
    PAFFT_INDEX_OUT_OF_RANGE = 6,   /* IndexOutOfRange (errors.hpp:42-44) */
    PAFFT_INVALID_ARGUMENT = 7,     /* pafft::Error (radix_from_value, core.cpp:55-62) */
    PAFFT_CUDA_ERROR = 8,
    PAFFT_NCCL_ERROR = 9,
    PAFFT_NO_DEVICE = 10
} pafft_status;

typedef enum { PAFFT_F64 = 0, PAFFT_F32 = 1 } pafft_precision;

typedef struct pafft_plan_s* pafft_plan_t;
typedef struct pafft_filter_s* pafft_filter_t;

/* Message of the last failure on this thread ("" if none). */
const char* pafft_last_error(void);
/* For PAFFT_NOT_A_POWER_OF_RADIX: offending dimension and extent
 * (NotAPowerOfRadix::dim / ::extent, errors.hpp:15-19). */
void pafft_last_error_dim(size_t* dim, size_t* extent);

/* ---------------------------------------------------------------- plan --
 * Replaces Plan::Plan / plan_create (core.cpp:93-129, core.hpp:98-132).
 * radix in {2, 3, 4, 5, 8} (the reference accepts 2, 4, 8: core.cpp:55-62).
 * Builds the device twiddle tables and pass schedule for that shape on
 * `device` (-1 = current device). */
pafft_status pafft_plan_create(unsigned radix, const size_t* dims, int rank, int precision, int device,
                               pafft_plan_t* out);
/* Per-axis radices: axis q is a
 * power of radices[q] and runs its own radix-radices[q] ladders; the prepared
 * filter is the per-axis digit reversal (P_{r_d,n_d} (x) ... (x) P_{r_1,n_1}) g.
 * pafft_plan_create(r, ...) == pafft_plan_create_mixed({r, r, ...}, ...). */
pafft_status pafft_plan_create_mixed(const unsigned* radices, const size_t* dims, int rank, int precision,
                                     int device, pafft_plan_t* out);
/* radices: rank entries. */
pafft_status pafft_plan_radices(pafft_plan_t plan, unsigned* radices);
pafft_status pafft_plan_destroy(pafft_plan_t plan);
/* Plan::radix/shape/total/depth (core.hpp:104-112). dims/depths: rank entries. */
pafft_status pafft_plan_info(pafft_plan_t plan, unsigned* radix, int* rank, size_t* dims, unsigned* depths,
                             size_t* total, int* precision, int* device);
/* Number of kernel launches one convolve_permfree of `batch` signals issues. */
pafft_status pafft_plan_num_passes(pafft_plan_t plan, int* permfree_passes);
/* Human-readable pass schedule (for DESIGN.md / profiling). */
pafft_status pafft_plan_describe(pafft_plan_t plan, char* buf, size_t len);

/* digit_reverse (permutation.cpp:27-37). */
pafft_status pafft_digit_reverse(uint64_t j, unsigned radix, unsigned digits, uint64_t* out);

/* ------------------------------------------------------------- filters --
 * prepare_filter (convolution.cpp:9-14): digit-reverses a natural-order
 * spectrum g once (one permutation pass, counted) and binds it to the plan.
 * The observable ghat (PreparedFilter::ghat) is kept bit-exact. */
pafft_status pafft_prepare_filter_split(pafft_plan_t plan, const double* g_re, const double* g_im,
                                        pafft_filter_t* out);
/* A filter whose spectrum is ALREADY digit-reversed (a PreparedFilter::ghat
 * the caller built or edited, convolution.hpp:9-12): uploaded as is, no
 * reordering pass.  The C++ shim uses it for aggregate-initialised or edited
 * PreparedFilter objects, since the reference reads ghat directly
 * (convolution.cpp:45-52). */
pafft_status pafft_filter_from_prepared_split(pafft_plan_t plan, const double* ghat_re, const double* ghat_im,
                                              pafft_filter_t* out);
/* Same from a device-resident interleaved spectrum (same precision as plan). */
pafft_status pafft_prepare_filter_device(pafft_plan_t plan, const void* g_dev, void* stream,
                                         pafft_filter_t* out);
/* Prepared directly from a device impulse response h: ghat = A^T h (the DIF
 * ladder leaves P*DFT(h)), zero permutation passes.
 * Equals prepare_filter(filter_from_impulse(h)) up to rounding. */
pafft_status pafft_prepare_filter_from_impulse_device(pafft_plan_t plan, const void* h_dev, void* stream,
                                                      pafft_filter_t* out);
/* Filter-spectrum cache across plans: as
 * pafft_prepare_filter_from_impulse_device, but a spectrum already prepared
 * for the same plan key (radices, dims, precision, device) from the same
 * impulse bytes (128-bit device content hash) is shared instead of
 * recomputed; *hit (may be NULL) says which.  Cached spectra are held weakly:
 * they live while any filter handle uses them.  The returned handle is owned
 * by the caller as usual (pafft_filter_destroy). */
pafft_status pafft_prepare_filter_from_impulse_cached(pafft_plan_t plan, const void* h_dev, void* stream,
                                                      pafft_filter_t* out, int* hit);
void pafft_filter_cache_stats(uint64_t* hits, uint64_t* misses, uint64_t* live);
pafft_status pafft_filter_destroy(pafft_filter_t filter);
/* PreparedFilter::ghat readback (split, double). */
pafft_status pafft_filter_ghat_split(pafft_filter_t filter, double* re, double* im);
/* Device buffer holding the interleaved ghat the kernels read (pre-scaled by
 * 1/N) and the unscaled one; both plan->total elements of the plan precision.
 * Used to broadcast a prepared filter to other GPUs (ncclBroadcast /
 * torch.distributed.broadcast); call pafft_filter_sync_scaled after writing
 * the unscaled buffer on a receiving rank. */
void* pafft_filter_device_ghat(pafft_filter_t filter);
void* pafft_filter_device_ghat_scaled(pafft_filter_t filter);
pafft_status pafft_filter_sync_scaled(pafft_filter_t filter, void* stream);
/* An empty filter bound to `plan`, to receive a broadcast ghat. */
pafft_status pafft_filter_create_empty(pafft_plan_t plan, pafft_filter_t* out);
/* Multi-GPU filter distribution: broadcast the prepared
 * filter of NCCL rank `root` into every other filter over NCCL (NVLink), once
 * per filter -- no per-call collective.  filters[i] sit on distinct devices,
 * all with the same plan key (the receivers from pafft_filter_create_empty);
 * comms[i] is the ncclComm_t of filters[i]'s device.  One process per GPU:
 * each rank passes its own filter (ndev = 1) and communicator.  comms == NULL:
 * single-process call over ndev devices, the library creates and caches the
 * communicator clique (ncclCommInitAll; rank i = filters[i]).  streams may be
 * NULL (legacy stream).  Receivers rebuild their kernel copy locally.  NCCL is
 * resolved at first use (libnccl.so.2; the process's own copy if loaded);
 * PAFFT_NCCL_ERROR if absent. */
pafft_status pafft_filter_broadcast(pafft_filter_t* filters, int ndev, int root, void* const* comms,
                                    void* const* streams);
/* PreparedFilter::key == plan.key() (convolution.cpp:46). */
int pafft_filter_matches(pafft_filter_t filter, pafft_plan_t plan);

/* -------------------------------------------------------- the hot path --
 * convolve_permfree (convolution.cpp:45-52): x <- A-bar(ghat o A^T x)/N for
 * `batch` device-resident signals, asynchronous on `stream` (cudaStream_t or
 * NULL), zero permutation passes.  In place (x_dev) or out of place
 * (x_dev -> y_dev; x is not modified).  FilterPlanMismatch if the filter was
 * prepared under another plan. */
pafft_status pafft_convolve_permfree(pafft_plan_t plan, pafft_filter_t filter, void* x_dev, size_t batch,
                                     void* stream);
pafft_status pafft_convolve_permfree_oop(pafft_plan_t plan, pafft_filter_t filter, const void* x_dev,
                                         void* y_dev, size_t batch, void* stream);
/* One pass of the same schedule (0 <= i < pafft_plan_num_passes): pass 0
 * reads x_dev and writes y_dev, later passes work in place on y_dev.  Running
 * i = 0..n-1 in order equals pafft_convolve_permfree_oop; used to time the
 * passes individually with CUDA events (bench.py roofline). */
pafft_status pafft_convolve_permfree_pass(pafft_plan_t plan, pafft_filter_t filter, const void* x_dev,
                                          void* y_dev, size_t batch, int i, void* stream);
/* kind: 0 DIF (A^T group), 1 DIT forward, 2 DIT conjugate, 3 CONV middle
 * (DIF + x ghat + DIT-conj); axis, R = radix^stages of the pass. */
pafft_status pafft_plan_pass_info(pafft_plan_t plan, int i, int* kind, int* axis, int* R, int* stages);
/* Drop-in host path: split host arrays (ComplexBuffer), synchronous, H2D and
 * D2H inside.  Mirrors convolve_permfree(ComplexBuffer&, ...) exactly. */
pafft_status pafft_convolve_permfree_split(pafft_plan_t plan, pafft_filter_t filter, double* re, double* im,
                                           size_t batch);
/* As pafft_convolve_permfree_split, but once the device result is ready the
 * library calls commit(ctx) and writes re/im back only if it returns nonzero
 * (*committed says which; re/im are untouched otherwise).  The C++ drop-in
 * uses it to check, concurrently with the upload and the convolution, that
 * the device spectrum still equals PreparedFilter::ghat (the reference reads
 * ghat on every call, convolution.cpp:49) without a serial pass over it. */
pafft_status pafft_convolve_permfree_split_if(pafft_plan_t plan, pafft_filter_t filter, double* re, double* im,
                                              size_t batch, int (*commit)(void*), void* ctx, int* committed);
/* Host interleaved buffers (pinned or pageable), pipelined in chunks over
 * copy/compute streams; synchronous. In place on x_host. */
pafft_status pafft_convolve_permfree_host(pafft_plan_t plan, pafft_filter_t filter, void* x_host,
                                          size_t batch);
/* Same, out of place: reads x_host, writes y_host (bench.py e2e leg). */
pafft_status pafft_convolve_permfree_host_oop(pafft_plan_t plan, pafft_filter_t filter, const void* x_host,
                                              void* y_host, size_t batch);

/* ------------------------------------------- comparator and transforms --
 * convolve_standard (convolution.cpp:37-43): permute, A, o g, permute,
 * A-bar, 1/N -- two permutation passes per call.  g is natural order. */
pafft_status pafft_convolve_standard(pafft_plan_t plan, const void* g_dev, void* x_dev, size_t batch,
                                     void* stream);
pafft_status pafft_convolve_standard_split(pafft_plan_t plan, const double* g_re, const double* g_im,
                                           double* re, double* im, size_t batch);
/* transform.cpp:8-26 */
pafft_status pafft_fft_forward(pafft_plan_t plan, void* x_dev, size_t batch, void* stream);
pafft_status pafft_fft_backward(pafft_plan_t plan, void* x_dev, size_t batch, void* stream);
pafft_status pafft_fft_forward_unordered(pafft_plan_t plan, void* x_dev, size_t batch, void* stream);
pafft_status pafft_fft_backward_unordered(pafft_plan_t plan, void* x_dev, size_t batch, void* stream);
/* A^T alone (DIF ladder, digit-reversed output). */
pafft_status pafft_fft_transposed(pafft_plan_t plan, void* x_dev, size_t batch, void* stream);
/* permute_tensor (permutation.cpp:46-90) on device; counted. */
pafft_status pafft_permute(pafft_plan_t plan, void* x_dev, size_t batch, void* stream);
/* Host split variants of the transforms (module.cpp:91-99 semantics). op:
 * 0 fft_forward, 1 fft_backward, 2 fft_forward_unordered,
 * 3 fft_backward_unordered, 4 fft_transposed (A^T), 5 permute,
 * 6 conjugate ladder A-bar without the 1/n (butterfly_conjugate). */
pafft_status pafft_transform_split(pafft_plan_t plan, int op, double* re, double* im, size_t batch);
/* filter_from_impulse (convolution.cpp:16-21): g = fft_forward(h), split host. */
pafft_status pafft_filter_from_impulse_split(pafft_plan_t plan, const double* h_re, const double* h_im,
                                             double* g_re, double* g_im);

/* ---------------------------------------------------------- counters --
 * permutation_pass_count (permutation.hpp:22-27): whole-buffer reordering
 * passes issued by this thread (one per permute of one signal batch). */
uint64_t pafft_permutation_pass_count(void);
void pafft_reset_permutation_pass_count(void);
/* Kernel launches issued by this library on this thread (all kinds). */
uint64_t pafft_kernel_launch_count(void);
/* Pass launches on this thread whose tiles were handed out dynamically (a
 * per-stream counter) instead of in the static round-robin order. */
uint64_t pafft_dynamic_launch_count(void);

/* ------------------------------------------------------- workload gen --
 * SplitMix64 (bench.cpp:22-42), interleaved output, n complex elements.
 * uniform: re, im ~ U(-1, 1) as bench.cpp:36-49; normal: Box-Muller. */
void pafft_fill_uniform(uint64_t seed, size_t n, double* out_interleaved);
void pafft_fill_normal(uint64_t seed, size_t n, double* out_interleaved);

/* Library version / build string. */
const char* pafft_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* PAFFT_B200_H */
