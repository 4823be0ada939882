"""B200-native permutation-avoiding FFT convolution (arxiv 2506.12718 hot path).

Drop-in mirror of the reference's Python module ``pafft``
(python/pafft/__init__.py, python/src/module.cpp:73-149): the same names,
argument meanings and error behaviour (every library error is a
``RuntimeError`` subclass, README.md:138-143), computed by hand-written
sm_100a kernels behind the C ABI ``include/pafft_b200.h``.

Host-array functions take numpy arrays in natural C order, like module.cpp,
and repack them to the library's vec layout (first index fastest,
core.cpp:131-178).  The device API (``DevicePlan``-style helpers at the end)
takes torch CUDA tensors of shape (batch, *dims) or (batch, N) already in vec
order and runs asynchronously on the current torch stream: that is the hot
path ``bench.py`` measures.

Extensions over the reference: radix 3 and 5 (the reference's Radix enum is
closed over {2, 4, 8}, core.hpp:14-19), fp32 plans, batched calls.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from ._lib import lib, EXPORTED  # noqa: F401  (raises if the .so is missing)

__all__ = [
    "Plan", "PreparedFilter", "convolve_permfree", "convolve_standard", "digit_reverse", "estimate_ai",
    "estimate_flop", "fft_backward", "fft_backward_unordered", "fft_forward", "fft_forward_unordered",
    "filter_from_impulse", "prepare_filter", "fft_transposed", "permute",
    "Error", "NotAPowerOfRadix", "EmptyShape", "LengthMismatch", "ShapeMismatch", "FilterPlanMismatch",
    "IndexOutOfRange", "CudaError", "NoDevice",
    "permutation_pass_count", "reset_permutation_pass_count", "kernel_launch_count", "dynamic_launch_count",
    "F64", "F32",
]

F64, F32 = 0, 1


# ------------------------------------------------------------------ errors
class Error(RuntimeError):
    """pafft::Error (errors.hpp:10-12)."""


class NotAPowerOfRadix(Error):
    def __init__(self, msg, dim=None, extent=None):
        super().__init__(msg)
        self.dim, self.extent = dim, extent


class EmptyShape(Error):
    pass


class LengthMismatch(Error):
    pass


class ShapeMismatch(Error):
    pass


class FilterPlanMismatch(Error):
    pass


class IndexOutOfRange(Error):
    pass


class CudaError(Error):
    pass


class NoDevice(Error):
    pass


_STATUS = {1: NotAPowerOfRadix, 2: EmptyShape, 3: LengthMismatch, 4: ShapeMismatch, 5: FilterPlanMismatch,
           6: IndexOutOfRange, 7: Error, 8: CudaError, 9: Error, 10: NoDevice}


def _check(status):
    if status == 0:
        return
    msg = lib.pafft_last_error().decode()
    cls = _STATUS.get(status, Error)
    if cls is NotAPowerOfRadix:
        d, e = C.c_size_t(), C.c_size_t()
        lib.pafft_last_error_dim(C.byref(d), C.byref(e))
        raise NotAPowerOfRadix(msg, d.value, e.value)
    raise cls(msg)


_dp = C.POINTER(C.c_double)


def _p(a):
    return a.ctypes.data_as(_dp)


# -------------------------------------------------------------------- plan
class Plan:
    """Plan(radix, dims[, precision, device]) -- module.cpp:76-85.

    ``dims`` follow the numpy axis order of the arrays passed in (numpy axis q
    is pafft dim q, module.cpp:30-35).  ``radix`` may also be a sequence with
    one radix per axis (mixed per-axis plans)."""

    def __init__(self, radix, dims, precision=F64, device=-1):
        dims = [int(d) for d in dims]
        arr = (C.c_size_t * max(len(dims), 1))(*dims)
        h = C.c_void_p()
        if isinstance(radix, (list, tuple)):
            if len(radix) != len(dims):
                raise Error(f"{len(radix)} radices for {len(dims)} dimensions")
            rs = (C.c_uint * max(len(radix), 1))(*[int(r) for r in radix])
            _check(lib.pafft_plan_create_mixed(rs, arr, len(dims), int(precision), int(device), C.byref(h)))
            self._radices = [int(r) for r in radix]
            radix = self._radices[0] if len(set(self._radices)) == 1 else list(self._radices)
        else:
            _check(lib.pafft_plan_create(int(radix), arr, len(dims), int(precision), int(device), C.byref(h)))
            self._radices = [int(radix)] * len(dims)
        self._h = h
        self._radix = radix if isinstance(radix, list) else int(radix)
        self._dims = dims
        self._precision = int(precision)
        dev = C.c_int()
        lib.pafft_plan_info(h, None, None, None, None, None, None, C.byref(dev))
        self._device = dev.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # (module globals may be gone at interpreter exit)
            lib.pafft_plan_destroy(h)
            self._h = None

    @property
    def radix(self):
        return self._radix

    @property
    def radices(self):
        """Per-axis radices (all equal for a pafft Radix plan)."""
        return list(self._radices)

    @property
    def dims(self):
        return list(self._dims)

    @property
    def total(self):
        return int(np.prod(self._dims))

    @property
    def precision(self):
        return self._precision

    @property
    def device(self):
        return self._device

    @property
    def depths(self):
        return [round(math.log(d, r)) if d > 1 else 0 for d, r in zip(self._dims, self._radices)]

    def describe(self):
        buf = C.create_string_buffer(8192)
        _check(lib.pafft_plan_describe(self._h, buf, 8192))
        return buf.value.decode()

    def num_passes(self):
        n = C.c_int()
        _check(lib.pafft_plan_num_passes(self._h, C.byref(n)))
        return n.value

    def key(self):
        return (tuple(self._radices), tuple(self._dims), self._precision, self._device)


class PreparedFilter:
    """Filter spectrum digit-reversed once for reuse (convolution.hpp:9-12)."""

    cache_hit = False

    def __init__(self, handle, plan):
        self._h = handle
        self._plan = plan  # keeps the plan (and its device tables) alive

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:
            lib.pafft_filter_destroy(h)
            self._h = None

    @property
    def ghat(self):
        """PreparedFilter::ghat in vec order, complex128 (bit-exact P*g)."""
        n = self._plan.total
        re, im = np.empty(n), np.empty(n)
        _check(lib.pafft_filter_ghat_split(self._h, _p(re), _p(im)))
        return re + 1j * im

    @property
    def key(self):
        return self._plan.key()

    def device_ghat_ptr(self, scaled=False):
        return (lib.pafft_filter_device_ghat_scaled if scaled else lib.pafft_filter_device_ghat)(self._h)


# ----------------------------------------------------- host array helpers
def _shape_text(dims):
    return "(" + ", ".join(str(d) for d in dims) + ")"


def _vec_split(a, plan):
    """module.cpp:46-52 buffer_for_plan: shape check + C order -> vec repack."""
    a = np.asarray(a)
    if list(a.shape) != plan.dims:
        raise Error(f"array shape {_shape_text(a.shape)} does not match plan shape {_shape_text(plan.dims)}")
    v = np.asarray(a, dtype=np.complex128).ravel(order="F")
    return np.ascontiguousarray(v.real), np.ascontiguousarray(v.imag)


def _from_vec(re, im, plan):
    """module.cpp:54-62 array_from_buffer: vec -> C order."""
    v = re + 1j * im
    return np.ascontiguousarray(v.reshape(plan.dims, order="F"))


def _transform(op, a, plan):
    re, im = _vec_split(a, plan)
    _check(lib.pafft_transform_split(plan._h, op, _p(re), _p(im), 1))
    return _from_vec(re, im, plan)


def fft_forward(a, plan):
    """Forward DFT in natural order (transform.cpp:8-11)."""
    return _transform(0, a, plan)


def fft_backward(a, plan):
    """Inverse DFT in natural order, normalized by 1/n (transform.cpp:13-16)."""
    return _transform(1, a, plan)


def fft_forward_unordered(a, plan):
    """Forward stage ladders only; expects digit-reversed input (transform.cpp:18-20)."""
    return _transform(2, a, plan)


def fft_backward_unordered(a, plan):
    """Conjugate stage ladders plus 1/n; expects digit-reversed input (transform.cpp:22-26)."""
    return _transform(3, a, plan)


def fft_transposed(a, plan):
    """A^T alone: the DIF ladder, spectrum left digit-reversed."""
    return _transform(4, a, plan)


def permute(a, plan):
    """permute_tensor (permutation.cpp:46-90)."""
    return _transform(5, a, plan)


def prepare_filter(g, plan):
    """Digit-reverse a natural-order filter spectrum once, offline (convolution.cpp:9-14)."""
    re, im = _vec_split(g, plan)
    h = C.c_void_p()
    _check(lib.pafft_prepare_filter_split(plan._h, _p(re), _p(im), C.byref(h)))
    return PreparedFilter(h, plan)


def filter_from_impulse(h, plan):
    """Spectrum of an impulse response: g = fft_forward(h) (convolution.cpp:16-21)."""
    return fft_forward(h, plan)


def convolve_standard(x, g, plan):
    """Transform, pointwise multiply, inverse transform: two reorderings (convolution.cpp:37-43)."""
    xr, xi = _vec_split(x, plan)
    gr, gi = _vec_split(g, plan)
    _check(lib.pafft_convolve_standard_split(plan._h, _p(gr), _p(gi), _p(xr), _p(xi), 1))
    return _from_vec(xr, xi, plan)


def convolve_permfree(x, filter, plan):
    """Circular convolution with zero reordering passes (convolution.cpp:45-52)."""
    if not isinstance(filter, PreparedFilter):
        raise TypeError("filter must be a PreparedFilter")
    xr, xi = _vec_split(x, plan)
    _check(lib.pafft_convolve_permfree_split(plan._h, filter._h, _p(xr), _p(xi), 1))
    return _from_vec(xr, xi, plan)


def digit_reverse(j, radix, digits):
    """Reverse j's base-radix digit string of the given width (permutation.cpp:27-37)."""
    out = C.c_uint64()
    _check(lib.pafft_digit_reverse(int(j), int(radix), int(digits), C.byref(out)))
    return out.value


# ------------------------------------------------------------- cost models
_PER_LOG2 = {2: 5.0, 4: 4.25, 8: 4.08}


def estimate_flop(n, radix):
    """Butterfly FLOP model for one transform (bench.cpp:111-117); radix 3/5 use
    the generic (core_r + 6(r-1))/r per point per stage."""
    n = int(n)
    if n < 2:
        return 0.0
    if radix in _PER_LOG2:
        return _PER_LOG2[radix] * n * math.log2(n)
    core = {3: 16.0, 5: 48.0}[radix]
    return (core + 6.0 * (radix - 1)) / radix * n * math.log(n, radix)


def estimate_ai(n, radix, permutation_free):
    """Arithmetic-intensity model, FLOP per byte (bench.cpp:119-126)."""
    n = int(n)
    if n < 2:
        return 0.0
    logr = math.log2(n) / math.log2(radix)
    elements = 2.0 * n * logr if permutation_free else 2.0 * n * (1.0 + logr)
    return estimate_flop(n, radix) / (16.0 * elements)


# ---------------------------------------------------------------- counters
def permutation_pass_count():
    return lib.pafft_permutation_pass_count()


def reset_permutation_pass_count():
    lib.pafft_reset_permutation_pass_count()


def kernel_launch_count():
    return lib.pafft_kernel_launch_count()


def dynamic_launch_count():
    return lib.pafft_dynamic_launch_count()


# ============================================================= device API
def _torch():
    import torch

    return torch


def _stream_ptr(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _dtype_ok(t, plan):
    torch = _torch()
    want = torch.complex128 if plan.precision == F64 else torch.complex64
    if t.dtype != want or not t.is_cuda or not t.is_contiguous():
        raise Error(f"expected a contiguous CUDA {want} tensor, got {t.dtype} on {t.device}")
    if t.numel() % plan.total:
        raise LengthMismatch(f"buffer length {t.numel()} is not a multiple of plan total {plan.total}")
    return t.numel() // plan.total


def convolve_permfree_(x, filter, plan, stream=None):
    """In-place device hot path: x (batch x N, vec order) <- conv(x). Async."""
    b = _dtype_ok(x, plan)
    _check(lib.pafft_convolve_permfree(plan._h, filter._h, C.c_void_p(x.data_ptr()), b, _stream_ptr(stream)))
    return x


def convolve_permfree_out(x, y, filter, plan, stream=None):
    """Out-of-place device hot path: y <- conv(x); x unchanged. Async."""
    b = _dtype_ok(x, plan)
    if _dtype_ok(y, plan) != b:
        raise LengthMismatch("x and y batch differ")
    _check(lib.pafft_convolve_permfree_oop(plan._h, filter._h, C.c_void_p(x.data_ptr()),
                                           C.c_void_p(y.data_ptr()), b, _stream_ptr(stream)))
    return y


def convolve_permfree_host(x, filter, plan):
    """Host-buffer path (numpy complex, vec order, ideally pinned): H2D, conv, D2H
    pipelined in chunks; synchronous; in place."""
    want = np.complex128 if plan.precision == F64 else np.complex64
    if x.dtype != want or not x.flags.c_contiguous:
        raise Error(f"expected a C-contiguous {want} array")
    if x.size % plan.total:
        raise LengthMismatch("host buffer is not a whole number of signals")
    _check(lib.pafft_convolve_permfree_host(plan._h, filter._h, C.c_void_p(x.ctypes.data), x.size // plan.total))
    return x


def convolve_standard_(x, g, plan, stream=None):
    """Device standard-order comparator: g natural-order spectrum (N,), x in place."""
    b = _dtype_ok(x, plan)
    _check(lib.pafft_convolve_standard(plan._h, C.c_void_p(g.data_ptr()), C.c_void_p(x.data_ptr()), b,
                                       _stream_ptr(stream)))
    return x


def _dev_op(fn, x, plan, stream=None):
    b = _dtype_ok(x, plan)
    _check(fn(plan._h, C.c_void_p(x.data_ptr()), b, _stream_ptr(stream)))
    return x


def fft_forward_(x, plan, stream=None):
    return _dev_op(lib.pafft_fft_forward, x, plan, stream)


def fft_backward_(x, plan, stream=None):
    return _dev_op(lib.pafft_fft_backward, x, plan, stream)


def fft_forward_unordered_(x, plan, stream=None):
    return _dev_op(lib.pafft_fft_forward_unordered, x, plan, stream)


def fft_backward_unordered_(x, plan, stream=None):
    return _dev_op(lib.pafft_fft_backward_unordered, x, plan, stream)


def fft_transposed_(x, plan, stream=None):
    return _dev_op(lib.pafft_fft_transposed, x, plan, stream)


def permute_(x, plan, stream=None):
    return _dev_op(lib.pafft_permute, x, plan, stream)


def prepare_filter_device(g, plan, stream=None):
    """prepare_filter from a device natural-order spectrum (one device permutation)."""
    _dtype_ok(g, plan)
    h = C.c_void_p()
    _check(lib.pafft_prepare_filter_device(plan._h, C.c_void_p(g.data_ptr()), _stream_ptr(stream), C.byref(h)))
    return PreparedFilter(h, plan)


def prepare_filter_from_impulse(h, plan, stream=None, cache=False):
    """ghat = A^T h directly on the device: zero permutation passes.

    cache=True: reuse a spectrum already prepared from the same impulse bytes
    for any plan with the same key (filter-spectrum cache across plans); the
    returned filter's ``cache_hit`` says whether it was shared."""
    _dtype_ok(h, plan)
    out = C.c_void_p()
    if cache:
        hit = C.c_int()
        _check(lib.pafft_prepare_filter_from_impulse_cached(plan._h, C.c_void_p(h.data_ptr()), _stream_ptr(stream),
                                                             C.byref(out), C.byref(hit)))
        f = PreparedFilter(out, plan)
        f.cache_hit = bool(hit.value)
        return f
    _check(lib.pafft_prepare_filter_from_impulse_device(plan._h, C.c_void_p(h.data_ptr()), _stream_ptr(stream),
                                                         C.byref(out)))
    return PreparedFilter(out, plan)


def filter_cache_stats():
    """(hits, misses, live entries) of the filter-spectrum cache."""
    a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
    lib.pafft_filter_cache_stats(C.byref(a), C.byref(b), C.byref(c))
    return a.value, b.value, c.value


def empty_filter(plan):
    """A filter bound to `plan` with uninitialised ghat (to receive a broadcast)."""
    h = C.c_void_p()
    _check(lib.pafft_filter_create_empty(plan._h, C.byref(h)))
    return PreparedFilter(h, plan)


def filter_device_tensor(filter, scaled=False):
    """Zero-copy torch view of a filter's device ghat (for NCCL broadcast)."""
    torch = _torch()
    plan = filter._plan
    ptr = filter.device_ghat_ptr(scaled)
    typestr = "<c16" if plan.precision == F64 else "<c8"

    class _View:
        __cuda_array_interface__ = {"shape": (plan.total,), "typestr": typestr, "data": (ptr, False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_View(), device=f"cuda:{plan.device}")


def broadcast_filter_nccl(filters, root=0, comms=None, streams=None):
    """pafft_filter_broadcast: NCCL broadcast of filters[root]'s prepared
    spectrum into the other filters (distinct devices, same plan key).
    Single process: comms=None lets the library build the communicator clique.
    One process per GPU: pass this rank's filter and its ncclComm_t handle."""
    n = len(filters)
    arr = (C.c_void_p * n)(*[f._h for f in filters])
    cm = (C.c_void_p * n)(*comms) if comms is not None else None
    ss = (C.c_void_p * n)(*[_stream_ptr(s) for s in streams]) if streams is not None else None
    _check(lib.pafft_filter_broadcast(arr, n, int(root), cm, ss))


def filter_sync_scaled(filter, stream=None):
    _check(lib.pafft_filter_sync_scaled(filter._h, _stream_ptr(stream)))


def fill_uniform(seed, n):
    """SplitMix64 U(-1,1) re/im, interleaved complex128 (bench.cpp:22-49)."""
    out = np.empty(n, dtype=np.complex128)
    lib.pafft_fill_uniform(int(seed), int(n), out.ctypes.data_as(_dp))
    return out


def fill_normal(seed, n):
    """SplitMix64 + Box-Muller N(0,1) re/im, interleaved complex128."""
    out = np.empty(n, dtype=np.complex128)
    lib.pafft_fill_normal(int(seed), int(n), out.ctypes.data_as(_dp))
    return out
