"""Test-side checkers for the permutation-avoiding convolution path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package, and only as the checker (or the timed CPU comparator).  The product
package ``paper_2506_12718_b200`` never imports it.

Two checkers live here, both over ctypes:

* :class:`Oracle` -- ``liboracle.so``, the C restatement of the reference's
  ladders / permutation / convolution at general radix (``pafft_oracle.c``;
  each function cites the reference file:line it restates).
* :class:`Ref` -- ``_ref/libpafft_ref.so``, the UNMODIFIED reference library
  compiled from ``/root/reference/proj/src`` (radix 2/4/8 only, as in the
  reference).  Absent when the reference was never built here.

All arrays are flat complex128 numpy arrays in vec order (first index
fastest, core.hpp:26-27).  Split re/im conversion happens here.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libpafft_ref.so")

FORWARD, CONJUGATE, TRANSPOSED = 0, 1, 2

_dp = C.POINTER(C.c_double)
_sz = C.c_size_t


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle status {code} {msg}".strip())
        self.code = code


def build():
    """Compile liboracle.so (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "-f", "Makefile"], check=True)


def _split(x):
    x = np.ascontiguousarray(x, dtype=np.complex128).reshape(-1)
    return np.ascontiguousarray(x.real), np.ascontiguousarray(x.imag)


def _p(a):
    return a.ctypes.data_as(_dp)


def _dims(dims):
    arr = (_sz * len(dims))(*dims)
    return arr, len(dims)


class _OrcPlan(C.Structure):
    _fields_ = [("radix", C.c_uint), ("rank", C.c_int), ("dims", _sz * 8), ("depth", C.c_uint * 8),
                ("total", _sz), ("tw_re", _dp * 8), ("tw_im", _dp * 8), ("rev", C.POINTER(C.c_uint32) * 8),
                ("radices", C.c_uint * 8)]


class Oracle:
    """ctypes view of liboracle.so (the restatement)."""

    def __init__(self, path=LIB):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.L = L
        L.orc_plan_create.argtypes = [C.c_uint, C.POINTER(_sz), C.c_int, C.POINTER(C.POINTER(_OrcPlan))]
        L.orc_plan_create_mixed.argtypes = [C.POINTER(C.c_uint), C.POINTER(_sz), C.c_int,
                                             C.POINTER(C.POINTER(_OrcPlan))]
        L.orc_plan_destroy.argtypes = [C.POINTER(_OrcPlan)]
        for name in ("orc_permute_tensor", "orc_convolve_permfree_batch"):
            pass
        L.orc_permute_tensor.argtypes = [C.POINTER(_OrcPlan), _dp, _dp]
        L.orc_butterfly_line.argtypes = [C.POINTER(_OrcPlan), _sz, C.c_int, _dp, _dp, _sz]
        L.orc_butterfly_tensor.argtypes = [C.POINTER(_OrcPlan), C.c_int, _dp, _dp]
        L.orc_prepare_filter.argtypes = [C.POINTER(_OrcPlan), _dp, _dp, _dp, _dp]
        L.orc_filter_from_impulse.argtypes = [C.POINTER(_OrcPlan), _dp, _dp, _dp, _dp]
        L.orc_convolve_permfree.argtypes = [C.POINTER(_OrcPlan), _dp, _dp, _dp, _dp]
        L.orc_convolve_standard.argtypes = [C.POINTER(_OrcPlan), _dp, _dp, _dp, _dp]
        L.orc_fft_forward.argtypes = [C.POINTER(_OrcPlan), _dp, _dp]
        L.orc_fft_backward.argtypes = [C.POINTER(_OrcPlan), _dp, _dp]
        L.orc_convolve_permfree_batch.argtypes = [C.POINTER(_OrcPlan), _dp, _dp, _dp, _dp, _sz, C.c_int]
        L.orc_convolve_permfree_fast_batch.argtypes = [C.POINTER(_OrcPlan), _dp, _dp, _dp, _dp, _sz, C.c_int]
        L.orc_naive_dft_tensor.argtypes = [C.POINTER(_sz), C.c_int, C.c_int, _dp, _dp, _dp, _dp]
        L.orc_naive_circular_convolution.argtypes = [C.POINTER(_sz), C.c_int, _dp, _dp, _dp, _dp, _dp, _dp]
        L.orc_digit_reverse.argtypes = [C.c_uint64, C.c_uint, C.c_uint, C.POINTER(C.c_uint64)]
        L.orc_permutation_pass_count.restype = C.c_uint64
        L.orc_fill_uniform.argtypes = [C.c_uint64, _sz, _dp, _dp]
        L.orc_fill_normal.argtypes = [C.c_uint64, _sz, _dp, _dp]
        L.orc_splitmix64_next.argtypes = [C.POINTER(C.c_uint64)]
        L.orc_splitmix64_next.restype = C.c_uint64

    # -- plans -----------------------------------------------------------
    def plan(self, radix, dims):
        return OraclePlan(self, radix, dims)

    # -- plan-free helpers ------------------------------------------------
    def digit_reverse(self, j, radix, digits):
        out = C.c_uint64()
        st = self.L.orc_digit_reverse(j, radix, digits, C.byref(out))
        if st:
            raise OracleError(st, "digit_reverse")
        return out.value

    def naive_dft(self, x, dims, backward=False):
        xr, xi = _split(x)
        yr, yi = np.empty_like(xr), np.empty_like(xi)
        d, rank = _dims(dims)
        self.L.orc_naive_dft_tensor(d, rank, int(backward), _p(xr), _p(xi), _p(yr), _p(yi))
        return yr + 1j * yi

    def naive_conv(self, x, h, dims):
        xr, xi = _split(x)
        hr, hi = _split(h)
        yr, yi = np.empty_like(xr), np.empty_like(xi)
        d, rank = _dims(dims)
        self.L.orc_naive_circular_convolution(d, rank, _p(xr), _p(xi), _p(hr), _p(hi), _p(yr), _p(yi))
        return yr + 1j * yi

    def fill_uniform(self, seed, n):
        re, im = np.empty(n), np.empty(n)
        self.L.orc_fill_uniform(seed, n, _p(re), _p(im))
        return re + 1j * im

    def fill_normal(self, seed, n):
        re, im = np.empty(n), np.empty(n)
        self.L.orc_fill_normal(seed, n, _p(re), _p(im))
        return re + 1j * im

    def fill_signals_split(self, uniform, seeds, n, threads=None):
        """Signals seeds[i] -> rows i of (re, im) float64 arrays (SplitMix64,
        the same bytes as the product generator), generated across threads."""
        import concurrent.futures as cf
        count = len(seeds)
        re, im = np.empty((count, n)), np.empty((count, n))
        fn = self.L.orc_fill_uniform if uniform else self.L.orc_fill_normal

        def one(i):
            fn(seeds[i], n, _p(re[i]), _p(im[i]))

        if count <= 1:
            for i in range(count):
                one(i)
        else:
            with cf.ThreadPoolExecutor(threads or min(count, os.cpu_count() or 4)) as ex:
                list(ex.map(one, range(count)))
        return re, im

    def pass_count(self):
        return self.L.orc_permutation_pass_count()

    def reset_pass_count(self):
        self.L.orc_reset_permutation_pass_count()


class OraclePlan:
    def __init__(self, orc, radix, dims):
        self.orc, self.L = orc, orc.L
        self.radix, self.dims = radix, list(dims)
        self.total = int(np.prod(self.dims)) if self.dims else 0
        d, rank = _dims(self.dims)
        ptr = C.POINTER(_OrcPlan)()
        if isinstance(radix, (list, tuple)):  # per-axis radices
            rs = (C.c_uint * max(1, len(radix)))(*radix)
            if len(radix) != rank:
                raise OracleError(-1, f"{len(radix)} radices for {rank} dims")
            st = self.L.orc_plan_create_mixed(rs, d, rank, C.byref(ptr))
        else:
            st = self.L.orc_plan_create(radix, d, rank, C.byref(ptr))
        if st:
            raise OracleError(st, f"plan_create(r={radix}, dims={dims})")
        self.ptr = ptr

    def __del__(self):
        if getattr(self, "ptr", None):
            self.L.orc_plan_destroy(self.ptr)
            self.ptr = None

    def _inplace(self, fn, x, *extra):
        xr, xi = _split(x)
        st = fn(self.ptr, *extra, _p(xr), _p(xi))
        if st:
            raise OracleError(st)
        return xr + 1j * xi

    def permute(self, x):
        return self._inplace(self.L.orc_permute_tensor, x)

    def butterfly_tensor(self, x, variant):
        return self._inplace(self.L.orc_butterfly_tensor, x, variant)

    def butterfly_line(self, x, dim, variant):
        xr, xi = _split(x)
        st = self.L.orc_butterfly_line(self.ptr, dim, variant, _p(xr), _p(xi), len(xr))
        if st:
            raise OracleError(st)
        return xr + 1j * xi

    def prepare_filter(self, g):
        gr, gi = _split(g)
        orr, oi = np.empty_like(gr), np.empty_like(gi)
        self.L.orc_prepare_filter(self.ptr, _p(gr), _p(gi), _p(orr), _p(oi))
        return orr + 1j * oi

    def filter_from_impulse(self, h):
        hr, hi = _split(h)
        gr, gi = np.empty_like(hr), np.empty_like(hi)
        self.L.orc_filter_from_impulse(self.ptr, _p(hr), _p(hi), _p(gr), _p(gi))
        return gr + 1j * gi

    def fft_forward(self, x):
        return self._inplace(self.L.orc_fft_forward, x)

    def fft_backward(self, x):
        return self._inplace(self.L.orc_fft_backward, x)

    def convolve_permfree(self, x, ghat):
        gr, gi = _split(ghat)
        return self._inplace(self.L.orc_convolve_permfree, x, _p(gr), _p(gi))

    def convolve_standard(self, x, g):
        gr, gi = _split(g)
        return self._inplace(self.L.orc_convolve_standard, x, _p(gr), _p(gi))

    def convolve_permfree_batch_split(self, ghat_re, ghat_im, re, im, batch, threads):
        """In place on caller-owned split arrays (no copies): the CPU comparator."""
        return self.L.orc_convolve_permfree_batch(self.ptr, _p(ghat_re), _p(ghat_im), _p(re), _p(im),
                                                  batch, threads)

    def convolve_permfree_fast_batch_split(self, ghat_re, ghat_im, re, im, batch, threads):
        """Reference-style specialised ladders (fast_ladders.c; 1-D, radix 2/3/4/5):
        the CPU stand-in for pafft at radix 3/5."""
        st = self.L.orc_convolve_permfree_fast_batch(self.ptr, _p(ghat_re), _p(ghat_im), _p(re), _p(im),
                                                     batch, threads)
        if st:
            raise OracleError(st, "convolve_permfree_fast_batch")
        return st


class Ref:
    """ctypes view of the reference library compiled into oracle/_ref."""

    @staticmethod
    def available(path=REF_LIB):
        return os.path.exists(path)

    def __init__(self, path=REF_LIB):
        L = C.CDLL(path)
        self.L = L
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_plan_create.argtypes = [C.c_uint, C.POINTER(_sz), C.c_int, C.POINTER(vp)]
        L.ref_plan_destroy.argtypes = [vp]
        L.ref_digit_reverse.argtypes = [C.c_uint64, C.c_uint, C.c_uint, C.POINTER(C.c_uint64)]
        L.ref_permutation_pass_count.restype = C.c_uint64
        L.ref_permute_tensor.argtypes = [vp, _dp, _dp]
        L.ref_butterfly_line.argtypes = [vp, _sz, C.c_int, _dp, _dp, _sz]
        L.ref_butterfly_tensor.argtypes = [vp, C.c_int, _dp, _dp]
        L.ref_prepare_filter.argtypes = [vp, _dp, _dp, _dp, _dp]
        L.ref_filter_from_impulse.argtypes = [vp, _dp, _dp, _dp, _dp]
        L.ref_convolve_permfree.argtypes = [vp, _dp, _dp, _dp, _dp]
        L.ref_convolve_standard.argtypes = [vp, _dp, _dp, _dp, _dp]
        L.ref_naive_circular_convolution.argtypes = [C.POINTER(_sz), C.c_int, _dp, _dp, _dp, _dp, _dp, _dp]
        L.ref_naive_dft_tensor.argtypes = [C.POINTER(_sz), C.c_int, C.c_int, _dp, _dp, _dp, _dp]
        L.ref_batch_create.argtypes = [vp, _dp, _dp, _dp, _dp, _sz]
        L.ref_batch_create.restype = vp
        L.ref_batch_run.argtypes = [vp, C.c_int]
        L.ref_batch_run.restype = C.c_double
        L.ref_batch_read.argtypes = [vp, _sz, _dp, _dp]
        L.ref_batch_destroy.argtypes = [vp]

    def _check(self, st, what):
        if st:
            raise OracleError(st, f"{what}: {self.L.ref_last_error().decode()}")

    def plan(self, radix, dims):
        return RefPlan(self, radix, dims)

    def digit_reverse(self, j, radix, digits):
        out = C.c_uint64()
        self._check(self.L.ref_digit_reverse(j, radix, digits, C.byref(out)), "digit_reverse")
        return out.value

    def naive_conv(self, x, h, dims):
        xr, xi = _split(x)
        hr, hi = _split(h)
        yr, yi = np.empty_like(xr), np.empty_like(xi)
        d, rank = _dims(dims)
        self._check(self.L.ref_naive_circular_convolution(d, rank, _p(xr), _p(xi), _p(hr), _p(hi), _p(yr), _p(yi)),
                    "naive_conv")
        return yr + 1j * yi

    def naive_dft(self, x, dims, backward=False):
        xr, xi = _split(x)
        yr, yi = np.empty_like(xr), np.empty_like(xi)
        d, rank = _dims(dims)
        self._check(self.L.ref_naive_dft_tensor(d, rank, int(backward), _p(xr), _p(xi), _p(yr), _p(yi)), "dft")
        return yr + 1j * yi


class RefPlan:
    def __init__(self, ref, radix, dims):
        self.ref, self.L = ref, ref.L
        self.radix, self.dims = radix, list(dims)
        self.total = int(np.prod(self.dims))
        d, rank = _dims(self.dims)
        h = C.c_void_p()
        ref._check(self.L.ref_plan_create(radix, d, rank, C.byref(h)), f"plan_create({radix},{dims})")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_plan_destroy(self.h)
            self.h = None

    def _inplace(self, fn, x, *extra):
        xr, xi = _split(x)
        self.ref._check(fn(self.h, *extra, _p(xr), _p(xi)), fn.__name__)
        return xr + 1j * xi

    def permute(self, x):
        return self._inplace(self.L.ref_permute_tensor, x)

    def butterfly_tensor(self, x, variant):
        return self._inplace(self.L.ref_butterfly_tensor, x, variant)

    def prepare_filter(self, g):
        gr, gi = _split(g)
        orr, oi = np.empty_like(gr), np.empty_like(gi)
        self.ref._check(self.L.ref_prepare_filter(self.h, _p(gr), _p(gi), _p(orr), _p(oi)), "prepare_filter")
        return orr + 1j * oi

    def filter_from_impulse(self, h):
        hr, hi = _split(h)
        gr, gi = np.empty_like(hr), np.empty_like(hi)
        self.ref._check(self.L.ref_filter_from_impulse(self.h, _p(hr), _p(hi), _p(gr), _p(gi)), "ffi")
        return gr + 1j * gi

    def convolve_permfree(self, x, ghat):
        gr, gi = _split(ghat)
        return self._inplace(self.L.ref_convolve_permfree, x, _p(gr), _p(gi))

    def convolve_standard(self, x, g):
        gr, gi = _split(g)
        return self._inplace(self.L.ref_convolve_standard, x, _p(gr), _p(gi))

    def batch(self, ghat, signals):
        """Stage `signals` (batch x total complex) for timed batched runs."""
        s = np.ascontiguousarray(signals, dtype=np.complex128).reshape(-1)
        return self.batch_split(ghat, np.ascontiguousarray(s.real), np.ascontiguousarray(s.imag))

    def batch_split(self, ghat, re, im):
        """Stage split signals (re, im: batch x total float64, C-contiguous)."""
        gr, gi = _split(ghat)
        re = np.ascontiguousarray(re, dtype=np.float64)
        im = np.ascontiguousarray(im, dtype=np.float64)
        n = re.size // self.total
        h = self.L.ref_batch_create(self.h, _p(gr), _p(gi), _p(re), _p(im), n)
        if not h:
            raise OracleError(-1, "ref_batch_create: " + self.L.ref_last_error().decode())
        return RefBatch(self, h, n)


class RefBatch:
    def __init__(self, plan, h, n):
        self.plan, self.h, self.n = plan, h, n

    def run(self, threads):
        return self.plan.L.ref_batch_run(self.h, threads)

    def read(self, i):
        re, im = np.empty(self.plan.total), np.empty(self.plan.total)
        self.plan.L.ref_batch_read(self.h, i, _p(re), _p(im))
        return re + 1j * im

    def __del__(self):
        if getattr(self, "h", None):
            self.plan.L.ref_batch_destroy(self.h)
            self.h = None


def rel_l2(a, b):
    a = np.asarray(a).reshape(-1)
    b = np.asarray(b).reshape(-1)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))
