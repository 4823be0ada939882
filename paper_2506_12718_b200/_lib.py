"""ctypes binding of libpafft_b200.so (the C ABI in include/pafft_b200.h).

The library is built in-tree by ``paper_2506_12718_b200.build``.  If it is
missing this module raises immediately: there is no CPU fallback for any
operation of this package.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PAFFT_LIB") or os.path.join(HERE, "libpafft_b200.so")  # PAFFT_LIB: A/B builds
if not os.path.isabs(LIB_PATH) and not os.path.exists(LIB_PATH):
    # a relative PAFFT_LIB names a file under the repo root (e.g. ab/lib<tag>.so)
    LIB_PATH = os.path.join(os.path.dirname(HERE), LIB_PATH)

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(or python paper_2506_12718_b200/build.py); this package has no CPU fallback")

lib = C.CDLL(LIB_PATH)

_vp = C.c_void_p
_sz = C.c_size_t
_dp = C.POINTER(C.c_double)
_st = C.c_int

# name -> (argtypes, restype)
_SIGS = {
    "pafft_last_error": ([], C.c_char_p),
    "pafft_last_error_dim": ([C.POINTER(_sz), C.POINTER(_sz)], None),
    "pafft_build_info": ([], C.c_char_p),
    "pafft_plan_create": ([C.c_uint, C.POINTER(_sz), C.c_int, C.c_int, C.c_int, C.POINTER(_vp)], _st),
    "pafft_plan_create_mixed": ([C.POINTER(C.c_uint), C.POINTER(_sz), C.c_int, C.c_int, C.c_int, C.POINTER(_vp)],
                                _st),
    "pafft_plan_radices": ([_vp, C.POINTER(C.c_uint)], _st),
    "pafft_plan_destroy": ([_vp], _st),
    "pafft_plan_info": ([_vp, C.POINTER(C.c_uint), C.POINTER(C.c_int), C.POINTER(_sz), C.POINTER(C.c_uint),
                         C.POINTER(_sz), C.POINTER(C.c_int), C.POINTER(C.c_int)], _st),
    "pafft_plan_num_passes": ([_vp, C.POINTER(C.c_int)], _st),
    "pafft_plan_describe": ([_vp, C.c_char_p, _sz], _st),
    "pafft_digit_reverse": ([C.c_uint64, C.c_uint, C.c_uint, C.POINTER(C.c_uint64)], _st),
    "pafft_prepare_filter_split": ([_vp, _dp, _dp, C.POINTER(_vp)], _st),
    "pafft_filter_from_prepared_split": ([_vp, _dp, _dp, C.POINTER(_vp)], _st),
    "pafft_convolve_permfree_split_if": ([_vp, _vp, _dp, _dp, _sz, _vp, _vp, C.POINTER(C.c_int)], _st),
    "pafft_prepare_filter_device": ([_vp, _vp, _vp, C.POINTER(_vp)], _st),
    "pafft_prepare_filter_from_impulse_device": ([_vp, _vp, _vp, C.POINTER(_vp)], _st),
    "pafft_prepare_filter_from_impulse_cached": ([_vp, _vp, _vp, C.POINTER(_vp), C.POINTER(C.c_int)], _st),
    "pafft_filter_cache_stats": ([C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)], None),
    "pafft_filter_destroy": ([_vp], _st),
    "pafft_filter_ghat_split": ([_vp, _dp, _dp], _st),
    "pafft_filter_device_ghat": ([_vp], _vp),
    "pafft_filter_device_ghat_scaled": ([_vp], _vp),
    "pafft_filter_sync_scaled": ([_vp, _vp], _st),
    "pafft_filter_create_empty": ([_vp, C.POINTER(_vp)], _st),
    "pafft_filter_broadcast": ([C.POINTER(_vp), C.c_int, C.c_int, C.POINTER(_vp), C.POINTER(_vp)], _st),
    "pafft_filter_matches": ([_vp, _vp], C.c_int),
    "pafft_convolve_permfree": ([_vp, _vp, _vp, _sz, _vp], _st),
    "pafft_convolve_permfree_oop": ([_vp, _vp, _vp, _vp, _sz, _vp], _st),
    "pafft_convolve_permfree_pass": ([_vp, _vp, _vp, _vp, _sz, C.c_int, _vp], _st),
    "pafft_plan_pass_info": ([_vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                              C.POINTER(C.c_int)], _st),
    "pafft_convolve_permfree_split": ([_vp, _vp, _dp, _dp, _sz], _st),
    "pafft_convolve_permfree_host": ([_vp, _vp, _vp, _sz], _st),
    "pafft_convolve_permfree_host_oop": ([_vp, _vp, _vp, _vp, _sz], _st),
    "pafft_convolve_standard": ([_vp, _vp, _vp, _sz, _vp], _st),
    "pafft_convolve_standard_split": ([_vp, _dp, _dp, _dp, _dp, _sz], _st),
    "pafft_fft_forward": ([_vp, _vp, _sz, _vp], _st),
    "pafft_fft_backward": ([_vp, _vp, _sz, _vp], _st),
    "pafft_fft_forward_unordered": ([_vp, _vp, _sz, _vp], _st),
    "pafft_fft_backward_unordered": ([_vp, _vp, _sz, _vp], _st),
    "pafft_fft_transposed": ([_vp, _vp, _sz, _vp], _st),
    "pafft_permute": ([_vp, _vp, _sz, _vp], _st),
    "pafft_transform_split": ([_vp, C.c_int, _dp, _dp, _sz], _st),
    "pafft_filter_from_impulse_split": ([_vp, _dp, _dp, _dp, _dp], _st),
    "pafft_permutation_pass_count": ([], C.c_uint64),
    "pafft_reset_permutation_pass_count": ([], None),
    "pafft_kernel_launch_count": ([], C.c_uint64),
    "pafft_dynamic_launch_count": ([], C.c_uint64),
    "pafft_fill_uniform": ([C.c_uint64, _sz, _dp], None),
    "pafft_fill_normal": ([C.c_uint64, _sz, _dp], None),
}

for _name, (_args, _res) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)
