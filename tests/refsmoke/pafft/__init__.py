"""`pafft` alias of the product package, so the reference's own Python smoke
test (tests/python/test_smoke.py, copied unchanged into oracle/_ref/ by
oracle/Makefile) runs against the GPU path: the reference module's names
(python/pafft/__init__.py, python/src/module.cpp:73-149) all come from
paper_2506_12718_b200."""
from paper_2506_12718_b200 import (  # noqa: F401
    Plan,
    PreparedFilter,
    convolve_permfree,
    convolve_standard,
    digit_reverse,
    estimate_ai,
    estimate_flop,
    fft_backward,
    fft_backward_unordered,
    fft_forward,
    fft_forward_unordered,
    filter_from_impulse,
    prepare_filter,
)
