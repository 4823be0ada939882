#!/bin/bash
# Profiling build with the per-CTA pass trace compiled in: ab/libtrace.so
# (use: PAFFT_LIB=ab/libtrace.so PAFFT_PASS_TRACE=1 python tools/pass_trace.py --config 2)
PAFFT_BUILD_TAG=trace PAFFT_NVCC_EXTRA=-DPAFFT_TRACE=1 python paper_2506_12718_b200/build.py
