#!/bin/bash
# Device-assert build (PAFFT_DEBUG: tile geometry + shared-memory index checks)
# into ab/libdebug.so (its own object dir), then the GPU suite against it:
#   bash tools/debug_build.sh && PAFFT_LIB=ab/libdebug.so python -m pytest tests -m gpu
set -e
cd "$(dirname "$0")/.."
PAFFT_BUILD_TAG=debug PAFFT_NVCC_EXTRA="-DPAFFT_DEBUG" python paper_2506_12718_b200/build.py
