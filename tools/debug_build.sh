#!/bin/bash
# Device-assert build (PAFFT_DEBUG: tile geometry + shared-memory index checks)
# into ab/libdebug.so, then the GPU suite against it:
#   bash tools/debug_build.sh && PAFFT_LIB=ab/libdebug.so python -m pytest tests -m gpu
set -e
cd "$(dirname "$0")/.."
PAFFT_NVCC_EXTRA="-DPAFFT_DEBUG" python -c "import __graft_entry__ as g; g.build()"
mkdir -p ab && cp paper_2506_12718_b200/libpafft_b200.so ab/libdebug.so
python -c "import __graft_entry__ as g; g.build()"   # restore the release build
