# the GPU suite against the device-assert build (tile geometry + shared-memory index checks)
PAFFT_LIB=ab/libdebug.so timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/debug_suite.log 2>&1; echo "rc=$?" >> gpurun_out/debug_suite.log
