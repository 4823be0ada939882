bash tools/ab.sh "2 5 1 3 4" paper_2506_12718_b200/libpafft_b200.so ab/libdirect.so > gpurun_out/r2j_ab.log 2>&1
PAFFT_LIB=ab/libdirect.so timeout 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -x > gpurun_out/r2j_pytest.log 2>&1
