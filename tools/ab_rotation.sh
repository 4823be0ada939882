bash tools/ab.sh "4 1" paper_2506_12718_b200/libpafft_b200.so ab/libnorot.so > gpurun_out/rotc_ab.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py -m gpu -q -x > gpurun_out/rotc_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rotc_pytest.log
