mkdir -p gpurun_out
bash tools/ab.sh "2" paper_2506_12718_b200/libpafft_b200.so ab/libgdiv3.so > gpurun_out/s5k_gdiv_ab.log 2>&1
cat gpurun_out/s5k_gdiv_ab.log
PAFFT_LIB=ab/libgdiv3.so timeout 600 python -m pytest tests/test_gpu_configs.py -x -q -m gpu -k "config2 or 2" > gpurun_out/s5k_pytest.log 2>&1; tail -3 gpurun_out/s5k_pytest.log
