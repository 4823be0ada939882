bash tools/ab.sh "3" paper_2506_12718_b200/libpafft_b200.so ab/libnorot.so > gpurun_out/r2m_ab.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2m_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_pytest.log
bash tools/env_sweep.sh 3 f32 "PAFFT_X=1" >> gpurun_out/r2m_ab.log 2>&1
PAFFT_LIB=ab/libnorot.so bash tools/env_sweep.sh 3 f32 "PAFFT_X=0" >> gpurun_out/r2m_ab.log 2>&1
