# PDL on/off A/B for configs 1, 2, 5 (+ f32), twice each
for rep in 1 2; do
bash tools/env_sweep.sh 1 f64 "PAFFT_PDL=0" "PAFFT_PDL=1"
bash tools/env_sweep.sh 2 f64 "PAFFT_PDL=0" "PAFFT_PDL=1"
bash tools/env_sweep.sh 5 f64 "PAFFT_PDL=0" "PAFFT_PDL=1"
bash tools/env_sweep.sh 3 f64 "PAFFT_PDL=0" "PAFFT_PDL=1"
bash tools/env_sweep.sh 1 f32 "PAFFT_PDL=0" "PAFFT_PDL=1"
done > gpurun_out/r2i_pdl.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_fuzz.py -m gpu -q -x > gpurun_out/r2i_pytest.log 2>&1
