for rep in 1 2; do
for c in 4 1 2 3; do bash tools/env_sweep.sh $c f64 "PAFFT_WIDE=1" "PAFFT_WIDE=0"; done
done > gpurun_out/wide_ab.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/wide_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/wide_pytest.log
