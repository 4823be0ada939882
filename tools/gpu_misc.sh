timeout 600 python -m pytest tests/test_gpu_edges.py -m gpu -q -k wide > gpurun_out/misc_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/misc_pytest.log
bash tools/ops_table.sh
