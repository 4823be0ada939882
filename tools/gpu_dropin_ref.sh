timeout 1200 python -m pytest tests/test_gpu_dropin_ref.py tests/test_gpu_configs.py::test_cpp_dropin_program -m gpu -q -rs > gpurun_out/dropin_ref_pytest.log 2>&1
