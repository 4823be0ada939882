# GPU suite (with per-test durations) + the reference acceptance gate log.
set -x
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=25 > gpurun_out/r2c_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2c_pytest.log
