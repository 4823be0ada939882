set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/first_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/first_pytest.log 2>&1
for c in 2 1 3 4 5; do timeout 600 python bench.py --config $c --no-e2e --no-cpu > gpurun_out/first_bench_c$c.json 2> gpurun_out/first_bench_c$c.err; done
timeout 600 python bench.py --config 5 --precision f32 --no-e2e --no-cpu > gpurun_out/first_bench_c5f32.json 2> gpurun_out/first_bench_c5f32.err
