# Round-2 evidence on the final code: GPU suite, smoke, default bench (+ sub-configs), reference arm,
# launch list of the headline step and one ncu --set full capture of its three pass kernels.
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=15 > gpurun_out/r2z_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2z_pytest.log
timeout 900 python bench.py > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2z_ref.json 2> gpurun_out/r2z_ref.err
CMD="python bench.py --config 2 --steps 3 --warmup 3 --no-e2e --no-cpu --no-sub"
timeout 300 $CMD > gpurun_out/r2z_plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pass_kernel -c 40 --csv --log-file gpurun_out/r2z_launches.csv $CMD > gpurun_out/r2z_ncu_launch.log 2>&1
CMD1="python bench.py --config 2 --steps 1 --warmup 1 --no-e2e --no-cpu --no-sub"
timeout 300 $CMD1 > gpurun_out/r2z_plain1.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pass_kernel -s 2 -c 3 -o gpurun_out/r2z_c2 $CMD1 > gpurun_out/r2z_ncu_full.log 2>&1
