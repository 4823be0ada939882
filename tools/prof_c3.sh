set -x
CMD="python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pass_kernel -s 3 -c 3 -o gpurun_out/prof_c3 $CMD > gpurun_out/ncu_c3.log 2>&1
