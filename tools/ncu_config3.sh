CMD="python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-sub"
timeout 300 $CMD > gpurun_out/r2l_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pass_kernel -s 2 -c 3 -o gpurun_out/r2l_c3 $CMD > gpurun_out/r2l_ncu.log 2>&1
