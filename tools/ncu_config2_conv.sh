# ncu --set full of the config-2 CONV kernel (source view for shared-memory conflicts)
CMD="python bench.py --config 2 --steps 1 --warmup 1 --no-e2e --no-cpu --no-sub"
timeout 300 $CMD > gpurun_out/r2g_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pass_kernel -s 3 -c 1 -o gpurun_out/r2g_conv2187 $CMD > gpurun_out/r2g_ncu.log 2>&1
