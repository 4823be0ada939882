# One ncu --set full capture of the three config-2 pass kernels (after the
# same command ran clean without ncu), plus per-config bench lines.
set -x
CMD="python bench.py --config 2 --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/plain_c2.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pass_kernel -s 3 -c 3 -o gpurun_out/prof_c2_final $CMD > gpurun_out/ncu_c2_final.log 2>&1
for c in 2 3 4; do timeout 600 python bench.py --config $c > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
