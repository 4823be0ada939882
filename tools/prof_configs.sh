# ncu --set full of the pass kernels of configs 5 and 1 (after each bench
# command ran clean without ncu), summarised by tools/ncu_summary.py
set -x
for c in 5 1; do
  CMD="python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu --graph 0"
  timeout 300 $CMD > gpurun_out/plain_c$c.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:pass_kernel -s 3 -c 3 -o gpurun_out/prof_c${c}_final $CMD > gpurun_out/ncu_c${c}_final.log 2>&1
done
