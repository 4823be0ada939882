# ncu --set full (source view) of the pass kernels of configs 1, 4, 5 (one step each)
for c in 1 4 5; do
  CMD="python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu --no-sub --graph 0"
  n=3; [ $c = 4 ] && n=5
  skip=2; [ $c = 4 ] && skip=3; [ $c = 1 ] && skip=2
  timeout 300 $CMD > gpurun_out/r2n_plain_c$c.log 2>&1 && \
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:pass_kernel -s $skip -c $n -o gpurun_out/r2n_c$c $CMD > gpurun_out/r2n_ncu_c$c.log 2>&1
done
