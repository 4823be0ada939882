# Round-2 final evidence (after the dynamic tile order and the packed fp32 path): smoke, GPU suite,
# default bench (+ sub-configs), reference arm, launch list of the headline step, ncu --set full of
# every config's pass kernels (each only after the same command ran clean without ncu), per-CTA trace.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/r2f_smi.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=15 > gpurun_out/r2f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_pytest.log
timeout 900 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2f_ref.json 2> gpurun_out/r2f_ref.err
CMD="python bench.py --config 2 --steps 3 --warmup 3 --no-e2e --no-cpu --no-sub"
timeout 300 $CMD > gpurun_out/r2f_plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pass_kernel -c 40 --csv --log-file gpurun_out/r2f_launches.csv $CMD > gpurun_out/r2f_ncu_launch.log 2>&1
for spec in "2 f64 3" "5 f64 3" "5 f32 3" "3 f64 3" "4 f64 5" "1 f64 3"; do
  set -- $spec
  C1="python bench.py --config $1 --precision $2 --steps 1 --warmup 1 --no-e2e --no-cpu --no-sub --graph 0"
  skip=2; [ $1 = 4 ] && skip=3  # the filter preparation launches that many DIF passes first
  timeout 300 $C1 > gpurun_out/r2f_plain_c$1$2.log 2>&1 && \
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:pass_kernel -s $skip -c $3 -o gpurun_out/r2f_c$1$2 $C1 > gpurun_out/r2f_ncu_c$1$2.log 2>&1
  # summarise on the box: the reports together exceed what gpurun copies back
  python tools/ncu_summary.py gpurun_out/r2f_c$1$2.ncu-rep > gpurun_out/r2f_ncu_c$1$2.txt 2>&1
  [ "$1$2" = 2f64 ] || rm -f gpurun_out/r2f_c$1$2.ncu-rep
done
for c in "2 f64" "3 f64" "4 f64" "5 f64" "5 f32"; do set -- $c; PAFFT_LIB=ab/libtrace.so timeout 300 python tools/pass_trace.py --config $1 --precision $2; done > gpurun_out/r2f_pass_trace.log 2>&1
bash tools/ops_table.sh > gpurun_out/r2f_ops_table.log 2>&1
