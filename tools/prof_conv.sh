# One ncu --set full capture (source-level) of one pass kernel.
# usage: bash tools/prof_conv.sh '<demangled-name regex>' out_name [bench args]
set -x
RX=${1:-'pass_kernel<double, 3, 9, 9, 9, 3, 3, 1>'}
OUT=${2:-conv_c2}
shift 2
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu $*"
timeout 300 $CMD > gpurun_out/plain_$OUT.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$RX" -s 1 -c 1 -o gpurun_out/$OUT $CMD > gpurun_out/ncu_$OUT.log 2>&1
tail -3 gpurun_out/ncu_$OUT.log
