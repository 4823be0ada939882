mkdir -p gpurun_out
for c in "2 f64" "5 f64" "5 f32" "3 f64" "4 f64"; do set -- $c; timeout 300 python tools/pass_trace.py --config $1 --precision $2; done > gpurun_out/s5e_pass_trace.log 2>&1
cat gpurun_out/s5e_pass_trace.log
