mkdir -p gpurun_out
export PAFFT_LIB=ab/libtrace.so
for c in "2 f64" "3 f64" "4 f64" "5 f64" "5 f32" "1 f64"; do set -- $c; timeout 300 python tools/pass_trace.py --config $1 --precision $2; done > gpurun_out/s5j_pass_trace.log 2>&1
grep -A3 "TILES=2" gpurun_out/s5j_pass_trace.log | sed 's/CTA retire times (us after first start) //' | cut -c1-260
