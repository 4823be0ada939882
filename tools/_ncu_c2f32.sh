mkdir -p gpurun_out
C1="python bench.py --config 2 --precision f32 --steps 1 --warmup 1 --no-e2e --no-cpu --no-sub --graph 0"
timeout 300 $C1 > gpurun_out/r2f_plain_c2f32.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:pass_kernel -s 3 -c 5 -o gpurun_out/r2f_c2f32 $C1 > gpurun_out/r2f_ncu_c2f32.log 2>&1
python tools/ncu_summary.py gpurun_out/r2f_c2f32.ncu-rep > gpurun_out/r2f_ncu_c2f32.txt 2>&1
rm -f gpurun_out/r2f_c2f32.ncu-rep gpurun_out/r2f_c2f64.ncu-rep
grep -E "^---|gpu__time_duration" gpurun_out/r2f_ncu_c2f32.txt
