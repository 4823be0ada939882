# session 5, call A: multi-stream L2-chunk probe + ncu of config 5 fp32
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/s5a_smi.log
{
timeout 600 python tools/l2_chunk_probe.py --config 5 --precision f32 --chunks 4096,512,256,128,64,32 --streams 1,2,3,4 --graph
timeout 600 python tools/l2_chunk_probe.py --config 5 --precision f64 --chunks 4096,512,128,64,32,16 --streams 1,2,3,4 --graph
timeout 600 python tools/l2_chunk_probe.py --config 2 --precision f64 --chunks 64,16,8,4,2 --streams 1,2,3,4 --graph
} > gpurun_out/s5a_chunk_streams.log 2>&1
CMD="python bench.py --config 5 --precision f32 --steps 1 --warmup 1 --no-e2e --no-cpu --no-sub --graph 0"
timeout 300 $CMD > gpurun_out/s5a_plain_c5f32.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:pass_kernel -s 3 -c 3 -o gpurun_out/s5a_c5f32 $CMD > gpurun_out/s5a_ncu_c5f32.log 2>&1
tail -3 gpurun_out/s5a_chunk_streams.log
