# session 5, call B: FFMA2 issue probe + multi-stream L2-chunk probe (fixed graph capture)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma2 tools/probes/ffma2.cu && /tmp/ffma2 > gpurun_out/s5b_ffma2.log 2>&1
{
timeout 600 python tools/l2_chunk_probe.py --config 5 --precision f32 --chunks 4096,512,256,128,64,32 --streams 1,2,3,4
timeout 600 python tools/l2_chunk_probe.py --config 5 --precision f64 --chunks 4096,512,128,64,32,16 --streams 1,2,3
timeout 600 python tools/l2_chunk_probe.py --config 2 --precision f64 --chunks 64,16,8,4,2 --streams 1,2,3
timeout 600 python tools/l2_chunk_probe.py --config 5 --precision f32 --chunks 4096,256,128,64,32 --streams 1,2,3 --graph
} > gpurun_out/s5b_chunk_streams.log 2>&1
cat gpurun_out/s5b_ffma2.log
