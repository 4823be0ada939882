# session 5, call C: co-resident software-pipelined passes (probe)
mkdir -p gpurun_out
{
timeout 900 python tools/corun_pipeline_probe.py --config 5 --precision f64 --chunks 1024,512,256,128 --caps 0:0,296:148,148:148,444:148,296:296
timeout 900 python tools/corun_pipeline_probe.py --config 5 --precision f32 --chunks 1024,512,256,128 --caps 0:0,444:148,296:148,592:148,888:148
timeout 900 python tools/corun_pipeline_probe.py --config 3 --precision f64 --chunks 8,4,2 --caps 0:0,148:148,148:296
} > gpurun_out/s5c_corun_pipeline.log 2>&1
tail -5 gpurun_out/s5c_corun_pipeline.log
