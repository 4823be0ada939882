timeout 120 tools/probes/dsmem_bw > gpurun_out/r2h_dsmem2.log 2>&1
