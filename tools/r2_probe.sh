timeout 120 tools/probes/dsmem_bw > gpurun_out/r2h_dsmem.log 2>&1
timeout 600 oracle/_ref/acceptance_dropin > gpurun_out/r2h_acceptance.log 2>&1
