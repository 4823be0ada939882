timeout 120 tools/probes/launch_gap > gpurun_out/r2k_gap.log 2>&1
