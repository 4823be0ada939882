timeout 300 python tools/diag_tensor_lines.py > gpurun_out/diag_tl.log 2>&1
