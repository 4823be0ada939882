# Full default bench (headline + per-config sub-results) and the reference arm.
set -x
free -g > gpurun_out/r2b_free.txt; nproc >> gpurun_out/r2b_free.txt; lscpu | head -20 >> gpurun_out/r2b_free.txt
timeout 900 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err
