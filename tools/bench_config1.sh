timeout 300 python bench.py --config 1 --no-cpu --no-e2e --no-sub > gpurun_out/c1_2s.json 2> gpurun_out/c1_2s.err; tail -3 gpurun_out/c1_2s.err
