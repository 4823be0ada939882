set -x
for c in 2 1 3 4 5; do timeout 600 python bench.py --config $c > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
timeout 600 python bench.py --config 5 --precision f32 > gpurun_out/bench_c5f32.json 2> gpurun_out/bench_c5f32.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_c2_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launch_c2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
