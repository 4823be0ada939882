# GPU op table (reference CSV layout + GPU columns) for the five BASELINE configs
out=gpurun_out/ops_table.md; : > $out
m="python -m paper_2506_12718_b200.bench_ops --op all --format md --reps 5"
$m --radix 2 --dims 1048576 --batch 1 >> $out 2>>gpurun_out/ops.err
$m --radix 3 --dims 1594323 --batch 64 >> $out 2>>gpurun_out/ops.err
$m --radix 2 --dims 2048x2048 --batch 16 >> $out 2>>gpurun_out/ops.err
$m --radix 4 --dims 256x256x256 --batch 8 >> $out 2>>gpurun_out/ops.err
$m --radix 5 --dims 78125 --batch 4096 >> $out 2>>gpurun_out/ops.err
