# CONV codelet-split sweep for configs 5 (R=3125) and 2 (R=2187), fp64 and fp32
set -x
bash tools/env_sweep.sh 5 f64 "PAFFT_MID_STAGES=4" "PAFFT_MID_STAGES=3" "PAFFT_SPLIT_3125=25x25x5" "PAFFT_SPLIT_3125=25x5x5x5" "PAFFT_SPLIT_3125=5x5x5x25" "PAFFT_SPLIT_3125=5x25x25" > gpurun_out/r2f_split.log 2>&1
bash tools/env_sweep.sh 5 f32 "PAFFT_MID_STAGES=4" "PAFFT_SPLIT_3125=25x25x5" "PAFFT_SPLIT_3125=25x5x5x5" "PAFFT_SPLIT_3125=5x5x5x25" "PAFFT_SPLIT_3125=5x25x25" >> gpurun_out/r2f_split.log 2>&1
bash tools/env_sweep.sh 2 f64 "PAFFT_SPLIT_2187=9x9x9x3" "PAFFT_SPLIT_2187=9x9x27" "PAFFT_SPLIT_2187=27x9x9" "PAFFT_SPLIT_2187=3x9x9x9" "PAFFT_SPLIT_2187=9x27x9" >> gpurun_out/r2f_split.log 2>&1
python - > gpurun_out/r2f_regs.txt 2>&1 <<'PY'
import sys; sys.path.insert(0,'.')
import os
import paper_2506_12718_b200 as pf
for r, d, sp in [(5,[5**7],"25x25x5"),(5,[5**7],"25x5x5x5"),(5,[5**7],"5x5x5x25"),(5,[5**7],"5x25x25"),(3,[3**13],"9x9x9x3"),(3,[3**13],"9x9x27"),(3,[3**13],"27x9x9"),(3,[3**13],"3x9x9x9"),(3,[3**13],"9x27x9")]:
    os.environ["PAFFT_SPLIT_%d" % (3125 if r == 5 else 2187)] = sp
    print(sp, pf.Plan(r, d).describe().splitlines()[1])
PY
# config 1: per-kernel device time inside the graph replay (warm caches: --cache-control none)
CMD="python bench.py --config 1 --steps 2 --warmup 3 --no-e2e --no-cpu --no-sub"
timeout 300 $CMD > gpurun_out/r2f_c1_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -k regex:pass_kernel -s 900 -c 60 --csv --log-file gpurun_out/r2f_c1_launches.csv $CMD > gpurun_out/r2f_c1_ncu.log 2>&1
