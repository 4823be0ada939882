set -x
python -c "
import sys; sys.path.insert(0,'.')
import paper_2506_12718_b200 as pf
for r,d in [(2,[1<<20]),(3,[3**13]),(5,[5**7]),(2,[2048,2048]),(4,[256,256,256])]:
    print(pf.Plan(r,d).describe())
" > gpurun_out/r2e_describe.txt 2>&1
bash tools/env_sweep.sh 1 f64 "PAFFT_NARROW=0" "PAFFT_NARROW=1 PAFFT_NARROW_W=4" "PAFFT_NARROW=1 PAFFT_NARROW_W=2" \
  "PAFFT_NARROW=0 PAFFT_MID_STAGES=11" "PAFFT_NARROW=1 PAFFT_MID_STAGES=11 PAFFT_NARROW_W=4" "PAFFT_NARROW=1 PAFFT_MID_STAGES=11 PAFFT_NARROW_W=2" \
  "PAFFT_NARROW=0 PAFFT_MID_STAGES=10" "PAFFT_NARROW=1 PAFFT_MID_STAGES=10 PAFFT_NARROW_W=4" "PAFFT_NARROW=1 PAFFT_MID_STAGES=10 PAFFT_NARROW_W=2" \
  "PAFFT_NARROW=0" > gpurun_out/r2e_c1sweep.log 2>&1
bash tools/env_sweep.sh 1 f32 "PAFFT_NARROW=0" "PAFFT_NARROW=1 PAFFT_NARROW_W=8" "PAFFT_NARROW=1 PAFFT_NARROW_W=4" >> gpurun_out/r2e_c1sweep.log 2>&1
timeout 600 oracle/_ref/acceptance_dropin > gpurun_out/r2e_acceptance.log 2>&1
timeout 300 tests/cpp/test_dropin > gpurun_out/r2e_dropin.log 2>&1
