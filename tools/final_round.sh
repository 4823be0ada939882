# Round-end evidence: smoke, config-5 group-size check, ncu launch list and
# one ncu --set full capture of the three config-2 pass kernels.
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
run() { echo "config $1 $2: $(env $2 timeout 300 python bench.py --config $1 $3 --steps 20 --warmup 5 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), ' '.join('%s%d=%.3f'%(p['kind'][:4],p['R'],p['ms']) for p in d.get('passes',[])))")"; }
for r in 1 2; do
  run 5 PAFFT_MID_STAGES=0 ""; run 5 PAFFT_MID_STAGES=4 ""
  run 5 PAFFT_MID_STAGES=0 "--precision f32"; run 5 PAFFT_MID_STAGES=4 "--precision f32"
done > gpurun_out/c5mid.log 2>&1
CMD="python bench.py --config 2 --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launch_c2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pass_kernel -s 3 -c 3 -o gpurun_out/prof_c2_final $CMD > gpurun_out/ncu_c2_final.log 2>&1
