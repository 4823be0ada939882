# contiguous (CONV) group size per config after the single-buffer change
run() { echo "config $1 $2: $(env $2 timeout 300 python bench.py --config $1 --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), ' '.join('%s%d=%.3f'%(p['kind'][:4],p['R'],p['ms']) for p in d.get('passes',[])))")"; }
run 1 PAFFT_MID_STAGES=0
run 1 PAFFT_MID_STAGES=13
run 1 PAFFT_MID_STAGES=11
run 1 PAFFT_MID_STAGES=10
run 3 PAFFT_MID_STAGES=0
run 3 PAFFT_MID_STAGES=10
run 4 PAFFT_MID_STAGES=0
run 4 PAFFT_MID_STAGES=3
run 5 PAFFT_MID_STAGES=0
run 5 PAFFT_MID_STAGES=4
run 2 PAFFT_MID_STAGES=0
run 2 PAFFT_MID_STAGES=8
