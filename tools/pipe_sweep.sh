# L2-resident chunk pipeline (PAFFT_PIPELINE=1) vs whole-batch launches
run() { echo "config $1 $2: $(env $2 timeout 300 python bench.py --config $1 --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],3))")"; }
for c in 5; do
  run $c PAFFT_PIPELINE=0
  for mb in 8 16 24 36 48 64; do run $c "PAFFT_PIPELINE=1 PAFFT_CHUNK_MB=$mb"; done
done
run 2 PAFFT_PIPELINE=0
for mb in 25 50; do run 2 "PAFFT_PIPELINE=1 PAFFT_CHUNK_MB=$mb"; done
