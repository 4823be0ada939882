# e2e (host-buffer C-ABI path) vs the host pipeline's chunk size / stream count
for s in 3 4 2; do for mb in 64 32 128 256; do
  v=$(PAFFT_HOST_STREAMS=$s PAFFT_HOST_CHUNK_MB=$mb timeout 300 python bench.py --config ${CFG:-2} --steps 3 --warmup 3 --no-cpu --e2e-steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['e2e']['value'],1))")
  echo "streams=$s chunk_mb=$mb e2e=$v"
done; done
