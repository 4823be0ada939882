# per-pass time per signal vs batch size (L2 residency of small batches)
run() { echo "config $1 batch $2: $(timeout 300 python bench.py --config $1 --batch $2 --steps 20 --warmup 5 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['config']['batch_per_gpu']
print(round(d['value'],1), ' '.join('%s=%.2fus/sig'%(p['kind'][:4],p['ms']*1e3/b) for p in d.get('passes',[])))")"; }
for b in 1 2 3 4 8 64; do run 2 $b; done
for b in 16 32 64 128 4096; do run 5 $b; done
