# usage: env_sweep.sh <config> <prec> "<ENV=.. ENV=..>" ...   -> one line per variant
# (bench.py device-resident value + per-pass ms; no e2e / CPU / sub-configs)
cfg=$1; prec=$2; shift 2
for v in "$@"; do
  out=$(env $v timeout 300 python bench.py --config $cfg --precision $prec --steps 20 --warmup 5 --no-e2e --no-cpu --no-sub 2>/dev/null | tail -1)
  echo "[$v] $(echo "$out" | python -c "import json,sys
try:
  d=json.loads(sys.stdin.read()); print(round(d['value'],1), ' '.join('%s%d=%.4f'%(p['kind'][:4],p['R'],p['ms']) for p in d['passes']))
except Exception as e: print('ERR', e)")"
done
