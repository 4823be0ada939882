#!/bin/bash
# A/B bench of prebuilt libraries: tools/ab.sh "2 3 5" ab/libA.so ab/libB.so ...
cfgs=$1; shift
for rep in 1 2; do
  for c in $cfgs; do
    for lib in "$@"; do
      v=$(PAFFT_LIB=$lib timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu --no-sub 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), ' '.join('%s=%.3f'%(p['kind'][:4],p['ms']) for p in d.get('passes',[])))")
      echo "rep$rep config$c $(basename $lib): $v"
    done
  done
done
