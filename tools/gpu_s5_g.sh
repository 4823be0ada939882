mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dynamic.py -x -q -m gpu > gpurun_out/s5g_pytest_dynamic.log 2>&1
tail -5 gpurun_out/s5g_pytest_dynamic.log
for m in 4 0 4 0; do
  PAFFT_DYN_MIN_TILES=$m timeout 900 python bench.py --no-cpu --no-e2e --steps 20 --warmup 5 > gpurun_out/s5g_bench_dyn$m.$RANDOM.json 2> gpurun_out/s5g_bench_dyn$m.err
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/s5g_bench_dyn*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f,'ERR',e); continue
    print(f, 'c2', round(d['value']), [round(p['ms'],3) for p in d['passes']], {k:round(v['value']) for k,v in d.get('configs',{}).items()})
PY
