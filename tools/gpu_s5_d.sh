# session 5, call D: dynamic tile order A/B (PAFFT_DYN_MIN_TILES) + parity with it on
mkdir -p gpurun_out
for m in 0 2 8 0 2; do
  PAFFT_DYN_MIN_TILES=$m timeout 900 python bench.py --no-cpu --no-e2e --steps 20 --warmup 5 > gpurun_out/s5d_bench_dyn$m.$RANDOM.json 2> gpurun_out/s5d_bench_dyn$m.err
done
PAFFT_DYN_MIN_TILES=2 timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_threads.py -x -q -m gpu > gpurun_out/s5d_pytest_dyn2.log 2>&1
tail -3 gpurun_out/s5d_pytest_dyn2.log
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/s5d_bench_dyn*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f,'ERR',e); continue
    print(f, 'c2', round(d['value']), [round(p['ms'],3) for p in d['passes']], {k:round(v['value']) for k,v in d.get('configs',{}).items()})
PY
