mkdir -p gpurun_out
for c in "2 f64" "5 f64" "5 f32" "3 f64" "4 f64"; do set -- $c; timeout 300 python tools/pass_trace.py --config $1 --precision $2; done > gpurun_out/s5f_pass_trace.log 2>&1
grep -A4 "TILES=2" gpurun_out/s5f_pass_trace.log | cut -c1-120
for m in 0 4 0 4; do
  PAFFT_DYN_MIN_TILES=$m timeout 900 python bench.py --no-cpu --no-e2e --steps 20 --warmup 5 > gpurun_out/s5f_bench_dyn$m.$RANDOM.json 2> gpurun_out/s5f_bench_dyn$m.err
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/s5f_bench_dyn*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f,'ERR',e); continue
    print(f, 'c2', round(d['value']), [round(p['ms'],3) for p in d['passes']], {k:round(v['value']) for k,v in d.get('configs',{}).items()})
PY
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/s5f_pytest.log 2>&1
tail -3 gpurun_out/s5f_pytest.log
