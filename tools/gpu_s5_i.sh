mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_mixed.py tests/test_gpu_dynamic.py -x -q -m gpu > gpurun_out/s5i_pytest.log 2>&1
tail -3 gpurun_out/s5i_pytest.log
for rep in 1 2; do
for lib in paper_2506_12718_b200/libpafft_b200.so ab/libnolomajor.so; do
  for c in 5; do
    v=$(PAFFT_LIB=$lib timeout 300 python bench.py --config $c --precision f32 --steps 20 --warmup 5 --no-e2e --no-cpu --no-sub 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), ' '.join('%s=%.3f'%(p['kind'][:4],p['ms']) for p in d.get('passes',[])))")
    echo "rep$rep config$c f32 $(basename $lib): $v"
  done
done
done > gpurun_out/s5i_lomajor_ab.log 2>&1
cat gpurun_out/s5i_lomajor_ab.log
