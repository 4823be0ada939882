# packed fp32 (FFMA2) A/B and parity
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/s5h_pytest.log 2>&1
tail -3 gpurun_out/s5h_pytest.log
for rep in 1 2; do
for lib in paper_2506_12718_b200/libpafft_b200.so ab/libnof32x2.so; do
  for c in 5 2 1 3 4; do
    v=$(PAFFT_LIB=$lib timeout 300 python bench.py --config $c --precision f32 --steps 20 --warmup 5 --no-e2e --no-cpu --no-sub 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), ' '.join('%s=%.3f'%(p['kind'][:4],p['ms']) for p in d.get('passes',[])))")
    echo "rep$rep config$c f32 $(basename $lib): $v"
  done
done
done > gpurun_out/s5h_f32x2_ab.log 2>&1
cat gpurun_out/s5h_f32x2_ab.log
python tools/accuracy_probe.py > gpurun_out/s5h_accuracy.log 2>&1; tail -20 gpurun_out/s5h_accuracy.log
