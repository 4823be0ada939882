# Multi-rank bench flow on one GPU (gloo; both ranks share cuda:0 -- plumbing only, not a measurement)
export PAFFT_BENCH_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
  bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --sub-steps 3 > gpurun_out/mr_bench.json 2> gpurun_out/mr_bench.err
echo "rc=$?" >> gpurun_out/mr_bench.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 \
  bench.py --impl reference --gpus 2 --steps 1 --warmup 0 --no-sub > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err
echo "rc=$?" >> gpurun_out/mr_ref.err
