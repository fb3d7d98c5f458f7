# the N>1 bench path with two ranks sharing the one GPU (gloo for the host collectives)
for t in nccl p2p; do
  NSG_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 50 --warmup 3 --no-cpu-baseline --transport $t > gpurun_out/bench_N2_$t.json 2> gpurun_out/bench_N2_$t.err
  NSG_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --path trace --transport $t > gpurun_out/bench_N2_trace_$t.json 2> gpurun_out/bench_N2_trace_$t.err
done
