# IP sets on two batch lanes: vectors parity, per-window parity, traffic of this build, C2 and vectors bench lines
set -u
timeout 600 python -m pytest tests/test_gpu_vectors.py tests/test_gpu_parity.py tests/test_gpu_capacity.py tests/test_gpu_aggregation.py -x -q > gpurun_out/lanes_tests.log 2>&1; tail -2 gpurun_out/lanes_tests.log
bash tools/gpu/run.sh traffic bench
timeout 600 python bench.py --steps 200 --warmup 10 --outputs vectors > gpurun_out/bench_C2_vectors.json 2> gpurun_out/bench_C2_vectors.err; tail -c 200 gpurun_out/bench_C2_vectors.json
