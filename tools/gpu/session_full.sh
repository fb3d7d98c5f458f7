set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo pytest rc $?
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; echo bench rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fast_kernel -s 3 -c 1 -f -o gpurun_out/fast_C2 python bench.py --steps 3 --warmup 3 --workload C2 --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo ncu rc $?
ncu -i gpurun_out/fast_C2.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/fast_C2_source.csv 2>/dev/null; echo src rc $?
