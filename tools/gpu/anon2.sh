timeout 900 python -m pytest tests/test_gpu_anon.py tests/test_gpu_trace.py -x -q > gpurun_out/anon.txt 2>&1; echo rc $? >> gpurun_out/anon.txt
timeout 300 python bench.py --path anonymize --no-cpu-baseline --steps 50 > gpurun_out/bench_C2_anonymize.json 2> gpurun_out/bench_C2_anonymize.err
timeout 300 python bench.py --path trace --no-cpu-baseline --steps 50 > gpurun_out/bench_C2_trace.json 2> gpurun_out/bench_C2_trace.err
