timeout 900 python -m pytest tests/test_gpu_trace.py -x -q > gpurun_out/trace.txt 2>&1; echo rc $? >> gpurun_out/trace.txt
timeout 600 python tools/trace_time.py > gpurun_out/trace_time.txt 2>&1
