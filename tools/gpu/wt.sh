timeout 900 python -m pytest tests/test_gpu_weighted.py -x -q > gpurun_out/wt.txt 2>&1; echo rc $? >> gpurun_out/wt.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo rc $? >> gpurun_out/pytest_gpu.txt
timeout 300 python tools/gpu_prof.py C2 > gpurun_out/prof.txt 2>&1
