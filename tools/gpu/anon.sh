timeout 900 python -m pytest tests/test_gpu_anon.py -x -q > gpurun_out/anon.txt 2>&1; echo rc $? >> gpurun_out/anon.txt
