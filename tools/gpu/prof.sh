for c in C2 U2 C3; do timeout 300 python tools/gpu_prof.py $c; done > gpurun_out/prof.txt 2>&1
