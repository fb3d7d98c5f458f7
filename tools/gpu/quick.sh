# parity spread + per-phase profile of the product build
timeout 600 python tools/gpu_quick.py > gpurun_out/quick.txt 2>&1; echo quick rc $? >> gpurun_out/quick.txt
for c in ${CFGS:-C2 U2 C3}; do timeout 300 python tools/gpu_prof.py $c; done > gpurun_out/prof.txt 2>&1
