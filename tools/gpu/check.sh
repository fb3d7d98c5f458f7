timeout 900 python -m pytest tests/test_gpu_anon.py tests/test_gpu_parity.py tests/test_gpu_vectors.py -x -q > gpurun_out/check.txt 2>&1; echo rc $? >> gpurun_out/check.txt
for c in ${CFGS:-C2 U2 C3}; do timeout 300 python tools/gpu_prof.py $c; done > gpurun_out/prof.txt 2>&1
timeout 300 python bench.py --path anonymize --no-cpu-baseline --steps 50 > gpurun_out/bench_C2_anonymize.json 2> gpurun_out/bench_C2_anonymize.err
