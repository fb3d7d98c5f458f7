# every bench line of this round (ALL=1 adds C3/C1 and the reference arm)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo rc $? >> gpurun_out/pytest_gpu.txt
timeout 300 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
timeout 300 python bench.py --outputs vectors --no-cpu-baseline --steps 200 > gpurun_out/bench_C2_vectors.json 2> gpurun_out/bench_C2_vectors.err
timeout 300 python bench.py --input weighted --no-cpu-baseline --steps 200 > gpurun_out/bench_C2_weighted.json 2> gpurun_out/bench_C2_weighted.err
timeout 300 python bench.py --path trace --no-cpu-baseline --steps 50 > gpurun_out/bench_C2_trace.json 2> gpurun_out/bench_C2_trace.err
if [ -n "$ALL" ]; then
  for w in C3 C1; do timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
  timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
fi
timeout 300 python bench.py --path anonymize --no-cpu-baseline --steps 50 > gpurun_out/bench_C2_anonymize.json 2> gpurun_out/bench_C2_anonymize.err
