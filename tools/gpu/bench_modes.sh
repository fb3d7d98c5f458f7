# default bench line + the vectors mode, C2 (and C3/C1 when ALL=1)
timeout 300 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
timeout 300 python bench.py --outputs vectors --no-cpu-baseline --steps 200 > gpurun_out/bench_C2_vectors.json 2> gpurun_out/bench_C2_vectors.err
if [ -n "$ALL" ]; then
  for w in C3 C1; do timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
  timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
fi
