# last evidence pass of round 2 on the final build: DRAM traffic of the per-window path (profiles/ncu_traffic.json,
# read by bench.py), smoke, and compute-sanitizer memcheck / racecheck of the anonymiser on 4 windows of C2
# (the sanitizer legs exit 86 on pools where compute-sanitizer is closed)
set -u
bash tools/gpu/run.sh traffic
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo smoke rc=$? >> gpurun_out/smoke.txt; tail -1 gpurun_out/smoke.txt
for tool in memcheck racecheck; do
  log=gpurun_out/sanitize_${tool}_C2r_anon.txt
  PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 400 compute-sanitizer --tool $tool python tools/sanitize_case.py C2r anon > $log 2>&1
  echo "rc=$?" >> $log
  echo "$tool anon: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|parity|rc=' $log | tr '\n' ' ')"
done
