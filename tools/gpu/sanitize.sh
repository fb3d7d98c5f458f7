#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the per-window kernels (C1 and 4 windows of C2;
# round-2 kernels, the round-1 kernel, and the vector path).  Logs: gpurun_out/sanitize_<tool>_<case>_<path>.txt
# PYTORCH_NO_CUDA_MEMORY_CACHING=1: every tensor is its own cudaMalloc, so memcheck sees each buffer's bounds
# (torch's caching pool would hide overruns); tools/sanitizer_check/ is the positive control.
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  for cs in C1 C2r; do
    for p in flat legacy vectors; do
      log=gpurun_out/sanitize_${tool}_${cs}_${p}.txt
      extra=""
      [ $tool = racecheck ] && extra="--racecheck-report all"
      t0=$(date +%s); PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 900 compute-sanitizer --tool $tool $extra \
        python tools/sanitize_case.py $cs $p > $log 2>&1
      echo "rc=$? seconds=$(( $(date +%s) - t0 ))" >> $log
      echo "$tool $cs $p: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|parity|rc=' $log | tr '\n' ' ')"
    done
  done
done
