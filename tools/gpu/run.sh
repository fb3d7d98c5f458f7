#!/bin/bash
# The GPU-side evidence of this repo, one subcommand per kind (run from the repo root on a B200, e.g.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/gpu/run.sh tests bench').
# Outputs land in gpurun_out/ (scratch); the summaries that are judged are copied into profiles/.
#
#   tests       pytest -m gpu (the parity suite)                       -> gpurun_out/gpu_tests.log
#   (order matters: run `traffic` before `bench`, so that the bench line reports the traffic of its own build)
#   bench       bench.py C2 line (200 steps)                           -> gpurun_out/bench_C2.json
#   benches     the C1 / C3 / vectors / weighted / L2-warm / Zipf-exponent lines and the reference arm
#                                                                       -> gpurun_out/bench_*.json
#   quick       parity spot set + C2 call time vs the round-1 kernel (tools/r2_quick.py), C1/C2/C3 call times
#               (tools/c3_time.py)                                     -> gpurun_out/quick.log
#   profiles    launch list of a bench run + ncu --set full of part/link/side on a C2 call, summarised by
#               tools/r02_summaries.py                                 -> gpurun_out/r02/, profiles/r02/
#   traffic     per-kernel DRAM bytes over a sequence of C2 / C3 calls (ncu --cache-control none)
#                                                                       -> profiles/ncu_traffic.json
#   sanitize    compute-sanitizer memcheck / racecheck / synccheck on C1 and 4 windows of C2, three paths
#               (round-2 kernels, round-1 kernel, vectors + IP sets, weighted rows) -> gpurun_out/sanitize_*.txt
#   batch-sweep rebuild libnsg with NSG_FLAT_BATCH = 16 / 32 / 64: C2 call time and DRAM bytes per call
#               (leaves the last build in place: rebuild afterwards)   -> gpurun_out/fb_*.csv
set -u
mkdir -p gpurun_out
# ncu per-kernel time + DRAM bytes, no cache flush between launches
NCU_LIST=(ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none
          --cache-control none -k "regex:part_kernel|link_kernel|side_kernel|discard_kernel" --csv --log-file)
for cmd in "$@"; do
  case $cmd in
  tests)
    timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log ;;
  bench)
    timeout 900 python bench.py --steps 200 --warmup 10 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
    tail -c 400 gpurun_out/bench_C2.json ;;
  benches)  # the other bench lines of profiles/r02/ (workloads, output modes, the reference arm)
    for spec in "C1:--workload C1" "C3:--workload C3" "C2_vectors:--outputs vectors" "C2_weighted:--input weighted" \
                "C2_l2warm:--l2 warm" "Z08:--workload Z08" "Z13:--workload Z13" "Z15:--workload Z15"; do
      name=${spec%%:*}; a=${spec#*:}
      timeout 600 python bench.py --steps 200 --warmup 10 $a > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err
      echo "$name: $(tail -c 300 gpurun_out/bench_$name.json | head -c 300)"
    done
    timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
    tail -c 200 gpurun_out/bench_reference.json ;;
  quick)
    { timeout 300 python tools/r2_quick.py --reps 20; timeout 300 python tools/c3_time.py; } > gpurun_out/quick.log 2>&1
    grep -v "parity OK" gpurun_out/quick.log ;;
  profiles)
    mkdir -p gpurun_out/r02
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/r02/launches_C2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline \
      > gpurun_out/r02/launches_bench_stdout.txt 2>&1
    REPS=4 timeout 900 ncu --set full --clock-control none --import-source on \
      -k "regex:part_kernel|link_kernel|side_kernel" -s 6 -c 3 -o gpurun_out/r02/full_C2 python tools/one_call.py \
      > /dev/null 2>&1
    ncu -i gpurun_out/r02/full_C2.ncu-rep --page raw --csv > gpurun_out/r02/full_C2_raw.csv 2>/dev/null
    for k in part link side; do
      ncu -i gpurun_out/r02/full_C2.ncu-rep --page source --csv --print-source=cuda,sass -k regex:${k}_kernel \
        > gpurun_out/r02/src_${k}.csv 2>/dev/null
    done
    python tools/r02_summaries.py gpurun_out/r02 gpurun_out/r02_summaries > /dev/null ;;
  traffic)
    for wl in C2 C3; do
      timeout 600 "${NCU_LIST[@]}" gpurun_out/traffic_$wl.csv python tools/traffic_case.py 12 $wl > /dev/null 2>&1
    done
    python tools/traffic_json.py C2=gpurun_out/traffic_C2.csv C3=gpurun_out/traffic_C3.csv
    cp profiles/ncu_traffic.json gpurun_out/ ;;
  sanitize)
    # PYTORCH_NO_CUDA_MEMORY_CACHING=1: every tensor is its own cudaMalloc, so memcheck sees each buffer's
    # bounds (torch's caching pool would hide overruns); tools/sanitizer_check/ is the positive control.
    for tool in memcheck racecheck synccheck; do
      for cs in C1 C2r; do
        for p in flat legacy vectors weighted; do
          log=gpurun_out/sanitize_${tool}_${cs}_${p}.txt
          extra=""
          [ $tool = racecheck ] && extra="--racecheck-report all"
          t0=$(date +%s)
          PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 900 compute-sanitizer --tool $tool $extra \
            python tools/sanitize_case.py $cs $p > $log 2>&1
          echo "rc=$? seconds=$(( $(date +%s) - t0 ))" >> $log
          echo "$tool $cs $p: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|parity|rc=' $log | tr '\n' ' ')"
        done
      done
    done
    PYTORCH_NO_CUDA_MEMORY_CACHING=1 compute-sanitizer --tool memcheck python tools/sanitizer_check/run.py \
      > gpurun_out/san_ctl_mem.txt 2>&1
    compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitizer_check/run.py \
      > gpurun_out/san_ctl_race.txt 2>&1 ;;
  batch-sweep)
    for B in 16 32 64; do
      nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
        -DNSG_FLAT_BATCH=$B -I include -o paper_2509_03653_b200/libnsg.so paper_2509_03653_b200/csrc/nsg.cu || exit 1
      echo "== FLAT_BATCH=$B"
      timeout 300 python tools/r2_quick.py --skip-parity --reps 20 2>&1 | grep "^r2" | head -1
      timeout 600 "${NCU_LIST[@]}" gpurun_out/fb_$B.csv python tools/traffic_case.py 12 C2 > /dev/null 2>&1
      LAUNCHES_PER_CALL=$(( 3 * (64 / B) + 1 )) python tools/traffic_json.py --print-only C2=gpurun_out/fb_$B.csv
    done ;;
  *) echo "unknown subcommand $cmd"; exit 2 ;;
  esac
done
