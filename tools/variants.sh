#!/bin/bash
# Build libnsg variants (-D flags) in place one after the other and time C1/C2/C3 calls for each, with a parity
# spot check and per-call DRAM traffic (ncu) of C2.  usage (GPU box): bash tools/variants.sh "NAME:-DA=1 -DB=2" ...
# Leaves the LAST variant built: rebuild afterwards.
mkdir -p gpurun_out
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared $flags \
    -I include -o paper_2509_03653_b200/libnsg.so paper_2509_03653_b200/csrc/nsg.cu || exit 1
  echo "== $name ($flags)"
  timeout 300 python tools/r2_quick.py --reps 20 2>&1 | grep -E "FAIL|^r2" | head -3
  timeout 300 python tools/c3_time.py 2>&1 | grep " r2:"
  if [ -n "${TRAFFIC:-}" ]; then
    timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --cache-control none -k "regex:part_kernel|link_kernel|side_kernel|discard_kernel" --csv \
      --log-file gpurun_out/var_$name.csv python tools/traffic_case.py 12 C2 > /dev/null 2>&1
    LAUNCHES_PER_CALL=7 python tools/traffic_json.py --print-only C2=gpurun_out/var_$name.csv 2>&1 | tail -3
  fi
done
