#!/bin/bash
# Per-kernel DRAM traffic of the per-window path on a sequence of C2 / C3 calls -> profiles/ncu_traffic.json
for wl in C2 C3; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --cache-control none -k "regex:part_kernel|link_kernel|side_kernel|discard_kernel" --csv --log-file gpurun_out/traffic_$wl.csv \
    python tools/traffic_case.py 12 $wl > /dev/null 2>&1
done
python tools/traffic_json.py C2=gpurun_out/traffic_C2.csv C3=gpurun_out/traffic_C3.csv
