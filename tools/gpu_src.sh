#!/bin/bash
# Source-level ncu capture of the link and side kernels (one C2 call): gpurun_out/{link,side}_src.csv
REPS=1 timeout 300 ncu --set full --import-source on --clock-control none -k "regex:link_kernel|side_kernel" -c 2 -o gpurun_out/fl python tools/one_call.py > /dev/null 2>&1
for k in link side; do
  ncu -i gpurun_out/fl.ncu-rep --page source --csv --print-source=cuda,sass -k regex:${k}_kernel > gpurun_out/${k}_src.csv 2>/dev/null
done
