#!/bin/bash
# One GPU iteration of the per-window kernel work (design tool): parity + C2 timing (tools/r2_quick.py)
# and the per-kernel launch list with instruction counts.  Usage on the box: bash tools/gpu_iter.sh
timeout 300 python tools/r2_quick.py --reps 20 > gpurun_out/q.log 2>&1
REPS=2 timeout 200 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k "regex:part_kernel|link_kernel|side_kernel" --csv --log-file gpurun_out/l.csv python tools/one_call.py > /dev/null 2>&1
cat gpurun_out/q.log
