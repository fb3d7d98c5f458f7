#!/bin/bash
# Batch-size sweep of the round-2 kernels (design tool): for each NSG_FLAT_BATCH, rebuild libnsg in place,
# time C2 (tools/r2_quick.py --skip-parity) and capture per-kernel DRAM bytes and time of one C2 call.
for B in ${BATCHES:-8 16 32 64}; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -DNSG_FLAT_BATCH=$B \
    -I include -o paper_2509_03653_b200/libnsg.so paper_2509_03653_b200/csrc/nsg.cu || exit 1
  echo "== FLAT_BATCH=$B"
  timeout 300 python tools/r2_quick.py --skip-parity --reps 20 2>&1 | grep "^r2" | head -1
  REPS=6 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
    -k "regex:part_kernel|link_kernel|side_kernel" --csv --log-file gpurun_out/fb_$B.csv python tools/one_call.py > /dev/null 2>&1
  python tools/ncu_sum.py gpurun_out/fb_$B.csv
done
