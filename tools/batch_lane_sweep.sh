#!/bin/bash
# C2 bench line (value, roofline fraction) for FLAT_BATCH x bench streams, with the batch lanes of the build
# (calls of >= 3 batches run on two lanes).  usage (GPU box): bash tools/batch_lane_sweep.sh "16 32" "1 2 3"
for B in $1; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -DNSG_FLAT_BATCH=$B \
    -I include -o paper_2509_03653_b200/libnsg.so paper_2509_03653_b200/csrc/nsg.cu || exit 1
  for st in $2; do
    v=$(timeout 300 python bench.py --steps 200 --warmup 10 --streams $st --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.2f G/s frac %.4f' % (d['value']/1e9, d['roofline']['frac']))")
    echo "batch=$B streams=$st: $v"
  done
done
