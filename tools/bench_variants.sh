#!/bin/bash
# Rebuild libnsg with each variant's -D flags and print the default bench line's value / e2e / roofline
# fraction (200 steps).  usage (GPU box): bash tools/bench_variants.sh "NAME:-DX=1" ...  (leaves the last built)
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared $flags \
    -I include -o paper_2509_03653_b200/libnsg.so paper_2509_03653_b200/csrc/nsg.cu || exit 1
  for a in "" "--workload C3" "--workload C1"; do
    timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline $a 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
print('$name', '${a:-C2}', 'value %.2f G/s' % (d['value'] / 1e9), 'e2e %.2f' % (d['e2e']['value'] / 1e9),
      'frac %.4f' % d['roofline']['frac'], 'ms/step %.4f' % d['ms_per_step'])"
  done
done
