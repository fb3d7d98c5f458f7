#!/bin/bash
# Batch-size sweep of the round-2 kernels (design tool): for each NSG_FLAT_BATCH, rebuild libnsg in place,
# time C2 (tools/r2_quick.py --skip-parity) and measure DRAM bytes per C2 call over a call sequence
# (tools/traffic_case.py under ncu --cache-control none).
for B in ${BATCHES:-16 32 64}; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -DNSG_FLAT_BATCH=$B \
    -I include -o paper_2509_03653_b200/libnsg.so paper_2509_03653_b200/csrc/nsg.cu || exit 1
  echo "== FLAT_BATCH=$B"
  timeout 300 python tools/r2_quick.py --skip-parity --reps 20 2>&1 | grep "^r2" | head -1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --cache-control none -k "regex:part_kernel|link_kernel|side_kernel|discard_kernel" --csv --log-file gpurun_out/fb_$B.csv \
    python tools/traffic_case.py 12 C2 > /dev/null 2>&1
  python - "$B" <<'PY'
import csv, sys
B = int(sys.argv[1]); per = 3 * (64 // B) + 1
rows = list(csv.reader(open(f"gpurun_out/fb_{B}.csv"))); hdr = None; L = {}
for r in rows:
    if "Kernel Name" in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r)); L.setdefault(int(x["ID"]), {})[x["Metric Name"]] = float(x["Metric Value"].replace(",", ""))
seq = [L[k] for k in sorted(L)]; calls = [seq[i:i + per] for i in range(0, len(seq) - per + 1, per)][6:]
f = lambda m: sum(sum(l.get(m, 0) for l in c) for c in calls) / len(calls)
print(f"B={B}: DRAM read {f('dram__bytes_read.sum')/1e6:.1f} MB write {f('dram__bytes_write.sum')/1e6:.1f} MB per call; "
      f"kernel time sum {f('gpu__time_duration.sum')/1e3:.1f} us (serialised under ncu)")
PY
done
