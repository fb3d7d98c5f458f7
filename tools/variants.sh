#!/bin/bash
# Build libnsg variants in place one after the other and time C1/C2/C3 calls for each, with a parity spot
# check and (TRAFFIC=1) per-kernel time and DRAM bytes per C2 call (ncu, --cache-control none).
# usage (GPU box): bash tools/variants.sh "NAME:-DA=1 -DB=2" "NAME2:@path/to/nsg.cu -DX=1" ...
#   a token @FILE builds FILE instead of paper_2509_03653_b200/csrc/nsg.cu (e.g. an older revision's copy)
# Leaves the LAST variant built: rebuild afterwards.
mkdir -p gpurun_out
for spec in "$@"; do
  name=${spec%%:*}
  src=paper_2509_03653_b200/csrc/nsg.cu
  flags=""
  for tok in ${spec#*:}; do
    case $tok in @*) src=${tok#@} ;; *) flags="$flags $tok" ;; esac
  done
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared $flags \
    -I include -o paper_2509_03653_b200/libnsg.so $src || exit 1
  echo "== $name ($src$flags)"
  timeout 300 python tools/r2_quick.py --reps 20 2>&1 | grep -E "FAIL|^r2" | head -3
  timeout 300 python tools/c3_time.py 2>&1 | grep " r2:"
  if [ -n "${TRAFFIC:-}" ]; then
    timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --cache-control none -k "regex:part_kernel|link_kernel|side_kernel|side_split_kernel|discard_kernel" --csv \
      --log-file gpurun_out/var_$name.csv python tools/traffic_case.py 12 C2 > /dev/null 2>&1
    python - gpurun_out/var_$name.csv <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, L = None, {}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        d = L.setdefault(int(x["ID"]), {"k": x["Kernel Name"].split("(")[0].split()[-1].split("<")[0]})
        d[x["Metric Name"]] = float(x["Metric Value"].replace(",", ""))
seq = [L[k] for k in sorted(L)]
tail = seq[len(seq) // 2:]  # the second half of the 12 calls
calls = 6
agg = {}
for d in tail:
    a = agg.setdefault(d["k"], [0.0, 0.0])
    a[0] += d.get("gpu__time_duration.sum", 0) / calls
    a[1] += (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / calls
print("  C2 per call: DRAM %.1f MB, " % (sum(v[1] for v in agg.values()) / 1e6) +
      ", ".join("%s %.1f us" % (k, v[0] / 1e3) for k, v in agg.items()))
PY
  fi
done
