"""Write profiles/ncu_traffic.json from ncu launch lists of tools/traffic_case.py (per-kernel
dram__bytes_read.sum + dram__bytes_write.sum, --cache-control none, so the traffic is what a sequence of
calls really moves): DRAM bytes per call = the mean over the last half of the calls of the sum over that
call's launches.  usage: traffic_json.py WORKLOAD=list.csv [...]"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_03653_b200 import _lib  # noqa: E402

out_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
res = json.load(open(out_path)) if os.path.exists(out_path) else {}
print_only = "--print-only" in sys.argv
for arg in [a for a in sys.argv[1:] if a != "--print-only"]:
    name, path = arg.split("=", 1)
    rows = list(csv.reader(open(path)))
    hdr, launches = None, {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            x = dict(zip(hdr, r))
            d = launches.setdefault(int(x["ID"]), {"kernel": x["Kernel Name"].split("(")[0]})
            d[x["Metric Name"]] = float(x["Metric Value"].replace(",", ""))
    seq = [launches[k] for k in sorted(launches)]
    # one call = its batches' (part, link, side) launches, closed by the scratch discards (one per batch lane)
    def is_discard(L):
        return L["kernel"].split("::")[-1].startswith("discard_kernel")

    calls, cur = [], []
    for i, L in enumerate(seq):
        cur.append(L)
        if is_discard(L) and (i + 1 == len(seq) or not is_discard(seq[i + 1])):
            calls.append(cur)
            cur = []
    per_call = len(calls[-1])
    tail = calls[len(calls) // 2:]

    def tot(c, m):
        return sum(L.get(m, 0.0) for L in c)

    rd = sum(tot(c, "dram__bytes_read.sum") for c in tail) / len(tail)
    wr = sum(tot(c, "dram__bytes_write.sum") for c in tail) / len(tail)
    t = sum(tot(c, "gpu__time_duration.sum") for c in tail) / len(tail)
    by_kernel = {}
    for c in tail:
        for L in c:
            k = L["kernel"].split("::")[-1]
            e = by_kernel.setdefault(k, [0.0, 0.0, 0.0])
            e[0] += L.get("dram__bytes_read.sum", 0.0) / len(tail)
            e[1] += L.get("dram__bytes_write.sum", 0.0) / len(tail)
            e[2] += L.get("gpu__time_duration.sum", 0.0) / len(tail)
    res[name] = {"dram_bytes_per_call": rd + wr, "dram_read_per_call": rd, "dram_write_per_call": wr,
                 "kernel_ns_per_call": t, "launches_per_call": per_call, "calls_averaged": len(tail),
                 "by_kernel": {k: {"read": v[0], "write": v[1], "ns": v[2]} for k, v in by_kernel.items()},
                 "build_id": _lib.build_id(),
                 "source": f"ncu --cache-control none --clock-control none, {len(calls)} calls of tools/traffic_case.py"}
    print(name, json.dumps(res[name]))
if not print_only:
    json.dump(res, open(out_path, "w"), indent=1)
