"""Summarise the round's ncu captures from gpurun_out/ into profiles/ (tracked).

usage: python tools/update_profiles.py ROUND_TAG [workload]
Reads gpurun_out/launches.csv (ncu --metrics gpu__time_duration.sum launch list of bench.py) and
gpurun_out/prof_bench.ncu-rep (ncu --set full capture of nsg::fast_kernel), writes
profiles/<tag>_launches_<wl>.txt, profiles/<tag>_ncu_fast_kernel_<wl>.txt and updates
profiles/ncu_traffic.json (dram bytes per launch, read by bench.py's roofline.traffic).
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
wl = sys.argv[2] if len(sys.argv) > 2 else "C2"
go = os.path.join(ROOT, "gpurun_out")
prof = os.path.join(ROOT, "profiles")

rows = [r for r in csv.reader(open(os.path.join(go, "launches.csv"))) if len(r) > 5]
h = rows[0]
I = {k: i for i, k in enumerate(h)}
out = ["# ncu --metrics gpu__time_duration.sum --clock-control none -c 60 python bench.py --steps 5 --warmup 3 "
       "--no-cpu-baseline", "# cold-cache, serialised launches: compare shares, not absolutes.  id, kernel, duration (ns)"]
tot = {}
for r in rows[1:]:
    k = r[I["Kernel Name"]].split("(")[0]
    v = float(r[I["Metric Value"]])
    out.append(f"{r[I['ID']]:>4} {k:28s} {v:12.1f}")
    if "gen_kernel" not in k:
        tot[k] = tot.get(k, 0.0) + v
s = sum(tot.values())
out.append("# share of the nsg step (input generator excluded): " + ", ".join(f"{k} {100 * v / s:.1f}%" for k, v in tot.items()))
open(os.path.join(prof, f"{tag}_launches_{wl}.txt"), "w").write("\n".join(out) + "\n")

raw = subprocess.run(["ncu", "-i", os.path.join(go, "prof_bench.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, units, vals = r[0], r[1], r[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"]
lines = [f"# ncu --set full --clock-control none -k regex:fast_kernel -s 3 -c 1 python bench.py --steps 3 --warmup 3 "
         f"--workload {wl} (one bench step: 64 windows x 2^17 packets)"]
for k in keys:
    if k in h:
        lines.append(f"{k:75s} {vals[h.index(k)]:>18s} {units[h.index(k)]}")
open(os.path.join(prof, f"{tag}_ncu_fast_kernel_{wl}.txt"), "w").write("\n".join(lines) + "\n")
mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = float(vals[h.index("dram__bytes_read.sum")]) * mul[units[h.index("dram__bytes_read.sum")]]
wr = float(vals[h.index("dram__bytes_write.sum")]) * mul[units[h.index("dram__bytes_write.sum")]]
tj = os.path.join(prof, "ncu_traffic.json")
t = json.load(open(tj)) if os.path.exists(tj) else {}
t[wl] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
         "source": f"profiles/{tag}_ncu_fast_kernel_{wl}.txt"}
json.dump(t, open(tj, "w"), indent=1)
print("\n".join(lines))
print(out[-1])
