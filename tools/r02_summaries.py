"""Summaries of the round-2 profile set (tools/gpu/profiles_r02.sh) for profiles/r02/:
launch shares of the bench run, and the key counters of each per-window kernel's ncu --set full capture."""
import collections
import csv
import os
import sys

D = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/r02"
OUT = sys.argv[2] if len(sys.argv) > 2 else "profiles/r02"
os.makedirs(OUT, exist_ok=True)

# 1. launch list: share of device time by kernel (ncu serialises launches: compare shares)
rows = list(csv.reader(open(os.path.join(D, "launches_C2.csv"))))
hdr, agg, cnt = None, collections.Counter(), collections.Counter()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        if x["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = x["Kernel Name"].split("(")[0]
        agg[k] += float(x["Metric Value"].replace(",", ""))
        cnt[k] += 1
tot = sum(agg.values())
with open(os.path.join(OUT, "launches_C2.txt"), "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 over `python bench.py --steps 20 "
            "--warmup 3 --no-cpu-baseline` (C2, build of this commit); launches are serialised and cold under ncu,\n"
            "# so compare shares, not absolutes.  Columns: kernel, launches, total us, share of all device time\n")
    for k, v in agg.most_common():
        f.write(f"{k:60s} {cnt[k]:5d} {v / 1e3:10.1f} {100 * v / tot:6.2f}%\n")
    flat = sum(v for k, v in agg.items() if "flat::" in k)
    f.write(f"# the per-window kernels (nsg::flat::*): {100 * flat / tot:.2f}% of device time "
            f"(the rest: input generation, e2e copies, the L2-path check, torch)\n")

# 2. full captures: selected raw counters per kernel
rows = list(csv.reader(open(os.path.join(D, "full_C2_raw.csv"))))
hdr = rows[0]
units = rows[1]
want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_shared_mem", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
        "smsp__sass_inst_executed_op_shared.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed"]
idx = {h: i for i, h in enumerate(hdr)}
W = 1 << 17
with open(os.path.join(OUT, "ncu_full_C2.txt"), "w") as f:
    f.write("# ncu --set full --clock-control none on one C2 call (64 windows x 2^17 packets = 2^23 packets); the "
            "capture holds one launch of each kernel = one batch\n# (8 windows for this call size; the packets of a "
            "launch follow from its grid: part 32 CTAs, link and side 128 CTAs per window)\n")
    for r in rows[2:]:
        name = r[idx["Kernel Name"]].split("(")[0]
        grid = int(float(r[idx["launch__grid_size"]].replace(",", "")))
        pk = grid // (32 if "part" in name else 128) * W  # packets of this launch
        f.write(f"\n== {name}\n")
        for m in want:
            if m in idx:
                f.write(f"  {m:75s} {r[idx[m]]:>16s} {units[idx[m]]}\n")
        if "smsp__inst_executed.sum" in idx:
            inst = float(r[idx["smsp__inst_executed.sum"]].replace(",", ""))
            f.write(f"  warp-instructions per packet (per launch / {pk} packets): {inst / pk:.2f}\n")
        for m, label in (("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts"),
                         ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "  of which atomics")):
            if m in idx:
                v = float(r[idx[m]].replace(",", ""))
                f.write(f"  {label} per packet: {v / pk:.2f}\n")
print(open(os.path.join(OUT, "launches_C2.txt")).read())
print(open(os.path.join(OUT, "ncu_full_C2.txt")).read())
