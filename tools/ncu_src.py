"""Summarise `ncu -i X --page source --csv --print-source=cuda,sass [-k regex:K]` output across all
source files: CUDA lines by stall samples and executed instructions.  usage: ncu_src.py dump.csv [N] [minline maxline]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
lo, hi_l = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 10 ** 9)
agg, inst, fname, h, I, sc, cur = {}, {}, "", None, None, None, None
for r in rows:
    if len(r) >= 2 and r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 3 and "Warp Stall Sampling (All Samples)" in r:
        h = r
        I = {k: i for i, k in enumerate(h)}
        sc = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
        continue
    if h is None or len(r) < len(h):
        continue
    if r[0]:
        try:
            cur = (fname, int(r[0]), r[1][:60])
        except ValueError:
            cur = None
        continue
    if cur is None:
        continue
    try:
        s = int(r[I["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    d = agg.setdefault(cur, {})
    inst[cur] = inst.get(cur, 0) + int(r[I["Instructions Executed"]] or 0)
    for k in sc:
        d[k[6:]] = d.get(k[6:], 0) + int(r[I[k]] or 0)
tot = sum(sum(v.values()) for v in agg.values()) or 1
ti = sum(inst.values()) or 1
print(f"samples {tot} inst {ti}")
items = sorted(((sum(v.values()), k, v) for k, v in agg.items() if lo <= k[1] <= hi_l), key=lambda x: -x[0])
for s, k, v in items[:N]:
    top = sorted(v.items(), key=lambda x: -x[1])[:3]
    print(f"{100*s/tot:5.1f}% {100*inst[k]/ti:5.1f}%i {k[0][:14]}:{k[1]} {k[2]:55s} {top}")
