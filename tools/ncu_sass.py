"""SASS rows of an `ncu --page source --print-source=cuda,sass` CSV in address order with executed
counts (warp-level) and average active threads.  usage: ncu_sass.py src.csv [min_count]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
mn = int(sys.argv[2]) if len(sys.argv) > 2 else 0
I, seen, out = None, set(), []
for r in rows:
    if r and r[0] == "Line No":
        I = {k: i for i, k in enumerate(r)}
        continue
    if I is None or len(r) < len(I) or r[0] != "" or not r[2].startswith("0x"):
        continue
    if r[2] in seen:
        continue
    seen.add(r[2])
    n = int(r[I["Instructions Executed"]] or 0)
    out.append((int(r[2], 16), n, r[I["Avg. Threads Executed"]], r[3]))
out.sort()
base = out[0][0] if out else 0
tot = sum(o[1] for o in out)
print("total", tot)
for a, n, th, s in out:
    if n >= mn:
        print(f"{a - base:6x} {n:10d} {th:>5s}  {s[:70]}")
