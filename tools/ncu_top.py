"""Summarise an ncu --page source --csv --print-source=cuda,sass dump: top CUDA lines and top SASS
instructions by stall samples, with their dominant stall reasons.  usage: ncu_top.py dump.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[2]
I = {k: i for i, k in enumerate(h)}
sc = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
lines, sass, cur = [], [], None
for r in rows[3:]:
    if len(r) < len(h):
        continue
    if r[0]:
        cur = (r[0], r[1][:90])
        try:
            lines.append((int(r[I["Warp Stall Sampling (All Samples)"]] or 0), int(r[I["Instructions Executed"]] or 0), cur))
        except ValueError:
            pass
        continue
    try:
        s = int(r[I["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    st = sorted(((k[6:], int(r[I[k]] or 0)) for k in sc), key=lambda x: -x[1])[:3]
    sass.append((s, cur, r[3].strip()[:58], st))
ts = sum(x[0] for x in lines) or 1
ti = sum(x[1] for x in lines) or 1
print(f"samples {ts}  warp-inst {ti}")
print("--- CUDA lines by stall samples")
for s, i, c in sorted(lines, key=lambda x: -x[0])[:N]:
    print(f"{100*s/ts:5.1f}% {100*i/ti:5.1f}%i L{c[0]:>4} {c[1]}")
print("--- SASS by stall samples")
for s, c, ins, st in sorted(sass, key=lambda x: -x[0])[:N]:
    print(f"{100*s/ts:5.1f}% L{c[0]:>4} {ins:58s} {st}")
