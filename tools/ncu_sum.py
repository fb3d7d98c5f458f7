"""Mean of each metric per kernel in an `ncu --csv --metrics ...` launch list. usage: ncu_sum.py list.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, d = None, collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        d[(x["Kernel Name"].split("(")[0][-14:], x["Metric Name"])].append(float(x["Metric Value"].replace(",", "")))
for k, v in sorted(d.items()):
    print(f"{k[0]:14s} {k[1]:60s} n={len(v)} mean={sum(v) / len(v):.2f}")
