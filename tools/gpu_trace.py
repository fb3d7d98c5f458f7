"""Item timeline of one fast-kernel launch (build a variant with -DNSG_EXP_TRACE, run with
NSG_LIB_PATH_DEV pointing at it).  Prints occupancy over time by item type and per-window latencies.
usage: NSG_LIB_PATH_DEV=tools/libnsg_tr.so python tools/gpu_trace.py [config]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import paper_2509_03653_b200 as nsg
from paper_2509_03653_b200 import _lib
from gen.configs import CONFIGS, Config

EXTRA = {"U2": Config("U2", 1 << 23, gen.Dist("uniform"), 2),
         "C2x4": Config("C2x4", 1 << 25, gen.Dist("zipf", 1.1, 1 << 20), 2)}
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = CONFIGS.get(name) or EXTRA[name]
dev = torch.device("cuda", 0)
kd = torch.empty(cfg.n_packets, dtype=torch.int64, device=dev)
gen.generate_device(cfg.dist, cfg.seed, 0, cfg.n_packets, keys=kd)
ws = nsg.Workspace(cfg.n_packets, cfg.window)
nw = nsg.num_windows(cfg.n_packets, cfg.window)
out = torch.empty((nw, 9), dtype=torch.int64, device=dev)
lib = _lib.load()
lib.nsg_debug_trace.restype = ctypes.c_uint
lib.nsg_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_uint]
cap = 1 << 18
buf = np.zeros((cap, 4), dtype=np.uint64)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
for _ in range(3):
    nsg.window_stats_packed(kd, cfg.window, out=out, workspace=ws)
torch.cuda.synchronize()
flush.zero_()
lib.nsg_debug_trace(buf.ctypes.data, cap)  # reset
nsg.window_stats_packed(kd, cfg.window, out=out, workspace=ws)
torch.cuda.synchronize()
n = lib.nsg_debug_trace(buf.ctypes.data, cap)
tr = buf[:n]
typ = (tr[:, 0] >> np.uint64(56)).astype(int)
win = ((tr[:, 0] >> np.uint64(32)) & np.uint64(0xFFFFFF)).astype(int)
t0 = tr[:, 1].astype(np.int64)
t1 = tr[:, 2].astype(np.int64)
base = t0.min()
t0 = (t0 - base) / 1e3
t1 = (t1 - base) / 1e3
span = t1.max()
print(f"{name}: {n} items, span {span:.1f} us")
names = {0: "P", 1: "L", 2: "S0", 3: "S1", 4: "F", 5: "nop"}
for k, v in names.items():
    m = typ == k
    if m.any():
        print(f"  {v:3s}: {m.sum():6d} items, mean {np.mean(t1[m] - t0[m]):7.2f} us, total {np.sum(t1[m] - t0[m]) / 1e3:8.2f} CTA-ms")
ncta = len(np.unique(tr[:, 3])) * 2
busy = np.sum(t1 - t0) / 1e3
print(f"  busy {busy:.2f} CTA-ms of {ncta * span / 1e3:.2f} ({100 * busy / (ncta * span / 1e3):.1f}%)")
bins = np.arange(0, span + 10, 10.0)
print("  time(us)  active items by type (P L S F nop) per 10 us bin (average concurrency)")
for b0 in bins[:-1]:
    b1 = b0 + 10
    row = []
    for k in (0, 1, 2, 4, 5):
        m = (typ == k) if k != 2 else ((typ == 2) | (typ == 3))
        ov = np.clip(np.minimum(t1[m], b1) - np.maximum(t0[m], b0), 0, None).sum() / 10
        row.append(ov)
    print(f"  {b0:7.0f}  " + " ".join(f"{x:6.1f}" for x in row) + f"   sum {sum(row):6.1f}")
print("  window  P_start P_end  L_start L_end  S_start S_end  F_end")
for w in list(range(0, nw, max(1, nw // 16))) + [nw - 1]:
    def rng(k):
        m = (win == w) & (typ == k) if k != 2 else (win == w) & ((typ == 2) | (typ == 3))
        return (t0[m].min(), t1[m].max()) if m.any() else (float("nan"), float("nan"))
    p, l, s, f = rng(0), rng(1), rng(2), rng(4)
    print(f"  {w:6d} {p[0]:7.1f} {p[1]:6.1f} {l[0]:7.1f} {l[1]:6.1f} {s[0]:7.1f} {s[1]:6.1f} {f[1]:6.1f}")
if "--last" in sys.argv:
    for k, v in ((0, "P"), (1, "L"), (2, "S0"), (3, "S1")):
        m = (win == nw - 1) & (typ == k)
        o = np.argsort(t0[m])
        print(f"  last window {v}: " + " ".join(f"{a:.0f}-{b:.0f}" for a, b in zip(t0[m][o], t1[m][o])))
