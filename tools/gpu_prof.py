"""Per-work-item-type cycle breakdown of the fast kernel (NSG_FLAG_PROFILE) + plain timing.
usage: python tools/gpu_prof.py [config] [--once]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import paper_2509_03653_b200 as nsg
from gen.configs import CONFIGS

FLAG_PROFILE = 8
from gen.configs import Config
EXTRA = {"U2": Config("U2", 1 << 23, gen.Dist("uniform"), 2), "Z08": Config("Z08", 1 << 23, gen.Dist("zipf", 0.8, 1 << 20), 2),
         "C2x4": Config("C2x4", 1 << 25, gen.Dist("zipf", 1.1, 1 << 20), 2), "C2x16": Config("C2x16", 1 << 27, gen.Dist("zipf", 1.1, 1 << 20), 2),
         "C2h": Config("C2h", 1 << 22, gen.Dist("zipf", 1.1, 1 << 20), 2),
         "Z13": Config("Z13", 1 << 23, gen.Dist("zipf", 1.3, 1 << 20), 2)}
name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "C2"
cfg = CONFIGS.get(name) or EXTRA[name]
once = "--once" in sys.argv
dev = torch.device("cuda", 0)
kd = torch.empty(cfg.n_packets, dtype=torch.int64, device=dev)
gen.generate_device(cfg.dist, cfg.seed, 0, cfg.n_packets, keys=kd)
ws = nsg.Workspace(cfg.n_packets, cfg.window)
nw = nsg.num_windows(cfg.n_packets, cfg.window)
out = torch.empty((nw, 9), dtype=torch.int64, device=dev)
if once:
    nsg.window_stats_packed(kd, cfg.window, out=out, workspace=ws)
    torch.cuda.synchronize()
    sys.exit(0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def timed(flags, reps=20):
    for _ in range(3):
        nsg.window_stats_packed(kd, cfg.window, out=out, workspace=ws, flags=flags)
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        nsg.window_stats_packed(kd, cfg.window, out=out, workspace=ws, flags=flags)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


t = timed(0)
print(f"{cfg.name}: {t*1e3:.1f} us  {cfg.n_packets / t / 1e6:.1f} Gpkt/s")
tp = timed(FLAG_PROFILE, reps=1)
off = ws.offset + 128
prof = ws.buffer[off:off + 896].view(torch.int64).cpu().numpy()
clk = 1.9e9
print(f"profiled run: {tp*1e3:.1f} us")
for i, name in enumerate(["partition", "link", "side"]):
    n, cyc, wait, mx = prof[i * 4:i * 4 + 4]
    if n:
        print(f"  {name:9s}: {n:7d} items, avg {cyc / n:9.0f} cyc ({cyc / n / clk * 1e6:6.2f} us), avg wait {wait / n:8.0f} cyc; max work {mx:8d};"
              f" total {cyc / clk * 1e3:8.2f} CTA-ms")
        ph = prof[16 + 16 * i:16 + 16 * i + 12]
        print("     phases (avg cyc/item):", " ".join(f"{x / n:8.0f}" for x in ph if x))
        pm = prof[64 + 16 * i:64 + 16 * i + 12]
        print("     phases (max cyc/item):", " ".join(f"{x:8d}" for x in pm if x))
        if prof[16 + 16 * i + 12]:
            print(f"     first-wave pending entries: avg {prof[16 + 16 * i + 12] / n:.1f}, max {prof[64 + 16 * i + 12]}")
if prof[13]:
    print(f"item boundary (thread 0: end of item -> start of next): avg {prof[12] / prof[13]:.0f} cyc over {prof[13]} boundaries")
if "--items" in sys.argv:
    det = ws.buffer[ws.offset + 128:ws.offset + 128 + 8 * 256].view(torch.int64).cpu().numpy()
    print("window 0 side items (side*B2+sb: cycles / records):")
    print("  " + " ".join(f"{i}:{det[128 + i]}/{det[192 + i]}" for i in range(64) if det[192 + i]))
print("diag", ws.diag())
