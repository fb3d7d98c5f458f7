"""Timing experiment: per-CTA cycle breakdown of win_kernel (variant built with -DNSG_WIN_PROF).
usage (GPU box): NSG_LIB_PATH_DEV=tools/libnsg_prof.so python tools/win_prof.py [--cfg C2] [--reps 5]"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2509_03653_b200 as nsg  # noqa: E402
from paper_2509_03653_b200 import api  # noqa: E402
from gen.configs import CONFIGS  # noqa: E402

NAMES = {0: "cons wait full", 1: "cons P", 2: "cons L part", 3: "cons L final", 4: "cons S part", 5: "cons S final",
         6: "cons done", 8: "prod stage-free", 9: "prod deps+offsets", 11: "prod desc", 12: "prod issue",
         16: "sig idle", 18: "sig signal", 20: "L wave0 (warp0)", 21: "L wave0 barrier", 22: "L rounds",
         27: "L rounds count"}

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="C2")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
c = CONFIGS[a.cfg]
dev = torch.device("cuda", 0)
keys = gen.generate_host(c.dist, c.seed, 0, c.n_packets, packed=True)
kd = torch.from_numpy(keys.view(np.int64)).to(dev)
lib = api._lib
lib.nsg_debug_win_prof.restype = ctypes.c_uint
lib.nsg_debug_win_prof.argtypes = [ctypes.c_void_p]
buf = np.zeros((1024, 32), dtype=np.uint64)
nsg.window_stats_packed(kd, c.window)
torch.cuda.synchronize()
lib.nsg_debug_win_prof(buf.ctypes.data)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    nsg.window_stats_packed(kd, c.window)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
lib.nsg_debug_win_prof(buf.ctypes.data)
ctas = int((buf.sum(axis=1) > 0).sum())
tot = buf[:ctas].astype(np.float64).sum(axis=0) / a.reps
print(f"{a.cfg}: {ms * 1e3:.1f} us per call, {ctas} CTAs; per-CTA mean cycles per call (x1e3):")
items = {k: tot[k] for k in (24, 25, 26)}
print("  items per call: P %d L %d S %d" % (items[24], items[25], items[26]))
for k, nm in NAMES.items():
    print(f"  {nm:16s} {tot[k] / ctas / 1e3:10.1f}k   per item-of-type: "
          + (f"{tot[k] / max(1, items[24]):.0f}" if k == 1 else f"{tot[k] / max(1, items[25]):.0f}" if k in (2, 3) else
             f"{tot[k] / max(1, items[26]):.0f}" if k in (4, 5) else ""))
