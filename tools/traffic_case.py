"""Calls of the per-window path as bench.py makes them (C2 batches from a ring of 8 distinct 64 MiB batches,
so inputs are not L2-resident), for an ncu capture of per-kernel DRAM traffic (tools/gpu/traffic.sh).
usage: python tools/traffic_case.py [calls] [workload C2|C3]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import gen  # noqa: E402
import paper_2509_03653_b200 as nsg  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 12
wl = sys.argv[2] if len(sys.argv) > 2 else "C2"
dist, seed = (gen.Dist("zipf", 1.1, 1 << 20), 2) if wl == "C2" else (gen.Dist("heavy"), 3)
W, n = 1 << 17, 64 << 17
ring = torch.empty((8, n), dtype=torch.int64, device="cuda")
for i in range(8):
    gen.generate_device(dist, seed, i * n, n, keys=ring[i])
ws = nsg.Workspace(n, W)
out = torch.empty((64, 9), dtype=torch.int64, device="cuda")
for i in range(calls):
    nsg.window_stats_packed(ring[i % 8], W, out=out, workspace=ws)
torch.cuda.synchronize()
print("calls", calls, "launches per call", nsg.last_launches())
