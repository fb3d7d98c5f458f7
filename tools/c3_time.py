"""C3 (heavy hitter) call time of the per-window path vs the round-1 kernel (design check)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2509_03653_b200 as nsg  # noqa: E402

for wl, dist, seed in (("C3", gen.Dist("heavy"), 3), ("C2", gen.Dist("zipf", 1.1, 1 << 20), 2),
                       ("C1-like", gen.Dist("uniform"), 1)):
    n = 64 << 17
    ring = torch.empty((4, n), dtype=torch.int64, device="cuda")
    for i in range(4):
        gen.generate_device(dist, seed, i * n, n, keys=ring[i])
    ws = nsg.Workspace(n, 1 << 17)
    out = torch.empty((64, 9), dtype=torch.int64, device="cuda")
    for flags, name in ((0, "r2"), (nsg.api._FLAG_LEGACY_FAST, "r1")):
        for i in range(3):
            nsg.window_stats_packed(ring[i % 4], 1 << 17, out=out, workspace=ws, flags=flags)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for i in range(20):
            nsg.window_stats_packed(ring[i % 4], 1 << 17, out=out, workspace=ws, flags=flags)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / 20
        print(f"{wl} {name}: {ms * 1e3:.1f} us/call = {n / ms / 1e6:.1f} Gpkt/s diag {ws.diag()}", flush=True)
