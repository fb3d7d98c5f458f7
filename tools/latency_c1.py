"""C1 (one 2^17-packet uniform window): latency of one call per window (CUDA events, median
and min of 200 calls after warm-up; input device-resident), and the oracle O1 / O2 time on the host."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2509_03653_b200 as nsg  # noqa: E402
from gen.configs import CONFIGS  # noqa: E402

c = CONFIGS["C1"]
keys = gen.generate_host(c.dist, c.seed, 0, c.n_packets, packed=True)
kd = torch.from_numpy(keys.view(np.int64)).cuda()
ws = nsg.Workspace(kd.numel(), c.window)
out = torch.empty((1, 9), dtype=torch.int64, device="cuda")
for _ in range(10):
    nsg.window_stats_packed(kd, c.window, out=out, workspace=ws)
torch.cuda.synchronize()
ms = []
for _ in range(200):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    nsg.window_stats_packed(kd, c.window, out=out, workspace=ws)
    b.record()
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
ok = np.array_equal(out.cpu().numpy().view(np.uint64), oracle.window_stats_sort(keys=keys, window=c.window))
t0 = time.perf_counter()
oracle.window_stats_sort(keys=keys, window=c.window, threads=1)
t2 = time.perf_counter() - t0
t0 = time.perf_counter()
oracle.window_stats_map(keys=keys, window=c.window, threads=1)
t1 = time.perf_counter() - t0
print(f"C1 one window: median {np.median(ms) * 1e3:.1f} us, min {min(ms) * 1e3:.1f} us per call (parity {ok}); "
      f"oracle O2 {t2 * 1e3:.1f} ms, O1 {t1 * 1e3:.1f} ms (1 thread)")
