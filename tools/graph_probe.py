"""Design check: one call of the per-window path captured in a CUDA graph and replayed, vs plain calls
(C2 ring of 8 batches, one stream; parity of the replayed output)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2509_03653_b200 as nsg  # noqa: E402

W, n = 1 << 17, 64 << 17
dist = gen.Dist("zipf", 1.1, 1 << 20)
ring = torch.empty((8, n), dtype=torch.int64, device="cuda")
for i in range(8):
    gen.generate_device(dist, 2, i * n, n, keys=ring[i])
ws = nsg.Workspace(n, W)
outs = [torch.empty((64, 9), dtype=torch.int64, device="cuda") for _ in range(8)]
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for i in range(3):
        nsg.window_stats_packed(ring[i], W, out=outs[i], workspace=ws, stream=s)
torch.cuda.synchronize()
graphs = []
for i in range(8):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        nsg.window_stats_packed(ring[i], W, out=outs[i], workspace=ws, stream=s)
    graphs.append(g)
torch.cuda.synchronize()
for name, fn in (("plain", lambda i: nsg.window_stats_packed(ring[i % 8], W, out=outs[i % 8], workspace=ws, stream=s)),
                 ("graph", lambda i: graphs[i % 8].replay())):
    with torch.cuda.stream(s):
        for i in range(5):
            fn(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for i in range(100):
            fn(i)
        e1.record(s)
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 100 * 1e3:.1f} us per call", flush=True)
for i in range(8):
    graphs[i].replay()
torch.cuda.synchronize()
keys = ring[3].cpu().numpy().view(np.uint64)
print("parity of a replayed call:", np.array_equal(outs[3].cpu().numpy().view(np.uint64),
                                                    oracle.window_stats_sort(keys=keys, window=W)))
