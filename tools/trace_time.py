"""Timing of the whole-trace path (nsg_trace_stats) on device-generated Zipf / uniform inputs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_2509_03653_b200 as nsg

dev = torch.device("cuda", 0)
for name, dist in (("zipf", gen.Dist("zipf", 1.1, 1 << 20)), ("uniform", gen.Dist("uniform"))):
    for logn in (23, 26, 28):
        n = 1 << logn
        kd = torch.empty(n, dtype=torch.int64, device=dev)
        gen.generate_device(dist, 5, 0, n, keys=kd)
        for _ in range(2):
            out = nsg.trace_stats(kd)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        a.record()
        for _ in range(reps):
            nsg.trace_stats(kd, out=out)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        print(f"{name} 2^{logn}: {ms:.3f} ms  {n / ms / 1e6:.2f} Gpkt/s  {out.cpu().tolist()}", flush=True)
        del kd
        torch.cuda.empty_cache()
