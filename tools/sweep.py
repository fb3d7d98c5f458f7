"""C5 scaling sweep on one GPU: n in {2^28 .. 2^32} packets x {uniform, zipf}, device-generated, one
launch over all windows (timed by CUDA events after a warm-up launch), plus sampled parity against
the CPU oracle (first, middle, last windows regenerated on the host).

usage: python tools/sweep.py [--max-log2 32] [--out profiles/r01_sweep_C5.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import oracle
import paper_2509_03653_b200 as nsg
from gen.configs import sweep_config

ap = argparse.ArgumentParser()
ap.add_argument("--min-log2", type=int, default=28)
ap.add_argument("--max-log2", type=int, default=32)
ap.add_argument("--out", default=None, help="JSON file (write it under gpurun_out/ to bring it back from the GPU box)")
args = ap.parse_args()
dev = torch.device("cuda", 0)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
rows = []
for lg in range(args.min_log2, args.max_log2 + 1):
    for dname in ("uniform", "zipf"):
        c = sweep_config(lg, dname)
        n, W = c.n_packets, c.window
        keys = torch.empty(n, dtype=torch.int64, device=dev)
        gen.generate_device(c.dist, c.seed, 0, n, keys=keys)
        ws = nsg.Workspace(n, W)
        nw = nsg.num_windows(n, W)
        out = torch.empty((nw, 9), dtype=torch.int64, device=dev)
        nsg.window_stats_packed(keys, W, out=out, workspace=ws)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            nsg.window_stats_packed(keys, W, out=out, workspace=ws, kernel_events=(a, b))
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        t = min(ts) / 1e3
        got = out.cpu().numpy().view(np.uint64)
        ok = True
        for w in sorted({0, nw // 2, nw - 1}):
            k = gen.generate_host(c.dist, c.seed, w * W, min(W, n - w * W), packed=True)
            ok &= got[w].tolist() == oracle.window_stats_sort(keys=k, window=W)[0].tolist()
        ok &= bool(np.all(got[:, 0] == W)) and ws.diag()[:2] == [0, 0]
        gbs = (n * 8 + nw * 72) / t / 1e9
        row = {"log2_n": lg, "dist": dname, "windows": nw, "kernel_ms": t * 1e3, "packets_per_s": n / t,
               "hbm_gbs_algorithmic": gbs, "roofline_frac": gbs / peak, "sampled_parity": bool(ok)}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del keys, ws, out
        torch.cuda.empty_cache()
if args.out:
    json.dump({"what": "C5 sweep, 1 B200, one launch per size, min of 3 CUDA-event timings", "rows": rows},
              open(args.out, "w"), indent=1)
