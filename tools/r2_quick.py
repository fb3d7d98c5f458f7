"""Quick GPU check of the per-window kernel: parity vs the oracle on C1-C3 (+ small windows) and
device time of one C2 launch, round-2 kernel vs the round-1 kernel (NSG_FLAG_LEGACY_FAST).
Usage (GPU box): python tools/r2_quick.py [--reps N]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2509_03653_b200 as nsg  # noqa: E402
from gen.configs import CONFIGS  # noqa: E402

LEGACY = 16


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--skip-parity", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    if not a.skip_parity:
        cases = [("C1", None, None), ("C2", None, None), ("C3", None, None)]
        for name, _, _ in cases:
            c = CONFIGS[name]
            keys = gen.generate_host(c.dist, c.seed, 0, c.n_packets, packed=True)
            want = oracle.window_stats_sort(keys=keys, window=c.window)
            kd = torch.from_numpy(keys.view(np.int64)).to(dev)
            t0 = time.time()
            got = nsg.window_stats_packed(kd, c.window).cpu().numpy().view(np.uint64)
            ok = np.array_equal(got, want)
            print(f"{name}: parity {'OK' if ok else 'FAIL'} ({time.time() - t0:.2f}s)", flush=True)
            if not ok:
                bad = np.nonzero((got != want).any(axis=1))[0]
                print("  bad windows", bad[:10].tolist(), "of", len(bad))
                print("  got ", got[bad[0]].tolist())
                print("  want", want[bad[0]].tolist())
        for window, n in [(1, 100), (7, 1000), (1000, 12345), (4096, 4096 * 3 + 5), (5000, 77777),
                          (1 << 16, (1 << 18) + 3), ((1 << 17) + 1, (1 << 19) + 9)]:
            keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 20), 9, 0, n, packed=True)
            want = oracle.window_stats_sort(keys=keys, window=window)
            kd = torch.from_numpy(keys.view(np.int64)).to(dev)
            got = nsg.window_stats_packed(kd, window).cpu().numpy().view(np.uint64)
            ok = np.array_equal(got, want)
            print(f"window {window} n {n}: parity {'OK' if ok else 'FAIL'}", flush=True)
            if not ok:
                bad = np.nonzero((got != want).any(axis=1))[0]
                print("  bad", bad[:10].tolist(), "got", got[bad[0]].tolist(), "want", want[bad[0]].tolist())
    # timing: C2 ring of 8 batches (inputs larger than L2 in aggregate)
    c = CONFIGS["C2"]
    ring = []
    for i in range(8):
        keys = gen.generate_host(c.dist, c.seed + 100 * i, 0, c.n_packets, packed=True)
        ring.append(torch.from_numpy(keys.view(np.int64)).to(dev))
    out = torch.empty((64, 9), dtype=torch.int64, device=dev)
    ws = nsg.Workspace(c.n_packets, c.window, dev)
    for flags, name in [(0, "r2"), (LEGACY, "r1-legacy"), (0, "r2")]:
        for i in range(3):
            nsg.window_stats_packed(ring[i % 8], c.window, out=out, workspace=ws, flags=flags)
        torch.cuda.synchronize()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.reps)]
        for r in range(a.reps):
            evs[2 * r].record()
            nsg.window_stats_packed(ring[r % 8], c.window, out=out, workspace=ws, flags=flags)
            evs[2 * r + 1].record()
        torch.cuda.synchronize()
        ms = [evs[2 * r].elapsed_time(evs[2 * r + 1]) for r in range(a.reps)]
        med = float(np.median(ms))
        print(f"{name}: C2 call median {med * 1e3:.1f} us  min {min(ms) * 1e3:.1f} us -> "
              f"{c.n_packets / med / 1e6:.1f} Gpkt/s (diag {ws.diag()})", flush=True)


if __name__ == "__main__":
    main()
