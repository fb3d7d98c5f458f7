"""Quick GPU check used during development: parity on a spread of cases + a rough C2 timing."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import oracle
import paper_2509_03653_b200 as nsg

dev = torch.device("cuda", 0)
fails = 0


def check(name, keys, window, flags=0, soa=False):
    global fails
    kd = torch.from_numpy(keys.view(np.int64)).to(dev)
    t0 = time.time()
    if soa:
        s = (kd >> 32).to(torch.int32).contiguous()
        d = (kd & 0xFFFFFFFF).to(torch.int32).contiguous()
        got = nsg.window_stats(s, d, window, flags=flags)
    else:
        got = nsg.window_stats_packed(kd, window, flags=flags)
    got = got.cpu().numpy().view(np.uint64)
    t1 = time.time()
    want = oracle.window_stats_sort(keys=keys, window=window)
    ok = np.array_equal(got, want)
    if not ok:
        fails += 1
        bad = np.nonzero((got != want).any(axis=1))[0]
        print(f"FAIL {name}: {len(bad)} bad windows of {len(want)}; first {bad[:5]}")
        for w in bad[:3]:
            print("   got ", got[w].tolist())
            print("   want", want[w].tolist())
    else:
        print(f"ok   {name}: {len(want)} windows ({t1 - t0:.3f}s) row0={got[0].tolist() if len(got) else []}")


W = 1 << 17
for name, dist, seed in [("C1-uniform", gen.Dist("uniform"), 1), ("C2-zipf", gen.Dist("zipf", 1.1, 1 << 20), 2),
                         ("C3-heavy", gen.Dist("heavy"), 3)]:
    n = W if name.startswith("C1") else 8 * W + 777
    keys = gen.generate_host(dist, seed, 0, n, packed=True)
    check(name, keys, W)
    check(name + "-soa", keys, W, soa=True)
    check(name + "-global", keys, W, flags=nsg.FLAG_FORCE_GLOBAL)
    check(name + "-inject", keys, W, flags=nsg.FLAG_INJECT_OVERFLOW)

rng = np.random.default_rng(0)
for window in [1, 2, 3, 7, 31, 1000, 4095, 4096, 4097, 9999, 65536, 1 << 20]:
    n = int(window * 3.5) + 1 if window < (1 << 20) else (1 << 21) + 5
    keys = rng.integers(0, 2**64, size=n, dtype=np.uint64) & np.uint64(0x000F000F000F000F)
    check(f"small-universe W={window}", keys, window)
    keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 12), 9, 0, n, packed=True)
    check(f"zipf-small W={window}", keys, window)
# adversarial keys
n = 3 * W
keys = np.full(n, 0xFFFFFFFFFFFFFFFF, dtype=np.uint64)
check("all ~0", keys, W)
keys[::3] = 0
keys[1::7] = 0xFFFFFFFF00000000
keys[2::11] = 0x00000000FFFFFFFF
check("adversarial sentinels", keys, W)
check("adversarial sentinels global", keys, W, flags=nsg.FLAG_FORCE_GLOBAL)
keys = np.full(n, 0x0A0000010A000002, dtype=np.uint64)
check("all same", keys, W)
keys = (np.arange(n, dtype=np.uint64) << np.uint64(32)) | np.uint64(7)
check("star-in", keys, W)
keys = np.uint64(5 << 32) | np.arange(n, dtype=np.uint64)
check("star-out", keys, W)
# window > fast max (global path only)
keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 20), 4, 0, (1 << 22) + 3, packed=True)
check("W=2^21 global", keys, 1 << 21)

# rough timing on C2 (64 windows)
keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 20), 2, 0, 1 << 23, packed=True)
kd = torch.from_numpy(keys.view(np.int64)).to(dev)
ws = nsg.Workspace(kd.numel(), W)
out = torch.empty((64, 9), dtype=torch.int64, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
for _ in range(3):
    nsg.window_stats_packed(kd, W, out=out, workspace=ws)
torch.cuda.synchronize()
times = []
for _ in range(20):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    nsg.window_stats_packed(kd, W, out=out, workspace=ws)
    b.record()
    torch.cuda.synchronize()
    times.append(a.elapsed_time(b))
t = float(np.median(times))
print(f"C2 timing: median {t*1e3:.1f} us, min {min(times)*1e3:.1f} us -> {(1<<23)/t/1e6:.1f} Gpkt/s; diag={ws.diag()}")
for flag in [nsg.FLAG_NO_FALLBACK_CHECK]:
    times = []
    for _ in range(20):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        nsg.window_stats_packed(kd, W, out=out, workspace=ws, flags=flag)
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    t = float(np.median(times))
    print(f"C2 timing (no fallback launch): median {t*1e3:.1f} us -> {(1<<23)/t/1e6:.1f} Gpkt/s")
print("FAILS:", fails)
sys.exit(1 if fails else 0)
