"""e2e (host input) timing of window_stats_from_host vs chunk size and the bare H2D copy (C2 batch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import paper_2509_03653_b200 as nsg
from gen.configs import CONFIGS

c = CONFIGS["C2"]
dev = torch.device("cuda", 0)
kd0 = torch.empty(c.n_packets, dtype=torch.int64, device=dev)
gen.generate_device(c.dist, c.seed, 0, c.n_packets, keys=kd0)
host = kd0.cpu().pin_memory()
kd = torch.empty_like(kd0)
ws = nsg.Workspace(c.n_packets, c.window)
out = torch.empty((64, 9), dtype=torch.int64, device=dev)
oh = torch.empty((64, 9), dtype=torch.int64, pin_memory=True)
want = nsg.window_stats_packed(kd0, c.window).cpu()


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


print(f"bare H2D 64 MiB: {t(lambda: kd.copy_(host, non_blocking=True)):.3f} ms")
for ch in (1, 2, 4, 8, 16, 64):
    ms = t(lambda: nsg.window_stats_from_host(host, c.window, keys_dev=kd, out=out, out_host=oh, workspace=ws,
                                               chunk_windows=ch))
    assert torch.equal(oh, want)
    print(f"from_host chunk {ch:3d}: {ms:.3f} ms  {c.n_packets / ms / 1e6:.2f} Gpkt/s")

# zero-copy: the kernel's partition items read the pinned host keys over PCIe (UVA pointer)
import ctypes
from paper_2509_03653_b200 import _lib
lib = _lib.load()
s = torch.cuda.current_stream(dev)


def zc():
    rc = lib.nsg_window_stats_timed(None, None, host.data_ptr(), c.n_packets, c.window, out.data_ptr(), ws.ptr,
                                    ws.nbytes, ctypes.c_void_p(s.cuda_stream), 0, None, None)
    assert rc == 0
    oh.copy_(out, non_blocking=True)


ms = t(zc)
assert torch.equal(oh, want)
print(f"zero-copy kernel on host keys: {ms:.3f} ms  {c.n_packets / ms / 1e6:.2f} Gpkt/s")
