"""The §8(b) boundary itself (-m gpu): nsg_window_stats (SoA) and nsg_window_stats_packed called directly
through ctypes on the C ABI of include/nsg.h (no Python binding in between; torch only provides device
memory and the stream), compared with the oracle O2 on C1 and C2.  Also the debug
build's readback of the device self-check as NSG_ERR_INTERNAL (include/nsg.h "Errors").
"""
import ctypes
import os

import numpy as np
import pytest
import torch

import gen
import oracle
from gen.configs import CONFIGS

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2509_03653_b200")
NSG_OK, NSG_ERR_INTERNAL = 0, 5
NSG_FLAG_INJECT_SELF_CHECK = 1 << 5  # include/nsg_internal.h
DIAG_WORDS = 4


def _lib(name):
    lib = ctypes.CDLL(os.path.join(PKG, name))
    u64, sz, vp, u32 = ctypes.c_uint64, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_uint32
    lib.nsg_workspace_bytes.restype = sz
    lib.nsg_workspace_bytes.argtypes = [u64, u64]
    lib.nsg_num_windows.restype = u64
    lib.nsg_num_windows.argtypes = [u64, u64]
    lib.nsg_window_stats.restype = ctypes.c_int
    lib.nsg_window_stats.argtypes = [vp, vp, u64, u64, vp, vp, sz, vp]
    lib.nsg_window_stats_packed.restype = ctypes.c_int
    lib.nsg_window_stats_packed.argtypes = [vp, u64, u64, vp, vp, sz, vp]
    lib.nsg_window_stats_ex.restype = ctypes.c_int
    lib.nsg_window_stats_ex.argtypes = [vp, vp, vp, u64, u64, vp, vp, sz, vp, u32]
    lib.nsg_diag_offset.restype = sz
    lib.nsg_diag_offset.argtypes = []
    return lib


class Call:
    """Device buffers for one (n, window) call: aligned workspace, output, the current stream."""

    def __init__(self, lib, n, window, device):
        self.n, self.window = n, window
        self.nw = int(lib.nsg_num_windows(n, window))
        self.wsb = int(lib.nsg_workspace_bytes(n, window))
        self.wsbuf = torch.empty(self.wsb + 256, dtype=torch.uint8, device=device)
        self.off = (-self.wsbuf.data_ptr()) % 256
        self.ws = self.wsbuf.data_ptr() + self.off
        self.out = torch.empty((self.nw, 9), dtype=torch.int64, device=device)
        self.stream = ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)
        self.diag_off = int(lib.nsg_diag_offset())

    def result(self):
        torch.cuda.synchronize()
        return self.out.cpu().numpy().view(np.uint64)

    def diag(self):
        torch.cuda.synchronize()
        o = self.off + self.diag_off
        return self.wsbuf[o:o + 4 * DIAG_WORDS].view(torch.int32).cpu().tolist()


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_packed_entry_point(cuda_device, cfg):
    lib = _lib("libnsg.so")
    c = CONFIGS[cfg]
    keys = gen.generate_host(c.dist, c.seed, 0, c.n_packets, packed=True)
    kd = torch.from_numpy(keys.view(np.int64)).to(cuda_device)
    call = Call(lib, c.n_packets, c.window, cuda_device)
    rc = lib.nsg_window_stats_packed(kd.data_ptr(), c.n_packets, c.window, call.out.data_ptr(), call.ws, call.wsb,
                                     call.stream)
    assert rc == NSG_OK
    assert call.result().tolist() == oracle.window_stats_sort(keys=keys, window=c.window).tolist()
    assert call.diag()[:2] == [0, 0]


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_soa_entry_point(cuda_device, cfg):
    lib = _lib("libnsg.so")
    c = CONFIGS[cfg]
    keys = gen.generate_host(c.dist, c.seed, 0, c.n_packets, packed=True)
    src = torch.from_numpy((keys >> np.uint64(32)).astype(np.uint32).view(np.int32)).to(cuda_device)
    dst = torch.from_numpy((keys & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.int32)).to(cuda_device)
    call = Call(lib, c.n_packets, c.window, cuda_device)
    rc = lib.nsg_window_stats(src.data_ptr(), dst.data_ptr(), c.n_packets, c.window, call.out.data_ptr(), call.ws,
                              call.wsb, call.stream)
    assert rc == NSG_OK
    assert call.result().tolist() == oracle.window_stats_sort(keys=keys, window=c.window).tolist()


def test_entry_points_reject_bad_arguments_before_launch(cuda_device):
    lib = _lib("libnsg.so")
    call = Call(lib, 1000, 100, cuda_device)
    kd = torch.zeros(1000, dtype=torch.int64, device=cuda_device)
    assert lib.nsg_window_stats_packed(None, 1000, 100, call.out.data_ptr(), call.ws, call.wsb, call.stream) == 1
    assert lib.nsg_window_stats_packed(kd.data_ptr(), 1000, 0, call.out.data_ptr(), call.ws, call.wsb, call.stream) == 1
    assert lib.nsg_window_stats_packed(kd.data_ptr(), 1000, 100, call.out.data_ptr(), call.ws, 16, call.stream) == 3
    assert lib.nsg_window_stats_packed(kd.data_ptr(), 1000, 100, call.out.data_ptr(), call.ws + 8, call.wsb,
                                       call.stream) == 1


def test_debug_build_reads_the_self_check_back(cuda_device):
    c = CONFIGS["C2"]
    n = 4 * c.window + 77
    keys = gen.generate_host(c.dist, c.seed, 0, n, packed=True)
    want = oracle.window_stats_sort(keys=keys, window=c.window).tolist()
    kd = torch.from_numpy(keys.view(np.int64)).to(cuda_device)
    for name, expect_rc in (("libnsg_debug.so", NSG_ERR_INTERNAL), ("libnsg.so", NSG_OK)):
        lib = _lib(name)
        call = Call(lib, n, c.window, cuda_device)
        # a normal call: OK in both builds, no self-check failure
        assert lib.nsg_window_stats_packed(kd.data_ptr(), n, c.window, call.out.data_ptr(), call.ws, call.wsb,
                                           call.stream) == NSG_OK
        assert call.result().tolist() == want and call.diag()[1] == 0
        # an injected self-check failure (window 0): the debug build returns NSG_ERR_INTERNAL, the product
        # build returns at once (asynchronous) and the failure is in the diagnostics
        rc = lib.nsg_window_stats_ex(None, None, kd.data_ptr(), n, c.window, call.out.data_ptr(), call.ws, call.wsb,
                                     call.stream, NSG_FLAG_INJECT_SELF_CHECK)
        assert rc == expect_rc, name
        assert call.diag()[1] == 1, name
        assert call.result().tolist() == want
