"""gen — seeded, counter-based synthetic packet generator shared by tests and bench.

Inputs only: this module holds none of the method's arithmetic (no group-by, no counting).  The
generator is defined once in gen/nsggen.cu (host and device instantiations of the same integer
code, recipe in its header and DESIGN.md "Input recipe"); ``generate_numpy`` is an independent
numpy restatement used only to cross-check it.

Distributions: ``uniform`` (independent 32-bit src/dst), ``zipf`` (Zipf(s) ranks over K addresses
per side, mapped through a bijective mixer), ``heavy`` (Bernoulli(1/2) hot source 10.0.0.1, else
uniform).  Packet i depends only on (dist, seed, i).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nsggen.cu")
_HDR = os.path.join(_HERE, "nsggen.h")
_LIB = os.path.join(_HERE, "libnsggen.so")
_lock = threading.Lock()
_lib = None
_tables: dict = {}

DISTS = {"uniform": 0, "zipf": 1, "heavy": 2}
NVCC_ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def build(force: bool = False) -> str:
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["nvcc", *NVCC_ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            lib.nsg_gen_zipf_table.restype = ctypes.c_int
            lib.nsg_gen_zipf_table.argtypes = [ctypes.c_double, ctypes.c_uint32, ctypes.c_void_p]
            lib.nsg_gen_host.restype = ctypes.c_int
            lib.nsg_gen_host.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_int]
            lib.nsg_gen_device.restype = ctypes.c_int
            lib.nsg_gen_device.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                           ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p]
            _lib = lib
    return _lib


@dataclass(frozen=True)
class Dist:
    """A packet distribution: name in DISTS, plus Zipf exponent s and per-side rank count K."""
    name: str = "uniform"
    zipf_s: float = 1.1
    zipf_k: int = 1 << 20

    @property
    def code(self) -> int:
        return DISTS[self.name]


def zipf_table(s: float, K: int) -> np.ndarray:
    """Zipf CDF table T[K] (u64), built once on the host in long double (nsggen.cu)."""
    key = (float(s), int(K))
    if key not in _tables:
        T = np.zeros(int(K), dtype=np.uint64)
        rc = _load().nsg_gen_zipf_table(float(s), int(K), T.ctypes.data)
        if rc:
            raise ValueError("bad zipf parameters")
        _tables[key] = T
    return _tables[key]


def _table_for(dist: Dist):
    if dist.name == "zipf":
        T = zipf_table(dist.zipf_s, dist.zipf_k)
        return T, T.ctypes.data, int(dist.zipf_k)
    return None, None, 0


def generate_host(dist: Dist, seed: int, first: int, count: int, *, packed: bool = False, threads: int = 0):
    """Packets [first, first+count) on the host: (src, dst) uint32 arrays, or uint64 keys if packed."""
    T, tp, K = _table_for(dist)
    lib = _load()
    if packed:
        keys = np.empty(count, dtype=np.uint64)
        rc = lib.nsg_gen_host(dist.code, seed, first, count, tp, K, None, None, keys.ctypes.data, threads)
        if rc:
            raise RuntimeError(f"nsg_gen_host failed ({rc})")
        return keys
    src = np.empty(count, dtype=np.uint32)
    dst = np.empty(count, dtype=np.uint32)
    rc = lib.nsg_gen_host(dist.code, seed, first, count, tp, K, src.ctypes.data, dst.ctypes.data, None, threads)
    if rc:
        raise RuntimeError(f"nsg_gen_host failed ({rc})")
    return src, dst


def generate_device(dist: Dist, seed: int, first: int, count: int, *, keys=None, src=None, dst=None, stream=None):
    """Fill torch CUDA tensors (keys: int64/uint64 [count]; src/dst: int32/uint32 [count]) on device."""
    import torch

    T, _, K = _table_for(dist)
    tdev = None
    if T is not None:
        dev = (keys if keys is not None else src).device
        cache_key = ("dev", dist.zipf_s, dist.zipf_k, str(dev))
        tdev = _tables.get(cache_key)
        if tdev is None:
            tdev = torch.from_numpy(T.view(np.int64)).to(dev)
            _tables[cache_key] = tdev
    s = stream if stream is not None else torch.cuda.current_stream()
    rc = _load().nsg_gen_device(dist.code, seed, first, count, None if tdev is None else tdev.data_ptr(), K,
                                None if src is None else src.data_ptr(), None if dst is None else dst.data_ptr(),
                                None if keys is None else keys.data_ptr(), ctypes.c_void_p(s.cuda_stream))
    if rc:
        raise RuntimeError(f"nsg_gen_device failed ({rc})")


# ---- independent numpy restatement (cross-check of the generator only) --------------------
_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30)); z = z * np.uint64(0xBF58476D1CE4E5B9)
    z = z ^ (z >> np.uint64(27)); z = z * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _lowbias32(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint32)
    x ^= x >> np.uint32(16); x *= np.uint32(0x7FEB352D)
    x ^= x >> np.uint32(15); x *= np.uint32(0x846CA68B)
    x ^= x >> np.uint32(16)
    return x


def generate_numpy(dist: Dist, seed: int, first: int, count: int):
    """Same packets as generate_host, computed with numpy (wrapping uint64 arithmetic)."""
    with np.errstate(over="ignore"):
        i = np.arange(first, first + count, dtype=np.uint64)
        g = np.uint64(0x9E3779B97F4A7C15)
        sd = np.uint64(seed)
        if dist.name == "uniform":
            k = _mix64(sd + (i + np.uint64(1)) * g)
            return (k >> np.uint64(32)).astype(np.uint32), (k & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        x = _mix64(sd + (np.uint64(2) * i + np.uint64(1)) * g)
        y = _mix64(sd + (np.uint64(2) * i + np.uint64(2)) * g)
        if dist.name == "zipf":
            T = zipf_table(dist.zipf_s, dist.zipf_k)
            rs = np.searchsorted(T, x, side="left").astype(np.uint32)
            rd = np.searchsorted(T, y, side="left").astype(np.uint32)
            return _lowbias32(rs ^ np.uint32(0x0A000000)), _lowbias32(rd ^ np.uint32(0xC0A80000))
        hot = (x >> np.uint64(63)).astype(bool)
        src = np.where(hot, np.uint32(0x0A000001), (x & np.uint64(0xFFFFFFFF)).astype(np.uint32)).astype(np.uint32)
        return src, (y & np.uint64(0xFFFFFFFF)).astype(np.uint32)


def pack(src: np.ndarray, dst: np.ndarray) -> np.ndarray:
    return (src.astype(np.uint64) << np.uint64(32)) | dst.astype(np.uint64)
