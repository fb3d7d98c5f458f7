"""oracle — TEST INFRASTRUCTURE ONLY: the plain CPU oracle of the nine per-window quantities.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  It shares no code with the CUDA path
(``paper_2509_03653_b200``) and the CUDA path never imports it.

Three procedures, each citing PAPER.md (= /root/reference/PAPER.md, arXiv 2509.03653) Table 2
(lines 171-193; destination mirrors by the caption, line 173):

* ``window_stats_map``  — O1, the literal definition over ``std::map`` (oracle.cpp).
* ``window_stats_sort`` — O2, the same definition via ``std::sort`` + run-length scans,
  thread-parallel over windows (oracle.cpp).
* ``window_distributions`` — O1d, the vector-valued rows of Table 2 (link packets :182, packets
  from source :185, source fan-out :187, their destination mirrors :173) and the four globally
  unique IP set counts (:209) per window, from the same ``std::map`` definition (oracle.cpp);
  ``window_distributions_dense`` is its dense O0 counterpart (dense.py).
* ``window_stats_weighted`` — O1w, O1 on weighted rows (src, dst, n_packets): the paper's three-column
  frame (:207; valid packets = sum of n_packets, :180); rows of weight 0 add nothing.
* ``anonymize`` — the IP anonymisation of PAPER.md:195-203 (unique, keyed permutation, gather; anon.py).
* ``window_stats_dense`` — O0, the "Matrix notation" column evaluated literally on a dense
  matrix after relabelling the (few) addresses of a tiny window (dense.py).

Output rows are in north_star order: valid packets, unique links, max link packets, unique
sources, max source packets, max source fan-out, unique destinations, max destination packets,
max destination fan-in.  Pinned by tests/test_oracle_*.py (worked examples, closed forms,
brute force, invariants, an independent pandas/scipy route); no function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

from .anon import anonymize  # noqa: F401
from .dense import window_distributions_dense, window_stats_dense  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

NUM_STATS = 9


def build(force: bool = False) -> str:
    """Compile oracle.cpp -> liboracle.so with g++ (plain -O2, no tuning)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-Wall", "-o", tmp, _SRC, "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            for name in ("nsg_oracle_window_stats_map", "nsg_oracle_window_stats_sort"):
                f = getattr(lib, name)
                f.restype = ctypes.c_int
                f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                              ctypes.c_void_p, ctypes.c_int]
            f = lib.nsg_oracle_window_stats_weighted
            f.restype = ctypes.c_int
            f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                          ctypes.c_void_p, ctypes.c_int]
            f = lib.nsg_oracle_window_distributions
            f.restype = ctypes.c_int
            f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64] + \
                [ctypes.c_void_p] * 10 + [ctypes.c_int]
            lib.nsg_oracle_hardware_threads.restype = ctypes.c_uint
            _lib = lib
    return _lib


def hardware_threads() -> int:
    return int(_load().nsg_oracle_hardware_threads())


def _u32(a) -> np.ndarray:
    a = np.ascontiguousarray(a)
    if a.dtype in (np.int32, np.uint32):
        return a.view(np.uint32)
    a64 = a.astype(np.int64)
    if a64.size and (a64.min() < 0 or a64.max() > 0xFFFFFFFF):
        raise ValueError("addresses must be 32-bit unsigned")
    return a64.astype(np.uint32)


def _split(src, dst, keys):
    if keys is not None:
        k = np.ascontiguousarray(keys).view(np.uint64)
        return (k >> np.uint64(32)).astype(np.uint32), (k & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    return _u32(src), _u32(dst)


def _run(fname, src, dst, keys, window, threads):
    s, d = _split(src, dst, keys)
    if s.shape != d.shape:
        raise ValueError("src and dst must have the same length")
    n = int(s.shape[0])
    if window < 1:
        raise ValueError("window must be >= 1")
    nw = 0 if n == 0 else (n + window - 1) // window
    out = np.zeros((nw, NUM_STATS), dtype=np.uint64)
    if n:
        rc = getattr(_load(), fname)(s.ctypes.data, d.ctypes.data, n, int(window), out.ctypes.data, int(threads))
        if rc != 0:
            raise ValueError(f"{fname} returned {rc}")
    if nw and int(out[:, 0].max()) == 0xFFFFFFFFFFFFFFFF:
        raise RuntimeError("oracle self-check failed")
    return out


def window_stats_map(src=None, dst=None, window: int = 1 << 17, *, keys=None, threads: int = 0) -> np.ndarray:
    """O1: literal std::map definition.  Returns uint64 [n_windows, 9]."""
    return _run("nsg_oracle_window_stats_map", src, dst, keys, window, threads)


def window_stats_sort(src=None, dst=None, window: int = 1 << 17, *, keys=None, threads: int = 0) -> np.ndarray:
    """O2: std::sort + run-length scans, a thread per window group.  Returns uint64 [n_windows, 9]."""
    return _run("nsg_oracle_window_stats_sort", src, dst, keys, window, threads)


IP_SETS = ("union", "src_only", "dst_only", "both")


def window_distributions(src=None, dst=None, window: int = 1 << 17, *, keys=None, weights=None,
                         threads: int = 0) -> dict:
    """O1d: per window, the nonzeros of A_t and the row/column sums and nnz, each in ascending key
    order, plus the four IP set counts.

    Returns a dict of numpy arrays:
      link_key u64[n], link_packets u64[n]         window w's links at [w*window, w*window + counts[w,0])
      src_node u32[n], src_packets u64[n], src_fan u64[n]     (counts[w,1] entries per window)
      dst_node u32[n], dst_packets u64[n], dst_fan u64[n]     (counts[w,2] entries per window)
      counts u64[nw, 3] = (links, sources, destinations); ip_sets u64[nw, 4] = IP_SETS order.
    `weights`: optional u32 [n] n_packets per row (weighted rows as O1w; weight 0 adds nothing).
    """
    s, d = _split(src, dst, keys)
    if s.shape != d.shape:
        raise ValueError("src and dst must have the same length")
    w8 = None if weights is None else _u32(weights)
    if w8 is not None and w8.shape != s.shape:
        raise ValueError("weights must have one entry per row")
    n = int(s.shape[0])
    if window < 1:
        raise ValueError("window must be >= 1")
    nw = 0 if n == 0 else (n + window - 1) // window
    r = {
        "link_key": np.zeros(n, np.uint64), "link_packets": np.zeros(n, np.uint64),
        "src_node": np.zeros(n, np.uint32), "src_packets": np.zeros(n, np.uint64), "src_fan": np.zeros(n, np.uint64),
        "dst_node": np.zeros(n, np.uint32), "dst_packets": np.zeros(n, np.uint64), "dst_fan": np.zeros(n, np.uint64),
        "counts": np.zeros((nw, 3), np.uint64), "ip_sets": np.zeros((nw, 4), np.uint64),
    }
    if n:
        order = ("link_key", "link_packets", "src_node", "src_packets", "src_fan", "dst_node", "dst_packets",
                 "dst_fan", "counts", "ip_sets")
        rc = _load().nsg_oracle_window_distributions(s.ctypes.data, d.ctypes.data,
                                                     None if w8 is None else w8.ctypes.data, n, int(window),
                                                     *[r[k].ctypes.data for k in order], int(threads))
        if rc != 0:
            raise ValueError(f"nsg_oracle_window_distributions returned {rc}")
    return r


def window_slices(r: dict, window: int, w: int) -> dict:
    """The entries of window w of a distributions dict (as returned by window_distributions)."""
    b = w * window
    nl, ns, nd = (int(x) for x in r["counts"][w])
    out = {"link_key": r["link_key"][b:b + nl], "link_packets": r["link_packets"][b:b + nl]}
    for k in ("src_node", "src_packets", "src_fan"):
        out[k] = r[k][b:b + ns]
    for k in ("dst_node", "dst_packets", "dst_fan"):
        out[k] = r[k][b:b + nd]
    out["ip_sets"] = r["ip_sets"][w]
    return out


def window_stats_weighted(src=None, dst=None, weights=None, window: int = 1 << 17, *, keys=None,
                          threads: int = 0) -> np.ndarray:
    """O1w: Table 2 on weighted rows, A_t(i,j) = sum of the weights of the window's rows i -> j.
    `weights` u32 [n].  Returns uint64 [n_windows, 9]."""
    s, d = _split(src, dst, keys)
    w8 = _u32(weights)
    if s.shape != d.shape or w8.shape != s.shape:
        raise ValueError("src, dst and weights must have the same length")
    n = int(s.shape[0])
    if window < 1:
        raise ValueError("window must be >= 1")
    nw = 0 if n == 0 else (n + window - 1) // window
    out = np.zeros((nw, NUM_STATS), dtype=np.uint64)
    if n:
        rc = _load().nsg_oracle_window_stats_weighted(s.ctypes.data, d.ctypes.data, w8.ctypes.data, n, int(window),
                                                      out.ctypes.data, int(threads))
        if rc != 0:
            raise ValueError(f"nsg_oracle_window_stats_weighted returned {rc}")
    return out
