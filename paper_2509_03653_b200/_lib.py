"""ctypes loader for libnsg.so (the C ABI declared in include/nsg.h).

The library is built in-tree by ``__graft_entry__.build()`` (``build_libnsg`` below).  There is no
fallback of any kind: if libnsg.so is missing or cannot be loaded, importing the binding raises.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

_PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(_PKG)
LIB_PATH = os.path.join(_PKG, "libnsg.so")
DEBUG_LIB_PATH = os.path.join(_PKG, "libnsg_debug.so")  # -DNSG_DEBUG_CHECKS: self-check read back (tests)
SOURCES = [os.path.join(_PKG, "csrc", f) for f in ("nsg.cu", "nsg_common.cuh", "nsg_fast.cuh", "nsg_global.cuh",
                                                   "nsg_trace.cuh", "nsg_anon.cuh", "nsg_flat.cuh")]
HEADER = os.path.join(ROOT, "include", "nsg.h")
INTERNAL_HEADER = os.path.join(ROOT, "include", "nsg_internal.h")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]

# Every symbol include/nsg.h and include/nsg_internal.h declare (checked by tests/test_abi.py).
EXPORTS = (
    "nsg_num_windows",
    "nsg_workspace_bytes",
    "nsg_window_stats",
    "nsg_window_stats_packed",
    "nsg_window_stats_ex",
    "nsg_window_stats_timed",
    "nsg_window_stats_from_host",
    "nsg_window_vectors",
    "nsg_window_vectors_weighted",
    "nsg_window_stats_weighted",
    "nsg_window_stats_mirrored",
    "nsg_trace_workspace_bytes",
    "nsg_trace_partition",
    "nsg_trace_links",
    "nsg_trace_nodes",
    "nsg_trace_stats_workspace_bytes",
    "nsg_trace_stats",
    "nsg_trace_stats_weighted",
    "nsg_ipc_handle_bytes",
    "nsg_ipc_alloc",
    "nsg_ipc_open",
    "nsg_ipc_close",
    "nsg_ipc_free",
    "nsg_trace_owner_counts",
    "nsg_trace_partition_peers",
    "nsg_trace_links_count",
    "nsg_trace_links_emit_peers",
    "nsg_anonymize_workspace_bytes",
    "nsg_anonymize",
    "nsg_diag_offset",
    "nsg_debug_trace_cas_first_slots",
    "nsg_last_launches",
    "nsg_status_string",
    "nsg_version",
)

STATUS = {
    0: "NSG_OK",
    1: "NSG_ERR_INVALID_ARGUMENT",
    2: "NSG_ERR_CUDA",
    3: "NSG_ERR_WORKSPACE_TOO_SMALL",
    4: "NSG_ERR_UNSUPPORTED_DEVICE",
    5: "NSG_ERR_INTERNAL",
}


def build_id() -> str:
    """Content hash of what libnsg.so is built from (sources, headers, nvcc flags): names the build that a
    committed measurement (e.g. profiles/ncu_traffic.json) belongs to."""
    import hashlib

    h = hashlib.sha256(" ".join(NVCC_FLAGS).encode())
    for p in SOURCES + [HEADER, INTERNAL_HEADER]:
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def build_libnsg(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    """nvcc -gencode arch=compute_100a,code=sm_100a ... -> paper_2509_03653_b200/libnsg.so
    (debug=True: libnsg_debug.so, the same sources with -DNSG_DEBUG_CHECKS)."""
    path = DEBUG_LIB_PATH if debug else LIB_PATH
    newest = max(os.path.getmtime(p) for p in SOURCES + [HEADER, INTERNAL_HEADER])
    if force or not os.path.exists(path) or os.path.getmtime(path) < newest:
        tmp = path + f".tmp{os.getpid()}"
        cmd = ["nvcc", *NVCC_FLAGS, *(["-DNSG_DEBUG_CHECKS"] if debug else []), "-I", os.path.join(ROOT, "include"),
               "-o", tmp, SOURCES[0]]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
        os.replace(tmp, path)
    return path


class NsgVectors(ctypes.Structure):
    """struct nsg_vectors (include/nsg.h): device pointers, NULL = not requested."""
    _fields_ = [(name, ctypes.c_void_p) for name in (
        "link_key", "link_packets", "src_node", "src_packets", "src_fanout", "dst_node", "dst_packets", "dst_fanin",
        "ip_sets")]


class NsgError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        super().__init__(f"{what}: {STATUS.get(status, status)}")
        self.status = status


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libnsg (the product library; tests may pass DEBUG_LIB_PATH)."""
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    u64, sz, vp, u32 = ctypes.c_uint64, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_uint32
    lib.nsg_num_windows.restype = u64
    lib.nsg_num_windows.argtypes = [u64, u64]
    lib.nsg_workspace_bytes.restype = sz
    lib.nsg_workspace_bytes.argtypes = [u64, u64]
    lib.nsg_window_stats.restype = ctypes.c_int
    lib.nsg_window_stats.argtypes = [vp, vp, u64, u64, vp, vp, sz, vp]
    lib.nsg_window_stats_packed.restype = ctypes.c_int
    lib.nsg_window_stats_packed.argtypes = [vp, u64, u64, vp, vp, sz, vp]
    lib.nsg_window_stats_ex.restype = ctypes.c_int
    lib.nsg_window_stats_ex.argtypes = [vp, vp, vp, u64, u64, vp, vp, sz, vp, u32]
    lib.nsg_window_stats_timed.restype = ctypes.c_int
    lib.nsg_window_stats_timed.argtypes = [vp, vp, vp, u64, u64, vp, vp, sz, vp, u32, vp, vp]
    lib.nsg_window_stats_from_host.restype = ctypes.c_int
    lib.nsg_window_stats_from_host.argtypes = [vp, u64, u64, vp, vp, vp, vp, sz, vp, vp, u32]
    lib.nsg_window_vectors.restype = ctypes.c_int
    lib.nsg_window_vectors.argtypes = [vp, vp, vp, u64, u64, vp, ctypes.POINTER(NsgVectors), vp, sz, vp, u32]
    lib.nsg_window_vectors_weighted.restype = ctypes.c_int
    lib.nsg_window_vectors_weighted.argtypes = [vp, vp, vp, vp, u64, u64, vp, ctypes.POINTER(NsgVectors), vp, sz, vp, u32]
    lib.nsg_window_stats_weighted.restype = ctypes.c_int
    lib.nsg_window_stats_weighted.argtypes = [vp, vp, vp, vp, u64, u64, vp, vp, sz, vp, u32]
    lib.nsg_trace_workspace_bytes.restype = sz
    lib.nsg_trace_workspace_bytes.argtypes = [u64, u64, u32]
    lib.nsg_trace_partition.restype = ctypes.c_int
    lib.nsg_trace_partition.argtypes = [vp, vp, vp, u64, u32, vp, vp, vp, sz, u64, u64, vp]
    lib.nsg_trace_links.restype = ctypes.c_int
    lib.nsg_trace_links.argtypes = [vp, vp, vp, u64, u32, vp, vp, vp, vp, vp, sz, u64, u64, vp]
    lib.nsg_trace_nodes.restype = ctypes.c_int
    lib.nsg_trace_nodes.argtypes = [vp, u64, vp, vp, sz, u64, u64, vp]
    lib.nsg_trace_stats_workspace_bytes.restype = sz
    lib.nsg_trace_stats_workspace_bytes.argtypes = [u64]
    lib.nsg_trace_stats_weighted.restype = ctypes.c_int
    lib.nsg_trace_stats_weighted.argtypes = [vp, vp, vp, vp, u64, vp, vp, sz, vp]
    lib.nsg_trace_stats.restype = ctypes.c_int
    lib.nsg_trace_stats.argtypes = [vp, vp, vp, u64, vp, vp, sz, vp]
    lib.nsg_anonymize_workspace_bytes.restype = sz
    lib.nsg_anonymize_workspace_bytes.argtypes = []
    lib.nsg_anonymize.restype = ctypes.c_int
    lib.nsg_anonymize.argtypes = [vp, vp, vp, u64, u64, u32, vp, vp, vp, vp, sz, vp]
    lib.nsg_debug_trace_cas_first_slots.restype = ctypes.c_int
    lib.nsg_debug_trace_cas_first_slots.argtypes = [u64]
    lib.nsg_ipc_handle_bytes.restype = sz
    lib.nsg_ipc_handle_bytes.argtypes = []
    lib.nsg_ipc_alloc.restype = ctypes.c_int
    lib.nsg_ipc_alloc.argtypes = [sz, ctypes.POINTER(vp), vp]
    lib.nsg_ipc_open.restype = ctypes.c_int
    lib.nsg_ipc_open.argtypes = [vp, ctypes.POINTER(vp)]
    lib.nsg_ipc_close.restype = ctypes.c_int
    lib.nsg_ipc_close.argtypes = [vp]
    lib.nsg_ipc_free.restype = ctypes.c_int
    lib.nsg_ipc_free.argtypes = [vp]
    lib.nsg_trace_owner_counts.restype = ctypes.c_int
    lib.nsg_trace_owner_counts.argtypes = [vp, vp, vp, u64, u32, vp, vp, sz, u64, u64, vp]
    lib.nsg_trace_partition_peers.restype = ctypes.c_int
    lib.nsg_trace_partition_peers.argtypes = [vp, vp, vp, u64, u32, vp, vp, vp, sz, u64, u64, vp]
    lib.nsg_trace_links_count.restype = ctypes.c_int
    lib.nsg_trace_links_count.argtypes = [vp, vp, vp, u64, u32, vp, vp, vp, sz, u64, u64, vp]
    lib.nsg_trace_links_emit_peers.restype = ctypes.c_int
    lib.nsg_trace_links_emit_peers.argtypes = [u32, vp, vp, vp, vp, vp, sz, u64, u64, vp]
    lib.nsg_window_stats_mirrored.restype = ctypes.c_int
    lib.nsg_window_stats_mirrored.argtypes = [vp, vp, vp, u64, u64, vp, vp, sz, vp, u32, vp, u32, u64]
    lib.nsg_diag_offset.restype = sz
    lib.nsg_diag_offset.argtypes = []
    lib.nsg_last_launches.restype = ctypes.c_uint
    lib.nsg_last_launches.argtypes = []
    lib.nsg_status_string.restype = ctypes.c_char_p
    lib.nsg_status_string.argtypes = [ctypes.c_int]
    lib.nsg_version.restype = ctypes.c_char_p
    lib.nsg_version.argtypes = []
    return lib
