"""Python binding of libnsg (include/nsg.h): argument marshalling only.

Every step of the per-window computation runs in libnsg's sm_100a kernels; this module only checks
tensors, hands raw device pointers and the current CUDA stream to the C ABI, and manages the
caller-owned workspace.  PyTorch supplies device memory and streams.

The nine output columns (north_star order; Table 2 lines 180-188 and the destination
mirrors of line 173):
"""
from __future__ import annotations

import ctypes
from typing import Optional

import torch

from ._lib import NsgError, NsgVectors, load

_lib = load()  # raises ImportError if libnsg.so is missing: there is no fallback

NUM_STATS = 9
STAT_NAMES = (
    "valid_packets",
    "unique_links",
    "max_link_packets",
    "unique_sources",
    "max_source_packets",
    "max_source_fanout",
    "unique_destinations",
    "max_destination_packets",
    "max_destination_fanin",
)
DEFAULT_WINDOW = 1 << 17
MAX_WINDOW = 1 << 31

# include/nsg.h fault-injection flags (tests of the L2-path hand-off)
FLAG_FORCE_GLOBAL = 1
FLAG_INJECT_OVERFLOW = 2
# include/nsg_internal.h: measurement / development switches, not part of the product interface
_FLAG_NO_FALLBACK_CHECK = 4
_FLAG_LEGACY_FAST = 16
_FLAG_INJECT_SELF_CHECK = 32

_U32_TYPES = (torch.int32, torch.uint32)
_U64_TYPES = (torch.int64, torch.uint64)


def num_windows(n_packets: int, window: int = DEFAULT_WINDOW) -> int:
    return int(_lib.nsg_num_windows(int(n_packets), int(window)))


def workspace_bytes(n_packets: int, window: int = DEFAULT_WINDOW) -> int:
    return int(_lib.nsg_workspace_bytes(int(n_packets), int(window)))


def version() -> str:
    return _lib.nsg_version().decode()


def last_launches() -> int:
    """Kernels launched by this thread's most recent window_stats* call."""
    return int(_lib.nsg_last_launches())


class Workspace:
    """Caller-owned device scratch for one (n_packets, window) shape, reusable across calls."""

    def __init__(self, n_packets: int, window: int = DEFAULT_WINDOW, device=None):
        self.n_packets, self.window = int(n_packets), int(window)
        self.nbytes = workspace_bytes(self.n_packets, self.window)
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        # + 256 so the pointer can be aligned to 256 B
        self.buffer = torch.empty(max(self.nbytes, 1) + 256, dtype=torch.uint8, device=dev)
        base = self.buffer.data_ptr()
        self.offset = (-base) % 256
        self.ptr = base + self.offset

    def fits(self, n_packets: int, window: int) -> bool:
        return workspace_bytes(n_packets, window) <= self.nbytes

    def diag(self) -> list:
        """u32[4] diagnostics of the last call (synchronises the buffer's device)."""
        off = self.offset + int(_lib.nsg_diag_offset())
        return [int(x) for x in self.buffer[off:off + 16].view(torch.int32).cpu().tolist()]


_ws_cache: dict = {}


def _workspace(n: int, window: int, device: torch.device, workspace: Optional[Workspace], stream=None) -> Workspace:
    """The caller's workspace, or an implicit one cached per (device, shape, stream): two calls on
    different streams never share scratch, and an evicted entry is dropped only after its stream has
    drained."""
    if workspace is not None:
        if not workspace.fits(n, window):
            raise NsgError(3, "workspace too small")
        return workspace
    s = stream if stream is not None else torch.cuda.current_stream(device)
    key = (device.index, n, window, s.cuda_stream)
    hit = _ws_cache.get(key)
    if hit is None:
        if len(_ws_cache) >= 8:
            for ws_old, s_old in _ws_cache.values():
                s_old.synchronize()
            _ws_cache.clear()
        hit = _ws_cache[key] = (Workspace(n, window, device), s)
    return hit[0]


def _check(t: torch.Tensor, name: str, dtypes) -> None:
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if t.dtype not in dtypes:
        raise TypeError(f"{name} has dtype {t.dtype}; expected one of {dtypes}")
    if t.dim() != 1 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous 1-D tensor")


def _keep(stream, *tensors) -> None:
    """The tensors are used by work enqueued on `stream`: the caching allocator must not hand their memory
    to another stream before that work completes (they may be temporaries of this call, or be freed by the
    caller while `stream` still runs)."""
    for t in tensors:
        if t is not None and t.is_cuda:
            t.record_stream(stream)


def _launch(src, dst, keys, n, window, out, workspace, stream, flags, device, events=None):
    window = int(window)
    if window < 1 or window > MAX_WINDOW:
        raise ValueError(f"window must be in [1, 2^31], got {window}")
    nw = num_windows(n, window)
    if out is None:
        out = torch.empty((nw, NUM_STATS), dtype=torch.int64, device=device)
    else:
        if out.dtype not in _U64_TYPES or not out.is_contiguous() or out.numel() < nw * NUM_STATS or not out.is_cuda:
            raise ValueError("out must be a contiguous CUDA int64/uint64 tensor with >= n_windows*9 elements")
    if n == 0:
        return out
    s = stream if stream is not None else torch.cuda.current_stream(device)
    ws = _workspace(n, window, device, workspace, s)
    _keep(s, out, ws.buffer, src, dst, keys)
    u64p = lambda t: None if t is None else t.data_ptr()  # noqa: E731
    if events is not None:  # measurement: nsg_window_stats_timed (include/nsg_internal.h)
        for e in events:
            if not e.cuda_event:  # torch creates the cudaEvent_t lazily, on first record
                e.record(s)
        ev0, ev1 = (ctypes.c_void_p(e.cuda_event) for e in events)
        rc, name = _lib.nsg_window_stats_timed(u64p(src), u64p(dst), u64p(keys), n, window, out.data_ptr(), ws.ptr,
                                               ws.nbytes, ctypes.c_void_p(s.cuda_stream), int(flags), ev0,
                                               ev1), "nsg_window_stats_timed"
    elif flags:
        rc, name = _lib.nsg_window_stats_ex(u64p(src), u64p(dst), u64p(keys), n, window, out.data_ptr(), ws.ptr,
                                            ws.nbytes, ctypes.c_void_p(s.cuda_stream), int(flags)), "nsg_window_stats_ex"
    elif keys is not None:
        rc, name = _lib.nsg_window_stats_packed(keys.data_ptr(), n, window, out.data_ptr(), ws.ptr, ws.nbytes,
                                                ctypes.c_void_p(s.cuda_stream)), "nsg_window_stats_packed"
    else:
        rc, name = _lib.nsg_window_stats(src.data_ptr(), dst.data_ptr(), n, window, out.data_ptr(), ws.ptr,
                                         ws.nbytes, ctypes.c_void_p(s.cuda_stream)), "nsg_window_stats"
    if rc != 0:
        raise NsgError(rc, name)
    return out


def window_stats(src: torch.Tensor, dst: torch.Tensor, window: int = DEFAULT_WINDOW, *, out=None,
                 workspace: Optional[Workspace] = None, stream=None, flags: int = 0) -> torch.Tensor:
    """Nine quantities per window of the SoA packet stream (src[i], dst[i]) (device int32/uint32).

    Returns a device int64 tensor [n_windows, 9], valid when `stream` (default: current) completes.
    """
    _check(src, "src", _U32_TYPES)
    _check(dst, "dst", _U32_TYPES)
    if src.numel() != dst.numel() or src.device != dst.device:
        raise ValueError("src and dst must have the same length and device")
    return _launch(src, dst, None, src.numel(), window, out, workspace, stream, flags, src.device)


def window_stats_packed(keys: torch.Tensor, window: int = DEFAULT_WINDOW, *, out=None,
                        workspace: Optional[Workspace] = None, stream=None, flags: int = 0,
                        kernel_events=None) -> torch.Tensor:
    """Nine quantities per window of packed keys[i] = src<<32 | dst (device int64/uint64).

    kernel_events: optional (start, end) torch.cuda.Event pair (created with enable_timing=True),
    recorded on the stream right around the main kernel (for measurement).
    """
    _check(keys, "keys", _U64_TYPES)
    return _launch(None, None, keys, keys.numel(), window, out, workspace, stream, flags, keys.device,
                   events=kernel_events)


_copy_streams = {}


def _copy_stream(device: torch.device):
    cs = _copy_streams.get(device.index)
    if cs is None:
        cs = _copy_streams[device.index] = torch.cuda.Stream(device)
    return cs


def window_stats_from_host(keys_host: torch.Tensor, window: int = DEFAULT_WINDOW, *, device=None,
                           keys_dev: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                           out_host: Optional[torch.Tensor] = None, workspace: Optional[Workspace] = None,
                           stream=None, copy_stream=None, chunk_windows: int = 8,
                           synchronize: bool = True) -> torch.Tensor:
    """End-to-end call on HOST packed keys (nsg_window_stats_from_host): chunked H2D copies on a copy
    stream overlapped with the device computation, then the D2H copy of the result.

    `keys_host` must be a pinned 1-D int64/uint64 CPU tensor.  Returns the pinned CPU int64
    [n_windows, 9] result (complete on return when `synchronize`, else once `stream` reaches it).
    """
    if (not isinstance(keys_host, torch.Tensor) or keys_host.is_cuda or keys_host.dtype not in _U64_TYPES
            or keys_host.dim() != 1 or not keys_host.is_contiguous()):
        raise ValueError("keys_host must be a contiguous 1-D host int64/uint64 tensor")
    if keys_host.numel() and not keys_host.is_pinned():
        raise ValueError("keys_host must be pinned (torch.Tensor.pin_memory())")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    window = int(window)
    if window < 1 or window > MAX_WINDOW:
        raise ValueError(f"window must be in [1, 2^31], got {window}")
    n = keys_host.numel()
    nw = num_windows(n, window)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    cs = copy_stream if copy_stream is not None else _copy_stream(dev)
    if keys_dev is None:
        keys_dev = torch.empty(n, dtype=keys_host.dtype, device=dev)
    elif not keys_dev.is_cuda or keys_dev.dtype not in _U64_TYPES or keys_dev.numel() < n or not keys_dev.is_contiguous():
        raise ValueError("keys_dev must be a contiguous CUDA int64/uint64 tensor with >= n elements")
    if out is None:
        out = torch.empty((nw, NUM_STATS), dtype=torch.int64, device=dev)
    elif out.dtype not in _U64_TYPES or not out.is_contiguous() or out.numel() < nw * NUM_STATS or not out.is_cuda:
        raise ValueError("out must be a contiguous CUDA int64/uint64 tensor with >= n_windows*9 elements")
    if out_host is None:
        out_host = torch.empty((nw, NUM_STATS), dtype=torch.int64, pin_memory=True)
    elif out_host.is_cuda or not out_host.is_pinned() or out_host.numel() < nw * NUM_STATS or not out_host.is_contiguous():
        raise ValueError("out_host must be a pinned contiguous CPU tensor with >= n_windows*9 elements")
    if n:
        ws = _workspace(n, window, dev, workspace, s)
        _keep(s, ws.buffer, keys_dev, out)
        _keep(cs, keys_dev)  # written by the copy stream
        rc = _lib.nsg_window_stats_from_host(
            keys_host.data_ptr(), n, window, keys_dev.data_ptr(), out.data_ptr(), out_host.data_ptr(), ws.ptr,
            ws.nbytes, ctypes.c_void_p(s.cuda_stream), ctypes.c_void_p(cs.cuda_stream), int(chunk_windows))
        if rc != 0:
            raise NsgError(rc, "nsg_window_stats_from_host")
    if synchronize:
        s.synchronize()
    return out_host[:nw] if out_host.dim() == 2 else out_host


IP_SET_NAMES = ("union", "src_only", "dst_only", "both")


def window_vectors(keys: Optional[torch.Tensor] = None, window: int = DEFAULT_WINDOW, *, src=None, dst=None,
                   links: bool = True, sources: bool = True, destinations: bool = True, ip_sets: bool = True,
                   out=None, workspace: Optional[Workspace] = None, stream=None, flags: int = 0,
                   buffers: Optional[dict] = None, n_packets: Optional[torch.Tensor] = None) -> dict:
    """The nine statistics plus the vector outputs of nsg_window_vectors.

    Input: packed `keys` (device int64/uint64) or SoA `src`, `dst` (device int32/uint32).  Returns a dict of
    device tensors (valid once `stream` completes): "stats" int64 [n_windows, 9]; when requested,
    "link_key" int64 [n] with "link_packets" int32 [n], "src_node"/"src_packets"/"src_fanout"
    int32 [n] (:185, :187), "dst_node"/"dst_packets"/"dst_fanin" int32 [n] (:173), "ip_sets" int64
    [n_windows, 4] = (|S u D|, |S \\ D|, |D \\ S|, |S n D|) (:209).  Window w's entries of a vector are at
    [w*window, w*window + count) with count = stats[w, 1] (links), stats[w, 3] (sources) or stats[w, 6]
    (destinations), in unspecified (hash) order; 32-bit values are the u32 bit patterns.
    `buffers`: optional preallocated output tensors (a dict as returned by an earlier call with the same
    n and window), reused instead of allocating.  `n_packets`: optional device int32/uint32 [n] weights of
    the rows (nsg_window_vectors_weighted; weighted rows as window_stats_weighted).
    """
    if keys is not None:
        if src is not None or dst is not None:
            raise ValueError("pass either keys or (src, dst)")
        _check(keys, "keys", _U64_TYPES)
        n, device = keys.numel(), keys.device
    else:
        _check(src, "src", _U32_TYPES)
        _check(dst, "dst", _U32_TYPES)
        if src.numel() != dst.numel() or src.device != dst.device:
            raise ValueError("src and dst must have the same length and device")
        n, device = src.numel(), src.device
    window = int(window)
    if window < 1 or window > MAX_WINDOW:
        raise ValueError(f"window must be in [1, 2^31], got {window}")
    nw = num_windows(n, window)
    if out is None:
        out = torch.empty((nw, NUM_STATS), dtype=torch.int64, device=device)
    elif out.dtype not in _U64_TYPES or not out.is_contiguous() or out.numel() < nw * NUM_STATS or not out.is_cuda:
        raise ValueError("out must be a contiguous CUDA int64/uint64 tensor with >= n_windows*9 elements")
    r = {"stats": out}
    v = NsgVectors()

    def alloc(name, shape, dtype):
        t = None if buffers is None else buffers.get(name)
        if t is None:
            return torch.empty(shape, dtype=dtype, device=device)
        if t.dtype != dtype or tuple(t.shape) != tuple(shape) or not t.is_contiguous() or t.device != device:
            raise ValueError(f"buffers[{name!r}] must be a contiguous {dtype} tensor of shape {shape} on {device}")
        return t

    if links:
        r["link_key"] = alloc("link_key", (n,), torch.int64)
        r["link_packets"] = alloc("link_packets", (n,), torch.int32)
        v.link_key, v.link_packets = r["link_key"].data_ptr(), r["link_packets"].data_ptr()
    if sources:
        for k in ("src_node", "src_packets", "src_fanout"):
            r[k] = alloc(k, (n,), torch.int32)
        v.src_node, v.src_packets, v.src_fanout = (r[k].data_ptr() for k in ("src_node", "src_packets", "src_fanout"))
    if destinations:
        for k in ("dst_node", "dst_packets", "dst_fanin"):
            r[k] = alloc(k, (n,), torch.int32)
        v.dst_node, v.dst_packets, v.dst_fanin = (r[k].data_ptr() for k in ("dst_node", "dst_packets", "dst_fanin"))
    if ip_sets:
        r["ip_sets"] = alloc("ip_sets", (nw, 4), torch.int64)
        v.ip_sets = r["ip_sets"].data_ptr()
    if n == 0:
        return r
    s = stream if stream is not None else torch.cuda.current_stream(device)
    ws = _workspace(n, window, device, workspace, s)
    _keep(s, ws.buffer, src, dst, keys, n_packets, *r.values())
    if n_packets is not None:
        _check(n_packets, "n_packets", _U32_TYPES)
        if n_packets.numel() != n or n_packets.device != device:
            raise ValueError("n_packets must have one entry per row, on the rows' device")
        rc = _lib.nsg_window_vectors_weighted(
            None if src is None else src.data_ptr(), None if dst is None else dst.data_ptr(),
            None if keys is None else keys.data_ptr(), n_packets.data_ptr(), n, window, out.data_ptr(),
            ctypes.byref(v), ws.ptr, ws.nbytes, ctypes.c_void_p(s.cuda_stream), int(flags))
        if rc != 0:
            raise NsgError(rc, "nsg_window_vectors_weighted")
        return r
    rc = _lib.nsg_window_vectors(
        None if src is None else src.data_ptr(), None if dst is None else dst.data_ptr(),
        None if keys is None else keys.data_ptr(), n, window, out.data_ptr(), ctypes.byref(v), ws.ptr, ws.nbytes,
        ctypes.c_void_p(s.cuda_stream), int(flags))
    if rc != 0:
        raise NsgError(rc, "nsg_window_vectors")
    return r


def window_stats_weighted(keys: Optional[torch.Tensor] = None, n_packets: Optional[torch.Tensor] = None,
                          window: int = DEFAULT_WINDOW, *, src=None, dst=None, out=None,
                          workspace: Optional[Workspace] = None, stream=None, flags: int = 0) -> torch.Tensor:
    """Nine quantities per window of WEIGHTED rows (src, dst, n_packets): the paper's three-column frame
    (PAPER.md:207; valid packets = sum of n_packets, :180).  Rows are packed `keys`
    (device int64/uint64) or SoA `src`, `dst` (device int32/uint32); `n_packets` device int32/uint32 (u32
    bit patterns).  Windows are cut by row index; a row of weight 0 adds nothing.  Returns a device int64
    tensor [n_windows, 9] (nsg_window_stats_weighted).
    """
    if keys is not None:
        if src is not None or dst is not None:
            raise ValueError("pass either keys or (src, dst)")
        _check(keys, "keys", _U64_TYPES)
        n, device = keys.numel(), keys.device
    else:
        _check(src, "src", _U32_TYPES)
        _check(dst, "dst", _U32_TYPES)
        if src.numel() != dst.numel() or src.device != dst.device:
            raise ValueError("src and dst must have the same length and device")
        n, device = src.numel(), src.device
    _check(n_packets, "n_packets", _U32_TYPES)
    if n_packets.numel() != n or n_packets.device != device:
        raise ValueError("n_packets must have one entry per row, on the rows' device")
    window = int(window)
    if window < 1 or window > MAX_WINDOW:
        raise ValueError(f"window must be in [1, 2^31], got {window}")
    nw = num_windows(n, window)
    if out is None:
        out = torch.empty((nw, NUM_STATS), dtype=torch.int64, device=device)
    elif out.dtype not in _U64_TYPES or not out.is_contiguous() or out.numel() < nw * NUM_STATS or not out.is_cuda:
        raise ValueError("out must be a contiguous CUDA int64/uint64 tensor with >= n_windows*9 elements")
    if n == 0:
        return out
    s = stream if stream is not None else torch.cuda.current_stream(device)
    ws = _workspace(n, window, device, workspace, s)
    _keep(s, ws.buffer, src, dst, keys, n_packets, out)
    rc = _lib.nsg_window_stats_weighted(
        None if src is None else src.data_ptr(), None if dst is None else dst.data_ptr(),
        None if keys is None else keys.data_ptr(), n_packets.data_ptr(), n, window, out.data_ptr(), ws.ptr,
        ws.nbytes, ctypes.c_void_p(s.cuda_stream), int(flags))
    if rc != 0:
        raise NsgError(rc, "nsg_window_stats_weighted")
    return out


# ---------------------------------------------------------------------------------------------------
# Whole-trace path: Table 2 on A = sum of the A_t, HBM-resident tables
# ---------------------------------------------------------------------------------------------------
class _Scratch:
    """Caller-owned, 256 B aligned device scratch of a given size."""

    def __init__(self, nbytes: int, device):
        self.nbytes = int(nbytes)
        self.buffer = torch.empty(max(self.nbytes, 1) + 256, dtype=torch.uint8, device=device)
        base = self.buffer.data_ptr()
        self.ptr = base + (-base) % 256


class TraceWorkspace(_Scratch):
    """Scratch of the trace steps for up to key_capacity keys per links call and record_capacity records
    per nodes call (nsg_trace_workspace_bytes)."""

    def __init__(self, key_capacity: int, record_capacity: int, world: int = 1, device=None):
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.key_capacity, self.record_capacity, self.world = int(key_capacity), int(record_capacity), int(world)
        nb = int(_lib.nsg_trace_workspace_bytes(self.key_capacity, self.record_capacity, self.world))
        if nb == 0:
            raise ValueError("world must be in [1, 1024]")
        super().__init__(nb, dev)


def _rows(keys, src, dst):
    if keys is not None:
        if src is not None or dst is not None:
            raise ValueError("pass either keys or (src, dst)")
        _check(keys, "keys", _U64_TYPES)
        return keys.numel(), keys.device
    _check(src, "src", _U32_TYPES)
    _check(dst, "dst", _U32_TYPES)
    if src.numel() != dst.numel() or src.device != dst.device:
        raise ValueError("src and dst must have the same length and device")
    return src.numel(), src.device


def _p(t):
    return None if t is None else t.data_ptr()


def trace_stats(keys: Optional[torch.Tensor] = None, *, src=None, dst=None, out=None, stream=None,
                n_packets: Optional[torch.Tensor] = None) -> torch.Tensor:
    """The nine statistics of the WHOLE input (A = sum of the A_t; nsg_trace_stats, one GPU).  Returns a
    device int64 [9] tensor, valid when `stream` completes.  `n_packets`: optional device int32/uint32 [n]
    weights of the rows (nsg_trace_stats_weighted)."""
    n, device = _rows(keys, src, dst)
    if out is None:
        out = torch.empty(NUM_STATS, dtype=torch.int64, device=device)
    if n == 0:
        return out.zero_()
    ws = _Scratch(_lib.nsg_trace_stats_workspace_bytes(n), device)
    s = stream if stream is not None else torch.cuda.current_stream(device)
    _keep(s, ws.buffer, out, src, dst, keys, n_packets)
    if n_packets is not None:
        _check(n_packets, "n_packets", _U32_TYPES)
        if n_packets.numel() != n or n_packets.device != device:
            raise ValueError("n_packets must have one entry per row, on the rows' device")
        rc = _lib.nsg_trace_stats_weighted(_p(src), _p(dst), _p(keys), n_packets.data_ptr(), n, out.data_ptr(),
                                           ws.ptr, ws.nbytes, ctypes.c_void_p(s.cuda_stream))
        if rc != 0:
            raise NsgError(rc, "nsg_trace_stats_weighted")
        return out
    rc = _lib.nsg_trace_stats(_p(src), _p(dst), _p(keys), n, out.data_ptr(), ws.ptr, ws.nbytes,
                              ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise NsgError(rc, "nsg_trace_stats")
    return out


def trace_partition(keys: torch.Tensor, world: int, workspace: TraceWorkspace, stream=None):
    """Step 1: keys grouped by the rank owning their link.  Returns (send_keys int64 [n], send_counts int64
    [world]) on the device."""
    n, device = _rows(keys, None, None)
    send = torch.empty(n, dtype=torch.int64, device=device)
    counts = torch.zeros(world, dtype=torch.int64, device=device)
    s = stream if stream is not None else torch.cuda.current_stream(device)
    _keep(s, keys, send, counts, workspace.buffer)
    rc = _lib.nsg_trace_partition(None, None, keys.data_ptr(), n, int(world), send.data_ptr(), counts.data_ptr(),
                                  workspace.ptr, workspace.nbytes, workspace.key_capacity, workspace.record_capacity,
                                  ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise NsgError(rc, "nsg_trace_partition")
    return send, counts


def trace_links(keys: torch.Tensor, world: int, workspace: TraceWorkspace, stream=None):
    """Step 2: the owned links.  Returns (link_stats int64 [3] = valid, unique links, max link; rec_src,
    rec_dst int64 [n] records (node << 32 | packets) grouped by owner; rec_counts int64 [2, world])."""
    n, device = _rows(keys, None, None)
    stats = torch.zeros(3, dtype=torch.int64, device=device)
    rs = torch.empty(max(n, 1), dtype=torch.int64, device=device)
    rd = torch.empty(max(n, 1), dtype=torch.int64, device=device)
    rc_ = torch.zeros((2, world), dtype=torch.int64, device=device)
    s = stream if stream is not None else torch.cuda.current_stream(device)
    _keep(s, keys, stats, rs, rd, rc_, workspace.buffer)
    rc = _lib.nsg_trace_links(None, None, keys.data_ptr() if n else None, n, int(world), stats.data_ptr(), rs.data_ptr(),
                              rd.data_ptr(), rc_.data_ptr(), workspace.ptr, workspace.nbytes, workspace.key_capacity,
                              workspace.record_capacity, ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise NsgError(rc, "nsg_trace_links")
    return stats, rs, rd, rc_


def trace_nodes(records: torch.Tensor, workspace: TraceWorkspace, stream=None) -> torch.Tensor:
    """Step 3: int64 [3] = unique nodes, max packets, max fan of one side's records."""
    m, device = records.numel(), records.device
    stats = torch.zeros(3, dtype=torch.int64, device=device)
    s = stream if stream is not None else torch.cuda.current_stream(device)
    _keep(s, records, stats, workspace.buffer)
    rc = _lib.nsg_trace_nodes(records.data_ptr() if m else None, m, stats.data_ptr(), workspace.ptr, workspace.nbytes,
                              workspace.key_capacity, workspace.record_capacity, ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise NsgError(rc, "nsg_trace_nodes")
    return stats



# ---------------------------------------------------------------------------------------------------
# IP address anonymisation
# ---------------------------------------------------------------------------------------------------
_anon_ws: dict = {}


def anonymize(keys: Optional[torch.Tensor] = None, *, src=None, dst=None, seed: int = 0, rounds: int = 1,
              stream=None):
    """Relabel every address by pi(rank(address)) (nsg_anonymize): rank = index among the distinct addresses
    of src and dst (ascending), pi = the keyed permutation of DESIGN.md R15 (`rounds` Feistel rounds; 0 = the
    ranks themselves).  Returns (src_out int32 [n], dst_out int32 [n], n_unique int64 [1]) on the device."""
    n, device = _rows(keys, src, dst)
    so = torch.empty(n, dtype=torch.int32, device=device)
    do = torch.empty(n, dtype=torch.int32, device=device)
    nu = torch.zeros(1, dtype=torch.int64, device=device)
    s = stream if stream is not None else torch.cuda.current_stream(device)
    ws = _anon_ws.get((device.index, s.cuda_stream))  # one scratch per stream: concurrent calls never share it
    if ws is None:
        ws = _anon_ws[(device.index, s.cuda_stream)] = _Scratch(_lib.nsg_anonymize_workspace_bytes(), device)
    _keep(s, ws.buffer, so, do, nu, src, dst, keys)
    rc = _lib.nsg_anonymize(_p(src), _p(dst), _p(keys), n, int(seed) & (2 ** 64 - 1), int(rounds), so.data_ptr(),
                            do.data_ptr(), nu.data_ptr(), ws.ptr, ws.nbytes, ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise NsgError(rc, "nsg_anonymize")
    return so, do, nu



# ---------------------------------------------------------------------------------------------------
# Fused exchange over peer memory (include/nsg.h "Fused exchange"): IPC-exported receive buffers
# ---------------------------------------------------------------------------------------------------
class _DevArray:
    """A raw device allocation seen by torch through __cuda_array_interface__ (no copy)."""

    def __init__(self, ptr: int, n: int, device):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (int(ptr), False), "version": 3,
                                         "strides": None}
        self.device = device


def ipc_handle_bytes() -> int:
    return int(_lib.nsg_ipc_handle_bytes())


def ipc_alloc(capacity: int, device):
    """An IPC-exportable device buffer of `capacity` int64 elements: (pointer, handle bytes, tensor view)."""
    ptr = ctypes.c_void_p()
    handle = (ctypes.c_char * ipc_handle_bytes())()
    with torch.cuda.device(device):
        rc = _lib.nsg_ipc_alloc(max(1, int(capacity)) * 8, ctypes.byref(ptr), handle)
    if rc != 0:
        raise NsgError(rc, "nsg_ipc_alloc")
    view = torch.as_tensor(_DevArray(ptr.value, max(1, int(capacity)), device), device=device)
    return ptr.value, bytes(handle), view


def ipc_open(handle: bytes, device) -> int:
    ptr = ctypes.c_void_p()
    with torch.cuda.device(device):
        rc = _lib.nsg_ipc_open(handle, ctypes.byref(ptr))
    if rc != 0:
        raise NsgError(rc, "nsg_ipc_open")
    return ptr.value


def ipc_close(ptr: int) -> None:
    _lib.nsg_ipc_close(ctypes.c_void_p(ptr))


def ipc_free(ptr: int) -> None:
    _lib.nsg_ipc_free(ctypes.c_void_p(ptr))


def trace_owner_counts(keys: torch.Tensor, world: int, workspace: TraceWorkspace, stream=None) -> torch.Tensor:
    """Keys per link owner rank: int64 [world] on the device (nsg_trace_owner_counts)."""
    n, device = _rows(keys, None, None)
    counts = torch.zeros(world, dtype=torch.int64, device=device)
    s = stream if stream is not None else torch.cuda.current_stream(device)
    _keep(s, keys, counts, workspace.buffer)
    rc = _lib.nsg_trace_owner_counts(None, None, keys.data_ptr() if n else None, n, int(world), counts.data_ptr(),
                                     workspace.ptr, workspace.nbytes, workspace.key_capacity,
                                     workspace.record_capacity, ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise NsgError(rc, "nsg_trace_owner_counts")
    return counts


def trace_partition_peers(keys: torch.Tensor, world: int, peer_ptrs: torch.Tensor, peer_base: torch.Tensor,
                          workspace: TraceWorkspace, stream=None) -> None:
    """Scatter the keys straight into the owners' receive buffers (nsg_trace_partition_peers)."""
    n, device = _rows(keys, None, None)
    s = stream if stream is not None else torch.cuda.current_stream(device)
    _keep(s, keys, peer_ptrs, peer_base, workspace.buffer)
    rc = _lib.nsg_trace_partition_peers(None, None, keys.data_ptr() if n else None, n, int(world), peer_ptrs.data_ptr(),
                                        peer_base.data_ptr(), workspace.ptr, workspace.nbytes, workspace.key_capacity,
                                        workspace.record_capacity, ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise NsgError(rc, "nsg_trace_partition_peers")


def trace_links_count(keys: torch.Tensor, world: int, workspace: TraceWorkspace, stream=None):
    """The owned links' statistics (int64 [3]) and record counts per side and owner (int64 [2, world]); the
    table stays in `workspace` for trace_links_emit_peers."""
    n, device = _rows(keys, None, None)
    stats = torch.zeros(3, dtype=torch.int64, device=device)
    rc_ = torch.zeros((2, world), dtype=torch.int64, device=device)
    s = stream if stream is not None else torch.cuda.current_stream(device)
    _keep(s, keys, stats, rc_, workspace.buffer)
    rc = _lib.nsg_trace_links_count(None, None, keys.data_ptr() if n else None, n, int(world), stats.data_ptr(),
                                    rc_.data_ptr(), workspace.ptr, workspace.nbytes, workspace.key_capacity,
                                    workspace.record_capacity, ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise NsgError(rc, "nsg_trace_links_count")
    return stats, rc_


def trace_links_emit_peers(world: int, ptrs_src: torch.Tensor, ptrs_dst: torch.Tensor, base_src: torch.Tensor,
                           base_dst: torch.Tensor, workspace: TraceWorkspace, stream=None) -> None:
    """Emit the records of the table left by trace_links_count straight into the owners' buffers."""
    device = ptrs_src.device
    s = stream if stream is not None else torch.cuda.current_stream(device)
    _keep(s, ptrs_src, ptrs_dst, base_src, base_dst, workspace.buffer)
    rc = _lib.nsg_trace_links_emit_peers(int(world), ptrs_src.data_ptr(), ptrs_dst.data_ptr(), base_src.data_ptr(),
                                         base_dst.data_ptr(), workspace.ptr, workspace.nbytes, workspace.key_capacity,
                                         workspace.record_capacity, ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise NsgError(rc, "nsg_trace_links_emit_peers")



def window_stats_mirrored(keys: torch.Tensor, mirrors: torch.Tensor, row0: int, window: int = DEFAULT_WINDOW, *,
                          out=None, workspace: Optional[Workspace] = None, stream=None, flags: int = 0) -> torch.Tensor:
    """window_stats_packed whose rows are also stored by the kernels into every table of `mirrors` (device
    int64 [k] of device pointers, e.g. the IPC-mapped result tables of every rank) at row row0 + w
    (nsg_window_stats_mirrored).  Returns the local int64 [n_windows, 9] result."""
    _check(keys, "keys", _U64_TYPES)
    n, device = keys.numel(), keys.device
    window = int(window)
    nw = num_windows(n, window)
    if out is None:
        out = torch.empty((nw, NUM_STATS), dtype=torch.int64, device=device)
    if n == 0:
        return out
    s = stream if stream is not None else torch.cuda.current_stream(device)
    ws = _workspace(n, window, device, workspace, s)
    _keep(s, ws.buffer, keys, mirrors, out)
    rc = _lib.nsg_window_stats_mirrored(None, None, keys.data_ptr(), n, window, out.data_ptr(), ws.ptr, ws.nbytes,
                                        ctypes.c_void_p(s.cuda_stream), int(flags), mirrors.data_ptr(),
                                        mirrors.numel(), int(row0))
    if rc != 0:
        raise NsgError(rc, "nsg_window_stats_mirrored")
    return out
