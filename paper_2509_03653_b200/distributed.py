"""Multi-GPU drivers: window-sharded per-window statistics and the whole-trace
statistics with key-hash all-to-all exchanges.

Windows are independent units (Table 2 is evaluated per traffic matrix A_t, line 173), so
rank r of R owns the contiguous window block [floor(r*Nw/R), floor((r+1)*Nw/R)) and computes it
with no data-path collective.  The only exchange is the 72 B/window result rows: one
all_gather_into_tensor of an int64 [max_rows, 9] block per rank (NCCL over NVLink on GPUs, gloo in
the CPU tests), after which every rank holds the [Nw, 9] table — or, with transport "p2p", the kernels'
epilogues store every row into every rank's CUDA-IPC-mapped table themselves.  The whole trace
partitions links and nodes over the ranks and exchanges keys and link records (NCCL all-to-all, or the
scatter kernels storing into the owners' IPC-mapped buffers).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

NUM_STATS = 9


def window_block(n_windows: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of windows owned by `rank` (at most one window of imbalance)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (n_windows * rank) // world, (n_windows * (rank + 1)) // world


def packet_block(n_packets: int, window: int, rank: int, world: int) -> tuple[int, int]:
    """Packet range [p0, p1) of the windows `rank` owns; windows never straddle ranks."""
    nw = 0 if n_packets == 0 else (n_packets + window - 1) // window
    w0, w1 = window_block(nw, rank, world)
    return min(w0 * window, n_packets), min(w1 * window, n_packets)


def gather_window_stats(local: torch.Tensor, n_windows: int, group=None) -> torch.Tensor:
    """All-gather every rank's [rows_r, 9] int64 block (rows_r from window_block) into [n_windows, 9].

    `local` lives on the collective's device (CUDA for NCCL, CPU for gloo).
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    w0, w1 = window_block(n_windows, rank, world)
    if local.shape != (w1 - w0, NUM_STATS) or local.dtype != torch.int64:
        raise ValueError(f"rank {rank}: expected int64 [{w1 - w0}, 9], got {tuple(local.shape)} {local.dtype}")
    rows = max(window_block(n_windows, r, world)[1] - window_block(n_windows, r, world)[0] for r in range(world))
    home = local.device
    if dist.get_backend(group) == "gloo" and local.is_cuda:  # gloo gathers host tensors
        local = local.cpu()
    padded = torch.zeros((rows, NUM_STATS), dtype=torch.int64, device=local.device)
    padded[: w1 - w0].copy_(local)
    out = torch.empty((world * rows, NUM_STATS), dtype=torch.int64, device=local.device)
    dist.all_gather_into_tensor(out, padded, group=group)
    pieces = []
    for r in range(world):
        a, b = window_block(n_windows, r, world)
        pieces.append(out[r * rows: r * rows + (b - a)])
    return torch.cat(pieces, dim=0).to(home)


_result_tables: dict = {}


def distributed_window_stats(keys_local: torch.Tensor, n_windows: int, window: int, group=None,
                             workspace=None, transport: str = "nccl") -> torch.Tensor:
    """Per-rank CUDA computation of its window block (packed keys of exactly those windows) and the gather of
    the [n_windows, 9] result onto every rank.  transport="nccl": all_gather_into_tensor; "p2p": the kernels'
    epilogues store every row into every rank's CUDA-IPC-mapped result table (nsg_window_stats_mirrored), then
    a stream sync + barrier; the tables are kept across calls."""
    if transport == "nccl":
        from .api import window_stats_packed

        local = window_stats_packed(keys_local, window, workspace=workspace)
        return gather_window_stats(local, n_windows, group)
    if transport != "p2p":
        raise ValueError("transport must be 'nccl' or 'p2p'")
    from .api import window_stats_mirrored

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    device = keys_local.device
    key = (id(group), n_windows, device.index)
    tab = _result_tables.get(key)
    if tab is None:
        tab = _result_tables[key] = PeerBuffers(n_windows * NUM_STATS, group, device)
    w0, w1 = window_block(n_windows, rank, world)
    # The kernels below store into every peer's table: first let every rank finish reading its table
    # from the previous call (the clone below runs asynchronously on its stream).
    torch.cuda.synchronize(device)
    dist.barrier(group=group)
    window_stats_mirrored(keys_local, tab.ptrs, w0, window, workspace=workspace)
    torch.cuda.synchronize(device)
    dist.barrier(group=group)  # every rank's rows are in every table
    return tab.local[: n_windows * NUM_STATS].view(n_windows, NUM_STATS).clone()



# ---------------------------------------------------------------------------------------------------
# Whole trace: A = sum over t of A_t over every rank's packets.  Links and nodes are
# hash-partitioned over the ranks, so the only data-path collectives are the all-to-all exchanges of the
# keys and of the link records; every aggregation step runs in libnsg's kernels (nsg_trace_*).
# ---------------------------------------------------------------------------------------------------
def _trace_partition(keys, world, ws):
    from .api import trace_partition

    return trace_partition(keys, world, ws)


def _trace_links(keys, world, ws):
    from .api import trace_links

    return trace_links(keys, world, ws)


def _trace_nodes(records, ws):
    from .api import trace_nodes

    return trace_nodes(records, ws)


def _trace_workspace(key_cap, rec_cap, world, device):
    from .api import TraceWorkspace

    return TraceWorkspace(key_cap, rec_cap, world, device)


def _exchange(send: torch.Tensor, counts: torch.Tensor, group=None) -> torch.Tensor:
    """All-to-all of the owner-grouped `send` (segment o -> rank o, lengths `counts`): returns what every
    rank sent here, in rank order.  NCCL moves device tensors directly; gloo stages them through host memory."""
    world = dist.get_world_size(group)
    home = send.device
    gloo = dist.get_backend(group) == "gloo"
    c = counts.cpu() if gloo else counts
    rc = torch.empty_like(c)
    dist.all_to_all_single(rc, c.contiguous(), group=group)
    ins, outs = counts.cpu().tolist(), rc.cpu().tolist()
    src = send[: sum(ins)]
    if gloo:
        src = src.cpu()
    recv = torch.empty(sum(outs), dtype=send.dtype, device=src.device)
    if world == 1:
        recv.copy_(src)
    else:
        dist.all_to_all_single(recv, src.contiguous(), output_split_sizes=outs, input_split_sizes=ins, group=group)
    return recv.to(home)


def segment_plan(counts: torch.Tensor, rank: int):
    """Placement of the fused exchange from the all-gathered counts[r][o] (items rank r sends to owner o):
    (items this rank receives, where this rank's segment starts in each owner's buffer [world], the largest
    buffer any owner needs).  Owner o's buffer holds the senders' segments in rank order."""
    c = counts.to(torch.int64).cpu()
    recv = int(c[:, rank].sum())
    base = c[:rank, :].sum(dim=0) if rank else torch.zeros(c.shape[1], dtype=torch.int64)
    cap = int(c.sum(dim=0).max()) if c.numel() else 0
    return recv, base, cap


def _all_gather_rows(t: torch.Tensor, group=None) -> torch.Tensor:
    """[world, *t.shape] stack of every rank's `t` (gloo: through host memory)."""
    world = dist.get_world_size(group)
    src = t.cpu() if dist.get_backend(group) == "gloo" else t
    out = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(out, src.contiguous(), group=group)
    return torch.stack(out).to(t.device)


class PeerBuffers:
    """One IPC-exported receive buffer per rank, mapped into every rank (include/nsg.h "Fused exchange"):
    `local` is this rank's buffer (int64 view), `ptrs` the device array of every rank's buffer pointer as
    seen from here.  Collective: every rank constructs and closes it together."""

    def __init__(self, capacity: int, group, device):
        from .api import ipc_alloc, ipc_open

        self.group, self.device = group, device
        self.capacity = max(1, int(capacity))
        self.own, handle, self.local = ipc_alloc(self.capacity, device)
        h = torch.frombuffer(bytearray(handle), dtype=torch.uint8)
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        hs = _all_gather_rows(h.to(device) if dist.get_backend(group) != "gloo" else h, group).cpu()
        self.opened = []
        ptrs = []
        for r in range(world):
            if r == rank:
                ptrs.append(self.own)
            else:
                p = ipc_open(bytes(hs[r].numpy().tobytes()), device)
                self.opened.append(p)
                ptrs.append(p)
        self.ptrs = torch.tensor(ptrs, dtype=torch.int64, device=device)

    def close(self):
        from .api import ipc_close, ipc_free

        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)  # nobody reads or writes the buffers any more
        for p in self.opened:
            ipc_close(p)
        ipc_free(self.own)
        self.opened = []


_trace_buffers: dict = {}


def _peer_buffers(name: str, capacity: int, group, device) -> "PeerBuffers":
    """Receive buffers kept across calls, re-created (collectively: every rank computes the same capacity
    from the same gathered counts) only when a call needs more than they hold."""
    key = (id(group), name, device.index)
    b = _trace_buffers.get(key)
    if b is None or b.capacity < max(1, capacity):
        if b is not None:
            b.close()
        b = _trace_buffers[key] = PeerBuffers(max(capacity, 1) * 5 // 4 + 1024, group, device)
    return b


def _trace_stats_p2p(keys_local: torch.Tensor, group=None) -> torch.Tensor:
    """distributed_trace_stats with the fused exchange: the partition and emission kernels store straight
    into the owners' receive buffers over peer memory, so no all-to-all collective moves the data."""
    from .api import trace_links_count, trace_links_emit_peers, trace_owner_counts, trace_partition_peers

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    device = keys_local.device
    n = keys_local.numel()
    ws = _trace_workspace(max(n, 1), 1, world, device)
    counts = trace_owner_counts(keys_local, world, ws)
    recv, base, cap = segment_plan(_all_gather_rows(counts, group), rank)
    kbuf = _peer_buffers("keys", cap, group, device)
    dist.barrier(group=group)  # the previous call's readers are done with the buffers
    trace_partition_peers(keys_local, world, kbuf.ptrs, base.to(device), ws)
    torch.cuda.synchronize(device)
    dist.barrier(group=group)  # every sender's stores into this rank's buffer are complete
    mine = kbuf.local[:recv]
    ws = _trace_workspace(max(recv, 1), 1, world, device)
    link_stats, rc = trace_links_count(mine, world, ws)
    R = _all_gather_rows(rc, group)  # [world, 2, world]
    plans = [segment_plan(R[:, s, :], rank) for s in (0, 1)]
    rbufs = [_peer_buffers(f"records{s}", plans[s][2], group, device) for s in (0, 1)]
    dist.barrier(group=group)
    trace_links_emit_peers(world, rbufs[0].ptrs, rbufs[1].ptrs, plans[0][1].to(device), plans[1][1].to(device), ws)
    torch.cuda.synchronize(device)
    dist.barrier(group=group)
    wsn = _trace_workspace(1, max(plans[0][0], plans[1][0], 1), 1, device)
    ns = _trace_nodes(rbufs[0].local[:plans[0][0]], wsn)
    nd = _trace_nodes(rbufs[1].local[:plans[1][0]], wsn)
    return _trace_combine(link_stats, ns, nd, group)


def _trace_combine(link_stats, ns, nd, group=None) -> torch.Tensor:
    """Sum / max over ranks of the per-rank partials into the nine statistics (north_star order)."""
    world = dist.get_world_size(group)
    device = link_stats.device
    sums = torch.stack([link_stats[0], link_stats[1], ns[0], nd[0]])
    maxes = torch.stack([link_stats[2], ns[1], ns[2], nd[1], nd[2]])
    if world > 1:
        gloo = dist.get_backend(group) == "gloo"
        sums_c, maxes_c = (sums.cpu(), maxes.cpu()) if gloo else (sums, maxes)
        dist.all_reduce(sums_c, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(maxes_c, op=dist.ReduceOp.MAX, group=group)
        sums, maxes = sums_c.to(device), maxes_c.to(device)
    return torch.stack([sums[0], sums[1], maxes[0], sums[2], maxes[1], maxes[2], sums[3], maxes[3], maxes[4]])


def distributed_trace_stats(keys_local: torch.Tensor, group=None, transport: str = "nccl") -> torch.Tensor:
    """The nine statistics of the whole trace held across the ranks (this rank's packets: packed int64 keys
    on its GPU).  Steps: partition by link owner -> all-to-all -> links -> all-to-all of the source and of the
    destination records -> nodes per side -> sum / max over ranks.  Returns int64 [9] on every rank (on the
    keys' device), north_star column order.  transport="nccl": the exchanges are NCCL all_to_all_single
    (gloo in CPU tests); "p2p": the partition and emission kernels write into the owners' IPC-mapped
    receive buffers themselves (fused compute + exchange over NVLink)."""
    if transport == "p2p":
        return _trace_stats_p2p(keys_local, group)
    if transport != "nccl":
        raise ValueError("transport must be 'nccl' or 'p2p'")
    world = dist.get_world_size(group)
    device = keys_local.device
    n = keys_local.numel()
    ws = _trace_workspace(max(n, 1), 1, world, device)
    send, counts = _trace_partition(keys_local, world, ws)
    mine = _exchange(send, counts, group)
    m = mine.numel()
    ws = _trace_workspace(max(m, 1), 1, world, device)
    link_stats, rs, rd, rc = _trace_links(mine, world, ws)
    rec_s = _exchange(rs, rc[0], group)
    rec_d = _exchange(rd, rc[1], group)
    ws = _trace_workspace(1, max(rec_s.numel(), rec_d.numel(), 1), 1, device)
    ns = _trace_nodes(rec_s, ws)
    nd = _trace_nodes(rec_d, ws)
    # sums: valid, unique links, unique sources, unique destinations; maxes: the rest
    return _trace_combine(link_stats, ns, nd, group)
