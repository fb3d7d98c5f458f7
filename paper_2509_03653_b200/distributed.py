"""Window-sharded multi-GPU driver.

Windows are independent units (Table 2 is evaluated per traffic matrix A_t, line 173), so
rank r of R owns the contiguous window block [floor(r*Nw/R), floor((r+1)*Nw/R)) and computes it
with no data-path collective.  The only exchange is the 72 B/window result rows: one
all_gather_into_tensor of an int64 [max_rows, 9] block per rank (NCCL over NVLink on GPUs, gloo in
the CPU tests), after which every rank holds the [Nw, 9] table.
"""
from __future__ import annotations

from typing import Optional

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


def distributed_window_stats(keys_local: torch.Tensor, n_windows: int, window: int, group=None,
                             workspace=None) -> torch.Tensor:
    """Per-rank CUDA computation of its window block (packed keys of exactly those windows) and the
    NCCL gather of the [n_windows, 9] result onto every rank."""
    from .api import window_stats_packed

    local = window_stats_packed(keys_local, window, workspace=workspace)
    return gather_window_stats(local, n_windows, group)
