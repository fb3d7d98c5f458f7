"""Multi-process host logic of the window-sharded driver (gloo, world_size 2, CPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle
from paper_2509_03653_b200.distributed import gather_window_stats, packet_block, window_block


@pytest.mark.parametrize("nw,world", [(0, 1), (1, 2), (7, 2), (8192, 8), (64, 3), (5, 8)])
def test_window_blocks_partition(nw, world):
    blocks = [window_block(nw, r, world) for r in range(world)]
    assert blocks[0][0] == 0 and blocks[-1][1] == nw
    for (a0, a1), (b0, b1) in zip(blocks, blocks[1:]):
        assert a1 == b0
    sizes = [b - a for a, b in blocks]
    assert max(sizes) - min(sizes) <= 1


def test_packet_blocks_align_to_windows():
    n, W = 10 * 1000 + 17, 1000
    covered = []
    for r in range(4):
        p0, p1 = packet_block(n, W, r, 4)
        assert p0 % W == 0
        covered.append((p0, p1))
    assert covered[0][0] == 0 and covered[-1][1] == n
    for (a0, a1), (b0, b1) in zip(covered, covered[1:]):
        assert a1 == b0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, W, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p0, p1 = packet_block(n, W, rank, world)
        keys = gen.generate_host(gen.Dist("heavy"), 3, p0, p1 - p0, packed=True)
        # the per-rank compute is the CUDA path on GPUs; here the oracle stands in for it (test only)
        local = torch.from_numpy(oracle.window_stats_sort(keys=keys, window=W).astype(np.int64))
        nw = (n + W - 1) // W
        full = gather_window_stats(local, nw)
        q.put((rank, full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [7 * 4096 + 123, 2 * 4096, 100])
def test_gather_matches_single_process(n):
    W, world = 4096, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, W, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    keys = gen.generate_host(gen.Dist("heavy"), 3, 0, n, packed=True)
    want = oracle.window_stats_sort(keys=keys, window=W).astype(np.int64)
    for r in range(world):
        assert np.array_equal(results[r], want)
