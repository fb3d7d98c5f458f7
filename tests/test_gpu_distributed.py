"""Multi-process drivers on the B200 (-m gpu): two ranks share the one GPU over gloo (the pod has one GPU).

The window-sharded statistics with both result transports: NCCL-style all-gather (gloo
here) and "p2p", where the kernels' epilogues store every result row into every rank's CUDA-IPC-mapped
table (nsg_window_stats_mirrored).  Checked bit-exactly against the oracle on every rank.
"""
import os
import socket

import numpy as np
import pytest
import torch

import gen
import oracle

pytestmark = pytest.mark.gpu

W = 1 << 17


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, transport, reps, q):
    import torch.distributed as dist

    import paper_2509_03653_b200 as nsg  # noqa: F401
    from paper_2509_03653_b200.distributed import distributed_window_stats, packet_block

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p0, p1 = packet_block(n, W, rank, world)
        nw = (n + W - 1) // W
        outs = []
        for rep in range(reps):  # the p2p tables are reused across calls
            keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 20), 30 + rep, p0, p1 - p0, packed=True)
            kd = torch.from_numpy(keys.view(np.int64)).cuda()
            outs.append(distributed_window_stats(kd, nw, W, transport=transport).cpu().numpy())
        q.put((rank, outs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
@pytest.mark.parametrize("world,n", [(2, 5 * W + 777), (3, 4 * W)])
def test_window_sharded_gather(cuda_device, transport, world, n):
    import torch.multiprocessing as mp

    reps = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, transport, reps, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rep in range(reps):
        keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 20), 30 + rep, 0, n, packed=True)
        want = oracle.window_stats_sort(keys=keys, window=W)
        for r in range(world):
            assert results[r][rep].view(np.uint64).tolist() == want.tolist(), (r, rep)


def _c4_worker(rank, world, port, q):
    import torch.distributed as dist

    from gen.configs import CONFIGS
    from paper_2509_03653_b200.distributed import distributed_window_stats, packet_block

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = CONFIGS["C4"]
        nw = c.n_packets // c.window
        p0, p1 = packet_block(c.n_packets, c.window, rank, world)
        kd = torch.empty(p1 - p0, dtype=torch.int64, device="cuda")
        gen.generate_device(c.dist, c.seed, p0, p1 - p0, keys=kd)  # this rank's windows only
        table = distributed_window_stats(kd, nw, c.window).cpu().numpy()
        q.put((rank, table if rank == 0 else int(table.sum())))
    finally:
        dist.destroy_process_group()


def test_c4_split_over_8_ranks(cuda_device):
    """C4 (2^30 packets, 8192 windows) as bench.py --gpus 8 splits it: 8 ranks (processes sharing the
    one GPU, gloo standing in for NCCL) each generate and compute their contiguous window block, then
    distributed_window_stats gathers the [8192, 9] table onto every rank; rank 0's table is compared
    with the oracle O2 on every window, the other ranks' tables by checksum."""
    import torch.multiprocessing as mp

    from gen.configs import CONFIGS

    world = 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_c4_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    table = results[0].view(np.uint64)
    assert all(results[r] == int(results[0].sum()) for r in range(1, world))
    c = CONFIGS["C4"]
    blk = 256 * c.window
    kd = torch.empty(blk, dtype=torch.int64, device=cuda_device)
    for b0 in range(0, c.n_packets, blk):
        gen.generate_device(c.dist, c.seed, b0, blk, keys=kd)
        want = oracle.window_stats_sort(keys=kd.cpu().numpy().view(np.uint64), window=c.window)
        w0 = b0 // c.window
        assert table[w0:w0 + want.shape[0]].tolist() == want.tolist(), w0
