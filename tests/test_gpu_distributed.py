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
