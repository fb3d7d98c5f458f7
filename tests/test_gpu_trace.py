"""CUDA whole-trace path (nsg_trace_*, through the C ABI) vs the CPU oracle, bit-exact (-m gpu).

SURVEY §8(f) row f4b: Table 2 on A = sum over t of A_t, i.e. the nine statistics of the whole input as
ONE window, computed by O2 (std::sort) with window = n.  Covers the one-GPU call (nsg_trace_stats), the
step API (partition / links / nodes) with several owner ranks on one GPU, and the multi-process driver
(two ranks sharing the GPU over gloo, which stages the all-to-all through host memory).
"""
import os
import socket

import numpy as np
import pytest
import torch

import gen
import oracle
from gen.configs import CONFIGS

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nsg(cuda_device):
    import paper_2509_03653_b200 as m

    return m


def whole(keys):
    return oracle.window_stats_sort(keys=keys, window=max(1, keys.size))[0].tolist()


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_trace_stats_configs(nsg, cuda_device, cfg):
    c = CONFIGS[cfg]
    keys = gen.generate_host(c.dist, c.seed, 0, c.n_packets, packed=True)
    kd = torch.from_numpy(keys.view(np.int64)).to(cuda_device)
    got = nsg.trace_stats(kd).cpu().numpy().view(np.uint64).tolist()
    assert got == whole(keys)


@pytest.mark.parametrize("n", [1, 2, 1000, 65_537])
def test_trace_small_and_soa(nsg, cuda_device, n):
    keys = gen.generate_host(gen.Dist("zipf", 1.2, 1 << 10), 71, 0, n, packed=True)
    kd = torch.from_numpy(keys.view(np.int64)).to(cuda_device)
    assert nsg.trace_stats(kd).cpu().numpy().view(np.uint64).tolist() == whole(keys)
    s = (kd >> 32).to(torch.int32).contiguous()
    d = (kd & 0xFFFFFFFF).to(torch.int32).contiguous()
    assert nsg.trace_stats(src=s, dst=d).cpu().numpy().view(np.uint64).tolist() == whole(keys)


def test_trace_adversarial(nsg, cuda_device):
    E = np.uint64(0xFFFFFFFF)
    rng = np.random.default_rng(8)
    keys = np.concatenate([np.full(777, (E << np.uint64(32)) | E, np.uint64),
                           (E << np.uint64(32)) | rng.integers(0, 40, 3000).astype(np.uint64),
                           (rng.integers(0, 40, 3000).astype(np.uint64) << np.uint64(32)) | E,
                           np.zeros(50, np.uint64)])
    rng.shuffle(keys)
    kd = torch.from_numpy(keys.view(np.int64)).to(cuda_device)
    assert nsg.trace_stats(kd).cpu().numpy().view(np.uint64).tolist() == whole(keys)


@pytest.mark.parametrize("world", [2, 5])
def test_trace_steps_on_one_gpu(nsg, cuda_device, world):
    """The step API with `world` owner ranks, all on this GPU: partitions are permutations grouped by owner,
    disjoint link sets per owner, and per-side node sets per owner; summed / maxed they give the whole trace."""
    n = 300_000
    keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 16), 72, 0, n, packed=True)
    kd = torch.from_numpy(keys.view(np.int64)).to(cuda_device)
    ws = nsg.TraceWorkspace(n, n, world, cuda_device)
    send, counts = nsg.trace_partition(kd, world, ws)
    counts = counts.cpu().tolist()
    assert sum(counts) == n
    assert np.array_equal(np.sort(send.cpu().numpy().view(np.uint64)), np.sort(keys))
    off = np.concatenate([[0], np.cumsum(counts)])
    parts = [send[off[o]:off[o + 1]] for o in range(world)]
    link_sets = [set(np.unique(p.cpu().numpy()).tolist()) for p in parts]
    for a in range(world):
        for b in range(a + 1, world):
            assert not (link_sets[a] & link_sets[b])
    ls, recs = [], [[[] for _ in range(world)] for _ in range(2)]
    for p in parts:
        st, rs, rd, rc = nsg.trace_links(p.contiguous(), world, ws)
        ls.append(st.cpu().numpy())
        rc = rc.cpu().numpy()
        for side, r in enumerate((rs, rd)):
            o = np.concatenate([[0], np.cumsum(rc[side])])
            for q in range(world):
                recs[side][q].append(r[o[q]:o[q + 1]])
    ns = [[nsg.trace_nodes(torch.cat(recs[side][q]), ws).cpu().numpy() for q in range(world)] for side in range(2)]
    ls = np.array(ls)
    got = [ls[:, 0].sum(), ls[:, 1].sum(), ls[:, 2].max(),
           sum(x[0] for x in ns[0]), max(x[1] for x in ns[0]), max(x[2] for x in ns[0]),
           sum(x[0] for x in ns[1]), max(x[1] for x in ns[1]), max(x[2] for x in ns[1])]
    assert [int(x) for x in got] == whole(keys)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _driver_worker(rank, world, port, n, q, transport="nccl"):
    import torch.distributed as dist

    import paper_2509_03653_b200 as nsg_mod  # noqa: F401  (loads libnsg)
    from paper_2509_03653_b200.distributed import distributed_trace_stats

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p0, p1 = (n * rank) // world, (n * (rank + 1)) // world
        keys = gen.generate_host(gen.Dist("heavy"), 73, p0, p1 - p0, packed=True)
        out = distributed_trace_stats(torch.from_numpy(keys.view(np.int64)).cuda(), transport=transport)
        q.put((rank, out.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_distributed_driver_two_ranks_one_gpu(cuda_device, transport):
    """Two ranks sharing the GPU over gloo.  transport="p2p": the partition / emission kernels store into the
    other rank's receive buffer through a CUDA IPC mapping (same device here; NVLink P2P across GPUs)."""
    import torch.multiprocessing as mp

    n, world = 200_003, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_driver_worker, args=(r, world, port, n, q, transport)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    keys = gen.generate_host(gen.Dist("heavy"), 73, 0, n, packed=True)
    for r in range(world):
        assert results[r].view(np.uint64).tolist() == whole(keys)


@pytest.mark.parametrize("n", [5000, 1 << 20])
def test_trace_weighted(nsg, cuda_device, n):
    """nsg_trace_stats_weighted: the whole trace of weighted rows vs O1w with window = n."""
    keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 16), 74, 0, n, packed=True)
    wt = np.random.default_rng(n).integers(0, 7, n).astype(np.uint32)
    kd = torch.from_numpy(keys.view(np.int64)).to(cuda_device)
    got = nsg.trace_stats(kd, n_packets=torch.from_numpy(wt.view(np.int32)).to(cuda_device))
    want = oracle.window_stats_weighted(keys=keys, weights=wt, window=n)[0]
    assert got.cpu().numpy().view(np.uint64).tolist() == want.tolist()


@pytest.mark.parametrize("dist", ["zipf", "uniform"])
def test_trace_cas_first_inserts_on_small_inputs(nsg, cuda_device, dist):
    """The CAS-as-probe inserts (used for DRAM-resident tables of >= 2^26 slots) forced on for every table
    size (nsg_debug_trace_cas_first_slots, include/nsg_internal.h), including the sentinel keys."""
    from paper_2509_03653_b200 import api

    d = gen.Dist("zipf", 1.1, 1 << 16) if dist == "zipf" else gen.Dist("uniform")
    keys = gen.generate_host(d, 72, 0, 300_007, packed=True)
    keys[::97] = np.uint64(0xFFFFFFFFFFFFFFFF)
    keys[5::101] = np.uint64(0xFFFFFFFF00000003)
    kd = torch.from_numpy(keys.view(np.int64)).to(cuda_device)
    assert api._lib.nsg_debug_trace_cas_first_slots(1) == 0
    try:
        got = nsg.trace_stats(kd).cpu().numpy().view(np.uint64).tolist()
    finally:
        assert api._lib.nsg_debug_trace_cas_first_slots(0) == 0
    assert got == whole(keys)


@pytest.mark.parametrize("dist", ["zipf", "uniform"])
def test_trace_at_2_25_keys(nsg, cuda_device, dist):
    """2^25 packets: link and node tables of >= 2^26 slots, where the CAS-as-probe inserts and the
    device-sized node tables run by default; checked against O2 (window = n)."""
    d = gen.Dist("zipf", 1.1, 1 << 20) if dist == "zipf" else gen.Dist("uniform")
    n = 1 << 25
    kd = torch.empty(n, dtype=torch.int64, device=cuda_device)
    gen.generate_device(d, 73, 0, n, keys=kd)
    got = nsg.trace_stats(kd).cpu().numpy().view(np.uint64).tolist()
    assert got == whole(kd.cpu().numpy().view(np.uint64))


def test_trace_rejects_2_32_packets(nsg, cuda_device):
    from paper_2509_03653_b200 import api

    kd = torch.zeros(8, dtype=torch.int64, device=cuda_device)
    out = torch.empty(9, dtype=torch.int64, device=cuda_device)
    rc = api._lib.nsg_trace_stats(None, None, kd.data_ptr(), 1 << 32, out.data_ptr(), None, 0, None)
    assert rc == 1  # NSG_ERR_INVALID_ARGUMENT before any allocation or launch
