"""CUDA path (libnsg, through the C ABI) vs the CPU oracle, element by element (-m gpu).

Bit-exact is the bar: every output is an integer.  Cases: the BASELINE configs
at full size (C1-C3 fully; C4 2^30 packets in bench.py's launch configuration, all 8192 windows), ragged tails, window sizes spanning one to
many partition chunks and link buckets, the L2 path (forced, and the overflow hand-off), adversarial
keys (the empty-slot sentinels, all-equal windows, stars), misaligned bases, both input layouts.
"""
import numpy as np
import pytest
import torch

import gen
import oracle
from gen.configs import CONFIGS

pytestmark = pytest.mark.gpu

W = 1 << 17


@pytest.fixture(scope="module")
def nsg(cuda_device):
    import paper_2509_03653_b200 as m

    return m


def run(nsg, keys_np, window, device, flags=0, layout="packed", offset=0):
    k = torch.from_numpy(np.ascontiguousarray(keys_np).view(np.int64))
    if layout == "packed":
        buf = torch.empty(k.numel() + offset, dtype=torch.int64, device=device)
        buf[offset:].copy_(k)
        out = nsg.window_stats_packed(buf[offset:], window, flags=flags)
    else:
        kd = k.to(device)
        s = torch.empty(kd.numel() + offset, dtype=torch.int32, device=device)
        d = torch.empty(kd.numel() + offset, dtype=torch.int32, device=device)
        s[offset:].copy_((kd >> 32).to(torch.int32))
        d[offset:].copy_((kd & 0xFFFFFFFF).to(torch.int32))
        out = nsg.window_stats(s[offset:], d[offset:], window, flags=flags)
    torch.cuda.synchronize(device)
    return out.cpu().numpy().view(np.uint64)


def assert_parity(got, want):
    assert got.shape == want.shape
    bad = np.nonzero((got != want).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} windows differ; first {bad[0]}: got {got[bad[0]].tolist()} want {want[bad[0]].tolist()}"


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
@pytest.mark.parametrize("layout", ["packed", "soa"])
def test_baseline_configs_full(nsg, cuda_device, cfg, layout):
    c = CONFIGS[cfg]
    keys = gen.generate_host(c.dist, c.seed, 0, c.n_packets, packed=True)
    want = oracle.window_stats_sort(keys=keys, window=c.window)
    assert_parity(run(nsg, keys, c.window, cuda_device, layout=layout), want)


@pytest.mark.parametrize("flags", ["FORCE_GLOBAL", "INJECT_OVERFLOW"])
@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_l2_path_and_overflow_handoff(nsg, cuda_device, cfg, flags):
    c = CONFIGS[cfg]
    n = 6 * W + 4321
    keys = gen.generate_host(c.dist, c.seed, 0, n, packed=True)
    want = oracle.window_stats_sort(keys=keys, window=W)
    flag = getattr(nsg, "FLAG_" + flags)
    assert_parity(run(nsg, keys, W, cuda_device, flags=flag), want)


def test_overflow_handoff_is_counted(nsg, cuda_device):
    keys = gen.generate_host(gen.Dist("uniform"), 5, 0, 5 * W, packed=True)
    kd = torch.from_numpy(keys.view(np.int64)).to(cuda_device)
    ws = nsg.Workspace(kd.numel(), W)
    nsg.window_stats_packed(kd, W, workspace=ws, flags=nsg.FLAG_INJECT_OVERFLOW)
    assert ws.diag()[:2] == [2, 0]       # odd windows 1 and 3 handed over; no self-check failure
    nsg.window_stats_packed(kd, W, workspace=ws)
    assert ws.diag()[:2] == [0, 0]


@pytest.mark.parametrize("window", [1, 2, 3, 7, 100, 1023, 1024, 1025, 4095, 4096, 4097, 8192 + 5, 65536,
                                    (1 << 17) - 1, (1 << 17) + 1, 1 << 20])
def test_window_sizes_and_ragged_tails(nsg, cuda_device, window):
    n = min(int(window * 3.5) + 3, (1 << 22) + 11)
    keys = gen.generate_host(gen.Dist("zipf", 1.2, 1 << 14), 17, 0, n, packed=True)
    want = oracle.window_stats_sort(keys=keys, window=window)
    assert_parity(run(nsg, keys, window, cuda_device), want)


@pytest.mark.parametrize("window", [(1 << 20) + 1, 1 << 21])
def test_large_windows_use_l2_path(nsg, cuda_device, window):
    n = 2 * window + 999
    keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 20), 4, 0, n, packed=True)
    assert_parity(run(nsg, keys, window, cuda_device), oracle.window_stats_sort(keys=keys, window=window))


def adversarial_cases():
    n = 3 * W + 77
    out = {}
    k = np.full(n, 0xFFFFFFFFFFFFFFFF, np.uint64)
    out["all-sentinel"] = k.copy()
    k[::3] = 0
    k[1::7] = 0xFFFFFFFF00000000
    k[2::11] = 0x00000000FFFFFFFF
    k[5::13] = 0xFFFFFFFF00000001
    out["sentinel-mix"] = k
    out["all-same"] = np.full(n, 0x0A0000010A000002, np.uint64)
    i = np.arange(n, dtype=np.uint64)
    out["star-in"] = (i << np.uint64(32)) | np.uint64(7)
    out["star-out"] = np.uint64(5 << 32) | i
    out["self-loops"] = (i % np.uint64(100)) * np.uint64(0x100000001)
    out["distinct"] = (i << np.uint64(32)) | (i + np.uint64(1 << 31))
    rng = np.random.default_rng(9)
    out["tiny-universe"] = rng.integers(0, 2 ** 64, n, dtype=np.uint64) & np.uint64(0x0000000300000003)
    return out


@pytest.mark.parametrize("name", sorted(adversarial_cases()))
@pytest.mark.parametrize("flags", [0, 1])
def test_adversarial_keys(nsg, cuda_device, name, flags):
    keys = adversarial_cases()[name]
    want = oracle.window_stats_sort(keys=keys, window=W)
    assert_parity(run(nsg, keys, W, cuda_device, flags=flags), want)


@pytest.mark.parametrize("offset", [1, 3])
@pytest.mark.parametrize("layout", ["packed", "soa"])
def test_misaligned_base(nsg, cuda_device, offset, layout):
    keys = gen.generate_host(gen.Dist("heavy"), 3, 0, 2 * W + 5, packed=True)
    want = oracle.window_stats_sort(keys=keys, window=W)
    assert_parity(run(nsg, keys, W, cuda_device, layout=layout, offset=offset), want)


def test_empty_input(nsg, cuda_device):
    out = nsg.window_stats_packed(torch.empty(0, dtype=torch.int64, device=cuda_device), W)
    assert tuple(out.shape) == (0, 9)


def test_repeat_calls_reuse_workspace(nsg, cuda_device):
    c = CONFIGS["C2"]
    keys = gen.generate_host(c.dist, c.seed, 0, 16 * W, packed=True)
    kd = torch.from_numpy(keys.view(np.int64)).to(cuda_device)
    ws = nsg.Workspace(kd.numel(), W)
    want = oracle.window_stats_sort(keys=keys, window=W)
    for _ in range(5):
        got = nsg.window_stats_packed(kd, W, workspace=ws).cpu().numpy().view(np.uint64)
        assert_parity(got, want)
    assert nsg.last_launches() >= 1


@pytest.mark.parametrize("n,window,chunk", [(3 * W + 777, W, 1), (8 * W, W, 3), (5 * W, W, 0), (100003, 4096, 5),
                                             (7 * W + 1, 3 * W, 2)])
def test_from_host_streamed(nsg, cuda_device, n, window, chunk):
    """nsg_window_stats_from_host: chunked H2D on a copy stream overlapped with the kernel (partition
    items wait on per-chunk arrival flags); parity with the oracle, and the staging buffer holds the
    input afterwards.  Ragged: partial last window, chunk counts that do not divide the windows."""
    c = CONFIGS["C2"]
    keys = gen.generate_host(c.dist, 11, 0, n, packed=True)
    host = torch.from_numpy(keys.view(np.int64)).pin_memory()
    kd = torch.empty(n, dtype=torch.int64, device=cuda_device)
    got = nsg.window_stats_from_host(host, window, device=cuda_device, keys_dev=kd, chunk_windows=chunk)
    assert_parity(got.numpy().view(np.uint64), oracle.window_stats_sort(keys=keys, window=window))
    assert torch.equal(kd.cpu(), host)


def test_from_host_repeated_and_forced_l2(nsg, cuda_device):
    c = CONFIGS["C3"]
    keys = gen.generate_host(c.dist, c.seed, 0, 6 * W + 5, packed=True)
    want = oracle.window_stats_sort(keys=keys, window=W)
    host = torch.from_numpy(keys.view(np.int64)).pin_memory()
    kd = torch.empty(host.numel(), dtype=torch.int64, device=cuda_device)
    ws = nsg.Workspace(host.numel(), W)
    for _ in range(3):
        assert_parity(nsg.window_stats_from_host(host, W, keys_dev=kd, workspace=ws).numpy().view(np.uint64), want)
    # a window above the fast path's limit goes to the L2 path after the copies
    keys2 = gen.generate_host(c.dist, 2, 0, (1 << 21) + 3, packed=True)
    host2 = torch.from_numpy(keys2.view(np.int64)).pin_memory()
    got = nsg.window_stats_from_host(host2, 1 << 21).numpy().view(np.uint64)
    assert_parity(got, oracle.window_stats_sort(keys=keys2, window=1 << 21))


def test_from_host_rejects_bad_arguments(nsg, cuda_device):
    host = torch.zeros(1000, dtype=torch.int64)
    with pytest.raises(ValueError):
        nsg.window_stats_from_host(host, W)  # not pinned
    hp = host.pin_memory()
    s = torch.cuda.current_stream(cuda_device)
    with pytest.raises(nsg.NsgError):
        nsg.window_stats_from_host(hp, W, stream=s, copy_stream=s)
    assert tuple(nsg.window_stats_from_host(torch.zeros(0, dtype=torch.int64).pin_memory(), W).shape) == (0, 9)


def test_device_generator_matches_host(nsg, cuda_device):
    for dist in (gen.Dist("uniform"), gen.Dist("zipf", 1.1, 1 << 20), gen.Dist("heavy")):
        kd = torch.empty(300000, dtype=torch.int64, device=cuda_device)
        gen.generate_device(dist, 5, (1 << 32) - 1000, 300000, keys=kd)
        host = gen.generate_host(dist, 5, (1 << 32) - 1000, 300000, packed=True)
        assert np.array_equal(kd.cpu().numpy().view(np.uint64), host)


def test_c4_full_size_all_windows(nsg, cuda_device):
    """C4: 2^30 packets generated on device, one launch over all 8192 windows (bench.py's launch
    configuration at N=1); EVERY window checked against the oracle O2.  The oracle's input is the same
    seeded generator's output (gen/, which holds none of the method's arithmetic and is pinned equal
    to the host generator by test_device_generator_matches_host), copied to the host block by block."""
    c = CONFIGS["C4"]
    kd = torch.empty(c.n_packets, dtype=torch.int64, device=cuda_device)
    gen.generate_device(c.dist, c.seed, 0, c.n_packets, keys=kd)
    got = nsg.window_stats_packed(kd, c.window).cpu().numpy().view(np.uint64)
    nw = c.n_packets // c.window
    assert got.shape == (nw, 9)
    blk = 256 * c.window
    host = torch.empty(blk, dtype=torch.int64).pin_memory()
    for b0 in range(0, c.n_packets, blk):
        host.copy_(kd[b0:b0 + blk])
        want = oracle.window_stats_sort(keys=host.numpy().view(np.uint64), window=c.window)
        w0 = b0 // c.window
        assert_parity(got[w0:w0 + want.shape[0]], want)
    del kd
    # a spot check that does not rely on the device generator: windows regenerated on the host
    for w in (0, nw // 2, nw - 1):
        k = gen.generate_host(c.dist, c.seed, w * c.window, c.window, packed=True)
        assert got[w].tolist() == oracle.window_stats_sort(keys=k, window=c.window)[0].tolist(), w
