"""CUDA path of nsg_window_stats_weighted (through the C ABI) vs the CPU oracles, bit-exact (-m gpu).

SURVEY §8(f) row f4a: weighted rows (src, dst, n_packets), the paper's three-column frame (PAPER.md:207,
valid packets = sum of n_packets :180).  Checked against O1w (oracle.window_stats_weighted) and, through
the raw / aggregated equivalence, against the raw-packet oracle O2 on the C2 stream
aggregated per window on the host.
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


def run_w(nsg, keys, wt, window, device, layout="packed", offset=0, flags=0, want_diag=False):
    k = torch.from_numpy(np.ascontiguousarray(keys).view(np.int64)).to(device)
    wb = torch.empty(wt.size + offset, dtype=torch.int32, device=device)
    wb[offset:].copy_(torch.from_numpy(np.ascontiguousarray(wt).view(np.int32)))
    ws = nsg.Workspace(max(1, keys.size), window, device)
    if layout == "packed":
        kb = torch.empty(k.numel() + offset, dtype=torch.int64, device=device)
        kb[offset:].copy_(k)
        out = nsg.window_stats_weighted(kb[offset:], wb[offset:], window, workspace=ws, flags=flags)
    else:
        s = (k >> 32).to(torch.int32).contiguous()
        d = (k & 0xFFFFFFFF).to(torch.int32).contiguous()
        out = nsg.window_stats_weighted(None, wb[offset:], window, src=s, dst=d, workspace=ws, flags=flags)
    torch.cuda.synchronize(device)
    got = out.cpu().numpy().view(np.uint64)
    return (got, ws.diag()) if want_diag else got


def aggregate(keys, window, rng):
    """Each window of raw packets -> its (key, count) rows, padded to `window` rows with weight-0 rows on
    random keys, rows shuffled."""
    K, C = [], []
    for b in range(0, keys.size, window):
        u, c = np.unique(keys[b:b + window], return_counts=True)
        pad = min(window, keys.size - b) - u.size
        ku = np.concatenate([u, rng.integers(0, 2 ** 63, pad, dtype=np.uint64)])
        cu = np.concatenate([c, np.zeros(pad, np.int64)]).astype(np.uint32)
        p = rng.permutation(ku.size)
        K.append(ku[p])
        C.append(cu[p])
    return np.concatenate(K), np.concatenate(C)


@pytest.mark.parametrize("cfg", ["C2", "C3", "C1"])
def test_raw_aggregated_equivalence(nsg, cuda_device, cfg):
    c = CONFIGS[cfg]
    keys = gen.generate_host(c.dist, c.seed, 0, c.n_packets, packed=True)
    raw = oracle.window_stats_sort(keys=keys, window=c.window)
    K, C = aggregate(keys, c.window, np.random.default_rng(3))
    assert run_w(nsg, K, C, c.window, cuda_device).tolist() == raw.tolist()


@pytest.mark.parametrize("layout,offset", [("packed", 0), ("soa", 0), ("packed", 1), ("soa", 3)])
def test_random_weights(nsg, cuda_device, layout, offset):
    n = 3 * W + 4321
    keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 20), 61, 0, n, packed=True)
    wt = np.random.default_rng(4).integers(0, 9, n).astype(np.uint32)
    want = oracle.window_stats_weighted(keys=keys, weights=wt, window=W)
    assert run_w(nsg, keys, wt, W, cuda_device, layout=layout, offset=offset).tolist() == want.tolist()


def test_unit_weights_equal_raw(nsg, cuda_device):
    keys = gen.generate_host(gen.Dist("heavy"), 62, 0, 2 * W + 77, packed=True)
    kd = torch.from_numpy(keys.view(np.int64)).to(cuda_device)
    raw = nsg.window_stats_packed(kd, W).cpu().numpy().view(np.uint64)
    assert run_w(nsg, keys, np.ones(keys.size, np.uint32), W, cuda_device).tolist() == raw.tolist()


@pytest.mark.parametrize("window", [1, 5, 4097, 100_000, (1 << 20) - 1, 1 << 21])
def test_window_sizes(nsg, cuda_device, window):
    n = max(3 * window + 11, 20_000) if window < (1 << 20) else window + 999
    keys = gen.generate_host(gen.Dist("zipf", 1.3, 1 << 10), 63, 0, n, packed=True)
    wt = np.random.default_rng(window).integers(0, 4, n).astype(np.uint32)
    want = oracle.window_stats_weighted(keys=keys, weights=wt, window=window)
    assert run_w(nsg, keys, wt, window, cuda_device).tolist() == want.tolist()


def test_heavy_weights_go_to_l2_path(nsg, cuda_device):
    """Bucket weight sums >= 2^20 do not fit the fast path's 20-bit record counts: those windows are handed
    to the L2 path (diag[0]) and stay exact."""
    n = 2 * W
    keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 20), 64, 0, n, packed=True)
    wt = np.random.default_rng(5).integers(1, 2048, n).astype(np.uint32)
    want = oracle.window_stats_weighted(keys=keys, weights=wt, window=W)
    got, diag = run_w(nsg, keys, wt, W, cuda_device, want_diag=True)
    assert got.tolist() == want.tolist()
    assert diag[0] == 2 and diag[1] == 0 and diag[2] == 0


def test_force_global_and_zero_windows(nsg, cuda_device):
    n = 4 * 3000
    keys = gen.generate_host(gen.Dist("uniform"), 65, 0, n, packed=True)
    wt = np.random.default_rng(6).integers(0, 3, n).astype(np.uint32)
    wt[3000:6000] = 0  # a window of zero-weight rows only: an all-zero A_t
    want = oracle.window_stats_weighted(keys=keys, weights=wt, window=3000)
    assert want[1].tolist() == [0] * 9
    for flags in (0, 1, 2):  # fast path, FORCE_GLOBAL, INJECT_OVERFLOW (odd windows handed to the L2 path)
        assert run_w(nsg, keys, wt, 3000, cuda_device, flags=flags).tolist() == want.tolist()


def test_sum_beyond_32_bits_is_reported(nsg, cuda_device):
    keys = np.array([5, 5, 6, 7], np.uint64)
    wt = np.array([0xFFFFFFFF, 0xFFFFFFFF, 1, 1], np.uint32)
    _, diag = run_w(nsg, keys, wt, 2, cuda_device, want_diag=True)
    assert diag[2] == 1  # window 0 exceeds the 32-bit counters; window 1 is fine
    got = run_w(nsg, keys[2:], wt[2:], 2, cuda_device)
    assert got.tolist() == oracle.window_stats_weighted(keys=keys[2:], weights=wt[2:], window=2).tolist()


@pytest.mark.parametrize("flags", [0, 1, 2])
def test_weighted_vectors(nsg, cuda_device, flags):
    """nsg_window_vectors_weighted: every vector and the IP sets of weighted rows vs the weighted O1d."""
    from test_gpu_vectors import window_entries

    n = 2 * W + 3001
    keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 18), 66, 0, n, packed=True)
    wt = np.random.default_rng(7).integers(0, 6, n).astype(np.uint32)
    kd = torch.from_numpy(keys.view(np.int64)).to(cuda_device)
    wd = torch.from_numpy(wt.view(np.int32)).to(cuda_device)
    r = nsg.window_vectors(kd, W, n_packets=wd, flags=flags)
    torch.cuda.synchronize(cuda_device)
    g = {k: (t.cpu().numpy().view(np.uint64) if t.dtype == torch.int64 else t.cpu().numpy().view(np.uint32))
         for k, t in r.items()}
    want = oracle.window_distributions(keys=keys, window=W, weights=wt)
    assert g["stats"].tolist() == oracle.window_stats_weighted(keys=keys, weights=wt, window=W).tolist()
    assert g["ip_sets"].tolist() == want["ip_sets"].tolist()
    for w in range(want["counts"].shape[0]):
        got, exp = window_entries(g, W, w), oracle.window_slices(want, W, w)
        for f in ("link_key", "link_packets", "src_node", "src_packets", "src_fan", "dst_node", "dst_packets",
                  "dst_fan"):
            assert got[f].astype(np.uint64).tolist() == exp[f].astype(np.uint64).tolist(), (w, f)


@pytest.mark.parametrize("delta", [-1, 0, 1])
def test_window_weight_sum_at_the_20_bit_edge(nsg, cuda_device, delta):
    """The round-2 kernels keep packets in 20-bit fields: a window whose weights sum to 2^20 or more is
    handed to the L2 path.  Sums 2^20 - 1 / 2^20 / 2^20 + 1 (hand-over count 0 / 1 / 1), bit-exact."""
    win = 4096
    keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 12), 66, 0, win, packed=True)
    wt = np.full(win, 256, np.uint32)  # sum 2^20
    wt[0] += np.uint32(delta) if delta >= 0 else np.uint32(0)
    if delta < 0:
        wt[0] -= np.uint32(1)
    assert int(wt.sum()) == (1 << 20) + delta
    want = oracle.window_stats_weighted(keys=keys, weights=wt, window=win)
    got, diag = run_w(nsg, keys, wt, win, cuda_device, want_diag=True)
    assert got.tolist() == want.tolist()
    assert diag[0] == (0 if delta < 0 else 1) and diag[1] == 0
