"""CUDA path of nsg_window_vectors (through the C ABI) vs the CPU oracle O1d, element by element (-m gpu).

SURVEY §8(f) rows f1 (vector-valued rows of Table 2: link packets PAPER.md:182, packets from source
:185, source fan-out :187, destination mirrors :173) and f3 (globally unique IPs :209, four counts).
The library returns each window's vector entries in hash order (include/nsg.h), so a window's entries
are sorted by key here before the comparison with the oracle, which emits them in ascending key order;
keys are unique within a window, so the sorted vectors are unique and compared bit-exactly, as are the
nine statistics (which must equal window_stats_packed's) and the IP set counts.
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


def gpu_vectors(nsg, keys_np, window, device, layout="packed", **kw):
    k = torch.from_numpy(np.ascontiguousarray(keys_np).view(np.int64)).to(device)
    if layout == "packed":
        r = nsg.window_vectors(k, window, **kw)
    else:
        r = nsg.window_vectors(None, window, src=(k >> 32).to(torch.int32).contiguous(),
                               dst=(k & 0xFFFFFFFF).to(torch.int32).contiguous(), **kw)
    torch.cuda.synchronize(device)
    out = {}
    for name, t in r.items():
        a = t.cpu().numpy()
        out[name] = a.view(np.uint64) if a.dtype == np.int64 else a.view(np.uint32)
    return out


def window_entries(g, window, w):
    """Window w's GPU entries, sorted by key (links) / node (sources, destinations)."""
    b = w * window
    nl, ns, nd = (int(x) for x in g["stats"][w, [1, 3, 6]])
    r = {}
    if "link_key" in g:
        k = g["link_key"][b:b + nl]
        o = np.argsort(k, kind="stable")
        r["link_key"], r["link_packets"] = k[o], g["link_packets"][b:b + nl][o]
    for side, n, names in (("src", ns, ("src_node", "src_packets", "src_fanout")),
                           ("dst", nd, ("dst_node", "dst_packets", "dst_fanin"))):
        if names[0] in g:
            node = g[names[0]][b:b + n]
            o = np.argsort(node, kind="stable")
            r[f"{side}_node"] = node[o]
            r[f"{side}_packets"] = g[names[1]][b:b + n][o]
            r[f"{side}_fan"] = g[names[2]][b:b + n][o]
    return r


def assert_vectors(g, keys, window, check=("links", "sources", "destinations", "ip_sets"), windows=None):
    want = oracle.window_distributions(keys=keys, window=window)
    stats = oracle.window_stats_sort(keys=keys, window=window)
    assert g["stats"].tolist() == stats.tolist()
    assert want["counts"].tolist() == stats[:, [1, 3, 6]].tolist()
    nw = stats.shape[0]
    if "ip_sets" in check:
        assert g["ip_sets"].tolist() == want["ip_sets"].tolist()
    for w in (range(nw) if windows is None else windows):
        got, exp = window_entries(g, window, w), oracle.window_slices(want, window, w)
        fields = []
        if "links" in check:
            fields += ["link_key", "link_packets"]
        if "sources" in check:
            fields += ["src_node", "src_packets", "src_fan"]
        if "destinations" in check:
            fields += ["dst_node", "dst_packets", "dst_fan"]
        for f in fields:
            a, b = got[f].astype(np.uint64), exp[f].astype(np.uint64)
            assert a.shape == b.shape and np.array_equal(a, b), (w, f, a.shape, b.shape)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_baseline_configs(nsg, cuda_device, cfg):
    c = CONFIGS[cfg]
    keys = gen.generate_host(c.dist, c.seed, 0, c.n_packets, packed=True)
    assert_vectors(gpu_vectors(nsg, keys, c.window, cuda_device), keys, c.window)


@pytest.mark.parametrize("n,window", [(3 * W + 12345, W), (10 ** 5, 4099), (50_000, 1), (20_000, 7),
                                      ((1 << 20) - 1 + 777, (1 << 20) - 1), (5000, 1 << 21)])
def test_ragged_and_window_sizes(nsg, cuda_device, n, window):
    keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 14), 41, 0, n, packed=True)
    windows = None if n // window < 64 else [0, 1, n // window // 2, (n - 1) // window]
    assert_vectors(gpu_vectors(nsg, keys, window, cuda_device), keys, window, windows=windows)


@pytest.mark.parametrize("flags", [1, 2])  # FORCE_GLOBAL (the L2 path), INJECT_OVERFLOW (odd windows handed off)
def test_l2_path_and_overflow_handoff(nsg, cuda_device, flags):
    keys = gen.generate_host(gen.Dist("heavy"), 42, 0, 4 * W + 999, packed=True)
    assert_vectors(gpu_vectors(nsg, keys, W, cuda_device, flags=flags), keys, W)


def test_adversarial_keys(nsg, cuda_device):
    """The empty-slot sentinels as addresses (255.255.255.255 as source, destination, both), all-equal
    windows, a star and self-loops, each a window of its own."""
    win = 4096
    rng = np.random.default_rng(5)
    E = np.uint64(0xFFFFFFFF)
    parts = [
        np.full(win, (E << np.uint64(32)) | E, np.uint64),                                         # ~0 -> ~0
        (E << np.uint64(32)) | rng.integers(0, 50, win).astype(np.uint64),                         # ~0 -> few
        (rng.integers(0, 50, win).astype(np.uint64) << np.uint64(32)) | E,                         # few -> ~0
        np.zeros(win, np.uint64),                                                                  # 0 -> 0
        (np.uint64(7) << np.uint64(32)) | np.arange(win, dtype=np.uint64),                         # star out
        (np.arange(win, dtype=np.uint64) << np.uint64(32)) | np.arange(win, dtype=np.uint64),      # self-loops
        np.where(rng.random(win) < 0.5, (E << np.uint64(32)) | E,
                 (rng.integers(0, 3, win).astype(np.uint64) << np.uint64(32)) | E),               # mixed ~0
    ]
    keys = np.concatenate(parts)
    for flags in (0, 1):
        assert_vectors(gpu_vectors(nsg, keys, win, cuda_device, flags=flags), keys, win)


def test_subsets_and_soa_layout(nsg, cuda_device):
    keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 20), 43, 0, 2 * W + 5, packed=True)
    g = gpu_vectors(nsg, keys, W, cuda_device, links=False, sources=False, destinations=False)
    assert set(g) == {"stats", "ip_sets"}
    assert_vectors(g, keys, W, check=("ip_sets",))
    g = gpu_vectors(nsg, keys, W, cuda_device, sources=False, ip_sets=False)
    assert_vectors(g, keys, W, check=("links", "destinations"))
    g = gpu_vectors(nsg, keys, W, cuda_device, layout="soa")
    assert_vectors(g, keys, W)


def test_stats_unchanged_by_vectors(nsg, cuda_device):
    c = CONFIGS["C2"]
    keys = gen.generate_host(c.dist, c.seed, 0, c.n_packets, packed=True)
    kd = torch.from_numpy(keys.view(np.int64)).to(cuda_device)
    a = nsg.window_stats_packed(kd, W).cpu()
    b = nsg.window_vectors(kd, W)["stats"].cpu()
    assert torch.equal(a, b)


def test_shared_address_pool(nsg, cuda_device):
    """Sources and destinations drawn from one Zipf-weighted pool of addresses, so most addresses are on both
    sides (the generated workloads use disjoint pools): exercises the S0 -> S1 list hand-off of |S n D|."""
    rng = np.random.default_rng(17)
    pool = rng.choice(2 ** 32, size=20_000, replace=False).astype(np.uint64)
    p = 1.0 / np.arange(1, pool.size + 1) ** 1.1
    p /= p.sum()
    n = 3 * W + 999
    keys = (pool[rng.choice(pool.size, n, p=p)] << np.uint64(32)) | pool[rng.choice(pool.size, n, p=p)]
    want = oracle.window_distributions(keys=keys, window=W)
    assert int(want["ip_sets"][:-1, 3].min()) > 1000   # full windows share most addresses
    for flags in (0, 1):
        assert_vectors(gpu_vectors(nsg, keys, W, cuda_device, flags=flags), keys, W)
