"""The input generator (not the method): host C == independent numpy restatement; Zipf table sanity."""
import numpy as np
import pytest

import gen
from gen.configs import CONFIGS


@pytest.mark.parametrize("dist", [gen.Dist("uniform"), gen.Dist("zipf", 1.1, 1 << 20), gen.Dist("heavy"),
                                  gen.Dist("zipf", 0.8, 1000)])
@pytest.mark.parametrize("first", [0, 12345, (1 << 32) - 100])
def test_host_matches_numpy(dist, first):
    s, d = gen.generate_host(dist, 7, first, 50000)
    s2, d2 = gen.generate_numpy(dist, 7, first, 50000)
    assert np.array_equal(s, s2) and np.array_equal(d, d2)
    k = gen.generate_host(dist, 7, first, 50000, packed=True)
    assert np.array_equal(k, gen.pack(s, d))


def test_counter_based_slices():
    dist = gen.Dist("zipf", 1.1, 1 << 20)
    s, d = gen.generate_host(dist, 2, 0, 100000)
    s2, d2 = gen.generate_host(dist, 2, 40000, 30000)
    assert np.array_equal(s[40000:70000], s2) and np.array_equal(d[40000:70000], d2)


def test_thread_count_independent():
    a = gen.generate_host(gen.Dist("heavy"), 3, 5, 300000, packed=True, threads=1)
    b = gen.generate_host(gen.Dist("heavy"), 3, 5, 300000, packed=True, threads=7)
    assert np.array_equal(a, b)


def test_zipf_table():
    s, K = 1.1, 1 << 20
    T = gen.zipf_table(s, K)
    assert T.dtype == np.uint64 and T.size == K
    assert int(T[-1]) == 2 ** 64 - 1
    assert np.all(np.diff(T.astype(np.float64)) >= 0)
    k = np.arange(1, K + 1, dtype=np.float64)
    F = np.cumsum(k ** -s) / np.sum((k ** -s)[::-1])
    assert np.max(np.abs(T.astype(np.float64) / 2.0 ** 64 - F)) < 1e-9


def test_distribution_shapes():
    W = 1 << 17
    s, d = gen.generate_host(gen.Dist("heavy"), 3, 0, W)
    hot = (s == 0x0A000001).mean()
    assert abs(hot - 0.5) < 0.01
    s, d = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 20), 2, 0, W)
    # rank-1 probability of Zipf(1.1, 2^20) is 1/H_{K,s} ~ 0.1237
    H = np.sum(np.arange(1, (1 << 20) + 1, dtype=np.float64) ** -1.1)
    top = np.bincount(np.unique(s, return_inverse=True)[1]).max() / W
    assert abs(top - 1.0 / H) < 0.005


def test_configs():
    assert CONFIGS["C2"].n_packets == 1 << 23 and CONFIGS["C2"].dist.name == "zipf"
    assert all(c.window == 1 << 17 for c in CONFIGS.values())
