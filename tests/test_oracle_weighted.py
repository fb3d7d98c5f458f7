"""Pins of the weighted-rows oracle O1w (oracle.window_stats_weighted; input rows
(src, dst, n_packets), the paper's three-column frame PAPER.md:207, valid packets = sum of n_packets
PAPER.md:180) to things other than itself (-m "not gpu"): worked examples (tests/golden,
SPEC.md:216 / :128), the raw / aggregated equivalence SPEC.md:142 against the independent raw oracle
O2 (std::sort), expansion of weights into raw packets, the weighted dense brute force O0, closed forms
with 64-bit sums, and zero-weight rows (reading R14).
"""
import numpy as np
import pytest

import gen
import oracle
from nsg_testutil import load_golden_weighted


def test_golden_examples():
    for window, s, d, wt, exp in load_golden_weighted("weighted_examples.txt"):
        assert oracle.window_stats_weighted(s, d, wt, window).tolist() == exp.tolist(), (window, wt.tolist())
        assert oracle.window_stats_dense(s, d, window, weights=wt).tolist() == exp.tolist()


def aggregate_windows(s, d, W, rows_per_window, rng):
    """Aggregate each W-packet window of a raw stream into (src, dst, count) rows, padded to
    rows_per_window rows with weight-0 rows on random addresses, in random row order."""
    S, D, C = [], [], []
    for b in range(0, s.size, W):
        k = (s[b:b + W].astype(np.uint64) << np.uint64(32)) | d[b:b + W].astype(np.uint64)
        u, c = np.unique(k, return_counts=True)
        pad = rows_per_window - u.size
        assert pad >= 0
        ku = np.concatenate([u, rng.integers(0, 2 ** 63, pad, dtype=np.uint64)])
        cu = np.concatenate([c, np.zeros(pad, np.int64)])
        p = rng.permutation(ku.size)
        S.append((ku[p] >> np.uint64(32)).astype(np.uint32))
        D.append((ku[p] & np.uint64(0xFFFFFFFF)).astype(np.uint32))
        C.append(cu[p].astype(np.uint32))
    return np.concatenate(S), np.concatenate(D), np.concatenate(C)


@pytest.mark.parametrize("dist", [gen.Dist("uniform"), gen.Dist("zipf", 1.1, 1 << 20), gen.Dist("heavy"),
                                  gen.Dist("zipf", 1.5, 1 << 8)])
def test_raw_aggregated_equivalence(dist):
    """every query on the raw rows equals the query on their aggregation.  The raw side is O2
    (std::sort, no code shared with O1w)."""
    W = 1 << 15
    s, d = gen.generate_host(dist, 51, 0, 3 * W)
    raw = oracle.window_stats_sort(s, d, W)
    rng = np.random.default_rng(1)
    S, D, C = aggregate_windows(s, d, W, W, rng)
    assert oracle.window_stats_weighted(S, D, C, W).tolist() == raw.tolist()


@pytest.mark.parametrize("seed", range(3))
def test_expansion_and_dense(seed):
    """Row i of weight n_i is n_i raw packets: O1w on the rows = O2 on the expanded packets (one window), and
    = the weighted dense O0."""
    rng = np.random.default_rng(300 + seed)
    for _ in range(150):
        V = int(rng.integers(1, 40))
        n = int(rng.integers(1, 300))
        labels = rng.choice(2 ** 32, size=V, replace=False).astype(np.uint64)
        s = labels[rng.integers(0, V, n)].astype(np.uint32)
        d = labels[rng.integers(0, V, n)].astype(np.uint32)
        wt = rng.integers(0, 6, n).astype(np.uint32)
        got = oracle.window_stats_weighted(s, d, wt, n)
        if wt.sum():
            assert got.tolist() == oracle.window_stats_sort(np.repeat(s, wt), np.repeat(d, wt), int(wt.sum())).tolist()
        else:
            assert got.tolist() == [[0] * 9]
        assert got.tolist() == oracle.window_stats_dense(s, d, n, weights=wt).tolist()


def test_unit_weights_equal_raw():
    s, d = gen.generate_host(gen.Dist("zipf", 1.2, 5000), 3, 0, 20000)
    assert oracle.window_stats_weighted(s, d, np.ones(20000, np.uint32), 3000).tolist() == \
        oracle.window_stats_map(s, d, 3000).tolist()


def test_closed_forms_and_wide_sums():
    # all rows a -> b with weights w_i: [sum, 1, sum, 1, sum, 1, 1, sum, 1]; sums beyond 2^32 stay exact
    for wt in (np.array([5], np.uint32), np.array([1, 2, 3, 4], np.uint32), np.full(4, 2 ** 31, np.uint32),
               np.full(7, 0xFFFFFFFF, np.uint32)):
        t = int(wt.astype(np.uint64).sum())
        n = wt.size
        got = oracle.window_stats_weighted(np.full(n, 9, np.uint32), np.full(n, 10, np.uint32), wt, n)
        assert got.tolist() == [[t, 1, t, 1, t, 1, 1, t, 1]]
    # star out with weights: source packets = sum, fan-out = #nonzero rows
    wt = np.array([3, 0, 2, 7, 0, 1], np.uint32)
    got = oracle.window_stats_weighted(np.full(6, 1, np.uint32), np.arange(6, dtype=np.uint32) + 100, wt, 6)
    assert got.tolist() == [[13, 4, 7, 1, 13, 4, 4, 7, 1]]


def test_zero_weight_rows_are_ignored():
    s, d = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 12), 7, 0, 9000)
    wt = (np.arange(9000) % 4).astype(np.uint32)
    base = oracle.window_stats_weighted(s, d, wt, 3000)
    # replace the addresses of every zero-weight row by fresh ones: nothing changes
    s2, d2 = s.copy(), d.copy()
    z = wt == 0
    s2[z] = 0xFFFFFFFF - np.arange(z.sum(), dtype=np.uint32)
    d2[z] = 0xFFFF0000 + np.arange(z.sum(), dtype=np.uint32)
    assert oracle.window_stats_weighted(s2, d2, wt, 3000).tolist() == base.tolist()


# ---------------------------------------------------------------- weighted distributions (f1 x f4a)
DKEYS = ("link_key", "link_packets", "src_node", "src_packets", "src_fan", "dst_node", "dst_packets", "dst_fan",
         "ip_sets")


def _dist_windows(r, W):
    return [oracle.window_slices(r, W, w) for w in range(r["counts"].shape[0])]


@pytest.mark.parametrize("dist", [gen.Dist("zipf", 1.1, 1 << 20), gen.Dist("heavy")])
def test_weighted_distributions_equal_raw(dist):
    """SPEC.md:142 for the vector-valued rows: the distributions of the per-window aggregated rows (weights =
    multiplicities, padded with weight-0 rows) equal the raw packets' distributions, window by window."""
    W = 1 << 14
    s, d = gen.generate_host(dist, 52, 0, 3 * W)
    raw = _dist_windows(oracle.window_distributions(s, d, W), W)
    S, D, C = aggregate_windows(s, d, W, W, np.random.default_rng(2))
    agg = _dist_windows(oracle.window_distributions(S, D, W, weights=C), W)
    for a, b in zip(agg, raw):
        for k in DKEYS:
            assert np.asarray(a[k]).tolist() == np.asarray(b[k]).tolist(), k


def test_weighted_distributions_expansion():
    rng = np.random.default_rng(9)
    for _ in range(100):
        n = int(rng.integers(1, 200))
        s = rng.integers(0, 30, n).astype(np.uint32)
        d = rng.integers(0, 30, n).astype(np.uint32)
        wt = rng.integers(0, 5, n).astype(np.uint32)
        if wt.sum() == 0:
            continue
        a = _dist_windows(oracle.window_distributions(s, d, n, weights=wt), n)[0]
        b = _dist_windows(oracle.window_distributions(np.repeat(s, wt), np.repeat(d, wt), int(wt.sum())),
                          int(wt.sum()))[0]
        for k in DKEYS:
            assert np.asarray(a[k]).tolist() == np.asarray(b[k]).tolist(), k
