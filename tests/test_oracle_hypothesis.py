"""Property-based pins of the oracles (hypothesis, -m "not gpu"): on arbitrary small packet streams
(arbitrary 32-bit addresses including the extremes, arbitrary window lengths and row weights), the three
independent procedures agree (O0 dense matrix = O1 std::map = O2 std::sort), the distributions oracle's
reductions equal the scalars, the weighted oracle equals the raw oracle on the weight-expanded stream, and
the invariants of SURVEY §8(c) hold.  Complements the fixed-seed brute force of test_oracle_pins.py.
"""
import numpy as np
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle

ADDR = st.one_of(st.integers(0, 7), st.sampled_from([0, 1, 0x7FFFFFFF, 0x80000000, 0xFFFFFFFE, 0xFFFFFFFF]),
                 st.integers(0, 2 ** 32 - 1))
PACKETS = st.lists(st.tuples(ADDR, ADDR), min_size=1, max_size=120)


def arrays(pk):
    s = np.array([p[0] for p in pk], dtype=np.uint32)
    d = np.array([p[1] for p in pk], dtype=np.uint32)
    return s, d


@settings(max_examples=300, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(PACKETS, st.integers(1, 130))
def test_three_oracles_agree(pk, W):
    s, d = arrays(pk)
    a = oracle.window_stats_map(s, d, W)
    assert a.tolist() == oracle.window_stats_sort(s, d, W).tolist()
    assert a.tolist() == oracle.window_stats_dense(s, d, W, max_vertices=512).tolist()


@settings(max_examples=200, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(PACKETS, st.integers(1, 130))
def test_invariants(pk, W):
    s, d = arrays(pk)
    out = oracle.window_stats_sort(s, d, W)
    for w, row in enumerate(out):
        v, L, mL, uS, mSP, mFO, uD, mDP, mFI = (int(x) for x in row)
        assert v == min(W, s.size - w * W)
        assert 1 <= L <= v and mFO <= uD and mFI <= uS and mL <= min(mSP, mDP)
        assert max(uS, uD) <= L <= uS * uD and -(-v // uS) <= mSP and -(-L // uS) <= mFO


@settings(max_examples=150, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(PACKETS, st.integers(1, 130))
def test_distribution_reductions(pk, W):
    s, d = arrays(pk)
    stats = oracle.window_stats_sort(s, d, W)
    r = oracle.window_distributions(s, d, W)
    assert r["counts"].tolist() == stats[:, [1, 3, 6]].tolist()
    for w in range(stats.shape[0]):
        g = oracle.window_slices(r, W, w)
        v, L, mL, uS, mSP, mFO, uD, mDP, mFI = (int(x) for x in stats[w])
        assert int(g["link_packets"].sum()) == v and int(g["link_packets"].max()) == mL
        assert (int(g["src_packets"].max()), int(g["src_fan"].max())) == (mSP, mFO)
        assert (int(g["dst_packets"].max()), int(g["dst_fan"].max())) == (mDP, mFI)
        u, so, do, b = (int(x) for x in g["ip_sets"])
        S = set(s[w * W:(w + 1) * W].tolist())
        D = set(d[w * W:(w + 1) * W].tolist())
        assert (u, so, do, b) == (len(S | D), len(S - D), len(D - S), len(S & D))


@settings(max_examples=150, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(st.lists(st.tuples(ADDR, ADDR, st.integers(0, 5)), min_size=1, max_size=60))
def test_weighted_equals_expanded(rows):
    s = np.array([r[0] for r in rows], np.uint32)
    d = np.array([r[1] for r in rows], np.uint32)
    wt = np.array([r[2] for r in rows], np.uint32)
    got = oracle.window_stats_weighted(s, d, wt, s.size)
    if wt.sum() == 0:
        assert got.tolist() == [[0] * 9]
    else:
        assert got.tolist() == oracle.window_stats_sort(np.repeat(s, wt), np.repeat(d, wt), int(wt.sum())).tolist()
