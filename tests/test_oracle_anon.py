"""Pins of the anonymisation oracle (oracle.anonymize), -m "not gpu".

The permutation itself is a defined reading (R15), so the pins fix what the paper fixes: the
unique/rank step on a hand example, N = |src u D| against the independent std::map union count (O1d), the
permutation property of pi for many N and seeds, and the paper's anonymisation argument (every Table 2
quantity of the relabelled stream equals the original's), checked with O2 per window and on the whole stream.
"""
import numpy as np
import pytest

import gen
import oracle
from oracle import anon


def test_ranks_hand_example():
    # addresses {3, 7, 10} -> U = [3, 7, 10]; with rounds = 0 the labels are the ranks
    s, d, N = oracle.anonymize([10, 3, 10, 7], [7, 7, 3, 10], rounds=0)
    assert N == 3 and s.tolist() == [2, 0, 2, 1] and d.tolist() == [1, 1, 0, 2]


@pytest.mark.parametrize("N", list(range(1, 70)) + [255, 256, 257, 1000, 4095, 65536, 100_003])
def test_permutation_is_a_bijection(N):
    for seed, rounds in ((0, 1), (12345, 2), (2 ** 63 + 7, 3)):
        p = anon.permutation(np.arange(N), N, seed, rounds)
        assert np.array_equal(np.sort(p), np.arange(N, dtype=np.uint64))


def test_permutation_depends_on_seed_and_rounds():
    N = 5000
    a = anon.permutation(np.arange(N), N, 1, 1)
    assert not np.array_equal(a, np.arange(N))
    assert not np.array_equal(a, anon.permutation(np.arange(N), N, 2, 1))
    assert not np.array_equal(a, anon.permutation(np.arange(N), N, 1, 2))
    # rounds compose: two rounds = the second network applied to the first's output
    b = anon.permutation(a, N, 1 + 1, 1)
    assert np.array_equal(anon.permutation(np.arange(N), N, 1, 2), b)


@pytest.mark.parametrize("dist", [gen.Dist("zipf", 1.1, 1 << 20), gen.Dist("heavy"), gen.Dist("uniform")])
def test_unique_count_equals_union_of_o1d(dist):
    n = 50_000
    s, d = gen.generate_host(dist, 81, 0, n)
    _, _, N = oracle.anonymize(s, d, seed=3)
    r = oracle.window_distributions(s, d, n)
    assert N == int(r["ip_sets"][0, 0])   # |S u D| of the whole stream (one window), std::map sets


@pytest.mark.parametrize("rounds", [0, 1, 2])
def test_statistics_invariant_under_anonymisation(rounds):
    """relabelling by a bijection keeps every Table 2 quantity."""
    W = 1 << 14
    s, d = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 16), 82, 0, 5 * W + 77)
    a, b, N = oracle.anonymize(s, d, seed=99, rounds=rounds)
    assert int(max(a.max(), b.max())) < N
    assert oracle.window_stats_sort(a, b, W).tolist() == oracle.window_stats_sort(s, d, W).tolist()
    assert oracle.window_stats_sort(a, b, s.size).tolist() == oracle.window_stats_sort(s, d, s.size).tolist()
    # the relabelling is one bijection on the addresses: equal addresses <-> equal labels
    both = np.concatenate([s, d])
    lab = np.concatenate([a, b])
    _, first = np.unique(both, return_index=True)
    assert np.unique(lab).size == N
    assert np.array_equal(lab, lab[first][np.searchsorted(np.unique(both), both)])
