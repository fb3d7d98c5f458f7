"""Pins of the CPU oracle to things other than itself (-m "not gpu").

Each pin cites what fixes it: a worked example (tests/golden, SPEC.md / hand counts from PAPER.md
Table 2), a closed form, brute force on the dense matrix, an independent library route (scipy.sparse
evaluation of the matrix notation; pandas with the DESIGN.md corrections of the dataframe column),
invariants and metamorphic relations.  A plausible bug in either oracle procedure (a dropped term, a
swapped src/dst, fan counted as packets, a max taken over the wrong axis) fails at least one pin.
"""
import numpy as np
import pytest

import gen
import oracle
from nsg_testutil import load_golden

ORACLES = {
    "map": lambda s, d, w: oracle.window_stats_map(s, d, w),
    "sort": lambda s, d, w: oracle.window_stats_sort(s, d, w),
    "sort1": lambda s, d, w: oracle.window_stats_sort(s, d, w, threads=1),
    "dense": lambda s, d, w: oracle.window_stats_dense(s, d, w, max_vertices=4096),
}


# ---------------------------------------------------------------- worked examples
@pytest.mark.parametrize("fixture", ["spec_s395_three_packets.txt", "survey_four_packets.txt",
                                     "spec_single_queries.txt"])
@pytest.mark.parametrize("which", sorted(ORACLES))
def test_golden_examples(fixture, which):
    for window, s, d, exp in load_golden(fixture):
        got = ORACLES[which](s, d, window)
        assert got.tolist() == exp.tolist(), (fixture, window)


def test_golden_concatenated_windows():
    # The single-query examples, concatenated, are separate windows only if each has the same length;
    # concatenate the two 3-packet cases of spec_single_queries.txt into one stream with window 3.
    cases = [c for c in load_golden("spec_single_queries.txt") if c[0] == 3]
    s = np.concatenate([c[1] for c in cases])
    d = np.concatenate([c[2] for c in cases])
    exp = np.concatenate([c[3] for c in cases])
    for which in ORACLES:
        assert ORACLES[which](s, d, 3).tolist() == exp.tolist()


# ---------------------------------------------------------------- closed forms
def closed_forms(W):
    """(name, src, dst, expected row) with the row fixed by hand from Table 2's definitions."""
    i = np.arange(W, dtype=np.uint64)
    out = []
    out.append(("all-same", np.full(W, 0x0A000001, np.uint32), np.full(W, 0x0A000002, np.uint32),
                [W, 1, W, 1, W, 1, 1, W, 1]))
    out.append(("self-loop", np.full(W, 0xC0A80001, np.uint32), np.full(W, 0xC0A80001, np.uint32),
                [W, 1, W, 1, W, 1, 1, W, 1]))
    out.append(("distinct", i.astype(np.uint32), (i + (1 << 31)).astype(np.uint32), [W, W, 1, W, 1, 1, W, 1, 1]))
    out.append(("star-out", np.full(W, 5, np.uint32), i.astype(np.uint32), [W, W, 1, 1, W, W, W, 1, 1]))
    out.append(("star-in", i.astype(np.uint32), np.full(W, 5, np.uint32), [W, W, 1, W, 1, 1, 1, W, W]))
    out.append(("extremes", np.full(W, 0xFFFFFFFF, np.uint32), np.full(W, 0xFFFFFFFF, np.uint32),
                [W, 1, W, 1, W, 1, 1, W, 1]))
    out.append(("zero", np.zeros(W, np.uint32), np.zeros(W, np.uint32), [W, 1, W, 1, W, 1, 1, W, 1]))
    return out


@pytest.mark.parametrize("W", [1, 2, 5, 64, 1000])
@pytest.mark.parametrize("which", sorted(ORACLES))
def test_closed_forms(W, which):
    for name, s, d, row in closed_forms(W):
        if which == "dense" and name in ("distinct", "star-out", "star-in") and W > 1000:
            continue
        got = ORACLES[which](s, d, W)
        assert got.tolist() == [row], name


@pytest.mark.parametrize("sdr", [(1, 1, 1), (2, 3, 1), (3, 2, 4), (5, 7, 3), (16, 1, 2), (1, 16, 2)])
@pytest.mark.parametrize("which", sorted(ORACLES))
def test_complete_bipartite(sdr, which):
    """s sources x d destinations, every pair r times: [W, s*d, r, s, d*r, d, d, s*r, s]."""
    S, D, r = sdr
    src = np.repeat(np.arange(S, dtype=np.uint32) + 100, D * r)
    dst = np.tile(np.repeat(np.arange(D, dtype=np.uint32) + 7000, r), S)
    rng = np.random.default_rng(S * 100 + D * 10 + r)
    perm = rng.permutation(src.size)
    W = S * D * r
    got = ORACLES[which](src[perm], dst[perm], W)
    assert got.tolist() == [[W, S * D, r, S, D * r, D, D, S * r, S]]


@pytest.mark.parametrize("which", ["map", "sort"])
def test_window_one_and_window_ge_n(which):
    rng = np.random.default_rng(5)
    s = rng.integers(0, 50, 300).astype(np.uint32)
    d = rng.integers(0, 50, 300).astype(np.uint32)
    assert ORACLES[which](s, d, 1).tolist() == [[1] * 9] * 300
    whole = ORACLES[which](s, d, 300)
    assert ORACLES[which](s, d, 10 ** 6).tolist() == whole.tolist()


def test_empty_input():
    e = np.zeros(0, np.uint32)
    for which in ORACLES:
        assert ORACLES[which](e, e, 17).shape == (0, 9)


# ---------------------------------------------------------------- brute force (dense matrix)
@pytest.mark.parametrize("seed", range(4))
def test_bruteforce_dense_equals_map_equals_sort(seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(500):
        V = int(rng.integers(1, 65))
        W = int(rng.integers(1, 600))
        n = int(rng.integers(1, 3 * W + 2))
        if rng.random() < 0.5:  # skewed draw
            p = rng.zipf(1.5, size=V).astype(float)
            p /= p.sum()
            s = rng.choice(V, n, p=p)
            d = rng.choice(V, n, p=p[::-1])
        else:
            s = rng.integers(0, V, n)
            d = rng.integers(0, V, n)
        labels = rng.choice(2 ** 32, size=V, replace=False).astype(np.uint64)  # arbitrary 32-bit addresses
        s = labels[s].astype(np.uint32)
        d = labels[d].astype(np.uint32)
        a = oracle.window_stats_dense(s, d, W)
        b = oracle.window_stats_map(s, d, W)
        c = oracle.window_stats_sort(s, d, W)
        assert a.tolist() == b.tolist() == c.tolist(), (V, W, n)


# ---------------------------------------------------------------- independent library routes
def scipy_route(s, d):
    """Table 2's matrix notation evaluated with scipy.sparse on one window (no code shared)."""
    import scipy.sparse as sp

    labels, inv = np.unique(np.concatenate([s, d]), return_inverse=True)
    V = labels.size
    A = sp.coo_matrix((np.ones(s.size, np.int64), (inv[: s.size], inv[s.size:])), shape=(V, V)).tocsr()
    A.sum_duplicates()
    nz = A.copy()
    nz.data = np.ones_like(nz.data)
    rs, cs = np.asarray(A.sum(1)).ravel(), np.asarray(A.sum(0)).ravel()
    rn, cn = np.asarray(nz.sum(1)).ravel(), np.asarray(nz.sum(0)).ravel()
    return [int(A.sum()), int(nz.sum()), int(A.max()), int((rs > 0).sum()), int(rs.max()), int(rn.max()),
            int((cs > 0).sum()), int(cs.max()), int(cn.max())]


def pandas_route(s, d):
    """Table 2's dataframe column with the DESIGN.md corrections R3 (fan = distinct neighbours, not
    value_counts on one column) and R8 (unique links = number of rows of drop_duplicates, not .size)."""
    import pandas as pd

    df = pd.DataFrame({"src": s.astype(np.int64), "dst": d.astype(np.int64)})
    links = df.groupby(["src", "dst"]).size()
    return [len(df), len(df[["src", "dst"]].drop_duplicates()), int(links.max()),
            int(df["src"].nunique()), int(df.groupby("src").size().max()), int(df.groupby("src")["dst"].nunique().max()),
            int(df["dst"].nunique()), int(df.groupby("dst").size().max()), int(df.groupby("dst")["src"].nunique().max())]


@pytest.mark.parametrize("cfg", ["uniform", "zipf", "heavy", "zipf-small"])
def test_library_routes_on_full_windows(cfg):
    W = 1 << 17
    dist = {"uniform": gen.Dist("uniform"), "zipf": gen.Dist("zipf", 1.1, 1 << 20), "heavy": gen.Dist("heavy"),
            "zipf-small": gen.Dist("zipf", 1.3, 1 << 10)}[cfg]
    s, d = gen.generate_host(dist, 11, 0, 2 * W + 999)
    o1 = oracle.window_stats_map(s, d, W)
    o2 = oracle.window_stats_sort(s, d, W)
    assert o1.tolist() == o2.tolist()
    for w in range(o2.shape[0]):
        sl = slice(w * W, (w + 1) * W)
        assert o2[w].tolist() == scipy_route(s[sl], d[sl]), w
    assert o2[0].tolist() == pandas_route(s[:W], d[:W])


# ---------------------------------------------------------------- invariants
def check_invariants(row, wlen):
    v, L, mL, uS, mSP, mFO, uD, mDP, mFI = [int(x) for x in row]
    assert v == wlen
    assert 1 <= L <= v and mL >= 1
    assert mFO <= uD and mFI <= uS
    assert mL <= min(mSP, mDP)
    assert mFO <= mSP and mFI <= mDP
    assert max(uS, uD) <= L <= uS * uD
    assert mFO <= L and mFI <= L
    assert -(-v // uS) <= mSP and -(-v // uD) <= mDP          # pigeonhole
    assert -(-L // uS) <= mFO and -(-L // uD) <= mFI
    assert mSP <= v and mDP <= v and mL <= v


@pytest.mark.parametrize("dist", [gen.Dist("uniform"), gen.Dist("zipf", 1.1, 1 << 20), gen.Dist("heavy"),
                                  gen.Dist("zipf", 0.8, 1 << 16), gen.Dist("zipf", 1.5, 1 << 20)])
def test_invariants_on_generated_windows(dist):
    W = 1 << 17
    n = 3 * W + 4321
    s, d = gen.generate_host(dist, 21, 0, n)
    out = oracle.window_stats_sort(s, d, W)
    for w, row in enumerate(out):
        check_invariants(row, min(W, n - w * W))


def test_row_and_column_sums_equal_valid():
    # sum of row sums = sum of column sums = valid packets (north_star invariant), on the dense matrix.
    rng = np.random.default_rng(3)
    s = rng.integers(0, 40, 5000).astype(np.uint32)
    d = rng.integers(0, 40, 5000).astype(np.uint32)
    labels, inv = np.unique(np.concatenate([s, d]), return_inverse=True)
    A = np.zeros((labels.size, labels.size), np.int64)
    np.add.at(A, (inv[:5000], inv[5000:]), 1)
    assert A.sum(1).sum() == A.sum(0).sum() == oracle.window_stats_map(s, d, 5000)[0, 0]


def test_uniform_statistics_sanity():
    # Not a pin: for uniform 32-bit addresses E[unique sources] = W - W^2/2^33 + O(W^3/2^64) = 131070.0
    W = 1 << 17
    s, d = gen.generate_host(gen.Dist("uniform"), 1, 0, 16 * W)
    out = oracle.window_stats_sort(s, d, W)
    assert abs(out[:, 3].astype(float).mean() - (W - W * W / 2 ** 33)) < 2.0
    assert abs(out[:, 6].astype(float).mean() - (W - W * W / 2 ** 33)) < 2.0


# ---------------------------------------------------------------- metamorphic relations
def _lowbias(x):
    x = x.astype(np.uint32)
    x ^= x >> np.uint32(16); x *= np.uint32(0x7FEB352D); x ^= x >> np.uint32(15); x *= np.uint32(0x846CA68B)
    x ^= x >> np.uint32(16)
    return x


@pytest.mark.parametrize("which", ["map", "sort"])
def test_metamorphic(which):
    f = ORACLES[which]
    W = 5000
    s, d = gen.generate_host(gen.Dist("zipf", 1.2, 3000), 8, 0, 3 * W + 17)
    base = f(s, d, W)
    # mirror: swap src and dst columns -> rows 3<->6, 4<->7, 5<->8 swap; 0-2 fixed
    mir = f(d, s, W)
    assert mir[:, [0, 1, 2, 6, 7, 8, 3, 4, 5]].tolist() == base.tolist()
    # relabel through a bijection (anonymisation): unchanged
    assert f(_lowbias(s), _lowbias(d), W).tolist() == base.tolist()
    # packet order inside a window: unchanged
    rng = np.random.default_rng(1)
    s2, d2 = s.copy(), d.copy()
    for w in range(0, s.size, W):
        p = rng.permutation(min(W, s.size - w)) + w
        s2[w:w + p.size], d2[w:w + p.size] = s[p], d[p]
    assert f(s2, d2, W).tolist() == base.tolist()
    # window concatenation: per-window results of a stream = separate runs on each window
    for w in range(base.shape[0]):
        assert f(s[w * W:(w + 1) * W], d[w * W:(w + 1) * W], W).tolist() == [base[w].tolist()]


def test_worker_count_independence():
    s, d = gen.generate_host(gen.Dist("heavy"), 4, 0, 20 * 4096 + 7)
    ref = oracle.window_stats_sort(s, d, 4096, threads=1)
    for t in (2, 3, 8):
        assert oracle.window_stats_sort(s, d, 4096, threads=t).tolist() == ref.tolist()


def test_packed_keys_equivalent():
    s, d = gen.generate_host(gen.Dist("uniform"), 3, 0, 10000)
    keys = gen.pack(s, d)
    assert oracle.window_stats_sort(keys=keys, window=999).tolist() == oracle.window_stats_sort(s, d, 999).tolist()


def test_distinguishes_plausible_mistakes():
    """The pins above must reject the garbled dataframe column literally (DESIGN R3/R8)."""
    window, s, d, exp = load_golden("survey_four_packets.txt")[0]
    row = exp[0].tolist()
    fan_as_packets = row[4]            # df[['src']].value_counts().max() = packets of the busiest source
    assert fan_as_packets != row[5]    # 3 != 2: fan-out is distinct destinations
    size_of_drop_duplicates = 2 * row[1]   # DataFrame.size = rows x 2 columns
    assert size_of_drop_duplicates != row[1]
