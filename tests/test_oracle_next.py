"""Pins of the distributions / IP-set oracle (O1d, oracle.window_distributions) to things other than
itself (-m "not gpu"): SURVEY §8(f) rows f1 (the vector-valued rows of Table 2: link packets
PAPER.md:182, packets from source :185, source fan-out :187, destination mirrors :173) and f3 (globally
unique IPs :209, all four set counts SPEC.md:239-245).

Pins: hand-counted worked examples (tests/golden/dist_examples.txt, SPEC.md:128/:216/:229/:243 and the
SURVEY four-packet table), closed forms, the dense-matrix brute force O0 on random tiny windows, the
independent sort-based scalar oracle O2 (every scalar of Table 2 is a reduction of a vector), an
independent library route (scipy.sparse + numpy set algebra) on full 2^17 windows, and the mirror /
relabel relations.  A swapped axis, a fan counted as packets, a dropped duplicate or a set-difference
taken the wrong way round fails at least one of them.
"""
import numpy as np
import pytest

import gen
import oracle
from nsg_testutil import load_golden_dist

KEYS = ("link_key", "link_packets", "src_node", "src_packets", "src_fan", "dst_node", "dst_packets", "dst_fan",
        "ip_sets")


def _eq(a: dict, b: dict, ctx=""):
    for k in KEYS:
        assert np.asarray(a[k]).astype(np.uint64).tolist() == np.asarray(b[k]).astype(np.uint64).tolist(), (ctx, k)


def o1d(s, d, W, threads=0):
    r = oracle.window_distributions(s, d, W, threads=threads)
    return [oracle.window_slices(r, W, w) for w in range(r["counts"].shape[0])], r


# ---------------------------------------------------------------- worked examples
def test_golden_examples_map_and_dense():
    for window, s, d, exp in load_golden_dist("dist_examples.txt"):
        got, _ = o1d(s, d, window)
        assert len(got) == 1
        _eq(got[0], exp, (window, s.tolist()))
        _eq(oracle.window_distributions_dense(s, d, window)[0], exp, "dense")


def test_golden_concatenated_stream():
    # the two 3-packet examples as one stream of two windows of 3
    cases = [c for c in load_golden_dist("dist_examples.txt") if c[0] == 3]
    s = np.concatenate([c[1] for c in cases])
    d = np.concatenate([c[2] for c in cases])
    got, _ = o1d(s, d, 3)
    for g, c in zip(got, cases):
        _eq(g, c[3])


# ---------------------------------------------------------------- closed forms
@pytest.mark.parametrize("W", [1, 2, 7, 300])
def test_closed_forms(W):
    i = np.arange(W, dtype=np.uint32)
    # star out: one source a to W distinct destinations
    a = np.uint32(0xFFFFFFF0)
    got, _ = o1d(np.full(W, a, np.uint32), i, W)
    g = got[0]
    assert g["link_packets"].tolist() == [1] * W
    assert g["src_node"].tolist() == [int(a)] and g["src_packets"].tolist() == [W] and g["src_fan"].tolist() == [W]
    assert g["dst_node"].tolist() == i.tolist() and g["dst_packets"].tolist() == [1] * W
    assert g["dst_fan"].tolist() == [1] * W
    assert g["ip_sets"].tolist() == [W + 1, 1, W, 0]
    # star in (the mirror)
    got, _ = o1d(i, np.full(W, a, np.uint32), W)
    g = got[0]
    assert g["src_node"].tolist() == i.tolist() and g["src_fan"].tolist() == [1] * W
    assert g["dst_packets"].tolist() == [W] and g["dst_fan"].tolist() == [W]
    assert g["ip_sets"].tolist() == [W + 1, W, 1, 0]
    # self-loop: one address, one link carrying every packet, on both sides
    got, _ = o1d(np.full(W, 9, np.uint32), np.full(W, 9, np.uint32), W)
    g = got[0]
    assert g["link_key"].tolist() == [(9 << 32) | 9] and g["link_packets"].tolist() == [W]
    assert g["src_packets"].tolist() == [W] and g["src_fan"].tolist() == [1]
    assert g["dst_packets"].tolist() == [W] and g["dst_fan"].tolist() == [1]
    assert g["ip_sets"].tolist() == [1, 0, 0, 1]


@pytest.mark.parametrize("sdr", [(1, 1, 1), (2, 3, 1), (3, 2, 4), (5, 7, 3)])
def test_complete_bipartite(sdr):
    """s sources x d destinations (disjoint), each pair r times: every link r, every source (d*r, d),
    every destination (s*r, s), IP sets (s+d, s, d, 0)."""
    S, D, r = sdr
    src = np.repeat(np.arange(S, dtype=np.uint32) + 100, D * r)
    dst = np.tile(np.repeat(np.arange(D, dtype=np.uint32) + 7000, r), S)
    perm = np.random.default_rng(S * 7 + D).permutation(src.size)
    W = S * D * r
    g = o1d(src[perm], dst[perm], W)[0][0]
    assert g["link_packets"].tolist() == [r] * (S * D)
    assert g["src_packets"].tolist() == [D * r] * S and g["src_fan"].tolist() == [D] * S
    assert g["dst_packets"].tolist() == [S * r] * D and g["dst_fan"].tolist() == [S] * D
    assert g["ip_sets"].tolist() == [S + D, S, D, 0]


def test_empty_input():
    e = np.zeros(0, np.uint32)
    r = oracle.window_distributions(e, e, 5)
    assert r["counts"].shape == (0, 3) and r["ip_sets"].shape == (0, 4)


# ---------------------------------------------------------------- brute force (dense matrix)
@pytest.mark.parametrize("seed", range(3))
def test_bruteforce_dense(seed):
    rng = np.random.default_rng(7000 + seed)
    for _ in range(300):
        V = int(rng.integers(1, 65))
        W = int(rng.integers(1, 400))
        n = int(rng.integers(1, 3 * W + 2))
        if rng.random() < 0.5:
            p = rng.zipf(1.5, size=V).astype(float)
            p /= p.sum()
            s, d = rng.choice(V, n, p=p), rng.choice(V, n, p=p[::-1])
        else:
            s, d = rng.integers(0, V, n), rng.integers(0, V, n)
        labels = rng.choice(2 ** 32, size=V, replace=False).astype(np.uint64)
        s, d = labels[s].astype(np.uint32), labels[d].astype(np.uint32)
        got, _ = o1d(s, d, W)
        want = oracle.window_distributions_dense(s, d, W)
        assert len(got) == len(want)
        for w, (g, x) in enumerate(zip(got, want)):
            _eq(g, x, (V, W, n, w))


# ---------------------------------------------------------------- against the independent scalar oracle O2
@pytest.mark.parametrize("dist", [gen.Dist("uniform"), gen.Dist("zipf", 1.1, 1 << 20), gen.Dist("heavy")])
def test_reductions_equal_scalar_oracle(dist):
    """Every Table 2 scalar is a reduction of a vector row: counts = unique links / sources / destinations,
    max = max link / source packets / fan-out (and mirrors); sum of link packets = sum of row sums = sum of
    column sums = valid; sum of fan-outs = sum of fan-ins = unique links.  O2 (std::sort) shares no code."""
    W = 1 << 16
    s, d = gen.generate_host(dist, 31, 0, 2 * W + 777)
    stats = oracle.window_stats_sort(s, d, W)
    got, r = o1d(s, d, W)
    assert r["counts"].tolist() == stats[:, [1, 3, 6]].tolist()
    for w, g in enumerate(got):
        v, L, mL, uS, mSP, mFO, uD, mDP, mFI = (int(x) for x in stats[w])
        assert int(g["link_packets"].sum()) == v == int(g["src_packets"].sum()) == int(g["dst_packets"].sum())
        assert int(g["src_fan"].sum()) == L == int(g["dst_fan"].sum())
        assert int(g["link_packets"].max()) == mL
        assert (int(g["src_packets"].max()), int(g["src_fan"].max())) == (mSP, mFO)
        assert (int(g["dst_packets"].max()), int(g["dst_fan"].max())) == (mDP, mFI)
        # ascending key order, no repeats
        for k in ("link_key", "src_node", "dst_node"):
            assert np.all(np.diff(g[k].astype(np.int64)) > 0), k
        u, so, do, b = (int(x) for x in g["ip_sets"])
        assert u == so + do + b and so + b == uS and do + b == uD


# ---------------------------------------------------------------- independent library route
def library_route(s, d):
    """scipy.sparse for the vectors (relabel -> COO -> sum_duplicates) and numpy set algebra for the IPs."""
    import scipy.sparse as sp

    labels, inv = np.unique(np.concatenate([s, d]), return_inverse=True)
    V = labels.size
    A = sp.coo_matrix((np.ones(s.size, np.int64), (inv[: s.size], inv[s.size:])), shape=(V, V)).tocsr()
    A.sum_duplicates()
    A.sort_indices()
    coo = A.tocoo()
    nz = A.copy()
    nz.data = np.ones_like(nz.data)
    rs, cs = np.asarray(A.sum(1)).ravel(), np.asarray(A.sum(0)).ravel()
    rn, cn = np.asarray(nz.sum(1)).ravel(), np.asarray(nz.sum(0)).ravel()
    rows, cols = np.nonzero(rs)[0], np.nonzero(cs)[0]
    lab = labels.astype(np.uint64)
    S, D = np.unique(s), np.unique(d)
    both = np.intersect1d(S, D).size
    return {"link_key": (lab[coo.row] << np.uint64(32)) | lab[coo.col], "link_packets": coo.data,
            "src_node": labels[rows], "src_packets": rs[rows], "src_fan": rn[rows],
            "dst_node": labels[cols], "dst_packets": cs[cols], "dst_fan": cn[cols],
            "ip_sets": [np.union1d(S, D).size, np.setdiff1d(S, D).size, np.setdiff1d(D, S).size, both]}


@pytest.mark.parametrize("cfg", ["uniform", "zipf", "heavy", "zipf-small"])
def test_library_route_on_full_windows(cfg):
    W = 1 << 17
    dist = {"uniform": gen.Dist("uniform"), "zipf": gen.Dist("zipf", 1.1, 1 << 20), "heavy": gen.Dist("heavy"),
            "zipf-small": gen.Dist("zipf", 1.3, 1 << 10)}[cfg]
    s, d = gen.generate_host(dist, 12, 0, W + 4099)
    got, _ = o1d(s, d, W)
    for w, g in enumerate(got):
        sl = slice(w * W, (w + 1) * W)
        _eq(g, library_route(s[sl], d[sl]), (cfg, w))


# ---------------------------------------------------------------- metamorphic relations
def _lowbias(x):
    x = x.astype(np.uint32)
    x ^= x >> np.uint32(16); x *= np.uint32(0x7FEB352D); x ^= x >> np.uint32(15); x *= np.uint32(0x846CA68B)
    x ^= x >> np.uint32(16)
    return x


def test_mirror_and_relabel():
    W = 3000
    s, d = gen.generate_host(gen.Dist("zipf", 1.2, 2000), 9, 0, 2 * W + 5)
    base, _ = o1d(s, d, W)
    mir, _ = o1d(d, s, W)
    for b, m in zip(base, mir):
        # swapping the columns transposes A_t: source and destination vectors swap,
        # links are transposed, src-only and dst-only swap
        for a, c in (("src", "dst"), ("dst", "src")):
            for f in ("node", "packets", "fan"):
                assert m[f"{a}_{f}"].tolist() == b[f"{c}_{f}"].tolist()
        t = ((b["link_key"] & np.uint64(0xFFFFFFFF)) << np.uint64(32)) | (b["link_key"] >> np.uint64(32))
        o = np.argsort(t)
        assert m["link_key"].tolist() == t[o].tolist() and m["link_packets"].tolist() == b["link_packets"][o].tolist()
        assert m["ip_sets"].tolist() == b["ip_sets"][[0, 2, 1, 3]].tolist()
    # relabel through a bijection (the anonymisation argument): every vector is the
    # correspondingly permuted vector, the IP set counts are unchanged
    rel, _ = o1d(_lowbias(s), _lowbias(d), W)
    for b, x in zip(base, rel):
        for side in ("src", "dst"):
            m = dict(zip(_lowbias(b[f"{side}_node"]).tolist(), zip(b[f"{side}_packets"].tolist(), b[f"{side}_fan"].tolist())))
            assert dict(zip(x[f"{side}_node"].tolist(), zip(x[f"{side}_packets"].tolist(), x[f"{side}_fan"].tolist()))) == m
        assert x["ip_sets"].tolist() == b["ip_sets"].tolist()


def test_worker_count_independence():
    s, d = gen.generate_host(gen.Dist("heavy"), 4, 0, 9 * 2048 + 3)
    _, ref = o1d(s, d, 2048, threads=1)
    for t in (2, 5):
        _, r = o1d(s, d, 2048, threads=t)
        for k in ref:
            assert r[k].tolist() == ref[k].tolist(), k
