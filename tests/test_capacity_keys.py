"""The crafted capacity windows (tests/capacity_keys.py) put exactly the intended number of distinct
links / nodes in bucket 0 of the kernels' hashes, keep ~0 outside, and fill the whole window (CPU)."""
import numpy as np
import pytest

import capacity_keys as ck

W = 1 << 17


def _params():
    f, g = ck.flat_params(), ck.legacy_params()
    return [("flat", f["MUL_L"], f["MUL_N"], ck._log2_buckets(W, f["BK"]), ck._log2_buckets(W, f["BK"]), f["FILL_L"],
             f["TS"]),
            ("legacy", g["MUL_L"], g["MUL_S"], ck._log2_buckets(W, g["BUCKET_KEYS"]),
             ck._log2_buckets(W, g["TCAP_S"] // 2), g["TCAP"], g["TCAP_S"])]


def test_constants_parsed():
    f, g = ck.flat_params(), ck.legacy_params()
    assert f["MUL_L"] % 2 == 1 and f["MUL_N"] % 2 == 1 and g["MUL_L"] % 2 == 1 and g["MUL_S"] % 2 == 1
    assert ck._log2_buckets(W, f["BK"]) == 7 and ck._log2_buckets(W, g["BUCKET_KEYS"]) == 5
    assert f["FILL_L"] < f["TS"] * 2 and g["TCAP"] >= g["BUCKET_KEYS"]


@pytest.mark.parametrize("path,mul_l,mul_n,logb,logbs,cap_l,cap_n", _params())
@pytest.mark.parametrize("delta", [-1, 0, 1])
def test_link_window(path, mul_l, mul_n, logb, logbs, cap_l, cap_n, delta):
    k = ck.link_capacity_window(cap_l + delta, W, mul_l, logb, True, seed=1)
    assert k.shape == (W,)
    u = np.unique(k)
    assert np.uint64(ck.M64) in u
    inner = u[u != np.uint64(ck.M64)]
    assert inner.size == cap_l + delta
    assert np.all(ck.link_bucket(inner, mul_l, logb) == 0)


@pytest.mark.parametrize("path,mul_l,mul_n,logb,logbs,cap_l,cap_n", _params())
@pytest.mark.parametrize("delta", [-1, 0, 1])
def test_node_window(path, mul_l, mul_n, logb, logbs, cap_l, cap_n, delta):
    k = ck.node_capacity_window(cap_n + delta, W, mul_n, logbs, True, seed=2)
    src = np.unique(k >> np.uint64(32))
    assert np.uint64(ck.M32) in src
    inner = src[src != np.uint64(ck.M32)]
    assert inner.size == cap_n + delta
    assert np.all(ck.node_bucket(inner, mul_n, logbs) == 0)
    assert np.unique(k).size == cap_n + delta + 1  # one link per source
