"""Property-based parity of the CUDA path (hypothesis, -m gpu): arbitrary small streams with arbitrary
32-bit addresses (the empty-slot sentinels 0xFFFFFFFF included), arbitrary window lengths, both the fast
path and the forced L2 path, raw and weighted rows, the stats and the IP sets — bit-exact against the oracle.
"""
import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle

pytestmark = pytest.mark.gpu

ADDR = st.one_of(st.integers(0, 5), st.sampled_from([0, 0xFFFFFFFE, 0xFFFFFFFF]), st.integers(0, 2 ** 32 - 1))
SETTINGS = settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow,
                                                                          HealthCheck.function_scoped_fixture])


def _keys(rows):
    s = np.array([r[0] for r in rows], np.uint64)
    d = np.array([r[1] for r in rows], np.uint64)
    return (s << np.uint64(32)) | d


@SETTINGS
@given(st.lists(st.tuples(ADDR, ADDR), min_size=1, max_size=3000), st.integers(1, 5000), st.sampled_from([0, 1]))
def test_stats_and_ip_sets(cuda_device, rows, window, flags):
    import paper_2509_03653_b200 as nsg

    keys = _keys(rows)
    kd = torch.from_numpy(keys.view(np.int64)).to(cuda_device)
    r = nsg.window_vectors(kd, window, links=False, sources=False, destinations=False, flags=flags)
    torch.cuda.synchronize(cuda_device)
    assert r["stats"].cpu().numpy().view(np.uint64).tolist() == oracle.window_stats_map(keys=keys, window=window).tolist()
    want = oracle.window_distributions(keys=keys, window=window)["ip_sets"]
    assert r["ip_sets"].cpu().numpy().view(np.uint64).tolist() == want.tolist()


@SETTINGS
@given(st.lists(st.tuples(ADDR, ADDR, st.integers(0, 9)), min_size=1, max_size=3000), st.integers(1, 5000),
       st.sampled_from([0, 1]))
def test_weighted_rows(cuda_device, rows, window, flags):
    import paper_2509_03653_b200 as nsg

    keys = _keys(rows)
    wt = np.array([r[2] for r in rows], np.uint32)
    kd = torch.from_numpy(keys.view(np.int64)).to(cuda_device)
    wd = torch.from_numpy(wt.view(np.int32)).to(cuda_device)
    got = nsg.window_stats_weighted(kd, wd, window, flags=flags).cpu().numpy().view(np.uint64)
    assert got.tolist() == oracle.window_stats_weighted(keys=keys, weights=wt, window=window).tolist()
