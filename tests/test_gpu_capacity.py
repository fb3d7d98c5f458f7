"""Genuine shared-memory table overflow (-m gpu): crafted windows that fill one link bucket or one node
bucket to its capacity -1, = and +1 (tests/capacity_keys.py), with 255.255.255.255 present.

At -1 and = the window stays on the shared-memory path (diag[0] = 0 windows handed over); at +1 it is
handed to the L2 path (diag[0] = 1).  In every case the nine statistics equal the oracle's (PAPER.md
:180-188, destination mirrors :173) bit-exactly; the node-bucket cases also request the vector outputs
and the IP sets (:209) — for the round-1 kernel, whose side-0 node lists need one entry beyond a full
table for the address ~0, and for the round-2 kernels.
"""
import numpy as np
import pytest
import torch

import capacity_keys as ck
import oracle

pytestmark = pytest.mark.gpu

W = 1 << 17
LEGACY_FAST = 16


@pytest.fixture(scope="module")
def nsg(cuda_device):
    import paper_2509_03653_b200 as m

    return m


def run_stats(nsg, keys, device, flags=0):
    kd = torch.from_numpy(keys.view(np.int64)).to(device)
    ws = nsg.Workspace(kd.numel(), W)
    got = nsg.window_stats_packed(kd, W, workspace=ws, flags=flags).cpu().numpy().view(np.uint64)
    return got, ws.diag()


def check(nsg, device, keys, cap_exceeded, flags=0):
    want = oracle.window_stats_sort(keys=keys, window=W)
    got, diag = run_stats(nsg, keys, device, flags)
    assert got.tolist() == want.tolist()
    assert diag[0] == (1 if cap_exceeded else 0), diag
    assert diag[1] == 0, diag


@pytest.mark.parametrize("delta", [-1, 0, 1])
def test_flat_link_bucket_capacity(nsg, cuda_device, delta):
    p = ck.flat_params()
    logb = ck._log2_buckets(W, p["BK"])
    keys = ck.link_capacity_window(p["FILL_L"] + delta, W, p["MUL_L"], logb, True, seed=100 + delta)
    check(nsg, cuda_device, keys, delta > 0)


@pytest.mark.parametrize("delta", [-1, 0, 1])
def test_flat_node_bucket_capacity(nsg, cuda_device, delta):
    p = ck.flat_params()
    logb = ck._log2_buckets(W, p["BK"]) - 1  # node buckets: half as many as link buckets
    keys = ck.node_capacity_window(p["TS"] + delta, W, p["MUL_N"], logb, True, seed=200 + delta)
    check(nsg, cuda_device, keys, delta > 0)


@pytest.mark.parametrize("delta", [-1, 0, 1])
def test_legacy_link_bucket_capacity(nsg, cuda_device, delta):
    p = ck.legacy_params()
    logb = ck._log2_buckets(W, p["BUCKET_KEYS"])
    keys = ck.link_capacity_window(p["TCAP"] + delta, W, p["MUL_L"], logb, True, seed=300 + delta)
    check(nsg, cuda_device, keys, delta > 0, flags=LEGACY_FAST)


@pytest.mark.parametrize("delta", [-1, 0, 1])
def test_legacy_side_bucket_capacity_with_ip_sets(nsg, cuda_device, delta):
    p = ck.legacy_params()
    logb = ck._log2_buckets(W, p["TCAP_S"] // 2)
    keys = ck.node_capacity_window(p["TCAP_S"] + delta, W, p["MUL_S"], logb, True, seed=400 + delta)
    check(nsg, cuda_device, keys, delta > 0, flags=LEGACY_FAST)
    # the vector path of the same kernel, with node lists and IP sets requested
    check_vectors(nsg, cuda_device, keys, delta > 0, flags=LEGACY_FAST)


@pytest.mark.parametrize("delta", [-1, 0, 1])
def test_flat_node_bucket_capacity_with_vectors(nsg, cuda_device, delta):
    p = ck.flat_params()
    logb = ck._log2_buckets(W, p["BK"]) - 1  # node buckets: half as many as link buckets
    keys = ck.node_capacity_window(p["TS"] + delta, W, p["MUL_N"], logb, True, seed=500 + delta)
    check(nsg, cuda_device, keys, delta > 0)
    check_vectors(nsg, cuda_device, keys, delta > 0)


def check_vectors(nsg, cuda_device, keys, cap_exceeded, flags=0):
    kd = torch.from_numpy(keys.view(np.int64)).to(cuda_device)
    ws = nsg.Workspace(kd.numel(), W)
    r = nsg.window_vectors(kd, W, workspace=ws, flags=flags)
    torch.cuda.synchronize(cuda_device)
    want = oracle.window_distributions(keys=keys, window=W)
    stats = oracle.window_stats_sort(keys=keys, window=W)
    assert r["stats"].cpu().numpy().view(np.uint64).tolist() == stats.tolist()
    assert r["ip_sets"].cpu().numpy().tolist() == want["ip_sets"].tolist()
    ns = int(stats[0, 3])
    got_src = np.sort(r["src_node"][:ns].cpu().numpy().view(np.uint32).astype(np.uint64))
    assert np.array_equal(got_src, np.sort(want["src_node"][:ns].astype(np.uint64)))
    assert ws.diag()[0] == (1 if cap_exceeded else 0)
