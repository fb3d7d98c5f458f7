"""Heavy groups of the round-2 link kernel (-m gpu): crafted windows that aim K links of one link bucket at
one node bucket of one side, at the aggregation threshold AGG_T -1, = and +1 and far beyond it, from one
node (a heavy hitter: its links reach the side item as one record per node) and from K distinct nodes (more
than the 128-slot aggregation table holds: the links that find no room send their own records, so one node
bucket's row mixes aggregated and single-link records).

A_t is defined over every (src, dst) pair, so an adversary can aim links at any bucket; the
bucket hashes are invertible multiplies (tests/capacity_keys.py reads their constants from the kernel
source).  Expected values come from the oracle only: the nine statistics (mirrors :173),
and with the vector outputs the per-node packets / fan-out / fan-in (:185, :187) and the IP sets (:209).
"""
import os
import re

import numpy as np
import pytest

import capacity_keys as ck
import oracle
from test_gpu_vectors import assert_vectors, gpu_vectors

pytestmark = pytest.mark.gpu

W = 1 << 17
_SRC = open(os.path.join(ck.CSRC, "nsg_flat.cuh")).read()
AGG_T = int(re.search(r"#define NSG_AGG_T (\d+)", _SRC).group(1))


@pytest.fixture(scope="module")
def nsg(cuda_device):
    import paper_2509_03653_b200 as m

    return m


def _buckets(keys, nodes, p):
    """link bucket of each key (top 7 bits of key * MUL_L), node bucket of each node (top 6 bits of node * MUL_N)."""
    lb = (keys * np.uint64(p["MUL_L"])) >> np.uint64(64 - 7)
    nb = ((nodes.astype(np.uint64) * np.uint64(p["MUL_N"])) & np.uint64(ck.M32)) >> np.uint64(32 - 6)
    return lb, nb


def heavy_group(k, side, distinct, seed, b0=5, q0=9):
    """k distinct links of link bucket b0 whose side-`side` node lies in node bucket q0: all from one node
    (distinct=False) or from k distinct nodes (distinct=True)."""
    p = ck.flat_params()
    rng = np.random.default_rng(seed)
    out = []
    if not distinct:  # one node in q0
        while True:
            node = rng.integers(0, 2 ** 32 - 1, dtype=np.uint64)
            if _buckets(np.zeros(1, np.uint64), np.array([node]), p)[1][0] == q0:
                break
        seen = set()
        while len(out) < k:
            other = rng.integers(0, 2 ** 32 - 1, 1 << 18, dtype=np.uint64)
            keys = (np.uint64(node) << np.uint64(32)) | other if side == 0 else (other << np.uint64(32)) | np.uint64(node)
            lb, _ = _buckets(keys, other, p)
            for x in keys[lb == b0]:
                if int(x) not in seen and len(out) < k:
                    seen.add(int(x))
                    out.append(x)
    else:
        seen = set()
        while len(out) < k:
            a = rng.integers(0, 2 ** 32 - 1, 1 << 22, dtype=np.uint64)
            b = rng.integers(0, 2 ** 32 - 1, 1 << 22, dtype=np.uint64)
            keys = (a << np.uint64(32)) | b
            node = a if side == 0 else b
            lb, nb = _buckets(keys, node, p)
            for x, nd in zip(keys[(lb == b0) & (nb == q0)], node[(lb == b0) & (nb == q0)]):
                if int(nd) not in seen and len(out) < k:
                    seen.add(int(nd))
                    out.append(x)
    return np.array(out, dtype=np.uint64)


def window_with(group, seed, reps=3):
    """One 2^17-packet window: the group's links (each repeated `reps` times, so the packets sums differ
    from the link counts), filler drawn from a pool of 20000 keys (so that the group's link bucket stays
    below its FILL_L distinct links; none of them in that bucket) and the address 255.255.255.255 as source
    and destination."""
    rng = np.random.default_rng(seed + 1000)
    g = np.repeat(group, reps)
    pool = rng.integers(0, 2 ** 64, 20000, dtype=np.uint64)
    pool = pool[_buckets(pool, pool, ck.flat_params())[0] != 5]  # none in the group's link bucket: exactly k links
    filler = pool[rng.integers(0, pool.size, W - g.size - 2)]
    E = np.uint64(0xFFFFFFFF)
    keys = np.concatenate([g, filler, np.array([(E << np.uint64(32)) | np.uint64(7), (np.uint64(7) << np.uint64(32)) | E], np.uint64)])
    rng.shuffle(keys)
    return keys


def check(nsg, device, keys, vectors, heavy_groups):
    import torch

    want = oracle.window_stats_sort(keys=keys, window=W)
    kd = torch.from_numpy(keys.view(np.int64)).to(device)
    ws = nsg.Workspace(kd.numel(), W)
    got = nsg.window_stats_packed(kd, W, workspace=ws).cpu().numpy().view(np.uint64)
    assert got.tolist() == want.tolist()
    assert ws.diag()[0] == 0  # stayed on the shared-memory path
    assert ws.diag()[3] == heavy_groups  # the group's links merged per node (or not, below AGG_T)
    if vectors:
        assert_vectors(gpu_vectors(nsg, keys, W, device), keys, W)


@pytest.mark.parametrize("side", [0, 1])
@pytest.mark.parametrize("k", [AGG_T - 1, AGG_T, AGG_T + 1, 1000])
def test_heavy_hitter_group(nsg, cuda_device, side, k):
    """One node with k links in one (link bucket, node bucket) group: aggregated into one record from
    AGG_T links on."""
    keys = window_with(heavy_group(k, side, distinct=False, seed=k + side), seed=k + side)
    check(nsg, cuda_device, keys, vectors=k in (AGG_T, 1000), heavy_groups=int(k >= AGG_T))


@pytest.mark.parametrize("side", [0, 1])
def test_distinct_nodes_overflow_aggregation_table(nsg, cuda_device, side):
    """600 links from 600 distinct nodes in one group: more nodes than the 128-slot aggregation table."""
    keys = window_with(heavy_group(600, side, distinct=True, seed=77 + side), seed=77 + side, reps=1)
    check(nsg, cuda_device, keys, vectors=True, heavy_groups=1)
