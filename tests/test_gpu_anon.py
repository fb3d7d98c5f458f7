"""CUDA anonymisation (nsg_anonymize, through the C ABI) vs the oracle, bit-exact (-m gpu).

SURVEY §8(f) row f2: every relabelled address and N must equal oracle.anonymize's; the
nine statistics of the relabelled stream (CUDA path) must equal the original's (the paper's argument).
"""
import numpy as np
import pytest
import torch

import gen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nsg(cuda_device):
    import paper_2509_03653_b200 as m

    return m


def gpu_anon(nsg, keys, device, layout="packed", **kw):
    kd = torch.from_numpy(np.ascontiguousarray(keys).view(np.int64)).to(device)
    if layout == "packed":
        s, d, nu = nsg.anonymize(kd, **kw)
    else:
        s, d, nu = nsg.anonymize(src=(kd >> 32).to(torch.int32).contiguous(),
                                 dst=(kd & 0xFFFFFFFF).to(torch.int32).contiguous(), **kw)
    torch.cuda.synchronize(device)
    return s.cpu().numpy().view(np.uint32), d.cpu().numpy().view(np.uint32), int(nu.item())


@pytest.mark.parametrize("dist,n", [(gen.Dist("zipf", 1.1, 1 << 20), 1 << 23), (gen.Dist("heavy"), 1 << 20),
                                    (gen.Dist("uniform"), 1 << 20), (gen.Dist("zipf", 1.5, 1 << 6), 1000), (None, 1),
                                    (gen.Dist("uniform"), 1 << 23)])  # the last: N > 2^23, direct ranks (no label table)
@pytest.mark.parametrize("seed,rounds", [(0, 0), (7, 1), (2 ** 64 - 1, 3)])
def test_anonymize_matches_oracle(nsg, cuda_device, dist, n, seed, rounds):
    keys = np.array([0x0A0000010A000002], np.uint64) if dist is None else gen.generate_host(dist, 91, 0, n, packed=True)
    s0, d0 = (keys >> np.uint64(32)).astype(np.uint32), (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    ws, wd, wN = oracle.anonymize(s0, d0, seed=seed, rounds=rounds)
    gs, gd, gN = gpu_anon(nsg, keys, cuda_device, seed=seed, rounds=rounds)
    assert gN == wN
    assert np.array_equal(gs, ws) and np.array_equal(gd, wd)


def test_extreme_addresses_and_soa(nsg, cuda_device):
    rng = np.random.default_rng(3)
    a = np.array([0, 1, 0xFFFFFFFF, 0xFFFFFFFE, 1023, 1024, 1025, 0x80000000], np.uint64)
    keys = (a[rng.integers(0, a.size, 5000)] << np.uint64(32)) | a[rng.integers(0, a.size, 5000)]
    s0, d0 = (keys >> np.uint64(32)).astype(np.uint32), (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    for rounds in (0, 2):
        ws, wd, wN = oracle.anonymize(s0, d0, seed=5, rounds=rounds)
        for layout in ("packed", "soa"):
            gs, gd, gN = gpu_anon(nsg, keys, cuda_device, layout=layout, seed=5, rounds=rounds)
            assert gN == wN and np.array_equal(gs, ws) and np.array_equal(gd, wd)


def test_statistics_invariant_on_gpu(nsg, cuda_device):
    W = 1 << 17
    keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 20), 2, 0, 8 * W, packed=True)
    kd = torch.from_numpy(keys.view(np.int64)).to(cuda_device)
    s, d, _ = nsg.anonymize(kd, seed=11, rounds=2)
    a = nsg.window_stats(s, d, W).cpu()
    b = nsg.window_stats_packed(kd, W).cpu()
    assert torch.equal(a, b)
