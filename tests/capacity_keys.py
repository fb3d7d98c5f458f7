"""Crafted inputs that fill one shared-memory table of the CUDA path to exactly its capacity -1, = and +1.

Every 2^64 key is a legal link (PAPER.md:182 defines A_t over all (src, dst) pairs), so an adversary can
aim a whole window at one link bucket or one node bucket.  The bucket hashes are invertible multiplies,
so the keys are built by inverting them: pick hash values with the bucket's top bits, multiply by the
inverse.  The constants (multipliers, capacities, bucket counts) are read from the kernel sources, so
the inputs follow the kernels if they are retuned; the expected values always come from the oracle.

Capacities:
- round-2 path (nsg_flat.cuh, W <= 2^17): a link bucket holds FILL_L distinct links (beyond that its
  records would not fit the record row); a node bucket's table holds TS distinct nodes (B = W / BK link
  buckets, B / 2 node buckets per side);
- round-1 path (nsg_fast.cuh; NSG_FLAG_LEGACY_FAST, windows 2^17 < W < 2^20, weighted rows): a link bucket holds TCAP
  distinct links, a side bucket TCAP_S distinct nodes.
The key ~0 (both addresses 255.255.255.255) and the node ~0 are kept outside the tables and never count.
"""
import os
import re

import numpy as np

CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2509_03653_b200", "csrc")
M64 = (1 << 64) - 1
M32 = (1 << 32) - 1


def _const(fname, pattern):
    src = open(os.path.join(CSRC, fname)).read()
    m = re.search(pattern, src)
    assert m, f"{pattern!r} not found in {fname}"
    return int(m.group(1), 0)


def flat_params():
    f = "nsg_flat.cuh"
    return {
        "MUL_L": _const(f, r"constexpr u64 MUL_L = (0x[0-9A-Fa-f]+)ull"),
        "MUL_N": _const(f, r"constexpr u32 MUL_N = (0x[0-9A-Fa-f]+)u"),
        "FILL_L": _const(f, r"constexpr u32 FILL_L = (\d+)"),
        "TS": 1 << _const(f, r"constexpr int LOG_TS = (\d+)"),
        "BK": _const(f, r"constexpr u64 BK = (\d+)"),
    }


def legacy_params():
    f = "nsg_fast.cuh"
    return {
        "MUL_L": _const(f, r"const u64 h = k \* (0x[0-9A-Fa-f]+)ull"),
        "MUL_S": _const(f, r"side_bucket\(u32 node, u32 logB\) \{ return logB \? \(node \* (0x[0-9A-Fa-f]+)u\)"),
        "TCAP": _const(f, r"#define NSG_TCAP (\d+)"),
        "TCAP_S": _const(f, r"#define NSG_TCAP_S (\d+)"),
        "BUCKET_KEYS": _const(f, r"#define NSG_BUCKET_KEYS (\d+)"),
    }


def _log2_buckets(window, per_bucket):
    b = 1
    while b * per_bucket < window:
        b *= 2
    return b.bit_length() - 1


def link_bucket(keys, mul, logb):
    """Top logb bits of key * mul (mod 2^64); for the round-1 kmix the xor-shift leaves them unchanged."""
    if logb == 0:
        return np.zeros(len(keys), np.uint64)
    return np.array([((int(k) * mul) & M64) >> (64 - logb) for k in keys], np.uint64)


def node_bucket(nodes, mul, logb):
    if logb == 0:
        return np.zeros(len(nodes), np.uint64)
    return np.array([((int(v) * mul) & M32) >> (32 - logb) for v in nodes], np.uint64)


def keys_in_link_bucket(count, mul, logb, rng):
    """`count` distinct keys, none equal to ~0, whose link bucket is 0."""
    inv = pow(mul, -1, 1 << 64)
    out = set()
    while len(out) < count:
        h = int(rng.integers(0, 1 << (64 - logb), dtype=np.uint64))
        k = (h * inv) & M64
        if k != M64:
            out.add(k)
    return np.array(sorted(out), np.uint64)


def nodes_in_node_bucket(count, mul, logb, rng):
    """`count` distinct nodes, none equal to ~0, whose node bucket is 0."""
    inv = pow(mul, -1, 1 << 32)
    out = set()
    while len(out) < count:
        h = int(rng.integers(0, 1 << (32 - logb)))
        v = (h * inv) & M32
        if v != M32:
            out.add(v)
    return np.array(sorted(out), np.uint64)


def fill_window(distinct, window, rng):
    """A window of `window` packets holding exactly the keys `distinct` (each at least once)."""
    assert len(distinct) <= window
    extra = rng.choice(distinct, window - len(distinct))
    k = np.concatenate([distinct, extra])
    rng.shuffle(k)
    return k


def link_capacity_window(count, window, mul, logb, with_sentinel, seed):
    """One window whose link bucket 0 holds `count` distinct links (plus the key ~0 if asked)."""
    rng = np.random.default_rng(seed)
    d = keys_in_link_bucket(count, mul, logb, rng)
    if with_sentinel:
        d = np.concatenate([d, np.array([M64], np.uint64)])
    return fill_window(d, window, rng)


def node_capacity_window(count, window, mul, logb, with_sentinel, seed, dst=12345):
    """One window whose source bucket 0 holds `count` distinct sources, each sending to `dst` (plus the
    source 255.255.255.255 if asked).  The links are distinct, one per source, spread over the link
    buckets by their own hash."""
    rng = np.random.default_rng(seed)
    src = nodes_in_node_bucket(count, mul, logb, rng)
    if with_sentinel:
        src = np.concatenate([src, np.array([M32], np.uint64)])
    d = (src << np.uint64(32)) | np.uint64(dst)
    return fill_window(d, window, rng)
