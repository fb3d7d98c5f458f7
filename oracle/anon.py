"""oracle/anon.py — TEST INFRASTRUCTURE ONLY.  IP address anonymisation.

Written from the paper's steps, in its order, with numpy (no code shared with the CUDA path):
  1. "unique": U = the distinct addresses of the src and dst columns, ascending (np.unique); N = |U|.
  2. the sequence 0..N-1 and its permutation pi: the shuffle is replaced by the keyed Feistel
     permutation of DESIGN.md reading R15 — per round k < rounds, with key K_k = splitmix64(seed + k): the
     smallest h >= 1 with 2^(2h) >= N (h = ceil(max(2, ceil(log2 N)) / 2)); x -> (L, R) = (x >> h, x & (2^h-1));
     four Feistel rounds (L, R) <- (R, L xor (splitmix64(K_k xor (j << 56) xor R) & (2^h-1))), j = 0..3;
     x <- L << h | R, repeated while x >= N (cycle walking); rounds = 0 is the identity.
  3. the gather: src' = pi[index of src in U], dst' = pi[index of dst in U].
Pinned by tests/test_oracle_anon.py: the hand example for the ranks, N against the union count of O1d,
bijectivity of pi for many N, and the paper's own argument — every Table 2 quantity of the relabelled
stream equals the original's, checked with O2.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(z):
    z = np.asarray(z, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def feistel(x, N: int, key) -> np.ndarray:
    """One keyed permutation of [0, N) applied to the array x (values in [0, N))."""
    x = np.asarray(x, dtype=np.uint64).copy()
    bits = max(2, int(N - 1).bit_length())
    h = (bits + 1) // 2
    mask = np.uint64((1 << h) - 1)
    key = np.uint64(key)
    todo = np.ones(x.shape, dtype=bool)
    with np.errstate(over="ignore"):
        while todo.any():
            v = x[todo]
            L, R = v >> np.uint64(h), v & mask
            for j in range(4):
                t = L ^ (splitmix64(key ^ (np.uint64(j) << np.uint64(56)) ^ R) & mask)
                L, R = R, t
            v = (L << np.uint64(h)) | R
            x[todo] = v
            todo[todo] = v >= np.uint64(N)
    return x


def permutation(r, N: int, seed: int, rounds: int) -> np.ndarray:
    r = np.asarray(r, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for k in range(rounds):
            r = feistel(r, N, splitmix64(np.uint64(seed) + np.uint64(k)))
    return r


def anonymize(src, dst, seed: int = 0, rounds: int = 1):
    """Returns (src' u32 [n], dst' u32 [n], N)."""
    s = np.asarray(src, dtype=np.uint32).ravel()
    d = np.asarray(dst, dtype=np.uint32).ravel()
    U = np.unique(np.concatenate([s, d]))                         # step 1
    N = int(U.size)
    rs = np.searchsorted(U, s).astype(np.uint64)                  # index in U
    rd = np.searchsorted(U, d).astype(np.uint64)
    ps = permutation(rs, N, seed, rounds) if N else rs            # steps 2-3
    pd = permutation(rd, N, seed, rounds) if N else rd
    return ps.astype(np.uint32), pd.astype(np.uint32), N
