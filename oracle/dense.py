"""oracle/dense.py — TEST INFRASTRUCTURE ONLY.  O0: Table 2's "Matrix notation" column evaluated
literally on a dense traffic matrix.

PAPER.md (arXiv 2509.03653) Table 2, defines the scalars on the traffic matrix A_t;
the caption (line 173) adds the destination mirrors by swapping src and dst.  Because every quantity
is invariant under a bijective relabelling of addresses (the paper's own anonymisation argument,
lines 195-203), the window's distinct addresses are relabelled 0..V-1 (np.unique) and A_t is built
as a dense V x V integer matrix by counting packets.  Then, literally:

    valid packets             sum_i sum_j A_t(i,j)          (:180)
    unique links              sum_i sum_j |A_t(i,j)|_0      (:181)
    max link packets          max_ij A_t(i,j)               (:183)
    unique sources            sum_i |sum_j A_t(i,j)|_0      (:184)
    max source packets        max_i sum_j A_t(i,j)          (:186)
    max source fan-out        max_i sum_j |A_t(i,j)|_0      (:188)
    unique destinations / max destination packets / max destination fan-in: the same on A_t^T (:173)

Only for tiny windows (V <= max_vertices).  Empty max = 0 (reading R7).
"""
from __future__ import annotations

import numpy as np


def _one_window(s: np.ndarray, d: np.ndarray, max_vertices: int, wt=None) -> list[int]:
    if s.size == 0:
        return [0] * 9
    labels, inv = np.unique(np.concatenate([s, d]), return_inverse=True)
    V = labels.size
    if V > max_vertices:
        raise ValueError(f"dense oracle is for tiny windows (V={V} > {max_vertices})")
    i, j = inv[: s.size], inv[s.size:]
    A = np.zeros((V, V), dtype=np.int64)
    np.add.at(A, (i, j), 1 if wt is None else wt)   # A_t(i,j) = packets (or summed n_packets) i -> j
    if not A.any():
        return [0] * 9
    nz = (A != 0).astype(np.int64)               # |A_t|_0
    row_sum, col_sum = A.sum(axis=1), A.sum(axis=0)          # A_t 1, 1^T A_t
    row_nnz, col_nnz = nz.sum(axis=1), nz.sum(axis=0)        # |A_t|_0 1, 1^T |A_t|_0
    return [
        int(A.sum()),
        int(nz.sum()),
        int(A.max()),
        int((row_sum != 0).sum()),
        int(row_sum.max()),
        int(row_nnz.max()),
        int((col_sum != 0).sum()),
        int(col_sum.max()),
        int(col_nnz.max()),
    ]


def window_stats_dense(src, dst, window: int, *, max_vertices: int = 256, weights=None) -> np.ndarray:
    """O0 over every window of (src, dst) (optionally weighted rows: A_t sums the weights, PAPER.md:180,
    :207).  Returns uint64 [n_windows, 9]."""
    s = np.asarray(src, dtype=np.int64).ravel()
    d = np.asarray(dst, dtype=np.int64).ravel()
    wt = None if weights is None else np.asarray(weights, dtype=np.int64).ravel()
    if s.shape != d.shape:
        raise ValueError("src and dst must have the same length")
    if window < 1:
        raise ValueError("window must be >= 1")
    n = s.size
    nw = 0 if n == 0 else (n + window - 1) // window
    out = np.zeros((nw, 9), dtype=np.uint64)
    for w in range(nw):
        sl = slice(w * window, (w + 1) * window)
        out[w] = _one_window(s[sl], d[sl], max_vertices, None if wt is None else wt[sl])
    return out


def _one_window_dist(s: np.ndarray, d: np.ndarray, max_vertices: int) -> dict:
    """Dense O0 of the vector-valued rows: A_t's nonzeros in (i, j) order, the row sums A_t 1 (:185) and
    row nnz |A_t|_0 1 (:187) of the nonzero rows, the column mirrors (:173), and the IP sets (:209)
    as index sets of the relabelled addresses."""
    if s.size == 0:
        e64, e32 = np.zeros(0, np.uint64), np.zeros(0, np.uint32)
        return {"link_key": e64, "link_packets": e64, "src_node": e32, "src_packets": e64, "src_fan": e64,
                "dst_node": e32, "dst_packets": e64, "dst_fan": e64, "ip_sets": np.zeros(4, np.uint64)}
    labels, inv = np.unique(np.concatenate([s, d]), return_inverse=True)   # ascending: labels keep key order
    V = labels.size
    if V > max_vertices:
        raise ValueError(f"dense oracle is for tiny windows (V={V} > {max_vertices})")
    i, j = inv[: s.size], inv[s.size:]
    A = np.zeros((V, V), dtype=np.int64)
    np.add.at(A, (i, j), 1)
    nz = (A != 0).astype(np.int64)
    ii, jj = np.nonzero(A)                                   # row-major: ascending (i, j)
    row_sum, col_sum = A.sum(axis=1), A.sum(axis=0)
    row_nnz, col_nnz = nz.sum(axis=1), nz.sum(axis=0)
    rows, cols = np.nonzero(row_sum)[0], np.nonzero(col_sum)[0]
    is_src, is_dst = row_sum != 0, col_sum != 0
    lab = labels.astype(np.uint64)
    return {
        "link_key": (lab[ii] << np.uint64(32)) | lab[jj], "link_packets": A[ii, jj].astype(np.uint64),
        "src_node": labels[rows].astype(np.uint32), "src_packets": row_sum[rows].astype(np.uint64),
        "src_fan": row_nnz[rows].astype(np.uint64),
        "dst_node": labels[cols].astype(np.uint32), "dst_packets": col_sum[cols].astype(np.uint64),
        "dst_fan": col_nnz[cols].astype(np.uint64),
        "ip_sets": np.array([(is_src | is_dst).sum(), (is_src & ~is_dst).sum(), (is_dst & ~is_src).sum(),
                             (is_src & is_dst).sum()], dtype=np.uint64),
    }


def window_distributions_dense(src, dst, window: int, *, max_vertices: int = 256) -> list:
    """O0 of the vector-valued rows for every window: a list of per-window dicts (keys as
    oracle.window_slices returns)."""
    s = np.asarray(src, dtype=np.int64).ravel()
    d = np.asarray(dst, dtype=np.int64).ravel()
    if s.shape != d.shape:
        raise ValueError("src and dst must have the same length")
    if window < 1:
        raise ValueError("window must be >= 1")
    n = s.size
    nw = 0 if n == 0 else (n + window - 1) // window
    return [_one_window_dist(s[w * window:(w + 1) * window], d[w * window:(w + 1) * window], max_vertices)
            for w in range(nw)]
