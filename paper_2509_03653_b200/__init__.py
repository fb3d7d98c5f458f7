"""paper_2509_03653_b200 — B200-native per-window Network Sensing Graph Challenge statistics.

For each window of N_V = 2^17 packets, the traffic matrix A_t (a group-by-count over (src, dst) IPv4
pairs; arXiv 2509.03653 Table 2) is reduced to nine integers: valid packets, unique
links, max link packets, unique sources, max source packets, max source fan-out, unique
destinations, max destination packets, max destination fan-in.  ``window_vectors`` adds the vector-valued
rows of Table 2 (link packets, per-source packets / fan-out and the destination mirrors) and the four
globally-unique-IP set counts per window.

The computation runs in libnsg.so (hand-written sm_100a CUDA behind the C ABI in include/nsg.h);
this package is its thin binding plus the window-sharded multi-GPU driver.
"""
from .api import (  # noqa: F401
    DEFAULT_WINDOW,
    FLAG_FORCE_GLOBAL,
    FLAG_INJECT_OVERFLOW,
    IP_SET_NAMES,
    NUM_STATS,
    STAT_NAMES,
    TraceWorkspace,
    Workspace,
    anonymize,
    last_launches,
    num_windows,
    trace_links,
    trace_links_count,
    trace_links_emit_peers,
    trace_nodes,
    trace_owner_counts,
    trace_partition,
    trace_partition_peers,
    trace_stats,
    version,
    window_stats,
    window_stats_from_host,
    window_stats_mirrored,
    window_stats_packed,
    window_stats_weighted,
    window_vectors,
    workspace_bytes,
)
from ._lib import NsgError  # noqa: F401
