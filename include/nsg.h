/* include/nsg.h — C ABI of libnsg, the B200 (sm_100a) per-window Network Sensing Graph Challenge path.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, arXiv 2509.03653):
 *   The packet stream (src_p, dst_p), p = 0..n-1, is cut into windows of `window` consecutive packets
 *   (window w holds packets [w*window, min((w+1)*window, n)); the last window may be shorter).  For
 *   window w, A_t is the traffic matrix of Table 2 (caption line 173):
 *       A_t(i,j) = number of packets of the window with src = i and dst = j      (raw packets, weight 1)
 *   and the library returns the nine scalars of Table 2 and its destination mirrors, in this column
 *   order (north_star order):
 *       [0] valid packets            1^T A_t 1
 *       [1] unique links             1^T |A_t|_0 1
 *       [2] max link packets         max(A_t)
 *       [3] unique sources           1^T |A_t 1|_0
 *       [4] max source packets       max(A_t 1)
 *       [5] max source fan-out       max(|A_t|_0 1)
 *       [6] unique destinations      mirror of [3]      PAPER.md:173 ("replace src and dst"), :241
 *       [7] max destination packets  mirror of [4]
 *       [8] max destination fan-in   mirror of [5]
 *   Readings of the paper where it is silent or garbled are listed in DESIGN.md ("Readings"): directed
 *   links, self-loops are ordinary entries, every 32-bit address value is a vertex, empty max = 0.
 *
 * Entry points: the nine statistics per window (nsg_window_stats*, raw packets; _weighted for rows
 * with n_packets; _mirrored to store the rows into other tables too); the vector-valued rows and the IP
 * set counts per window (nsg_window_vectors); the whole-trace statistics (nsg_trace_*, one GPU or the
 * steps of a multi-GPU exchange, with nsg_ipc_* buffers for the peer-memory variant); IP anonymisation
 * (nsg_anonymize).  SURVEY.md §8 maps them to the paper.
 *
 * Addresses are IPv4 in host integer order (a.b.c.d <-> a<<24|b<<16|c<<8|d).  The packed form of a
 * packet is the u64 key (src << 32) | dst.
 *
 * Conventions for every entry point:
 *   - Ownership: the caller allocates every buffer; the library never allocates device memory (except
 *     nsg_ipc_alloc, whose purpose is an IPC-exportable buffer) and keeps no pointer after returning.  Device work is ASYNCHRONOUS on `stream` (a cudaStream_t passed as
 *     void*; NULL = legacy default stream): buffers must stay alive and unmodified until the stream
 *     reaches that point.  out[] is only valid once the stream has completed the call.
 *   - Arguments: window >= 1 and window <= NSG_MAX_WINDOW; n_packets == 0 -> NSG_OK with no launch;
 *     NULL data/out/workspace pointers with n_packets > 0 -> NSG_ERR_INVALID_ARGUMENT, nothing launched.
 *     Pointers need only natural alignment (4 B for src/dst, 8 B for keys, 8 B for out, 256 B for the
 *     workspace); wider vector loads are used internally when the data happens to be 16 B aligned.
 *   - Output: out is device memory, row-major [nsg_num_windows(n, window)][NSG_NUM_STATS] u64.
 *   - Errors: argument errors and launch errors are returned synchronously; nothing is launched on an
 *     argument error.  Device-detected inconsistencies (the per-window self-check: the link counts of a
 *     window must sum to its length) are counted in the workspace diagnostics
 *     (nsg_diag_offset); a debug build of the library (-DNSG_DEBUG_CHECKS, libnsg_debug.so) synchronises
 *     `stream` after the nsg_window_stats* calls, reads them back and returns NSG_ERR_INTERNAL if any.  There is no CPU fallback: a device that is not sm_100 returns
 *     NSG_ERR_UNSUPPORTED_DEVICE.
 *   - Thread safety: calls are independent; two concurrent calls must not share a workspace.
 */
#ifndef NSG_H
#define NSG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { NSG_NUM_STATS = 9 };

/* Column index of each statistic in an out row. */
enum nsg_stat {
  NSG_VALID_PACKETS = 0,
  NSG_UNIQUE_LINKS = 1,
  NSG_MAX_LINK_PACKETS = 2,
  NSG_UNIQUE_SOURCES = 3,
  NSG_MAX_SOURCE_PACKETS = 4,
  NSG_MAX_SOURCE_FANOUT = 5,
  NSG_UNIQUE_DESTINATIONS = 6,
  NSG_MAX_DESTINATION_PACKETS = 7,
  NSG_MAX_DESTINATION_FANIN = 8
};

typedef enum {
  NSG_OK = 0,
  NSG_ERR_INVALID_ARGUMENT = 1,
  NSG_ERR_CUDA = 2,
  NSG_ERR_WORKSPACE_TOO_SMALL = 3,
  NSG_ERR_UNSUPPORTED_DEVICE = 4,
  NSG_ERR_INTERNAL = 5
} nsg_status;

/* Largest supported window (per-window counts are kept in 32 bits on the device). */
#define NSG_MAX_WINDOW (1ull << 31)

/* Flags for nsg_window_stats_ex (fault injection for tests; 0 = normal operation).  Measurement and
 * development switches live in nsg_internal.h (not part of the product interface). */
enum {
  NSG_FLAG_FORCE_GLOBAL = 1u << 0,     /* run every window on the L2 (global-table) path */
  NSG_FLAG_INJECT_OVERFLOW = 1u << 1   /* mark every odd window as overflowed on the shared-memory path, so
                                          the overflow hand-off to the L2 path is exercised */
};

/* Number of windows: ceil(n_packets / window); 0 if n_packets == 0 or window == 0. */
uint64_t nsg_num_windows(uint64_t n_packets, uint64_t window);

/* Device scratch (bytes) the caller must pass as `workspace` for (n_packets, window); 0 when
 * n_packets == 0.  Depends only on (n_packets, window) and the device's SM count. */
size_t nsg_workspace_bytes(uint64_t n_packets, uint64_t window);

/* SoA input: src[n_packets], dst[n_packets] device u32 arrays. */
nsg_status nsg_window_stats(const uint32_t* src, const uint32_t* dst, uint64_t n_packets, uint64_t window,
                            uint64_t* out, void* workspace, size_t workspace_bytes, void* stream);

/* Packed input: keys[n_packets] device u64 array, keys[p] = (u64)src_p << 32 | dst_p. */
nsg_status nsg_window_stats_packed(const uint64_t* keys, uint64_t n_packets, uint64_t window, uint64_t* out,
                                   void* workspace, size_t workspace_bytes, void* stream);

/* Either input form (exactly one of keys / (src,dst) non-NULL) plus test flags. */
nsg_status nsg_window_stats_ex(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n_packets,
                               uint64_t window, uint64_t* out, void* workspace, size_t workspace_bytes,
                               void* stream, uint32_t flags);

/* End-to-end call on HOST input, overlapping the host->device copy with the computation (PAPER.md
 * line 173: the per-window statistics of Table 2, as nsg_window_stats_packed).
 *   keys_host     host u64[n_packets] (packed as in nsg_window_stats_packed); must be page-locked
 *                 (cudaHostAlloc / cudaHostRegister) for the copies to be asynchronous; 8 B aligned.
 *   keys_dev      device u64[n_packets] staging buffer the library copies the input into.
 *   out           device u64[nsg_num_windows][9] result; out_host: optional (NULL: skipped) page-locked
 *                 host copy of it, written by a D2H copy on `stream` after the computation.
 *   copy_stream   a second stream (cudaStream_t as void*, != stream) for the host->device copies.
 *   chunk_windows windows per copy chunk (0: default 8; 8-16 measured best on the C2 batch).
 * The keys are copied in chunks on copy_stream, each followed by a stream write of a per-chunk
 * arrival flag in `workspace`; the persistent kernel is launched on `stream` at once and each of its
 * partition items waits for its chunk's flag, so the computation proceeds under the copies.  Before
 * the call returns, `stream` is made to wait for copy_stream's copies (keys_dev is complete once the
 * call's work on `stream` is).  Asynchronous like the other entry points: host buffers must stay alive
 * and unmodified until `stream` has completed the call.  Errors as nsg_window_stats_packed, plus
 * NSG_ERR_INVALID_ARGUMENT for a NULL keys_host / keys_dev / out / copy_stream or copy_stream == stream,
 * and NSG_ERR_CUDA if the driver's stream-memory-operation entry point is unavailable. */
nsg_status nsg_window_stats_from_host(const uint64_t* keys_host, uint64_t n_packets, uint64_t window,
                                      uint64_t* keys_dev, uint64_t* out, uint64_t* out_host, void* workspace,
                                      size_t workspace_bytes, void* stream, void* copy_stream, uint32_t chunk_windows);

/* nsg_window_stats_ex whose result rows are also stored, by the kernels' epilogues, into n_mirrors >= 1
 * further tables: row w goes to mirrors[j] + (mirror_row0 + w) * NSG_NUM_STATS for every j.  mirrors is a
 * device array of device pointers (8 B aligned) valid in this process — in the multi-GPU driver
 * (distributed.py, transport "p2p") the CUDA-IPC-mapped result tables of every rank, so the all-gather of
 * the 72 B/window results is done by the stores themselves over peer memory instead of a collective.
 * Rows of windows recomputed by the L2 path are rewritten there later in stream order. */
nsg_status nsg_window_stats_mirrored(const uint32_t* src, const uint32_t* dst, const uint64_t* keys,
                                     uint64_t n_packets, uint64_t window, uint64_t* out, void* workspace,
                                     size_t workspace_bytes, void* stream, uint32_t flags, uint64_t* const* mirrors,
                                     uint32_t n_mirrors, uint64_t mirror_row0);

/* Weighted rows: the paper's three-column frame src, dst, n_packets
 * (PAPER.md:207).  Row p adds its weight n_packets[p] to A_t(src_p, dst_p), so valid packets is the sum
 * of n_packets and a link is a nonzero of A_t: a row of weight 0 adds
 * nothing (R14).  Windows are cut by ROW index (window w = rows [w*window, ...)).  Raw packets
 * are the case n_packets = 1 (nsg_window_stats*).
 *   n_packets  device u32[n_rows], 4 B aligned; the input rows as for nsg_window_stats_ex (exactly one
 *              of keys / (src, dst)).
 * Per window the weights must sum to < 2^32 (32-bit device counters); a window that does not is counted
 * in diag[2] (nsg_diag_offset) and its row is unspecified.  Same workspace size, conventions and errors
 * as nsg_window_stats_ex, plus NSG_ERR_INVALID_ARGUMENT for a NULL or misaligned n_packets. */
nsg_status nsg_window_stats_weighted(const uint32_t* src, const uint32_t* dst, const uint64_t* keys,
                                     const uint32_t* n_packets, uint64_t n_rows, uint64_t window, uint64_t* out,
                                     void* workspace, size_t workspace_bytes, void* stream, uint32_t flags);

/* Optional per-window vector outputs of nsg_window_vectors.
 *   links        the nonzeros of A_t: key (src<<32 | dst) and A_t(src,dst)
 *                ("Link packets from i to j")
 *   sources      per source i with a nonzero row: i, (A_t 1)_i (packets from source i)
 *                and (|A_t|_0 1)_i (source fan-out from i)
 *   destinations the column mirrors (1^T A_t)_j and (1^T |A_t|_0)_j
 *   ip_sets      [n_windows][4] u64: |S u D|, |S \ D|, |D \ S|, |S n D| with S / D the window's source /
 *                destination address sets ("Globally unique IP addresses"; R13)
 * Every vector array is device memory with n_packets elements: window w's entries are at
 * [w*window, w*window + count), count = out[w][NSG_UNIQUE_LINKS] (links), out[w][NSG_UNIQUE_SOURCES]
 * (sources) or out[w][NSG_UNIQUE_DESTINATIONS] (destinations); elements past count are unspecified.
 * The ORDER of the entries inside a window is unspecified (hash order; it may differ between runs).
 * A group is requested by non-NULL pointers: link_key and link_packets together; src_node,
 * src_packets and src_fanout together; dst_* together; ip_sets alone.  Alignment: 8 B for link_key and
 * ip_sets, 4 B for the rest; a half-specified group or a misaligned array is NSG_ERR_INVALID_ARGUMENT. */
typedef struct {
  uint64_t* link_key;
  uint32_t* link_packets;
  uint32_t* src_node;
  uint32_t* src_packets;
  uint32_t* src_fanout;
  uint32_t* dst_node;
  uint32_t* dst_packets;
  uint32_t* dst_fanin;
  uint64_t* ip_sets;
} nsg_vectors;

/* nsg_window_stats_ex plus the vector outputs requested in `*vectors` (not NULL; every member may be
 * NULL).  out[][9] is written as by nsg_window_stats_ex.  Same conventions (asynchronous on `stream`,
 * caller-owned buffers, same workspace size); the arrays of *vectors are read when the call is made. */
nsg_status nsg_window_vectors(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n_packets,
                              uint64_t window, uint64_t* out, const nsg_vectors* vectors, void* workspace,
                              size_t workspace_bytes, void* stream, uint32_t flags);

/* ---- Whole-trace path ------------------------------------------------
 * Table 2 on the traffic matrix of the WHOLE input, A = sum over t of A_t (the paper's
 * frame holds the whole capture), i.e. the nine statistics with window = n_packets, but with HBM-resident
 * hash tables filled by every SM, so the input may be far larger than a window.  Per-link and per-node
 * sums are kept in 32 bits (n_packets < 2^32 per call).  The work is split into steps so that a multi-GPU
 * driver can exchange data between them (paper_2509_03653_b200/distributed.py, NCCL all-to-all):
 *   1. nsg_trace_partition: group this rank's keys by the rank that owns their link.
 *   2. (all-to-all of the keys)  nsg_trace_links: aggregate the owned links -> link_stats u64[3] =
 *      {valid packets (sum of A), unique links, max link packets} and one record
 *      (node << 32 | A(i,j)) per link and side, grouped by the node's owner rank.
 *   3. (all-to-all of the records)  nsg_trace_nodes, once per side: node_stats u64[3] = {unique nodes,
 *      max packets, max fan} (PAPER.md:184, :186, :188; the destination mirrors, :173).
 *   4. (sum / max over ranks).
 * Owners: link (key) -> top bits of a 64-bit mix of the key times world; node -> a 32-bit mix.  Every
 * pointer is device memory, 8 B aligned; all calls are asynchronous on `stream`; the workspace (256 B
 * aligned, nsg_trace_workspace_bytes) may be reused by the next step once this one is enqueued (steps on
 * one stream are ordered).  Capacities: n <= key_capacity keys per links call, m <= record_capacity
 * records per nodes call, 1 <= world <= 1024, fewer than 2^32 keys per links call (per-link and per-node
 * sums are 32-bit); violations are NSG_ERR_INVALID_ARGUMENT.  Weighted rows: the caller keeps the total
 * n_packets of a trace below 2^32 (the sums are not checked for wrap-around). */
size_t nsg_trace_workspace_bytes(uint64_t key_capacity, uint64_t record_capacity, uint32_t world);

/* send_keys u64[n] (device): the keys grouped by owner rank, rank o's segment at the exclusive prefix
 * of send_counts; send_counts u64[world] (device).  Input as nsg_window_stats_ex (keys or src/dst). */
nsg_status nsg_trace_partition(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n,
                               uint32_t world, uint64_t* send_keys, uint64_t* send_counts, void* workspace,
                               size_t workspace_bytes, uint64_t key_capacity, uint64_t record_capacity, void* stream);

/* link_stats u64[3]; rec_src, rec_dst u64[n] (at most one record per distinct link and side), grouped by
 * owner rank at the exclusive prefix of rec_counts[0][*] / rec_counts[1][*]; rec_counts u64[2][world]. */
nsg_status nsg_trace_links(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n, uint32_t world,
                           uint64_t* link_stats, uint64_t* rec_src, uint64_t* rec_dst, uint64_t* rec_counts,
                           void* workspace, size_t workspace_bytes, uint64_t key_capacity, uint64_t record_capacity,
                           void* stream);

/* node_stats u64[3] from m records (node << 32 | packets), each record one link of the node. */
nsg_status nsg_trace_nodes(const uint64_t* records, uint64_t m, uint64_t* node_stats, void* workspace,
                           size_t workspace_bytes, uint64_t key_capacity, uint64_t record_capacity, void* stream);

/* ---- Fused exchange over peer memory (one process per GPU, CUDA IPC) --------------------------------
 * The all-to-all steps above can skip the collective: the scatter kernels store every key / record
 * straight into the owner rank's receive buffer through a peer mapping (NVLink P2P on a multi-GPU node),
 * so the transfer overlaps the partition / emission tile by tile.  The driver (distributed.py) all-gathers
 * the per-owner counts first to place each rank's segment, and synchronises (stream + barrier) before an
 * owner reads its buffer.
 *   nsg_ipc_alloc   cudaMalloc `bytes` and export it: *dev_ptr, handle_out = nsg_ipc_handle_bytes() host
 *                   bytes to send to the peers; nsg_ipc_free releases it.  (The only entry points that
 *                   allocate device memory: the receive buffers must be IPC-exportable allocations.)
 *   nsg_ipc_open    map a peer's buffer from its handle (same node; the same GPU works too); nsg_ipc_close.
 *   nsg_trace_owner_counts     counts u64[world] (device): keys per link owner (as nsg_trace_partition).
 *   nsg_trace_partition_peers  scatter the keys: owner o's segment to peers[o] + peer_base[o] (peers: device
 *                              array of `world` device pointers valid in this process; peer_base: device
 *                              u64[world], in elements).
 *   nsg_trace_links_count      nsg_trace_links without the emission: link_stats u64[3], rec_counts
 *                              u64[2][world]; the table stays in the workspace for ...
 *   nsg_trace_links_emit_peers the records of the table left by nsg_trace_links_count (same workspace and
 *                              capacities, nothing in between on it), side s's owner-o segment to
 *                              peers_s[o] + base_s[o]. */
size_t nsg_ipc_handle_bytes(void);
nsg_status nsg_ipc_alloc(size_t bytes, void** dev_ptr, void* handle_out);
nsg_status nsg_ipc_open(const void* handle, void** dev_ptr);
nsg_status nsg_ipc_close(void* dev_ptr);
nsg_status nsg_ipc_free(void* dev_ptr);
nsg_status nsg_trace_owner_counts(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n,
                                  uint32_t world, uint64_t* counts, void* workspace, size_t workspace_bytes,
                                  uint64_t key_capacity, uint64_t record_capacity, void* stream);
nsg_status nsg_trace_partition_peers(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n,
                                     uint32_t world, uint64_t* const* peers, const uint64_t* peer_base,
                                     void* workspace, size_t workspace_bytes, uint64_t key_capacity,
                                     uint64_t record_capacity, void* stream);
nsg_status nsg_trace_links_count(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n,
                                 uint32_t world, uint64_t* link_stats, uint64_t* rec_counts, void* workspace,
                                 size_t workspace_bytes, uint64_t key_capacity, uint64_t record_capacity, void* stream);
nsg_status nsg_trace_links_emit_peers(uint32_t world, uint64_t* const* peers_src, uint64_t* const* peers_dst,
                                      const uint64_t* base_src, const uint64_t* base_dst, void* workspace,
                                      size_t workspace_bytes, uint64_t key_capacity, uint64_t record_capacity,
                                      void* stream);

/* One GPU: the nine whole-trace statistics into out u64[9] (device), north_star column order; the steps
 * above with world = 1 and no host synchronisation.  Workspace: nsg_trace_stats_workspace_bytes(n).
 * n_packets >= 2^32 is NSG_ERR_INVALID_ARGUMENT (32-bit per-link / per-node sums). */
size_t nsg_trace_stats_workspace_bytes(uint64_t n_packets);
nsg_status nsg_trace_stats(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n_packets,
                           uint64_t* out, void* workspace, size_t workspace_bytes, void* stream);

/* ---- IP address anonymisation ------------------------------
 * For the whole input: U = the distinct addresses of src and dst in ascending order, N = |U| (PAPER.md:199,
 * "the number of unique value of src and dest ids"); rank(a) = index of a in U; pi = a keyed pseudo-random
 * permutation of [0, N) standing for the paper's shuffle of 0..N-1 (reading R15:
 * per round k < rounds a 4-round Feistel network on the smallest even-bit domain >= N, keyed by
 * splitmix64(seed + k), cycle-walked into [0, N); rounds = 0 is the identity, i.e. labels = ranks); then
 * the gather: src_out[p] = pi(rank(src_p)), dst_out[p] = pi(rank(dst_p)).  Every Table 2
 * quantity of the relabelled stream equals the original's (the paper's anonymisation argument).
 *   src_out, dst_out  device u32[n_packets]; n_unique device u64[1] (N).  Input as nsg_window_stats_ex.
 *   workspace         device, 256 B aligned, nsg_anonymize_workspace_bytes() (a 2^32-bit bitmap of which only
 *                     the 128-bit groups holding input addresses are touched, a 4 MiB summary of those groups,
 *                     rank prefixes); contents on entry are irrelevant (the summary is zeroed by each call).
 * Asynchronous on `stream`; errors as nsg_window_stats_ex. */
size_t nsg_anonymize_workspace_bytes(void);
nsg_status nsg_anonymize(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n_packets,
                         uint64_t seed, uint32_t rounds, uint32_t* src_out, uint32_t* dst_out, uint64_t* n_unique,
                         void* workspace, size_t workspace_bytes, void* stream);

/* nsg_window_vectors on weighted rows (src, dst, n_packets) as nsg_window_stats_weighted: link packets,
 * source / destination packets are sums of n_packets; rows of weight 0 add nothing. */
nsg_status nsg_window_vectors_weighted(const uint32_t* src, const uint32_t* dst, const uint64_t* keys,
                                       const uint32_t* n_packets, uint64_t n_rows, uint64_t window, uint64_t* out,
                                       const nsg_vectors* vectors, void* workspace, size_t workspace_bytes,
                                       void* stream, uint32_t flags);

/* nsg_trace_stats on weighted rows (src, dst, n_packets; device u32 n_packets[n_rows], 4 B aligned): the
 * whole-trace statistics with A(i,j) = summed n_packets (as nsg_window_stats_weighted, one window = the
 * whole input); per-link and per-node sums must stay below 2^32.  Same workspace size as nsg_trace_stats. */
nsg_status nsg_trace_stats_weighted(const uint32_t* src, const uint32_t* dst, const uint64_t* keys,
                                    const uint32_t* n_packets, uint64_t n_rows, uint64_t* out, void* workspace,
                                    size_t workspace_bytes, void* stream);

/* Diagnostics of the last call that used `workspace` (device memory; read it after the stream has
 * completed the call): byte offset inside the workspace of a u32[4] =
 *   {windows the fast path handed to the L2 path because an SMEM table would overflow,
 *    windows whose self-check failed (sum of link counts != window length, or != the sum of n_packets;
 *    0 unless there is a bug), weighted windows whose n_packets sum to >= 2^32 (unsupported),
 *    heavy groups: (link bucket, node bucket) pairs of the windows <= 2^17 path whose links were merged into
 *    one record per node (heavy hitters; performance information, results are exact either way)}. */
size_t nsg_diag_offset(void);

/* Number of kernels the calling host thread's most recent nsg_window_stats* call launched. */
unsigned nsg_last_launches(void);

/* Human-readable name of a status code (static storage). */
const char* nsg_status_string(nsg_status s);

/* Library build identification (static storage), e.g. "libnsg sm_100a <date>". */
const char* nsg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* NSG_H */
