// nsg_fast.cuh — the fast path of libnsg: one persistent kernel, three kinds of work item per window.
//
// Window w (packets [w*W, min((w+1)*W, n))) is processed as
//   P(w,c)      c < cp   : a CH-key chunk is read from HBM once (128-bit streaming loads), counting-
//                          sorted in SMEM by link bucket b = top logB bits of kmix(key) and written
//                          to the window's L2-resident scratch slot, with its bucket offsets.
//   L(w,b)      b < B    : the keys of link bucket b (about W/B of them) are gathered from every chunk
//                          and aggregated in an SMEM hash table key -> count: this is A_t restricted to
//                          the bucket ("Link packets from i to j").  One scan gives the
//                          bucket's unique links (:181), max link packets (:183) and sum of counts
//                          (:180), and emits one record per link and side, node<<32 | count, into
//                          side buckets sb = top logB bits of node*0x9E3779B1.
//   S(w,side,sb)         : all records of side bucket sb (from every link bucket) are merged in an SMEM
//                          table node -> (sum of counts, number of records): the row sums A_t 1 (:185)
//                          and row nnz |A_t|_0 1 (:187) of those sources (or the column mirrors, :173).
//                          A scan gives unique nodes (:184), max packets (:186), max fan (:188).
//   F(w)                 : reduces the per-bucket partials of window w to the nine outputs.
// Items are handed out by one global ticket counter in steps of up to 1 + 2B2 + B + cp tickets:
// step k = F(k-LAG_F), S(k-LAG_S), L(k-LAG_L), P(k) (classes whose window is out of range take no
// ticket).  Every item
// waits only on items with smaller tickets, so the schedule cannot deadlock; a scratch slot is reused
// once its previous window is final (RSLOTS windows in flight).  Dependencies are counted
// semaphores: __syncthreads() + red.release.gpu by one thread to signal, ld.acquire.gpu spin by one
// thread + __syncthreads() to wait.
// Options of the same kernel (Geo): weighted rows (fast_kernel<true>: P and L items carry n_packets per
// key), vector outputs (L items append each link, S items each node; S1 items count |S n D| from the
// S0 item's node list), result mirrors (F writes its row into further tables, e.g. peer ranks').
#pragma once
#include "nsg_internal.h"
#include "nsg_common.cuh"

namespace nsg {

#ifndef NSG_FT
#define NSG_FT 512
#endif
#ifndef NSG_TCAP
#define NSG_TCAP 8192
#endif
#ifndef NSG_BUCKET_KEYS
#define NSG_BUCKET_KEYS 4096
#endif
#ifndef NSG_PCAP
#define NSG_PCAP 512
#endif
constexpr int FT = NSG_FT;                   // threads per CTA (default 512: 2 CTAs per SM)
constexpr int NWARP = FT / 32;
constexpr int KPT = 8;                       // elements per thread per round
constexpr int CH = FT * KPT;                 // 4096 keys per chunk / per gather round
constexpr int TCAP = NSG_TCAP;               // link-table slots (slot = (h * TCAP) >> 32)
#ifndef NSG_TCAP_S
#define NSG_TCAP_S 8192
#endif
#ifndef NSG_PCAP_S
#define NSG_PCAP_S 512
#endif
#ifndef NSG_LOG_FAST_WINDOW
#define NSG_LOG_FAST_WINDOW 20
#endif
constexpr int TCAP_S = NSG_TCAP_S;           // node-table slots of a side item
constexpr u32 S0LIST = TCAP_S + 1;           // a side-0 node list: a full table plus the address ~0
constexpr int NODE_BUCKET = TCAP_S / 2;      // side buckets are sized for <= 4096 nodes (load <= 1/2)
constexpr int PCAP_S = NSG_PCAP_S;           // side items' pending-list capacity
constexpr int BUCKET_KEYS = NSG_BUCKET_KEYS; // target keys per link bucket (table load factor <= 1/2)
constexpr int PCAP = NSG_PCAP;               // pending-list capacity (entries) per insertion wave
constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c(x >> 1); }
constexpr int MAX_LOGB = NSG_LOG_FAST_WINDOW - ilog2c(BUCKET_KEYS);  // B * BUCKET_KEYS <= 2^LOG_FAST_WINDOW
constexpr int MAXB = 1 << MAX_LOGB;
constexpr int MAXB2 = (1 << NSG_LOG_FAST_WINDOW) / NODE_BUCKET;  // side buckets for the largest fast window
constexpr u64 FAST_MAX_WINDOW = ((u64)BUCKET_KEYS << MAX_LOGB) - 1;  // 2^20 - 1: P fits a record's 20 bits
constexpr int MAXCP = (int)((FAST_MAX_WINDOW + CH) / CH);
// A link record: node << 32 | F << 20 | P (F = links merged into it, P = their packets; a window on
// the fast path has < 2^20 packets so P always fits, and F is split over several records if > 4095).
constexpr u32 REC_PBITS = 20, REC_FMAX = 4095;
__host__ __device__ __forceinline__ u64 make_rec(u32 node, u32 f, u32 p) {
  return ((u64)node << 32) | ((u64)f << REC_PBITS) | p;
}
static_assert(TCAP % FT == 0 && TCAP_S % FT == 0, "emission / vector loops are warp-uniform");
constexpr int LAG_L = 8, LAG_S = 20, LAG_F = 26;  // pipeline lags (steps) of L, S, F items behind P (measured plateau)
constexpr int LOG_RSLOTS = 5;
constexpr int RSLOTS = 1 << LOG_RSLOTS;      // scratch slots (windows in flight), > LAG_S
constexpr u32 RCAP = (2 * (TCAP + 1) + 15) & ~15u;  // records per link bucket (both sides); x8 B = whole 128-B lines



constexpr int MAX_REG = 10;  // ticket regions: <= 7 between the breakpoints 0, LAG_*, nw + LAG_*, +2 drain splits
static_assert(RSLOTS > LAG_F && LAG_F > LAG_S && LAG_S > LAG_L && LAG_L >= 1, "schedule lags");

struct Geo {
  u64 n, W, nw;
  u32 logB, B, cp, cp_last, R;
  u32 logB2, B2;    // side buckets per side: ceil(W / NODE_BUCKET) rounded up to a power of two
  // Ticket regions: steps [reg_k0[r], reg_k0[r+1]) all hold the same item classes (reg_mask bits:
  // 1 F, 2 S, 4 L, 8 P), reg_ips[r] tickets each, starting at ticket reg_t0[r].  Steps with a class
  // out of range (before its lag, or past the last window) simply have fewer tickets: no no-op items.
  u32 nreg;
  u32 reg_ips[MAX_REG], reg_mask[MAX_REG];
  u64 reg_k0[MAX_REG], reg_t0[MAX_REG + 1];
  u64 total_items;
  u32 flags;
  u64* ticket;
  u32* diag;
  u64* prof;  // [3 item types][4] = {count, cycles, wait cycles, -} when NSG_FLAG_PROFILE
  u32 *pdone, *ldone, *sdone, *fin, *ovf;
  const u32* arrived;  // streamed input (nsg_window_stats_from_host): arrived[w / chunk_w] != 0 once the
  u32 chunk_w;         // chunk holding window w has been copied to the device; NULL: input resident
  u64* kscr;  // [R][cp*CH]      keys, chunk-major, each chunk sorted by link bucket
  u32* koff;  // [R][cp][B+1]    bucket offsets inside each chunk
  u64* rscr;  // [R][B][RCAP]    link records of each link bucket, sorted by (side, side bucket)
  u32* roff;  // [R][B][2B+1]    start offsets of (side, side bucket) inside each link bucket's records
  u32* rend;  // [R][B][2B]      end offsets (records are aggregated per node, so segments may be short)
  u32* lres;  // [R][B][4]       per link bucket: unique links, max count, sum of counts
  u32* sres;  // [R][2][B][4]    per side bucket: unique nodes, max packets, max fan, |S n D| (side 1)
  // Optional vector outputs (nsg_window_vectors); NULL = not requested.  Window
  // w's entries go to [w*W, w*W + count) of each array, in hash order.
  u64* v_lkey; u32* v_lpk;                   // links: key, A_t(i,j)
  u32* v_node[2]; u32* v_pk[2]; u32* v_fan[2];  // per side: node, packets, fan              (:185, :187, :173)
  u64* v_ipsets;                             // [nw][4] |S u D|, |S \ D|, |D \ S|, |S n D|   (:209)
  u32* vfill;   // [nw][3] fill counters of the link / source / destination vectors
  u32* s0list;  // [R][B2][S0LIST] node list of each side-0 item (read by the side-1 item of the bucket)
  u32* s0cnt;   // [R][B2]
  u32* s0win;   // [R][B2]         w+1 once side item S0(w, sb) has published its list (release)
  // Weighted rows (nsg_window_stats_weighted): n_packets per row, or NULL.
  const u32* wgt;
  // Result mirrors (nsg_window_stats_mirrored): every row is also stored at mirror[j] + (row0 + w) * 9,
  // e.g. the IPC-mapped result tables of every rank (the multi-GPU gather done by the epilogue itself).
  u64* const* mirror;
  u32 n_mirror;
  u64 mirror_row0;
  u32* wscr;    // [R][cp*CH]      the weights, laid out like kscr
};

struct SmemP { u64 stage[CH]; u32 hist[MAXB + 1]; u32 stagew[CH]; };  // stagew: weighted rows only
// Per-warp gather tables: warp w gathers segments w, w + NWARP, ... (chunks for L, link buckets for S).
constexpr int WSEG_L = (MAXCP + NWARP - 1) / NWARP;
constexpr int WSEG_S = (MAXB + NWARP - 1) / NWARP;
static_assert(WSEG_L <= 32 && WSEG_S <= 32, "one segment per lane");
// Pending lists are SoA: a = the key (link item) or node<<32 | F<<20 | P (side item), p = next probe.
struct SmemL {
  u64 lkey[TCAP]; u32 lcnt[TCAP]; u64 pa[2][PCAP]; u16 pp[2][PCAP]; u32 wlo[NWARP][WSEG_L]; u32 wpre[NWARP][WSEG_L + 1];
  u32 hist[2 * MAXB2 + 1];
};
// The weighted-rows link item carries a weight per pending entry; its pending lists are half as long so
// that the CTA still fits two per SM.
constexpr int PCAP_W = NSG_PCAP / 2;
struct SmemLW {
  u64 lkey[TCAP]; u32 lcnt[TCAP]; u64 pa[2][PCAP_W]; u16 pp[2][PCAP_W]; u32 pw[2][PCAP_W]; u32 wlo[NWARP][WSEG_L];
  u32 wpre[NWARP][WSEG_L + 1];
  u32 hist[2 * MAXB2 + 1];
};
struct SmemS {
  u32 key[TCAP_S]; u32 P[TCAP_S]; u32 F[TCAP_S]; u64 pa[2][PCAP_S]; u16 pp[2][PCAP_S]; u32 wlo[NWARP][WSEG_S];
  u32 wpre[NWARP][WSEG_S + 1];
};
struct SmemMisc {
  u32 wtmp[10 * NWARP];
  u32 esc[4];  // [0] link-table escape count (key ~0); [1],[2] node-table escape P, F (node ~0)
  u32 flag, dep;
  u32 type, idx;
  u32 pcnt[2];  // pending-list fill counters
  u32 hot[2];   // link item: per side, a side bucket holding >= 8x the average records (or ~0u)
  u32 vbase, vcnt;  // vector outputs: the item's base inside its window's region, its fill counter
  u32 n0, both;     // side-1 item with IP sets: entries in S0's node list, nodes found on both sides
  u64 w;
  unsigned long long wsum;  // weighted link item: sum of the bucket's weights
};
constexpr size_t cmax(size_t a, size_t b) { return a > b ? a : b; }
constexpr size_t MISC_BYTES = (sizeof(SmemMisc) + 15) & ~size_t(15);
constexpr size_t FAST_SMEM = MISC_BYTES + cmax(cmax(sizeof(SmemP), sizeof(SmemLW)), cmax(sizeof(SmemL), sizeof(SmemS)));

// ------------------------------------------------------------------------------------------
// Block helpers
// ------------------------------------------------------------------------------------------
// In-place exclusive scan of a[0..n) by the whole CTA; afterwards a[n] = total.
__device__ void block_exclusive_scan(u32* a, int n, u32* wtmp) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int per = (n + FT - 1) / FT;
  const int b = min(t * per, n), e = min(b + per, n);
  u32 s = 0;
  for (int i = b; i < e; ++i) s += a[i];
  u32 x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wtmp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    u32 v = lane < NWARP ? wtmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    if (lane < NWARP) wtmp[lane] = v;
  }
  __syncthreads();
  u32 run = x - s + (wid ? wtmp[wid - 1] : 0);
  for (int i = b; i < e; ++i) {
    const u32 v = a[i];
    a[i] = run;
    run += v;
  }
  if (t == 0) a[n] = wtmp[NWARP - 1];
  __syncthreads();
}

// Exclusive scan of a[0..n) in place by warp 0 (a[n] = total).  The caller brackets it with
// __syncthreads(); n is small (chunks, buckets), so one warp beats a 3-barrier block scan.
__device__ __forceinline__ void warp0_exclusive_scan(u32* a, int n) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const int per = (n + 31) >> 5;
  const int b = min(lane * per, n), e = min(b + per, n);
  u32 sum = 0;
  for (int i = b; i < e; ++i) sum += a[i];
  u32 x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  u32 run = x - sum;
  for (int i = b; i < e; ++i) {
    const u32 v = a[i];
    a[i] = run;
    run += v;
  }
  if (lane == 31) a[n] = x;
}

// Largest c in [0, n) with pre[c] <= i (pre is an exclusive prefix with pre[n] > i).
__device__ __forceinline__ u32 find_seg(const u32* pre, u32 n, u32 i) {
  u32 lo = 0, hi = n - 1;
  while (lo < hi) {
    const u32 mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= i) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// ------------------------------------------------------------------------------------------
// SMEM hash tables, filled in dense "waves".  A claimed slot never changes key.  SMEM atomics
// cost per warp-instruction, so a per-lane probe loop (whose later iterations run with a few lanes
// active) is avoided: in wave 0 every entry tries its home slot with one full-warp CAS; entries
// that find another key there are appended (warp-aggregated) to a compact pending list, and the
// pending list is retried densely at the next probe position, wave after wave.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ u32 home_slot(u32 h) { return (u32)(((u64)h * (u64)TCAP) >> 32); }
__device__ __forceinline__ u32 probe_slot(u32 home, u32 probe) {
  const u32 x = home + probe;  // probe < TCAP
  return x >= (u32)TCAP ? x - TCAP : x;
}
__device__ __forceinline__ u32 probe_slot_s(u32 home, u32 probe) {
  const u32 x = home + probe;  // probe < TCAP_S (a power of two)
  return x & (TCAP_S - 1);
}
// Cheap multiplicative mixes (one multiply each; hashes only steer performance, never results):
// kmix's top bits pick the link bucket and its low 32 bits (which fold in the product's high half)
// the home slot; side buckets take the top bits of node * 0x9E3779B1 and node homes the top bits of
// an independent multiplier.
__device__ __forceinline__ u64 kmix(u64 k) {
  const u64 h = k * 0x9E3779B97F4A7C15ull;
  return h ^ (h >> 29);
}
__device__ __forceinline__ u32 link_home(u64 key) { return home_slot((u32)kmix(key)); }
__device__ __forceinline__ u32 node_home(u32 node) { return (u32)(((u64)(node * 0x85EBCA77u) * (u64)TCAP_S) >> 32); }

// one attempt: true if the key now owns `slot` (inserted or already there) and was counted
__device__ __forceinline__ bool link_try(u64* lkey, u32* lcnt, u64 key, u32 add, u32 slot) {
  const u64 old = atomicCAS(reinterpret_cast<unsigned long long*>(&lkey[slot]), EMPTY64, key);
  if (old == EMPTY64 || old == key) { atomicAdd(&lcnt[slot], add); return true; }
  return false;
}
__device__ __forceinline__ bool node_try(u32* key, u32* P, u32* F, u32 node, u32 p, u32 f, u32 slot) {
  const u32 old = atomicCAS(&key[slot], EMPTY32, node);
  if (old == EMPTY32 || old == node) {
    atomicAdd(&P[slot], p);
    if (f) atomicAdd(&F[slot], f);
    return true;
  }
  return false;
}
// rare path (pending list full): finish the probe sequence in this lane; false if the table is full
__device__ __noinline__ bool link_finish(u64* lkey, u32* lcnt, u64 key, u32 add, u32 probe) {
  const u32 home = link_home(key);
  for (; probe < (u32)TCAP; ++probe)
    if (link_try(lkey, lcnt, key, add, probe_slot(home, probe))) return true;
  return false;
}
__device__ __noinline__ bool node_finish(u32* key, u32* P, u32* F, u32 node, u32 p, u32 f, u32 probe) {
  const u32 home = node_home(node);
  for (; probe < (u32)TCAP_S; ++probe)
    if (node_try(key, P, F, node, p, f, probe_slot_s(home, probe))) return true;
  return false;
}

// merge a cached (node, P, F) aggregate into the node table (one lane); nothing if it saw no record
__device__ __noinline__ bool node_flush(u32* key, u32* P, u32* F, u32* esc, u32 node, u32 p, u32 f) {
  if (f == 0) return true;
  if (node == EMPTY32) { atomicAdd(&esc[1], p); atomicAdd(&esc[2], f); return true; }
  return node_finish(key, P, F, node, p, f, 0u);
}

// Warp-aggregated append of the lanes with `want` to pending list `list`; must be called by all
// lanes of the warp.  Returns false for a lane whose entry did not fit (the caller finishes it).
__device__ __forceinline__ bool pend_push(u64* la, u16* lp, u32* cnt, bool want, u64 a, u32 probe, u32 cap,
                                          u32* lw = nullptr, u32 wt = 0) {
  const u32 mask = __ballot_sync(0xffffffffu, want);
  if (mask == 0) return true;
  const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
  u32 base = 0;
  if (lane == leader) base = atomicAdd(cnt, (u32)__popc(mask));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (!want) return true;
  const u32 pos = base + __popc(mask & ((1u << lane) - 1u));
  if (pos >= cap) return false;
  la[pos] = a;
  lp[pos] = (u16)probe;
  if (lw) lw[pos] = wt;
  return true;
}

__device__ __forceinline__ u32 side_bucket(u32 node, u32 logB) { return logB ? (node * 0x9E3779B1u) >> (32 - logB) : 0u; }
__device__ __forceinline__ u32 link_bucket(u64 key, u32 logB) { return logB ? (u32)(kmix(key) >> (64 - logB)) : 0u; }

__device__ __forceinline__ void mark_overflow(const Geo& g, u64 w) {
  if (atomicExch(&g.ovf[w], 1u) == 0u) atomicAdd(&g.diag[0], 1u);
}

__device__ __forceinline__ u32 chunks_of(const Geo& g, u64 w) { return w + 1 == g.nw ? g.cp_last : g.cp; }
__device__ __forceinline__ u64 window_len(const Geo& g, u64 w) { return min(g.W, g.n - w * g.W); }
__device__ __forceinline__ u32 slot_of(const Geo& g, u64 w) { return (u32)w & (g.R - 1); }

// Spin (acquire) until *p >= v, starting from a first value `first` loaded earlier with
// ld_acquire32 so that its latency overlapped other work.
__device__ __forceinline__ long long wait_geq(const u32* p, u32 v, u32 first) {
  if (first >= v) return 0;
  const long long t0 = clock64();
  while (ld_acquire32(p) < v) __nanosleep(32);
  return clock64() - t0;
}

#ifdef NSG_PROFILE_BUILD
constexpr bool kProfile = true;
#else
constexpr bool kProfile = false;
#endif
#ifdef NSG_PROFILE_BUILD
// Phase timer (NSG_FLAG_PROFILE): thread 0 adds the cycles since the previous mark to
// prof[16 + type*16 + phase].  Marks are placed right after a __syncthreads().
// profiling: after the first wave, add the number of entries that wanted the pending list to
// prof[16 + 16*type + 12] and its max to prof[64 + 16*type + 12]
__device__ __forceinline__ void prof_pending(const Geo& g, int type, u32 n) {
  if ((g.flags & NSG_FLAG_PROFILE) && threadIdx.x == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&g.prof[16 + type * 16 + 12]), (unsigned long long)n);
    atomicMax(reinterpret_cast<unsigned long long*>(&g.prof[64 + type * 16 + 12]), (unsigned long long)n);
  }
}

struct PhaseTimer {
  long long last;
  __device__ __forceinline__ PhaseTimer() { last = clock64(); }
  __device__ __forceinline__ void mark(const Geo& g, int type, int phase) {
    if ((g.flags & NSG_FLAG_PROFILE) && threadIdx.x == 0) {
      const long long now = clock64();
      atomicAdd(reinterpret_cast<unsigned long long*>(&g.prof[16 + type * 16 + phase]), (unsigned long long)(now - last));
      atomicMax(reinterpret_cast<unsigned long long*>(&g.prof[64 + type * 16 + phase]), (unsigned long long)(now - last));
      last = now;
    }
  }
};

__device__ __forceinline__ void prof_add(const Geo& g, int type, long long cyc, long long wait) {
  if (g.flags & NSG_FLAG_PROFILE) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&g.prof[type * 4 + 0]), 1ull);
    atomicAdd(reinterpret_cast<unsigned long long*>(&g.prof[type * 4 + 1]), (unsigned long long)cyc);
    atomicAdd(reinterpret_cast<unsigned long long*>(&g.prof[type * 4 + 2]), (unsigned long long)wait);
    atomicMax(reinterpret_cast<unsigned long long*>(&g.prof[type * 4 + 3]), (unsigned long long)(cyc - wait));
  }
}
#else  // production build: no profiling code in the kernel
__device__ __forceinline__ void prof_pending(const Geo&, int, u32) {}
struct PhaseTimer {
  __device__ __forceinline__ void mark(const Geo&, int, int) {}
};
__device__ __forceinline__ void prof_add(const Geo&, int, long long, long long) {}
#endif

// ------------------------------------------------------------------------------------------
// P item: partition one chunk of window w by link bucket
// ------------------------------------------------------------------------------------------
// The scheduler thread's claim of the next ticket.  Items call now() late in their body (before their
// last phase), so that the claim's round trip overlaps that phase but a claimed ticket is not held for
// a whole item (which would delay the items on the critical path at the end of a launch).
constexpr int SCHED_THREAD = 32;
struct Claim {
  u64 tk;
  bool done;
  __device__ __forceinline__ void now(const Geo& g) {
    if (threadIdx.x == SCHED_THREAD && !done) {
      tk = atomicAdd(reinterpret_cast<unsigned long long*>(g.ticket), 1ull);
      done = true;
    }
  }
};

template <bool WT>
__device__ void item_partition(const Geo& g, const u32* __restrict__ src, const u32* __restrict__ dst,
                               const u64* __restrict__ keys, u64 w, u32 c, SmemP& s, SmemMisc& m, Claim& cl) {
  const int t = threadIdx.x;
  PhaseTimer pt;
  const long long tstart = clock64();
  long long waited = 0;
  if (g.arrived) {  // streamed input: wait until the copy engine has delivered this window's chunk
    if (t == 0) {
      const u32* f = &g.arrived[w / g.chunk_w];
      if (ld_acquire_sys32(f) == 0) {
        const long long t0 = clock64();
        while (ld_acquire_sys32(f) == 0) __nanosleep(128);
        waited += clock64() - t0;
      }
    }
    __syncthreads();
  }
  u32 dep = 1;
  if (t == 0 && w >= g.R) dep = ld_acquire32(&g.fin[w - g.R]);  // the slot's previous window is final
  for (int i = t; i <= (int)g.B; i += FT) s.hist[i] = 0;
  const u64 wbase = w * g.W;
  const u64 wlen = min(g.W, g.n - wbase);
  const u64 base = wbase + (u64)c * CH;
  const u32 len = (u32)min((u64)CH, wlen - (u64)c * CH);
  const u32 slot = slot_of(g, w);

  // Full chunks with 16 B aligned bases use 128-bit loads (key order inside the chunk is irrelevant);
  // otherwise element j of thread t is t + j*FT.
  const bool full = len == CH;
  u64 k[KPT];
  if (keys) {
    const u64* p = keys + base;
    if (full && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
      const ulonglong2* p2 = reinterpret_cast<const ulonglong2*>(p);
#pragma unroll
      for (int j = 0; j < KPT / 2; ++j) {
        const ulonglong2 v = __ldcs(p2 + t + j * FT);
        k[2 * j] = v.x; k[2 * j + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < KPT; ++j) k[j] = (t + j * FT < (int)len) ? __ldcs(p + t + j * FT) : 0ull;
    }
  } else {
    const u32* ps = src + base;
    const u32* pd = dst + base;
    if (full && ((reinterpret_cast<uintptr_t>(ps) & 15) == 0) && ((reinterpret_cast<uintptr_t>(pd) & 15) == 0)) {
      const uint4* s4 = reinterpret_cast<const uint4*>(ps);
      const uint4* d4 = reinterpret_cast<const uint4*>(pd);
#pragma unroll
      for (int j = 0; j < KPT / 4; ++j) {
        const uint4 a = __ldcs(s4 + t + j * FT);
        const uint4 b = __ldcs(d4 + t + j * FT);
        k[4 * j + 0] = ((u64)a.x << 32) | b.x;
        k[4 * j + 1] = ((u64)a.y << 32) | b.y;
        k[4 * j + 2] = ((u64)a.z << 32) | b.z;
        k[4 * j + 3] = ((u64)a.w << 32) | b.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < KPT; ++j)
        k[j] = (t + j * FT < (int)len) ? (((u64)__ldcs(ps + t + j * FT) << 32) | __ldcs(pd + t + j * FT)) : 0ull;
    }
  }
  // Weighted rows: the weight of each element (same element order as the key loads above); a row of
  // weight 0 is not an element (it adds nothing to A_t, R14).
  u32 wv[KPT];
  bool el[KPT];
  if constexpr (WT) {
#pragma unroll
    for (int j = 0; j < KPT; ++j) el[j] = full || t + j * FT < (int)len;
    const bool v2 = full && keys && ((reinterpret_cast<uintptr_t>(keys + base) & 15) == 0);
    const bool v4 = full && !keys && ((reinterpret_cast<uintptr_t>(src + base) & 15) == 0) &&
                    ((reinterpret_cast<uintptr_t>(dst + base) & 15) == 0);
    const u32* pw = g.wgt + base;
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      const int e = v2 ? 2 * (t + (j >> 1) * FT) + (j & 1) : v4 ? 4 * (t + (j >> 2) * FT) + (j & 3) : t + j * FT;
      wv[j] = el[j] ? __ldcs(pw + e) : 0u;
      el[j] = el[j] && wv[j] != 0u;
    }
  }
  if (t == 0 && w >= g.R) waited = wait_geq(&g.fin[w - g.R], 1u, dep);
  __syncthreads();  // hist cleared; thread 0's wait for the slot is published
  pt.mark(g, 0, 0);
#define NSG_ELEMENT(j) (WT ? el[j] : (full || t + (j) * FT < (int)len))
#pragma unroll
  for (int j = 0; j < KPT; ++j)
    if (NSG_ELEMENT(j)) atomicAdd(&s.hist[link_bucket(k[j], g.logB)], 1u);
  __syncthreads();
  pt.mark(g, 0, 1);
  warp0_exclusive_scan(s.hist, (int)g.B);  // warp 0 scans and publishes the chunk's bucket offsets
  if (t < 32) {
    __syncwarp();
    u32* off = g.koff + ((u64)slot * g.cp + c) * (g.B + 1);
    for (int i = t; i <= (int)g.B; i += 32) off[i] = s.hist[i];
  }
  __syncthreads();
  pt.mark(g, 0, 2);
  cl.now(g);
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    if (NSG_ELEMENT(j)) {
      const u32 pos = atomicAdd(&s.hist[link_bucket(k[j], g.logB)], 1u);
      s.stage[pos] = k[j];
      if constexpr (WT) s.stagew[pos] = wv[j];
    }
  }
#undef NSG_ELEMENT
  __syncthreads();
  pt.mark(g, 0, 3);
  u64* out = g.kscr + (u64)slot * g.cp * CH + (u64)c * CH;
  if (len == CH) {
    ulonglong2* o2 = reinterpret_cast<ulonglong2*>(out);
    const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(s.stage);
#pragma unroll
    for (int i = t; i < CH / 2; i += FT) o2[i] = s2[i];
  } else {
    for (u32 i = t; i < len; i += FT) out[i] = s.stage[i];
  }
  if constexpr (WT) {
    u32* ow = g.wscr + (u64)slot * g.cp * CH + (u64)c * CH;
    for (u32 i = t; i < len; i += FT) ow[i] = s.stagew[i];
  }
  __syncthreads();
  pt.mark(g, 0, 4);
  if (t == 0) { red_release_add32(&g.pdone[w], 1u); prof_add(g, 0, clock64() - tstart, waited); }
}

// ------------------------------------------------------------------------------------------
// L item: aggregate link bucket b of window w
// ------------------------------------------------------------------------------------------
// one attempt at `slot`; a new claim also counts the link's two records into the per-(side, side
// bucket) histogram used to lay out the bucket's record region
__device__ __forceinline__ bool link_try_h(u64* lkey, u32* lcnt, u32* hist, u32 B, u32 logB, u64 key, u32 add,
                                           u32 slot) {
  const u64 old = atomicCAS(reinterpret_cast<unsigned long long*>(&lkey[slot]), EMPTY64, key);
  if (old == EMPTY64) {
    atomicAdd(&hist[side_bucket((u32)(key >> 32), logB)], 1u);
    atomicAdd(&hist[B + side_bucket((u32)key, logB)], 1u);
  }
  if (old == EMPTY64 || old == key) { atomicAdd(&lcnt[slot], add); return true; }
  return false;
}
__device__ __noinline__ bool link_finish_h(u64* lkey, u32* lcnt, u32* hist, u32 B, u32 logB, u64 key, u32 add,
                                           u32 probe) {
  const u32 home = link_home(key);
  for (; probe < (u32)TCAP; ++probe)
    if (link_try_h(lkey, lcnt, hist, B, logB, key, add, probe_slot(home, probe))) return true;
  return false;
}

constexpr u32 WAVE_TAIL = 512; // pending entries (<= list capacity) finish per lane: measured faster than barrier-separated waves

// Drop the L2 lines lying entirely inside byte range [lo, hi) of `base` (this warp consumed them and
// nobody reads them again before the slot is rewritten), so dead scratch is never written back to DRAM.
// Lines shared with a neighbouring segment are kept.  All lanes of the warp call it.
__device__ __forceinline__ void discard_interior(const unsigned char* base, u64 lo, u64 hi) {
  const u64 first = (lo + 127) & ~127ull, last = hi & ~127ull;
  for (u64 a = first + (u64)(threadIdx.x & 31) * 128; a < last; a += 32 * 128) discard_l2_line(base + a);
}
__device__ __forceinline__ void discard_segments(const void* base, u32 esize, const u32* wlo, const u32* wpre,
                                                 u32 nseg) {
#ifdef NSG_DISCARD_CONSUMED
  for (u32 q = 0; q < nseg; ++q)
    discard_interior(reinterpret_cast<const unsigned char*>(base), (u64)wlo[q] * esize,
                     ((u64)wlo[q] + (wpre[q + 1] - wpre[q])) * esize);
#endif
}

// Warp-level gather setup: lane q < nseg describes segment q of this warp (global element offset `lo`,
// length `len`); the warp publishes segment starts and exclusive prefixes into its SMEM rows and
// returns the warp's element total.  No CTA barrier is involved.
__device__ __forceinline__ u32 warp_segments(u32* wlo, u32* wpre, u32 nseg, u32 lo, u32 len) {
  const int lane = threadIdx.x & 31;
  if ((u32)lane >= nseg) len = 0;
  u32 x = len;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  const u32 total = __shfl_sync(0xffffffffu, x, 31);
  if ((u32)lane < nseg) { wlo[lane] = lo; wpre[lane] = x - len; }
  if (lane == 0) wpre[nseg] = total;
  __syncwarp();
  return total;
}

// Vector output of one link (all lanes of the warp call it; `valid` lanes write).
__device__ __forceinline__ void emit_link(const Geo& g, u64 w, SmemMisc& m, bool valid, u64 key, u32 c) {
  const u32 r = warp_append(valid, &m.vcnt);
  if (valid) {
    const u64 p = w * g.W + m.vbase + r;
    g.v_lkey[p] = key;
    g.v_lpk[p] = c;
  }
}

template <bool WT, class SL>
__device__ void item_link(const Geo& g, u64 w, u32 b, SL& s, SmemMisc& m, Claim& cl) {
  constexpr int pcap = WT ? PCAP_W : PCAP;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  PhaseTimer pt;
  const u32 ncp = chunks_of(g, w);
  const u32 B = g.B, B2 = g.B2, logB2 = g.logB2;
  const long long tstart = clock64();
  long long waited = 0;
  const u32 slot = slot_of(g, w);
  const u32* koff = g.koff + (u64)slot * g.cp * (B + 1);
  const u64* ks = g.kscr + (u64)slot * g.cp * CH;
  bool ok = true;
  // The partition items of window w are complete (thread 0 waited at the previous item boundary), so
  // the gather starts at once: warp wid reads bucket b's segment of chunks wid, wid + NWARP, ... and
  // issues its first round of key loads; their L2 latency overlaps the table initialisation below.
  const u32 nseg = (u32)wid < ncp ? (ncp - 1 - wid) / NWARP + 1 : 0;
  u32* wlo = s.wlo[wid];
  u32* wpre = s.wpre[wid];
  u32 total;
  {
    u32 lo = 0, len = 0;
    if ((u32)lane < nseg) {
      const u32 c = wid + lane * NWARP;
      const u32* o = koff + (u64)c * (B + 1) + b;
      lo = ldcg32(o);
      len = ldcg32(o + 1) - lo;
      lo += c * CH;
    }
    total = warp_segments(wlo, wpre, nseg, lo, len);
  }
  pt.mark(g, 1, 5);
  u64 k[KPT];
  u32 wv[KPT];  // weighted rows: the weight of each gathered key
  const u32* wsc = WT ? g.wscr + (u64)slot * g.cp * CH : nullptr;
  u32* pwl[2] = {nullptr, nullptr};
  if constexpr (WT) { pwl[0] = s.pw[0]; pwl[1] = s.pw[1]; }
  unsigned long long wl = 0;  // this lane's sum of weights
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    const u32 e = lane + 32 * j;
    wv[j] = 1u;
    if (e < total) {
      const u32 q = find_seg(wpre, nseg, e);
      k[j] = ldcg64(ks + wlo[q] + (e - wpre[q]));
      if constexpr (WT) wv[j] = ldcg32(wsc + wlo[q] + (e - wpre[q]));
    }
  }
  pt.mark(g, 1, 6);
  {
    ulonglong2* k2 = reinterpret_cast<ulonglong2*>(s.lkey);
    uint4* c4 = reinterpret_cast<uint4*>(s.lcnt);
    for (int i = t; i < TCAP / 2; i += FT) k2[i] = make_ulonglong2(EMPTY64, EMPTY64);
    for (int i = t; i < TCAP / 4; i += FT) c4[i] = make_uint4(0, 0, 0, 0);
  }
  for (int i = t; i <= (int)(2 * B2); i += FT) s.hist[i] = 0;
  if (t < 4) m.esc[t] = 0;
  if (t == 0) { m.flag = 0; m.pcnt[0] = 0; m.wsum = 0; }
  pt.mark(g, 1, 7);
  __syncthreads();
  pt.mark(g, 1, 0);
#ifdef NSG_EXP_MARK_KEYS
#pragma unroll
  for (int j = 0; j < KPT; ++j) asm volatile("" ::"l"(k[j]));
  pt.mark(g, 1, 8);
#endif
  for (u32 base = 0; base < total; base += 32 * KPT) {  // warp-uniform rounds
    if (base) {
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        const u32 e = base + lane + 32 * j;
        if (e < total) {
          const u32 q = find_seg(wpre, nseg, e);
          k[j] = ldcg64(ks + wlo[q] + (e - wpre[q]));
          if constexpr (WT) wv[j] = ldcg32(wsc + wlo[q] + (e - wpre[q]));
        }
      }
    }
    // wave 0: one full-warp CAS per key at its home slot, then one at the next slot for the losers
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      if (base + 32 * j >= total) break;  // warp-uniform
      bool entry = base + lane + 32 * j < total;
      const u32 a = WT ? wv[j] : 1u;  // A_t(i,j) += n_packets of the row (1 for raw packets)
      if constexpr (WT) wl += entry ? a : 0u;
      if (entry && k[j] == EMPTY64) { atomicAdd(&m.esc[0], a); entry = false; }
      bool placed = true;
      u32 home = 0;
      if (entry) { home = link_home(k[j]); placed = link_try_h(s.lkey, s.lcnt, s.hist, B2, logB2, k[j], a, home); }
      if (!placed) placed = link_try_h(s.lkey, s.lcnt, s.hist, B2, logB2, k[j], a, probe_slot(home, 1u));
      if (!pend_push(s.pa[0], s.pp[0], &m.pcnt[0], !placed, k[j], 2u, pcap, pwl[0], a))
        ok = link_finish_h(s.lkey, s.lcnt, s.hist, B2, logB2, k[j], a, 2u) && ok;
    }
  }
  if constexpr (WT) {  // the bucket's weight sum bounds every count in it: records carry counts < 2^20
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wl += __shfl_xor_sync(0xffffffffu, wl, o);
    if (lane == 0 && wl) atomicAdd(&m.wsum, wl);
  }
  discard_segments(ks, 8, wlo, wpre, nseg);  // this warp's key segments are consumed
  if constexpr (WT) discard_segments(wsc, 4, wlo, wpre, nseg);
  __syncthreads();
  pt.mark(g, 1, 1);
  prof_pending(g, 1, m.pcnt[0]);
  {
    // waves 1..: the pending list, densely, one probe further each wave; a short tail finishes per lane
    int cur = 0;
    u32 n = min(m.pcnt[0], (u32)pcap);
    while (n) {
      if (n <= WAVE_TAIL) {
        if ((u32)t < n)
          ok = link_finish_h(s.lkey, s.lcnt, s.hist, B2, logB2, s.pa[cur][t], WT ? pwl[cur][t] : 1u, s.pp[cur][t]) && ok;
        break;
      }
      if (t == 0) m.pcnt[cur ^ 1] = 0;
      __syncthreads();
      for (u32 i0 = 0; i0 < n; i0 += FT) {
        const u32 i = i0 + t;
        u64 a = 0;
        u32 probe = 0, wt = 1u;
        bool placed = true;
        if (i < n) {
          a = s.pa[cur][i];
          probe = s.pp[cur][i];
          if constexpr (WT) wt = pwl[cur][i];
          if (probe >= (u32)TCAP) ok = false;
          else placed = link_try_h(s.lkey, s.lcnt, s.hist, B2, logB2, a, wt, probe_slot(link_home(a), probe));
        }
        probe += 1;
        if (!pend_push(s.pa[cur ^ 1], s.pp[cur ^ 1], &m.pcnt[cur ^ 1], !placed, a, probe, pcap, pwl[cur ^ 1], wt))
          ok = link_finish_h(s.lkey, s.lcnt, s.hist, B2, logB2, a, wt, probe) && ok;
      }
      __syncthreads();
      cur ^= 1;
      n = min(m.pcnt[cur], (u32)pcap);
    }
  }
  if (!ok) m.flag = 1;
  // weighted rows: a bucket whose weights sum to >= 2^20 cannot use 20-bit record counts: the window
  // goes to the L2 path (64-bit-safe sums there)
  if (WT && t == 0 && m.wsum >= (1ull << REC_PBITS)) m.flag = 1;
  if (t == 0 && m.esc[0]) {  // the key ~0 (255.255.255.255 -> 255.255.255.255) is one more link
    atomicAdd(&s.hist[side_bucket(EMPTY32, logB2)], 1u);
    atomicAdd(&s.hist[B2 + side_bucket(EMPTY32, logB2)], 1u);
  }
  __syncthreads();
  pt.mark(g, 1, 2);
  // A side bucket with >= 8x the average records (the heavy source's bucket) is "hot": its records
  // are merged per node by a warp register cache during emission (below).
  if (wid == 0) {
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      u32 mx = 0, mi = 0, tot = 0;
      for (u32 i = lane; i < B2; i += 32) {
        const u32 v = s.hist[side * B2 + i];
        tot += v;
        if (v > mx) { mx = v; mi = i; }
      }
      tot = warp_sum(tot);
      const u32 gmx = warp_max(mx);
      const u32 who = __ballot_sync(0xffffffffu, mx == gmx && gmx > 0);
      const u32 gmi = __shfl_sync(0xffffffffu, mi, who ? __ffs(who) - 1 : 0);
      if (lane == 0) m.hot[side] = (B2 > 1 && gmx >= 512 && gmx >= 8 * (tot / B2)) ? gmi : ~0u;
    }
  }
  // record region layout: offsets of every (side, side bucket), scanned and published by warp 0
  warp0_exclusive_scan(s.hist, (int)(2 * B2));
  if (t < 32) {
    __syncwarp();
    u32* off = g.roff + ((u64)slot * B + b) * (2 * B2 + 1);
    for (int i = t; i <= (int)(2 * B2); i += 32) off[i] = s.hist[i];
    if (t == 0 && g.v_lkey) {  // this bucket's links (two records each) get a contiguous part of the window's region
      m.vbase = atomicAdd(&g.vfill[w * 3], s.hist[2 * B2] / 2);
      m.vcnt = 0;
    }
  }
  __syncthreads();
  pt.mark(g, 1, 3);
  cl.now(g);
  // One pass over the bucket's part of A_t: unique links (:181), max link packets (:183), sum of counts
  // (:180); and one record per link and side, node<<32 | 1<<20 | count.
  u64* rec = g.rscr + ((u64)slot * B + b) * RCAP;
  u32 nl = 0, mx = 0, sm = 0;
#ifndef NSG_EXP_SKIP_EMIT  // timing experiment only: results are wrong when defined
  const u32 hot0 = m.hot[0], hot1 = m.hot[1];
  if (hot0 == ~0u && hot1 == ~0u) {  // CTA-uniform: no skewed side bucket (the common case)
    for (int i = t; i < TCAP; i += FT) {
      const u64 key = s.lkey[i];
      u32 c = 0;
      if (key != EMPTY64) {
        c = s.lcnt[i];
        nl += 1; mx = max(mx, c); sm += c;
        const u32 sn = (u32)(key >> 32), dn = (u32)key;
        rec[atomicAdd(&s.hist[side_bucket(sn, logB2)], 1u)] = make_rec(sn, 1u, c);
        rec[atomicAdd(&s.hist[B2 + side_bucket(dn, logB2)], 1u)] = make_rec(dn, 1u, c);
      }
      if (g.v_lkey) emit_link(g, w, m, key != EMPTY64, key, c);  // CTA-uniform
    }
  } else {
    // per side, a warp cache node (seeded from the hot bucket's first record of the warp while it has
    // had no hit) whose links are summed in lane registers and emitted as one record per warp
    u32 cn[2] = {0, 0}, ch[2] = {0, 0}, lp[2] = {0, 0}, lf[2] = {0, 0};
    for (int i = t; i < TCAP; i += FT) {  // TCAP % FT == 0: every lane runs the same iterations
      const u64 key = s.lkey[i];
      const bool valid = key != EMPTY64;
      const u32 c = valid ? s.lcnt[i] : 0u;
      if (valid) { nl += 1; mx = max(mx, c); sm += c; }
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const u32 node = side ? (u32)key : (u32)(key >> 32);
        const u32 sbk = side_bucket(node, logB2);
        const u32 hot = side ? hot1 : hot0;
        const bool inhot = valid && sbk == hot;
        const u32 hm = __ballot_sync(0xffffffffu, inhot);
        bool hit = false;
        if (hm) {
          if (ch[side] == 0) cn[side] = __shfl_sync(0xffffffffu, node, __ffs(hm) - 1);
          hit = inhot && node == cn[side];
          ch[side] += (u32)__popc(__ballot_sync(0xffffffffu, hit));
          if (hit) { lp[side] += c; lf[side] += 1; }
        }
        if (valid && !hit) rec[atomicAdd(&s.hist[side * B2 + sbk], 1u)] = make_rec(node, 1u, c);
      }
      if (g.v_lkey) emit_link(g, w, m, valid, key, c);
    }
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const u32 p = warp_sum(lp[side]);
      u32 f = warp_sum(lf[side]);
      if (lane == 0 && f) {  // one merged record (split when F > REC_FMAX)
        const u32 nrec = (f + REC_FMAX - 1) / REC_FMAX;
        const u32 pos = atomicAdd(&s.hist[side * B2 + side_bucket(cn[side], logB2)], nrec);
        for (u32 q = 0; q < nrec; ++q) {
          const u32 fr = min(f, REC_FMAX);
          rec[pos + q] = make_rec(cn[side], fr, q == 0 ? p : 0u);
          f -= fr;
        }
      }
    }
  }
#endif
  if (t == 0 && m.esc[0]) {
    const u32 c = m.esc[0];
    nl += 1; mx = max(mx, c); sm += c;
    const u64 r = make_rec(EMPTY32, 1u, c);
    rec[atomicAdd(&s.hist[side_bucket(EMPTY32, logB2)], 1u)] = r;
    rec[atomicAdd(&s.hist[B2 + side_bucket(EMPTY32, logB2)], 1u)] = r;
    if (g.v_lkey) {
      const u64 p = w * g.W + m.vbase + atomicAdd(&m.vcnt, 1u);
      g.v_lkey[p] = EMPTY64; g.v_lpk[p] = c;
    }
  }
  nl = warp_sum(nl); mx = warp_max(mx); sm = warp_sum(sm);
  if (lane == 0) { m.wtmp[4 * NWARP + wid] = nl; m.wtmp[5 * NWARP + wid] = mx; m.wtmp[6 * NWARP + wid] = sm; }
  __syncthreads();
  pt.mark(g, 1, 4);
  if (wid == 0) {
    u32 a = lane < NWARP ? m.wtmp[4 * NWARP + lane] : 0u;
    u32 bm = lane < NWARP ? m.wtmp[5 * NWARP + lane] : 0u;
    u32 cs = lane < NWARP ? m.wtmp[6 * NWARP + lane] : 0u;
    a = warp_sum(a); bm = warp_max(bm); cs = warp_sum(cs);
    u32* rend = g.rend + ((u64)slot * B + b) * (2 * B2);
    for (int i = lane; i < (int)(2 * B2); i += 32) rend[i] = s.hist[i];  // cursors = segment ends
    __syncwarp();
    if (lane == 0) {
      u32* r = g.lres + ((u64)slot * B + b) * 4;
      r[0] = a; r[1] = bm; r[2] = cs;
      if (m.flag) mark_overflow(g, w);
      __threadfence_block();
      red_release_add32(&g.ldone[w], 1u);  // after the CTA barrier; warp 0's writes precede it
      prof_add(g, 1, clock64() - tstart, waited);
      pt.mark(g, 1, 9);
    }
  }
}

// ------------------------------------------------------------------------------------------
// Window finalisation (run by the CTA that completes the window's last S item)
// ------------------------------------------------------------------------------------------
__device__ void item_finalize(const Geo& g, u64 w, SmemMisc& m, u64* __restrict__ out) {
  const int t = threadIdx.x;
  const u32 slot = slot_of(g, w);
  // all side items of window w are complete (waited for at the previous item boundary)
  // sums: 0 links, 1 sum of counts, 2 unique sources, 3 unique destinations;
  // maxes: 4 max link, 5 max source packets, 6 max fan-out, 7 max destination packets, 8 max fan-in
  u32 v[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};  // [9]: |S n D| (IP sets)
  for (u32 i = t; i < g.B; i += FT) {
    const u32* r = g.lres + ((u64)slot * g.B + i) * 4;
    v[0] += ldcg32(r); v[4] = max(v[4], ldcg32(r + 1)); v[1] += ldcg32(r + 2);
  }
  for (u32 i = t; i < g.B2; i += FT) {
    const u32* s0 = g.sres + (((u64)slot * 2 + 0) * g.B2 + i) * 4;
    const u32* s1 = g.sres + (((u64)slot * 2 + 1) * g.B2 + i) * 4;
    v[2] += ldcg32(s0); v[5] = max(v[5], ldcg32(s0 + 1)); v[6] = max(v[6], ldcg32(s0 + 2));
    v[3] += ldcg32(s1); v[7] = max(v[7], ldcg32(s1 + 1)); v[8] = max(v[8], ldcg32(s1 + 2));
    v[9] += ldcg32(s1 + 3);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) v[j] = warp_sum(v[j]);
#pragma unroll
  for (int j = 4; j < 9; ++j) v[j] = warp_max(v[j]);
  v[9] = warp_sum(v[9]);
  const int lane = t & 31, wid = t >> 5;
  __syncthreads();
  if (lane == 0)
    for (int j = 0; j < 10; ++j) m.wtmp[j * NWARP + wid] = v[j];
  __syncthreads();
  if (t == 0) {
    u32 r[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < NWARP; ++i) {
      for (int j = 0; j < 4; ++j) r[j] += m.wtmp[j * NWARP + i];
      for (int j = 4; j < 9; ++j) r[j] = max(r[j], m.wtmp[j * NWARP + i]);
      r[9] += m.wtmp[9 * NWARP + i];
    }
    const u64 wlen = min(g.W, g.n - w * g.W);
    const u64 row[NSG_NUM_STATS] = {r[1], r[0], r[4], r[2], r[5], r[6], r[3], r[7], r[8]};  // north_star order
    store_row(out + w * NSG_NUM_STATS, row);
    for (u32 j = 0; j < g.n_mirror; ++j) store_row(g.mirror[j] + (g.mirror_row0 + w) * NSG_NUM_STATS, row);
    if (g.v_ipsets) {  // |S u D|, |S \ D|, |D \ S|, |S n D|
      u64* ip = g.v_ipsets + w * 4;
      ip[0] = (u64)r[2] + r[3] - r[9]; ip[1] = r[2] - r[9]; ip[2] = r[3] - r[9]; ip[3] = r[9];
    }
    if (!g.wgt && (u64)r[1] != wlen && ld_acquire32(&g.ovf[w]) == 0) atomicAdd(&g.diag[1], 1u);
    if ((g.flags & NSG_FLAG_INJECT_OVERFLOW) && (w & 1)) mark_overflow(g, w);
    // The slot may now be reused: every reader of it has signalled sdone.  (Dropping its dead L2
    // lines with discard.global.L2 first halves DRAM writes but was measured 14% slower on C2.)
    st_release32(&g.fin[w], 1u);
  }
}

// ------------------------------------------------------------------------------------------
// S item: merge side bucket sb of one side of window w
// ------------------------------------------------------------------------------------------
// Is `node` in the (complete) node table?  Linear probing from its home slot; slots never empty again.
__device__ __forceinline__ bool node_present(const u32* key, u32 node) {
  const u32 home = node_home(node);
  for (u32 probe = 0; probe < (u32)TCAP_S; ++probe) {
    const u32 k = key[probe_slot_s(home, probe)];
    if (k == node) return true;
    if (k == EMPTY32) return false;
  }
  return false;
}

// Vector outputs of a side item (after its table is final and m.wtmp holds the per-warp node counts):
//  - the nodes with their packets and fan (A_t 1 / |A_t|_0 1 or the mirrors)
//    into the window's region of v_node/v_pk/v_fan[side];
//  - IP sets: side 0 publishes its node list; side 1 waits for the list of the side-0
//    item of the same bucket (same node hash partition: side_bucket() is one function of the address)
//    and counts the listed nodes present in its own table, i.e. |S n D| restricted to the bucket.
// S0(w, sb) holds a smaller ticket than S1(w, sb), so the wait cannot deadlock.
// (Takes its pointers by value: a Geo& to a __noinline__ function would put the kernel's parameter
// block in local memory.)
struct SideVec {
  u32 *node, *pk, *fan;  // this side's vectors (node NULL: not requested)
  bool ipsets;
  u32 *vfill, *s0list, *s0cnt, *s0win;
  u64 W;
  u32 B2;
};
__device__ __noinline__ void side_vectors(const SideVec g, u64 w, int side, u32 sb, u32 slot, SmemS& s, SmemMisc& m) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const bool nodes = g.node != nullptr;
  const bool list0 = side == 0 && g.ipsets;
  u32* list = g.s0list + ((u64)slot * g.B2 + sb) * S0LIST;
  if (t == 0) {
    u32 tot = 0;
    for (int i = 0; i < NWARP; ++i) tot += m.wtmp[4 * NWARP + i];
    m.vbase = nodes ? atomicAdd(&g.vfill[w * 3 + 1 + side], tot) : 0u;
    m.vcnt = 0;
  }
  __syncthreads();
  const u64 wb = w * g.W + m.vbase;
  if (nodes || list0) {
    for (int i = t; i < TCAP_S; i += FT) {  // TCAP_S % FT == 0: warp-uniform trip count
      const u32 node = s.key[i];
      const bool valid = node != EMPTY32;
      const u32 r = warp_append(valid, &m.vcnt);
      if (valid) {
        if (nodes) { g.node[wb + r] = node; g.pk[wb + r] = s.P[i]; g.fan[wb + r] = s.F[i]; }
        if (list0) list[r] = node;
      }
    }
    if (t == 0 && m.esc[2]) {  // the address ~0 (255.255.255.255), kept outside the table
      const u32 r = atomicAdd(&m.vcnt, 1u);
      if (nodes) { g.node[wb + r] = EMPTY32; g.pk[wb + r] = m.esc[1]; g.fan[wb + r] = m.esc[2]; }
      if (list0) list[r] = EMPTY32;
    }
    __syncthreads();
  }
  if (list0 && t == 0) {
    g.s0cnt[(u64)slot * g.B2 + sb] = m.vcnt;
    st_release32(&g.s0win[(u64)slot * g.B2 + sb], (u32)w + 1u);  // after the barrier: publishes every lane's list writes
  }
  if (side == 1 && g.ipsets) {
    if (t == 0) {
      const u32* f = &g.s0win[(u64)slot * g.B2 + sb];
      while (ld_acquire32(f) != (u32)w + 1u) __nanosleep(64);
      m.n0 = ldcg32(&g.s0cnt[(u64)slot * g.B2 + sb]);
    }
    __syncthreads();
    const u32 n0 = m.n0;
    u32 hits = 0;
    for (u32 i = t; i < n0; i += FT) {
      const u32 node = ldcg32(&list[i]);
      hits += node == EMPTY32 ? (m.esc[2] != 0u) : (u32)node_present(s.key, node);
    }
    hits = warp_sum(hits);
    if (lane == 0) m.wtmp[7 * NWARP + wid] = hits;
    __syncthreads();
    if (t == 0) {
      u32 b = 0;
      for (int i = 0; i < NWARP; ++i) b += m.wtmp[7 * NWARP + i];
      m.both = b;
    }
    __syncthreads();
  }
}

__device__ void item_side(const Geo& g, u64 w, int side, u32 sb, SmemS& s, SmemMisc& m, Claim& cl) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
#ifdef NSG_EXP_SKIP_S  // timing experiment only: results are wrong
  if (t == 0) { wait_geq(&g.ldone[w], g.B, 0); red_release_add32(&g.sdone[w], 1u); }
  __syncthreads();
  return;
#endif
  PhaseTimer pt;
  const u32 B = g.B, B2 = g.B2;
  const long long tstart = clock64();
  long long waited = 0;
  const u32 slot = slot_of(g, w);
  const u64* rs = g.rscr + (u64)slot * B * RCAP;
  bool ok = true;
  {
    // All link items of window w are complete (waited for at the previous item boundary): warp wid
    // gathers side bucket sb's records from link buckets wid, wid + NWARP, ... and issues its first
    // round of loads before the table initialisation, which hides their L2 latency.
    const u32 nseg = (u32)wid < B ? (B - 1 - wid) / NWARP + 1 : 0;
    u32 lo = 0, len = 0;
    if ((u32)lane < nseg) {
      const u32 lb = wid + lane * NWARP;
      lo = ldcg32(g.roff + ((u64)slot * B + lb) * (2 * B2 + 1) + side * B2 + sb);
      len = ldcg32(g.rend + ((u64)slot * B + lb) * (2 * B2) + side * B2 + sb) - lo;
      lo += lb * RCAP;
    }
    u32* wlo = s.wlo[wid];
    u32* wpre = s.wpre[wid];
    const u32 total = warp_segments(wlo, wpre, nseg, lo, len);
    if (kProfile && lane == 0 && (g.flags & NSG_FLAG_PROFILE) && w == 0 && side * B2 + sb < 64)
      atomicAdd(reinterpret_cast<unsigned long long*>(&g.prof[192 + side * B2 + sb]), (unsigned long long)total);
    u64 r[KPT];
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      const u32 e = lane + 32 * j;
      if (e < total) {
        const u32 q = find_seg(wpre, nseg, e);
        r[j] = ldcg64(rs + wlo[q] + (e - wpre[q]));
      }
    }
    {
      uint4* k4 = reinterpret_cast<uint4*>(s.key);
      uint4* p4 = reinterpret_cast<uint4*>(s.P);
      uint4* f4 = reinterpret_cast<uint4*>(s.F);
      for (int i = t; i < TCAP_S / 4; i += FT) {
        k4[i] = make_uint4(EMPTY32, EMPTY32, EMPTY32, EMPTY32);
        p4[i] = make_uint4(0, 0, 0, 0);
        f4[i] = make_uint4(0, 0, 0, 0);
      }
    }
    if (t < 4) m.esc[t] = 0;
    if (t == 0) { m.flag = 0; m.pcnt[0] = 0; }
    __syncthreads();
    pt.mark(g, 2, 0);
    // Warp-uniform register cache of one hot node (e.g. the heavy source): records of the cached node
    // are summed in lane registers across rounds and merged into the table once, when the entry is
    // evicted.  An entry is replaced only after a round in which it had fewer than 8 hits.
    bool c_has = false;
    u32 c_node = 0, c_p = 0, c_f = 0, c_hits = 0;
    for (u32 base = 0; base < total; base += 32 * KPT) {  // warp-uniform rounds
      if (base) {
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
          const u32 e = base + lane + 32 * j;
          if (e < total) {
            const u32 q = find_seg(wpre, nseg, e);
            r[j] = ldcg64(rs + wlo[q] + (e - wpre[q]));
          }
        }
      }
      if (!c_has || c_hits < 8) {  // (re)seed the cache with the first record of the round
        const u32 cand = __shfl_sync(0xffffffffu, (u32)(r[0] >> 32), 0);
        if (c_has && cand != c_node) {  // evict: merge the old entry (lane partial sums) into the table
          const u32 sp = warp_sum(c_p), sf = warp_sum(c_f);
          if (lane == 0) ok = node_flush(s.key, s.P, s.F, m.esc, c_node, sp, sf) && ok;
        }
        if (!c_has || cand != c_node) { c_node = cand; c_p = 0; c_f = 0; c_has = true; }
      }
      c_hits = 0;
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        if (base + 32 * j >= total) break;  // warp-uniform
        const bool valid = base + lane + 32 * j < total;
        const u32 node = (u32)(r[j] >> 32);
        const u32 p = (u32)r[j] & ((1u << REC_PBITS) - 1u);
        const u32 f = (u32)(r[j] >> REC_PBITS) & REC_FMAX;
        const bool hit = valid && node == c_node;
        c_hits += (u32)__popc(__ballot_sync(0xffffffffu, hit));
        if (hit) { c_p += p; c_f += f; }  // lane partial sums; reduced once, when the entry is flushed
        bool entry = valid && !hit;
        if (entry && node == EMPTY32) { atomicAdd(&m.esc[1], p); atomicAdd(&m.esc[2], f); entry = false; }
        bool placed = true;
        u32 home = 0;
        if (entry) { home = node_home(node); placed = node_try(s.key, s.P, s.F, node, p, f, home); }
        if (!placed) placed = node_try(s.key, s.P, s.F, node, p, f, probe_slot_s(home, 1u));
        if (!pend_push(s.pa[0], s.pp[0], &m.pcnt[0], !placed, make_rec(node, f, p), 2u, PCAP_S))
          ok = node_finish(s.key, s.P, s.F, node, p, f, 2u) && ok;
      }
    }
    if (c_has) {  // flush the cache
      const u32 sp = warp_sum(c_p), sf = warp_sum(c_f);
      if (lane == 0) ok = node_flush(s.key, s.P, s.F, m.esc, c_node, sp, sf) && ok;
    }
    discard_segments(rs, 8, wlo, wpre, nseg);  // this warp's record segments are consumed
  }
  __syncthreads();
  pt.mark(g, 2, 1);
  prof_pending(g, 2, m.pcnt[0]);
  {
    int cur = 0;
    u32 n = min(m.pcnt[0], (u32)PCAP_S);
    while (n) {
      if (n <= WAVE_TAIL) {
        if ((u32)t < n) {
          const u64 a = s.pa[cur][t];
          ok = node_finish(s.key, s.P, s.F, (u32)(a >> 32), (u32)a & ((1u << REC_PBITS) - 1u),
                           (u32)(a >> REC_PBITS) & REC_FMAX, s.pp[cur][t]) && ok;
        }
        break;
      }
      if (t == 0) m.pcnt[cur ^ 1] = 0;
      __syncthreads();
      for (u32 i0 = 0; i0 < n; i0 += FT) {
        const u32 i = i0 + t;
        u64 a = 0;
        u32 probe = 0;
        bool placed = true;
        const u32 nd = (u32)(s.pa[cur][min(i, n - 1)] >> 32);
        if (i < n) {
          a = s.pa[cur][i];
          probe = s.pp[cur][i];
          if (probe >= (u32)TCAP_S) ok = false;
          else placed = node_try(s.key, s.P, s.F, nd, (u32)a & ((1u << REC_PBITS) - 1u), (u32)(a >> REC_PBITS) & REC_FMAX,
                                 probe_slot_s(node_home(nd), probe));
        }
        probe += 1;
        if (!pend_push(s.pa[cur ^ 1], s.pp[cur ^ 1], &m.pcnt[cur ^ 1], !placed, a, probe, PCAP_S))
          ok = node_finish(s.key, s.P, s.F, nd, (u32)a & ((1u << REC_PBITS) - 1u), (u32)(a >> REC_PBITS) & REC_FMAX, probe) && ok;
      }
      __syncthreads();
      cur ^= 1;
      n = min(m.pcnt[cur], (u32)PCAP_S);
    }
  }
  if (!ok) m.flag = 1;
  __syncthreads();
  pt.mark(g, 2, 2);
  cl.now(g);
  // unique nodes (1^T|A_t 1|_0 or its mirror), max packets (max A_t 1), max fan (max |A_t|_0 1)
  u32 d = 0, mp = 0, mf = 0;
  for (int i = t; i < TCAP_S; i += FT) {
    if (s.key[i] != EMPTY32) { d += 1; mp = max(mp, s.P[i]); mf = max(mf, s.F[i]); }
  }
  if (t == 0 && m.esc[1]) { d += 1; mp = max(mp, m.esc[1]); mf = max(mf, m.esc[2]); }
  d = warp_sum(d); mp = warp_max(mp); mf = warp_max(mf);
  if (lane == 0) { m.wtmp[4 * NWARP + wid] = d; m.wtmp[5 * NWARP + wid] = mp; m.wtmp[6 * NWARP + wid] = mf; }
  __syncthreads();
  pt.mark(g, 2, 3);
  if ((side ? g.v_node[1] : g.v_node[0]) || g.v_ipsets) {  // CTA-uniform
    const SideVec sv{side ? g.v_node[1] : g.v_node[0], side ? g.v_pk[1] : g.v_pk[0], side ? g.v_fan[1] : g.v_fan[0],
                     g.v_ipsets != nullptr, g.vfill, g.s0list, g.s0cnt, g.s0win, g.W, g.B2};
    side_vectors(sv, w, side, sb, slot, s, m);
  }
  if (wid == 0) {
    u32 a = lane < NWARP ? m.wtmp[4 * NWARP + lane] : 0u;
    u32 bp = lane < NWARP ? m.wtmp[5 * NWARP + lane] : 0u;
    u32 cf = lane < NWARP ? m.wtmp[6 * NWARP + lane] : 0u;
    a = warp_sum(a); bp = warp_max(bp); cf = warp_max(cf);
    if (kProfile && lane == 0 && (g.flags & NSG_FLAG_PROFILE) && w == 0 && side * B2 + sb < 64) {  // window-0 detail
      g.prof[128 + side * B2 + sb] = (u64)(clock64() - tstart);
    }
    if (lane == 0) {
      u32* res = g.sres + (((u64)slot * 2 + side) * B2 + sb) * 4;
      res[0] = a; res[1] = bp; res[2] = cf; res[3] = (side == 1 && g.v_ipsets) ? m.both : 0u;
      if (m.flag) mark_overflow(g, w);
      red_release_add32(&g.sdone[w], 1u);  // thread 0 wrote res itself: program order + release
      prof_add(g, 2, clock64() - tstart, waited);
      pt.mark(g, 2, 9);
    }
  }
}

// ------------------------------------------------------------------------------------------
// Ticket decoding: step k holds F(k-LAG_F), S(k-LAG_S) [2*B2], L(k-LAG_L) [B], P(k) [cp], each class
// only while its window is in [0, nw).
// ------------------------------------------------------------------------------------------
enum : u32 { ITEM_P = 0, ITEM_L = 1, ITEM_S0 = 2, ITEM_S1 = 3, ITEM_F = 4, ITEM_NOP = 5, ITEM_DONE = 6 };

struct Item { u32 type, idx; u64 w; };

// Thread 0: block until the dependencies of `it` are complete (acquire).  Called before the barrier
// that starts the item, so the item's first loads can be issued at once.  An item only ever waits on
// items with smaller tickets, so the schedule cannot deadlock.
__device__ __forceinline__ long long wait_item_deps(const Geo& g, const Item& it) {
  switch (it.type) {
    case ITEM_P: return 0;  // waits inside, after issuing its HBM loads (slot reuse rarely blocks)
    case ITEM_L: return wait_geq(&g.pdone[it.w], g.cp, 0u);                       // all chunks partitioned
    case ITEM_S0:
    case ITEM_S1: return wait_geq(&g.ldone[it.w], g.B, 0u);                       // all link buckets emitted
    case ITEM_F: return wait_geq(&g.sdone[it.w], 2 * g.B2, 0u);                   // all side buckets merged
    default: return 0;
  }
}
__device__ __forceinline__ void prof_wait(const Geo& g, const Item& it, long long waited) {
  if ((g.flags & NSG_FLAG_PROFILE) && waited) {
    const int type = it.type == ITEM_P ? 0 : it.type == ITEM_L ? 1 : 2;
    if (it.type <= ITEM_S1)
      atomicAdd(reinterpret_cast<unsigned long long*>(&g.prof[type * 4 + 2]), (unsigned long long)waited);
  }
}

__device__ __forceinline__ Item decode_ticket(const Geo& g, u64 tk) {
  Item it{ITEM_DONE, 0, 0};
  if (tk >= g.total_items) return it;
  u32 r = 0;
  while (r + 1 < g.nreg && tk >= g.reg_t0[r + 1]) ++r;
  const u64 rel = tk - g.reg_t0[r];
  const u32 ips = g.reg_ips[r];
  u64 k, idx;
  if (rel <= 0xFFFFFFFFull) {  // 32-bit division when it fits (the usual case)
    const u32 q = (u32)rel / ips;
    k = q;
    idx = (u32)rel - q * ips;
  } else {
    k = rel / ips;
    idx = rel - k * ips;
  }
  k += g.reg_k0[r];
  const u32 mask = g.reg_mask[r];
  u64 w;
  u32 type;
  if ((mask & 1u) && idx == 0) { type = ITEM_F; w = k - LAG_F; }
  else {
    if (mask & 1u) idx -= 1;
    if ((mask & 2u) && idx < 2ull * g.B2) { type = idx < g.B2 ? ITEM_S0 : ITEM_S1; idx &= g.B2 - 1; w = k - LAG_S; }
    else {
      if (mask & 2u) idx -= 2ull * g.B2;
      if ((mask & 4u) && idx < g.B) { type = ITEM_L; w = k - LAG_L; }
      else {
        if (mask & 4u) idx -= g.B;
        type = ITEM_P; w = k;
      }
    }
  }
  it.type = type; it.w = w; it.idx = (u32)idx;
  return it;
}

#ifdef NSG_EXP_TRACE  // timing experiment: per-item (type|w|idx, start ns, end ns, smid) records
constexpr u32 TRACE_CAP = 1u << 18;
__device__ u64 g_trace[TRACE_CAP][4];
__device__ u32 g_trace_n;
#endif

template <bool WT>
__global__ void __launch_bounds__(FT, 1024 / FT)
fast_kernel(Geo g, const u32* __restrict__ src, const u32* __restrict__ dst, const u64* __restrict__ keys,
            u64* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SmemMisc& m = *reinterpret_cast<SmemMisc*>(smem_raw);
  unsigned char* u = smem_raw + MISC_BYTES;
  // The scheduler thread (lane 0 of warp 1) claims the next ticket late in the current item (Claim),
  // and at its end decodes it and waits for its dependencies (acquire) while warp 0 is still doing the
  // item's tail (result writes, release), so the round trips overlap and the boundary barrier only
  // publishes an already-decoded, ready descriptor.
  const bool sched = threadIdx.x == SCHED_THREAD;
  Claim cl{0, false};
  if (sched) {
    const Item first = decode_ticket(g, atomicAdd(reinterpret_cast<unsigned long long*>(g.ticket), 1ull));
    prof_wait(g, first, wait_item_deps(g, first));
    m.type = first.type; m.idx = first.idx; m.w = first.w;
  }
  long long t_end = 0;  // scheduler: clock at the end of the previous item (profiling)
  for (;;) {
    __syncthreads();
    const u32 type = m.type, idx = m.idx;
    const u64 w = m.w;
    if (type == ITEM_DONE) break;
    if (sched) {
      if ((g.flags & NSG_FLAG_PROFILE) && t_end) {  // boundary: tail/wait overlap + barrier
        atomicAdd(reinterpret_cast<unsigned long long*>(&g.prof[12]), (unsigned long long)(clock64() - t_end));
        atomicAdd(reinterpret_cast<unsigned long long*>(&g.prof[13]), 1ull);
      }
      cl.done = false;
    }
#ifdef NSG_EXP_TRACE
    u64 tr0 = 0;
    if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr0));
#endif
    // every item function passes a __syncthreads() before the scheduler can overwrite m.type/m.w/m.idx
    if (type == ITEM_P) {
      if (idx < chunks_of(g, w)) {
        item_partition<WT>(g, src, dst, keys, w, idx, *reinterpret_cast<SmemP*>(u), m, cl);
      } else {  // a chunk past the end of the last (short) window: count it done
        if (threadIdx.x == 0) red_release_add32(&g.pdone[w], 1u);
        __syncthreads();
      }
    } else if (type == ITEM_L) {
      if constexpr (WT) item_link<true>(g, w, idx, *reinterpret_cast<SmemLW*>(u), m, cl);
      else item_link<false>(g, w, idx, *reinterpret_cast<SmemL*>(u), m, cl);
    } else if (type == ITEM_S0 || type == ITEM_S1) {
      item_side(g, w, (int)(type - ITEM_S0), idx, *reinterpret_cast<SmemS*>(u), m, cl);
    } else if (type == ITEM_F) {
      item_finalize(g, w, m, out);
    } else {
      __syncthreads();  // no-op ticket
    }
#ifdef NSG_EXP_TRACE
    if (threadIdx.x == 0) {
      u64 tr1, smid;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr1));
      asm volatile("{ .reg .u32 r; mov.u32 r, %%smid; cvt.u64.u32 %0, r; }" : "=l"(smid));
      const u32 e = atomicAdd(&g_trace_n, 1u);
      if (e < TRACE_CAP) {
        g_trace[e][0] = ((u64)type << 56) | ((w & 0xFFFFFFull) << 32) | idx;
        g_trace[e][1] = tr0; g_trace[e][2] = tr1; g_trace[e][3] = smid;
      }
    }
#endif
    // every item function passed a __syncthreads() after all threads read m.type/m.w/m.idx
    if (sched) {
      t_end = clock64();
      cl.now(g);  // items that did not claim (F, short items)
      const Item nxt = decode_ticket(g, cl.tk);
      prof_wait(g, nxt, wait_item_deps(g, nxt));
      m.type = nxt.type; m.idx = nxt.idx; m.w = nxt.w;
    }
  }
}

}  // namespace nsg
