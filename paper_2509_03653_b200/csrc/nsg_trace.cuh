// nsg_trace.cuh — the whole-trace path of libnsg: Table 2 on the traffic
// matrix of the WHOLE input, A = sum over t of A_t (PAPER.md:145, :207 — the paper's cuDF frame holds the
// whole capture).  Its distinct links far exceed any SMEM, so the tables live in HBM (global-memory
// open addressing), and the path is split into steps that a multi-GPU driver interleaves with NCCL
// all-to-all exchanges (paper_2509_03653_b200/distributed.py):
//   partition  keys -> owner rank of the link  (o = top bits of hash64(key) * world)
//   links      this rank's links: A restricted to the owned keys -> valid, unique links, max link,
//              and one record (node << 32 | A(i,j)) per link and side, grouped by the node's owner rank
//   nodes      records of one side -> row sums A1 / row nnz |A|_0 1 of the owned nodes (PAPER.md:185,
//              :187; the column mirrors for destination records, :173) -> unique, max packets, max fan
// With world = 1 nothing is exchanged: nsg_trace_stats runs links -> nodes(src) -> nodes(dst).
#pragma once
#include "nsg_internal.h"
#include "nsg_common.cuh"
#include "nsg_global.cuh"

namespace nsg {

constexpr int TT = 512;          // threads per CTA of the trace kernels
constexpr u64 TRACE_CAS_FIRST_SLOTS = 1ull << 26;  // tables this large live in DRAM: probe by CAS (tl_insert)
// The threshold as the kernels read it (tests lower it to run the CAS-as-probe inserts on small inputs:
// nsg_debug_trace_cas_first_slots in nsg_internal.h).
__device__ u64 g_trace_cas_first_slots = TRACE_CAS_FIRST_SLOTS;
constexpr int TRACE_MAX_WORLD = 1024;

// owner rank of a link / of a node (independent of the table slots, which use the low bits)
__device__ __forceinline__ u32 link_owner(u64 key, u32 world) {
  return __umulhi((u32)(hash64(key) >> 32), world);  // floor(h * world / 2^32) < world
}
__device__ __forceinline__ u32 node_owner(u32 node, u32 world) {
  return __umulhi(hash32(node ^ 0x5BD1E995u), world);
}

// Slot range [lo, hi) of CTA b when `total` slots are split into gridDim.x contiguous ranges.
__device__ __forceinline__ void cta_range(u64 total, u64& lo, u64& hi) {
  const u64 per = (total + gridDim.x - 1) / gridDim.x;
  lo = min(total, (u64)blockIdx.x * per);
  hi = min(total, lo + per);
}

__device__ __forceinline__ u64 load_key(const u64* keys, const u32* src, const u32* dst, u64 i) {
  return keys ? keys[i] : (((u64)src[i] << 32) | dst[i]);
}

// HBM tables with one 16-byte slot per entry (key and counters in the same 32-byte sector: one DRAM
// access per probe instead of one per array)
struct __align__(16) LSlot { u64 key; u32 cnt; u32 pad; };
struct __align__(16) NSlot { u32 key, P, F, pad; };

// Node-table slots actually used: next_pow2(2m) for m records (m read from the device: the single-GPU
// trace knows its record count only there), at most the workspace's NC.
__device__ __forceinline__ u64 node_cap(u64 NC, const u64* m_dev) {
  if (!m_dev) return NC;
  const u64 m = *m_dev;
  u64 c = 2;
  while (c < 2 * m && c < NC) c <<= 1;
  return c < NC ? c : NC;
}

__global__ void __launch_bounds__(TT) trace_fill(LSlot* __restrict__ lt, u64 LC, NSlot* __restrict__ nt, u64 NC,
                                                 const u64* __restrict__ m_dev = nullptr) {
  NC = node_cap(NC, m_dev);
  for (u64 i = (u64)blockIdx.x * TT + threadIdx.x; i < LC; i += (u64)gridDim.x * TT)
    reinterpret_cast<ulonglong2*>(lt)[i] = make_ulonglong2(EMPTY64, 0ull);
  for (u64 i = (u64)blockIdx.x * TT + threadIdx.x; i < NC; i += (u64)gridDim.x * TT)
    reinterpret_cast<uint4*>(nt)[i] = make_uint4(EMPTY32, 0u, 0u, 0u);
}

// A free slot is claimed together with its first count by one 128-bit CAS ({~0, 0, 0} -> {key, add, 0}):
// a new entry costs one probe load and one atomic instead of a CAS and an add (random DRAM sectors).
typedef unsigned __int128 u128;
// cas_first: the CAS itself is the probe (it returns the slot's key when the claim fails) — fewer
// operations per new key, best when the table lives in DRAM; otherwise a load probes first and only a
// free slot is CASed — cheaper when occupied slots are L2 hits (measured crossover ~2^25 keys).
__device__ __forceinline__ void tl_insert(LSlot* t, u64 LC, u64 key, u32 add, bool cas_first = false) {
  u64 slot = hash64(key) & (LC - 1);
  const u128 empty = (u128)EMPTY64;
  for (;;) {
    u64 k = cas_first ? EMPTY64 : ldcg64(&t[slot].key);
    if (k == EMPTY64) {
      const u128 old = atomicCAS(reinterpret_cast<u128*>(&t[slot]), empty, (u128)key | ((u128)add << 64));
      if (old == empty) return;
      k = (u64)old;
    }
    if (k == key) { atomicAdd(&t[slot].cnt, add); return; }
    slot = (slot + 1) & (LC - 1);  // >= 2x the keys' slots: never full
  }
}

__device__ __forceinline__ void tn_upsert(NSlot* t, u64 NC, u32* esc, u32 node, u32 p, u32 f, bool cas_first = false) {
  if (node == EMPTY32) { atomicAdd(&esc[0], p); atomicAdd(&esc[1], f); return; }
  u64 slot = ((u64)hash32(node) * 0x9E3779B97F4A7C15ull >> 11) & (NC - 1);
  const u128 empty = (u128)EMPTY32;  // {key ~0, P 0, F 0, pad 0}
  for (;;) {  // claim with the first packets and links in one 128-bit CAS (the probe, when cas_first)
    u32 k = cas_first ? EMPTY32 : ldcg32(&t[slot].key);
    if (k == EMPTY32) {
      const u128 old = atomicCAS(reinterpret_cast<u128*>(&t[slot]), empty, (u128)node | ((u128)p << 32) | ((u128)f << 64));
      if (old == empty) return;
      k = (u32)old;
    }
    if (k == node) { atomicAdd(&t[slot].P, p); atomicAdd(&t[slot].F, f); return; }
    slot = (slot + 1) & (NC - 1);
  }
}

// ---- partition (world > 1): counts per (CTA, owner), then a scatter into owner-contiguous segments
__global__ void __launch_bounds__(TT) trace_part_count(const u64* __restrict__ keys, const u32* __restrict__ src,
                                                       const u32* __restrict__ dst, u64 n, u32 world,
                                                       u32* __restrict__ ccount) {
  __shared__ u32 h[TRACE_MAX_WORLD];
  for (u32 o = threadIdx.x; o < world; o += TT) h[o] = 0;
  __syncthreads();
  u64 lo, hi;
  cta_range(n, lo, hi);
  for (u64 i = lo + threadIdx.x; i < hi; i += TT) atomicAdd(&h[link_owner(load_key(keys, src, dst, i), world)], 1u);
  __syncthreads();
  for (u32 o = threadIdx.x; o < world; o += TT) ccount[(u64)blockIdx.x * world + o] = h[o];
}

// Exclusive offsets in (owner-major, CTA-minor) order for `sides` independent count tables
// ccount[b][side][o] -> coff[b][side][o]; totals[side][o].  One CTA of 1024 threads scans the world*grid
// counts of each side in chunks of 1024 (element e = o * grid + b).
__global__ void __launch_bounds__(TRACE_MAX_WORLD) trace_scan(const u32* __restrict__ ccount, u32 grid, u32 sides,
                                                              u32 world, u64* __restrict__ coff, u64* __restrict__ totals) {
  __shared__ u64 wsum[32];
  __shared__ u64 carry;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const u64 ne = (u64)world * grid;
  for (u32 sd = 0; sd < sides; ++sd) {
    if (t == 0) carry = 0;
    __syncthreads();
    for (u64 e0 = 0; e0 < ne; e0 += TRACE_MAX_WORLD) {
      const u64 e = e0 + t;
      const u32 o = (u32)(e / grid), b = (u32)(e - (u64)o * grid);
      const u64 idx = ((u64)b * sides + sd) * world + o;
      const u64 v = e < ne ? ccount[idx] : 0;
      u64 x = v;
#pragma unroll
      for (int k = 1; k < 32; k <<= 1) {
        const u64 y = __shfl_up_sync(0xffffffffu, x, k);
        if (lane >= k) x += y;
      }
      if (lane == 31) wsum[wid] = x;
      __syncthreads();
      if (wid == 0) {
        u64 w = wsum[lane];
#pragma unroll
        for (int k = 1; k < 32; k <<= 1) {
          const u64 y = __shfl_up_sync(0xffffffffu, w, k);
          if (lane >= k) w += y;
        }
        wsum[lane] = w;
      }
      __syncthreads();
      const u64 incl = x + (wid ? wsum[wid - 1] : 0ull) + carry;
      if (e < ne) coff[idx] = incl - v;
      __syncthreads();
      if (t == TRACE_MAX_WORLD - 1) carry = incl;
      __syncthreads();
    }
  }
  // totals per (side, owner): the difference of consecutive owner starts (totals may be NULL)
  if (totals)
  for (u32 sd = 0; sd < sides; ++sd)
    for (u32 o = t; o < world; o += TRACE_MAX_WORLD) {
      const u64 first = coff[((u64)0 * sides + sd) * world + o];
      const u64 lastb = (u64)(grid - 1);
      const u64 li = (lastb * sides + sd) * world + o;
      totals[(u64)sd * world + o] = coff[li] + ccount[li] - first;
    }
}

// Destination of owner o's segment: this rank's local array (out, at the scan's offsets), or, for the
// fused exchange, owner o's receive buffer in peer memory (peers[o], mapped here through CUDA IPC) at
// pbase[o] (where this rank's segment starts there, from the all-gathered counts): every store of the
// scatter then goes straight over NVLink into the owner's buffer.
__device__ __forceinline__ u64* seg_ptr(u64* out, u64* const* peers, const u64* pbase, u64 seg_start, u32 o) {
  return peers ? peers[o] + pbase[o] - seg_start : out;
}

__global__ void __launch_bounds__(TT) trace_part_scatter(const u64* __restrict__ keys, const u32* __restrict__ src,
                                                         const u32* __restrict__ dst, u64 n, u32 world,
                                                         const u64* __restrict__ coff, u64* __restrict__ out,
                                                         u64* const* __restrict__ peers, const u64* __restrict__ pbase) {
  // per owner: the CTA's u64 base (from the scan), a 32-bit local cursor (a CTA range has < 2^32 rows) and
  // the segment's destination pointer
  __shared__ u64 base[TRACE_MAX_WORLD];
  __shared__ u64* dstp[TRACE_MAX_WORLD];
  __shared__ u32 cur[TRACE_MAX_WORLD];
  for (u32 o = threadIdx.x; o < world; o += TT) {
    base[o] = coff[(u64)blockIdx.x * world + o];
    dstp[o] = seg_ptr(out, peers, pbase, coff[o], o);  // coff[0][o]: owner o's segment start
    cur[o] = 0;
  }
  __syncthreads();
  u64 lo, hi;
  cta_range(n, lo, hi);
  for (u64 i = lo + threadIdx.x; i < hi; i += TT) {
    const u64 k = load_key(keys, src, dst, i);
    const u32 o = link_owner(k, world);
    dstp[o][base[o] + atomicAdd(&cur[o], 1u)] = k;
  }
}

// ---- links: A restricted to this rank's keys in a global table, then records per side and owner
// Each CTA first aggregates in a direct-mapped SMEM cache (slot = top bits of an independent multiplicative
// mix of the key): a packet whose key holds (or claims) its cache slot costs one SMEM atomic, so hot
// links (Zipf) do not serialise on one global counter; the rest go to the global table at once, and the
// cache is flushed (one global upsert per cached key) at the end.  Every packet is counted exactly once.
constexpr int TCACHE = 4096;
__global__ void __launch_bounds__(TT) trace_link_insert(const u64* __restrict__ keys, const u32* __restrict__ src,
                                                        const u32* __restrict__ dst, u64 n, LSlot* __restrict__ lt,
                                                        u64 LC, u32* __restrict__ esc, const u32* __restrict__ wgt = nullptr) {
  // wgt: weighted rows (n_packets per row; 0 adds nothing), NULL for raw packets
  const bool cas_first = LC >= g_trace_cas_first_slots;
  __shared__ u64 ck[TCACHE];
  __shared__ u32 cc[TCACHE];
  for (int i = threadIdx.x; i < TCACHE; i += TT) { ck[i] = EMPTY64; cc[i] = 0; }
  __syncthreads();
  for (u64 i = (u64)blockIdx.x * TT + threadIdx.x; i < n; i += (u64)gridDim.x * TT) {
    const u32 a = wgt ? wgt[i] : 1u;
    if (a == 0) continue;
    const u64 k = load_key(keys, src, dst, i);
    if (k == EMPTY64) { atomicAdd(esc, a); continue; }  // the key ~0 is kept outside the table (reading R6)
    const u32 cs = (u32)((k * 0x9E3779B97F4A7C15ull) >> 52);  // an independent mix: owner and table use hash64
    u64 cur = ck[cs];
    if (cur == EMPTY64) {
      cur = atomicCAS(reinterpret_cast<unsigned long long*>(&ck[cs]), EMPTY64, k);
      if (cur == EMPTY64) cur = k;
    }
    if (cur == k) atomicAdd(&cc[cs], a);
    else tl_insert(lt, LC, k, a, cas_first);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < TCACHE; i += TT)
    if (ck[i] != EMPTY64) tl_insert(lt, LC, ck[i], cc[i], cas_first);
}

// Per CTA slot range: link statistics (valid = sum of counts, unique links, max link; PAPER.md:180, :181,
// :183) into acc[0..2] and the record counts per (side, owner) into ccount[b][2][world].  CTA 0 also
// accounts the escaped key ~0 (esc[0] packets).
__global__ void __launch_bounds__(TT) trace_link_count(const LSlot* __restrict__ lt, u64 LC,
                                                       const u32* __restrict__ esc, u32 world,
                                                       u32* __restrict__ ccount, unsigned long long* __restrict__ acc) {
  __shared__ u32 h[2][TRACE_MAX_WORLD];
  __shared__ unsigned long long s_sum, s_links, s_max;
  for (u32 o = threadIdx.x; o < world; o += TT) { h[0][o] = 0; h[1][o] = 0; }
  if (threadIdx.x == 0) { s_sum = 0; s_links = 0; s_max = 0; }
  __syncthreads();
  u64 lo, hi;
  cta_range(LC, lo, hi);
  unsigned long long sm = 0, nl = 0;
  u32 mx = 0;
  for (u64 i = lo + threadIdx.x; i < hi; i += TT) {
    const ulonglong2 e = __ldcg(reinterpret_cast<const ulonglong2*>(lt) + i);
    const u64 k = e.x;
    if (k != EMPTY64) {
      const u32 c = (u32)e.y;
      sm += c; nl += 1; mx = max(mx, c);
      atomicAdd(&h[0][node_owner((u32)(k >> 32), world)], 1u);
      atomicAdd(&h[1][node_owner((u32)k, world)], 1u);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && esc[0]) {
    const u32 c = esc[0];
    sm += c; nl += 1; mx = max(mx, c);
    atomicAdd(&h[0][node_owner(EMPTY32, world)], 1u);
    atomicAdd(&h[1][node_owner(EMPTY32, world)], 1u);
  }
  if (sm) atomicAdd(&s_sum, sm);
  if (nl) atomicAdd(&s_links, nl);
  if (mx) atomicMax(&s_max, (unsigned long long)mx);
  __syncthreads();
  for (u32 o = threadIdx.x; o < world; o += TT) {
    ccount[((u64)blockIdx.x * 2 + 0) * world + o] = h[0][o];
    ccount[((u64)blockIdx.x * 2 + 1) * world + o] = h[1][o];
  }
  if (threadIdx.x == 0) {
    if (s_sum) atomicAdd(&acc[0], s_sum);
    if (s_links) atomicAdd(&acc[1], s_links);
    if (s_max) atomicMax(&acc[2], s_max);
  }
}

__device__ __forceinline__ u64 link_rec(u32 node, u32 c) { return ((u64)node << 32) | c; }

__global__ void __launch_bounds__(TT) trace_link_emit(const LSlot* __restrict__ lt, u64 LC,
                                                      const u32* __restrict__ esc, u32 world,
                                                      const u64* __restrict__ coff, u64* __restrict__ rec_src_local,
                                                      u64* __restrict__ rec_dst_local, u64* const* __restrict__ peers_src,
                                                      u64* const* __restrict__ peers_dst, const u64* __restrict__ pbase_src,
                                                      const u64* __restrict__ pbase_dst) {
  __shared__ u64 base[2][TRACE_MAX_WORLD];
  __shared__ u64* dstp[2][TRACE_MAX_WORLD];
  __shared__ u32 cur[2][TRACE_MAX_WORLD];
  for (u32 o = threadIdx.x; o < world; o += TT) {
    base[0][o] = coff[((u64)blockIdx.x * 2 + 0) * world + o];
    base[1][o] = coff[((u64)blockIdx.x * 2 + 1) * world + o];
    dstp[0][o] = seg_ptr(rec_src_local, peers_src, pbase_src, coff[(u64)0 * world + o], o);
    dstp[1][o] = seg_ptr(rec_dst_local, peers_dst, pbase_dst, coff[(u64)1 * world + o], o);
    cur[0][o] = 0;
    cur[1][o] = 0;
  }
  __syncthreads();
  u64 lo, hi;
  cta_range(LC, lo, hi);
  for (u64 i = lo + threadIdx.x; i < hi; i += TT) {
    const ulonglong2 e = __ldcg(reinterpret_cast<const ulonglong2*>(lt) + i);
    const u64 k = e.x;
    if (k != EMPTY64) {
      const u32 c = (u32)e.y;
      const u32 s = (u32)(k >> 32), d = (u32)k;
      const u32 os = node_owner(s, world), od = node_owner(d, world);
      dstp[0][os][base[0][os] + atomicAdd(&cur[0][os], 1u)] = link_rec(s, c);
      dstp[1][od][base[1][od] + atomicAdd(&cur[1][od], 1u)] = link_rec(d, c);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && esc[0]) {
    const u32 o = node_owner(EMPTY32, world);
    dstp[0][o][base[0][o] + atomicAdd(&cur[0][o], 1u)] = link_rec(EMPTY32, esc[0]);
    dstp[1][o][base[1][o] + atomicAdd(&cur[1][o], 1u)] = link_rec(EMPTY32, esc[0]);
  }
}

// ---- one rank (nsg_trace_stats): statistics and records in a single pass over the link table.  Each
// CTA walks its slot range in tiles of TT*8 slots; a tile's links get consecutive record positions from
// one global cursor (one atomic per tile), the same position on both sides.
__global__ void __launch_bounds__(TT) trace_link_emit1(const LSlot* __restrict__ lt, u64 LC,
                                                       const u32* __restrict__ esc, u64* __restrict__ rec_src,
                                                       u64* __restrict__ rec_dst, unsigned long long* __restrict__ cursor,
                                                       unsigned long long* __restrict__ acc) {
  constexpr int PER = 8;
  __shared__ u32 wsum[TT / 32];
  __shared__ unsigned long long tile_base, s_sum, s_links, s_max;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  if (t == 0) { s_sum = 0; s_links = 0; s_max = 0; }
  u64 lo, hi;
  cta_range(LC, lo, hi);
  unsigned long long sm = 0, nl = 0;
  u32 mx = 0;
  for (u64 t0 = lo; t0 < hi; t0 += (u64)TT * PER) {
    ulonglong2 e[PER];
    u32 cnt = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const u64 i = t0 + (u64)t * PER + q;
      e[q] = i < hi ? __ldcg(reinterpret_cast<const ulonglong2*>(lt) + i) : make_ulonglong2(EMPTY64, 0ull);
      cnt += e[q].x != EMPTY64;
    }
    u32 x = cnt;  // block exclusive scan of the per-thread link counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      u32 w = lane < TT / 32 ? wsum[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      if (lane < TT / 32) wsum[lane] = w;
      if (lane == TT / 32 - 1) tile_base = w ? atomicAdd(cursor, (unsigned long long)w) : 0ull;
    }
    __syncthreads();
    u64 pos = tile_base + (x - cnt) + (wid ? wsum[wid - 1] : 0u);
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      if (e[q].x == EMPTY64) continue;
      const u32 c = (u32)e[q].y;
      sm += c; nl += 1; mx = max(mx, c);
      rec_src[pos] = link_rec((u32)(e[q].x >> 32), c);
      rec_dst[pos] = link_rec((u32)e[q].x, c);
      ++pos;
    }
    __syncthreads();  // wsum / tile_base are reused by the next tile
  }
  if (blockIdx.x == 0 && t == 0 && esc[0]) {  // the escaped key ~0 -> ~0
    const u32 c = esc[0];
    sm += c; nl += 1; mx = max(mx, c);
    const u64 p = atomicAdd(cursor, 1ull);
    rec_src[p] = link_rec(EMPTY32, c);
    rec_dst[p] = link_rec(EMPTY32, c);
  }
  if (sm) atomicAdd(&s_sum, sm);
  if (nl) atomicAdd(&s_links, nl);
  if (mx) atomicMax(&s_max, (unsigned long long)mx);
  __syncthreads();
  if (t == 0) {
    if (s_sum) atomicAdd(&acc[0], s_sum);
    if (s_links) atomicAdd(&acc[1], s_links);
    if (s_max) atomicMax(&acc[2], s_max);
  }
}

// ---- nodes: merge the records of one side; unique nodes, max packets (:186), max fan (:188)
// Records of a node are merged in a per-CTA SMEM cache first, as trace_link_insert does for links (hot
// sources / destinations would otherwise serialise on one global counter).
__device__ __forceinline__ void node_records(const u64* __restrict__ rec, u64 m, NSlot* __restrict__ nt, u64 NC,
                                             u32* __restrict__ esc, u32* ck, u32* cp, u32* cf) {
  for (int i = threadIdx.x; i < TCACHE; i += TT) { ck[i] = EMPTY32; cp[i] = 0; cf[i] = 0; }
  __syncthreads();
  for (u64 i = (u64)blockIdx.x * TT + threadIdx.x; i < m; i += (u64)gridDim.x * TT) {
    const u64 r = rec[i];
    const u32 node = (u32)(r >> 32), c = (u32)r;
    if (node == EMPTY32) { atomicAdd(&esc[0], c); atomicAdd(&esc[1], 1u); continue; }
    const u32 cs = (node * 0x9E3779B1u) >> (32 - 12);  // independent of the owner / table hashes (hash32)
    u32 cur = ck[cs];
    if (cur == EMPTY32) {
      cur = atomicCAS(&ck[cs], EMPTY32, node);
      if (cur == EMPTY32) cur = node;
    }
    if (cur == node) { atomicAdd(&cp[cs], c); atomicAdd(&cf[cs], 1u); }
    else tn_upsert(nt, NC, esc, node, c, 1u, NC >= g_trace_cas_first_slots);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < TCACHE; i += TT)
    if (ck[i] != EMPTY32) tn_upsert(nt, NC, esc, ck[i], cp[i], cf[i], NC >= g_trace_cas_first_slots);
}
static_assert(TCACHE == 4096, "node cache slot uses 12 hash bits");

__global__ void __launch_bounds__(TT) trace_node_insert(const u64* __restrict__ rec, u64 m, NSlot* __restrict__ nt,
                                                        u64 NC, u32* __restrict__ esc) {
  __shared__ u32 ck[TCACHE], cp[TCACHE], cf[TCACHE];
  node_records(rec, m, nt, NC, esc, ck, cp, cf);
}

// the same, with the record count read from device memory (single-rank trace: no host sync)
__global__ void __launch_bounds__(TT) trace_node_insert_dev(const u64* __restrict__ rec, const u64* __restrict__ m_dev,
                                                            NSlot* __restrict__ nt, u64 NC, u32* __restrict__ esc) {
  __shared__ u32 ck[TCACHE], cp[TCACHE], cf[TCACHE];
  node_records(rec, *m_dev, nt, node_cap(NC, m_dev), esc, ck, cp, cf);
}

__global__ void __launch_bounds__(TT) trace_node_scan(const NSlot* __restrict__ nt, u64 NC, const u32* __restrict__ esc,
                                                      unsigned long long* __restrict__ acc,
                                                      const u64* __restrict__ m_dev = nullptr) {
  NC = node_cap(NC, m_dev);
  __shared__ unsigned long long s_n, s_p, s_f;
  if (threadIdx.x == 0) { s_n = 0; s_p = 0; s_f = 0; }
  __syncthreads();
  unsigned long long nn = 0;
  u32 mp = 0, mf = 0;
  for (u64 i = (u64)blockIdx.x * TT + threadIdx.x; i < NC; i += (u64)gridDim.x * TT) {
    const uint4 e = __ldcg(reinterpret_cast<const uint4*>(nt) + i);
    if (e.x != EMPTY32) { nn += 1; mp = max(mp, e.y); mf = max(mf, e.z); }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && esc[1]) { nn += 1; mp = max(mp, esc[0]); mf = max(mf, esc[1]); }
  if (nn) atomicAdd(&s_n, nn);
  if (mp) atomicMax(&s_p, (unsigned long long)mp);
  if (mf) atomicMax(&s_f, (unsigned long long)mf);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_n) atomicAdd(&acc[0], s_n);
    if (s_p) atomicMax(&acc[1], s_p);
    if (s_f) atomicMax(&acc[2], s_f);
  }
}

// out[9] (north_star order) from the link partial [valid, links, max link] and the two node partials
__global__ void trace_finish(const unsigned long long* __restrict__ lacc, const unsigned long long* __restrict__ sacc,
                             const unsigned long long* __restrict__ dacc, u64* __restrict__ out) {
  if (threadIdx.x == 0) {
    out[NSG_VALID_PACKETS] = lacc[0];
    out[NSG_UNIQUE_LINKS] = lacc[1];
    out[NSG_MAX_LINK_PACKETS] = lacc[2];
    out[NSG_UNIQUE_SOURCES] = sacc[0];
    out[NSG_MAX_SOURCE_PACKETS] = sacc[1];
    out[NSG_MAX_SOURCE_FANOUT] = sacc[2];
    out[NSG_UNIQUE_DESTINATIONS] = dacc[0];
    out[NSG_MAX_DESTINATION_PACKETS] = dacc[1];
    out[NSG_MAX_DESTINATION_FANIN] = dacc[2];
  }
}

}  // namespace nsg
