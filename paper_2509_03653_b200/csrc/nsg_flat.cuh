// nsg_flat.cuh — the per-window statistics kernels of libnsg (round 2), windows <= 2^17.
//
// What it computes: for every window of W consecutive packets, the nine Table 2 scalars of the
// traffic matrix A_t (destination mirrors, line 173): valid packets (:180),
// unique links (:181), max link packets (:183), unique sources (:184), max source packets (:186), max
// source fan-out (:188) and the three destination mirrors; optionally the vector-valued rows (:182,
// :185, :187) and the four IP-set counts (:209).  Readings: DESIGN.md §2.
//
// How: three flat kernels per batch of 32 windows, one work item per CTA, several CTAs
// resident per SM so that the latency chains of independent items overlap:
//   part  (w, c)   4096 keys of window w (128-bit loads, L2 evict-first), counting-sorted by link bucket
//                  (top bits of key * phi64) into the batch's key scratch; one row of segment
//                  descriptors per item;
//   link  (w, b)   link bucket b (~1024 keys): each warp gathers its share of the chunks' segments
//                  straight into registers and inserts two keys per lane in lockstep into a 2048-slot
//                  SMEM table (A_t restricted to the bucket); a key that claims a free slot is a new link:
//                  it is listed (claim list) and counted in its two node buckets' histograms right then.
//                  The list gives unique links, max link, count sum (-> window accumulators) and one
//                  record (node << 32 | count) per link and side, stored by node bucket into the
//                  bucket's record row;
//   side  (w,s,q)  node bucket q of side s: the records of every link bucket merged per node in a
//                  4096-slot SMEM table of (node, packets | fan << 20); unique nodes (claimed slots), max
//                  packets and max fan come from the adds' return values (no table scan) -> window
//                  accumulators; the last side item of a window writes its row.
// Tables are probed with a plain load first (a hot key's repeats cost a broadcast read and an
// aggregated increment, never a CAS); collisions probe on with double hashing (odd steps).
#pragma once
#include "nsg_internal.h"
#include "nsg_common.cuh"

namespace nsg {
namespace flat {

constexpr int CH = 4096;                      // keys per partition item
constexpr int PTH = 256;                      // partition CTA threads
constexpr int LTH = 256;                      // link CTA threads
#ifndef NSG_STH
#define NSG_STH 256
#endif
constexpr int STH = NSG_STH;                  // side CTA threads
constexpr u64 BK = 1024;                      // target keys per link bucket / nodes per side bucket
constexpr u64 MAX_W = 1ull << 17;             // windows this path takes (<= 128 link / side buckets)
constexpr int MAXB = (int)(MAX_W / BK);          // link buckets of the largest window (= 2 x node buckets)
constexpr int LOG_TL = 11, TL = 1 << LOG_TL;  // link-table slots (load <= 5/8)
constexpr int LOG_TS = 12, TS = 1 << LOG_TS;  // node-table slots
constexpr u32 FILL_L = 1280;                  // distinct links of a bucket before the window goes to the L2 path
constexpr u32 RCAP = (2 * (FILL_L + 1) + 15) & ~15u;  // records per link bucket (both sides), whole lines
constexpr int PFS = 20;                       // node packets: 20-bit field (W < 2^20)
constexpr u32 PMASK = (1u << PFS) - 1;
constexpr u32 FMAX = 0xFFFu;                  // fan field: 12 bits; items with >= 4096 records track wraps
constexpr int WRAPCAP = 64;
#ifndef NSG_HEAVY_S
#define NSG_HEAVY_S 8192
#endif
constexpr u32 HEAVY_S = NSG_HEAVY_S;          // side items with more records cache a hot node per warp
#ifndef NSG_AGG_T
#define NSG_AGG_T 128
#endif
constexpr u32 AGG_T = NSG_AGG_T;              // a link bucket's node-bucket group with this many links sends one
                                              // record per node (P, F) instead of one per link (heavy hitters)
constexpr int LOG_TA = 7, TA = 1 << LOG_TA;   // per-side aggregation table slots of a link item
constexpr u64 MUL_L = 0x9E3779B97F4A7C15ull;  // link hash: top bits of key * phi64
constexpr u32 MUL_N = 0x9E3779B9u;            // node hash: top bits of node * phi32
static_assert((RCAP * 8) % 128 == 0, "record rows are whole 128-B lines (16-B stores, L2 discards)");

// Per-window state (64 B), zeroed by the host before the launches.
struct WinState {
  u32 sdone, ovf, links, maxc, sumc, vfill[3];  // vfill: vector entries reserved (links, sources, destinations)
  u32 nodes[2], maxp[2], maxf[2], both, wtot;   // both: |S n D| (IP sets); wtot: sum of n_packets (weighted rows)
};
static_assert(sizeof(WinState) == 64, "WinState is 64 B");

struct FGeo {
  u64 n, W, nw;
  u64 w0;                          // first window of the batch
  u32 nbw;                         // windows in the batch
  u32 logB, B, logBs, Bs, CP;
  WinState* ws;                    // [nw]
  u64* kscr;                       // [nbw][CP][CH]
  const u32* wgt;                  // weighted rows: n_packets per row (NULL: raw packets, weight 1)
  u32* wscr;                       // [nbw][CP][CH] the keys' weights, in kscr order (weighted rows)
  u32* koff;                       // [nbw][CP][B]    start << 16 | count of bucket b in chunk c
  u64* rscr;                       // [nbw][B][RCAP]
  u32* roff;                       // [nbw][B][2Bs]   start << 16 | count of side bucket (s,q) in link bucket b
  u32* diag;                       // [0] windows handed to the L2 path, [1] self-check failures,
                                   // [3] heavy groups aggregated
  u64* const* mirror;
  u32 n_mirror;
  u64 mirror_row0;
  u32 inject;                      // bit 0 NSG_FLAG_INJECT_OVERFLOW: odd windows are handed to the L2 path;
                                   // bit 1 NSG_FLAG_INJECT_SELF_CHECK: window 0 counts a self-check failure
  // nsg_window_vectors (NULL = not requested): window w's entries at [w*W, w*W + count) in reservation order
  u64* v_lkey;
  u32* v_lpk;
  u32* v_node[2];
  u32* v_pk[2];
  u32* v_fan[2];
  u64* v_ipsets;                   // [nw][4]
  u32* ipl;                        // [nbw][Bs][TS] side-0 node lists (IP sets)
  u32* ipc;                        // [nbw][Bs] side-0 list length + 1 (0 = not yet published) | esc << 31
};

__device__ __forceinline__ u32 link_bucket(u64 key, u32 logB) { return logB ? (u32)((key * MUL_L) >> (64 - logB)) : 0u; }
__device__ __forceinline__ u32 link_slot(u64 key, u32 logB) {
  return (u32)((key * MUL_L) >> (64 - logB - LOG_TL)) & (TL - 1);
}
__device__ __forceinline__ u32 link_step(u64 key) { return ((u32)(key * MUL_L) >> 9) | 1u; }  // odd
__device__ __forceinline__ u32 node_bucket(u32 node, u32 logBs) { return logBs ? (node * MUL_N) >> (32 - logBs) : 0u; }
__device__ __forceinline__ u32 node_slot(u32 node, u32 logBs) {
  return ((node * MUL_N) >> (32 - logBs - LOG_TS)) & (TS - 1);
}
__device__ __forceinline__ u32 node_step(u32 node) { return ((node * 0x85ebca6bu) >> 7) | 1u; }


// Input keys are read once: loaded with an L2 evict-first policy so that the stream does not push the
// (dirty, L2-resident) scratch of the batch pipeline out to HBM.
__device__ __forceinline__ u64 l2_evict_first() {
  u64 pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ u64 ld_stream64(const u64* p, u64 pol) {
  u64 v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ ulonglong2 ld_stream128(const u64* p, u64 pol) {
  ulonglong2 v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.u64 {%0,%1}, [%2], %3;" : "=l"(v.x), "=l"(v.y) : "l"(p), "l"(pol));
  return v;
}

// exclusive scan of (h[i] & mask), i < n, by one warp into o[0, n); fn(i, excl, count) for every
// entry; returns the total
template <class F>
__device__ __forceinline__ u32 warp_exscan(const u32* h, u32* o, u32 n, int lane, F fn, u32 mask = 0xFFFFFFFFu) {
  u32 carry = 0;
  for (u32 b0 = 0; b0 < n; b0 += 32) {
    const u32 i = b0 + lane;
    const u32 v = i < n ? (h[i] & mask) : 0u;
    u32 x = v;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, x, k);
      if (lane >= k) x += y;
    }
    const u32 ex = carry + x - v;
    if (i < n) { o[i] = ex; fn(i, ex, v); }
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  return carry;
}


__device__ __forceinline__ u64 warp_sum64(u64 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void warp_reduce4(u32& a, u32& b, u32& c, u32& d) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    c = max(c, __shfl_xor_sync(0xffffffffu, c, o));
    d += __shfl_xor_sync(0xffffffffu, d, o);
  }
}

template <int NTH>
__device__ __forceinline__ void copy_out(u64* __restrict__ dstp, const u64* st, u32 n) {
  const int t = threadIdx.x;
  if ((reinterpret_cast<uintptr_t>(dstp) & 15) == 0) {
    for (u32 e = 2 * t; e + 1 < n; e += 2 * NTH) {
      const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(st + e);
      *reinterpret_cast<ulonglong2*>(dstp + e) = v;
    }
    if ((n & 1u) && t == 0) dstp[n - 1] = st[n - 1];
  } else {
    for (u32 e = t; e < n; e += NTH) dstp[e] = st[e];
  }
}

// ---------------------------------------------------------------------------------------------
// Warp-owned gathers: warp v of the CTA owns segments v, v + NW, ... of an item (its share of the
// chunks / link buckets) and walks their concatenation 64 elements per step, loading each element
// straight from L2 into a register.  The segment list lives in registers (lane k: the warp's k-th
// non-empty segment), so locating an element's segment is a few bit operations, no search.  The
// inserts need no CTA barrier: a slot only ever goes from free to a key, so concurrent inserts from
// other warps are safe, and one barrier ends the whole insert phase.
// ---------------------------------------------------------------------------------------------
struct WarpSegs {
  u32 n;      // elements of the warp's concatenation
  u32 nseg;   // non-empty segments owned (<= 32)
  u32 pre;    // lane k < nseg: first element of segment k in the concatenation
  u32 d;      // lane k < nseg: element offset of segment k's storage minus pre
  u32 kb;     // segments that start before the current step
};

// desc(i) = start << 16 | count of segment i (i < nall), row(i) = element offset of segment i's row;
// scr: 64 words of this warp's shared memory (the non-empty segments are compacted through it); mid()
// runs while the descriptors are loading (the item's table initialisation hides their L2 latency).
template <class D, class R, class M>
__device__ __forceinline__ WarpSegs warp_segs(u32 nall, u32 nwarps, u32* scr, D desc, R row, M mid) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const u32 nraw = nall > (u32)wid ? (nall - 1 - wid) / nwarps + 1 : 0u;  // <= 32 by construction
  const u32 i = wid + lane * nwarps;
  const u32 v = (u32)lane < nraw ? desc(i) : 0u;
  mid();
  const u32 cnt = v & 0xFFFFu;
  u32 x = cnt;
#pragma unroll
  for (int k = 1; k < 32; k <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, x, k);
    if (lane >= k) x += y;
  }
  const u32 m = __ballot_sync(0xffffffffu, cnt != 0);
  if (cnt) {
    const u32 r = __popc(m & ((1u << lane) - 1u));
    scr[r] = x - cnt;
    scr[32 + r] = row(i) + (v >> 16) - (x - cnt);
  }
  __syncwarp();
  WarpSegs r;
  r.nseg = __popc(m);
  r.pre = scr[lane];
  r.d = scr[32 + lane];
  r.n = __shfl_sync(0xffffffffu, x, 31);
  r.kb = 0;
  return r;
}

// Element offsets of elements e0 + lane and e0 + 32 + lane (callers check e < n); advances ws.kb.
__device__ __forceinline__ void warp_seg_step(WarpSegs& ws, u32 e0, u32& oa, u32& ob) {
  const int lane = threadIdx.x & 31;
  const u32 rel = ((u32)lane < ws.nseg && ws.pre >= e0) ? ws.pre - e0 : 64u;
  const u32 mlo = __reduce_or_sync(0xffffffffu, rel < 32 ? 1u << rel : 0u);
  const u32 mhi = __reduce_or_sync(0xffffffffu, rel - 32 < 32 ? 1u << (rel - 32) : 0u);
  const u32 le = (2u << lane) - 1u;  // bits 0..lane
  const u32 ka = ws.kb + __popc(mlo & le) - 1;
  const u32 kb = ws.kb + __popc(mlo) + __popc(mhi & le) - 1;
  oa = __shfl_sync(0xffffffffu, ws.d, ka & 31) + e0 + lane;
  ob = __shfl_sync(0xffffffffu, ws.d, kb & 31) + e0 + 32 + lane;
  ws.kb += __popc(mlo) + __popc(mhi);
}

// ---------------------------------------------------------------------------------------------
// part(w, c): counting sort of one chunk by link bucket
// ---------------------------------------------------------------------------------------------
struct SmemP {
  u64 stage[CH];
  u32 hist[MAXB], offs[MAXB];
  u32 wraw[CH], wstage[CH];        // weighted rows only: the chunk's weights in row order, then sorted
};
// part_kernel<false> is launched with only the shared memory before wraw (33 KB instead of 66 KB)
__host__ __device__ constexpr size_t part_smem(bool wt) { return wt ? sizeof(SmemP) : offsetof(SmemP, wraw); }
constexpr u32 WTOT_MAX = 1u << 20;  // weighted windows summing to this or more go to the L2 path (20-bit packets)

template <bool WT>
#ifndef NSG_PART_MINB
#define NSG_PART_MINB 3
#endif
__global__ void __launch_bounds__(PTH, NSG_PART_MINB)
part_kernel(const FGeo g, const u32* __restrict__ src, const u32* __restrict__ dst, const u64* __restrict__ keys) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SmemP& s = *reinterpret_cast<SmemP*>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const u32 wb = blockIdx.x / g.CP, c = blockIdx.x % g.CP;
  const u64 w = g.w0 + wb;
  const u64 len = min(g.W, g.n - w * g.W);
  const u64 c0 = (u64)c * CH;
  const u32 n = c0 < len ? (u32)min((u64)CH, len - c0) : 0u;
  const u64 base = w * g.W + c0;
  const u32 B = g.B, logB = g.logB;
  for (u32 i = t; i < B; i += PTH) s.hist[i] = 0;
  constexpr int KPT = CH / PTH;
  u64 kk[KPT];
  const u64 pol = l2_evict_first();
  if (keys) {
    const u64* p = keys + base;
    if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < KPT / 2; ++i) {
        const u32 e = 2 * (i * PTH + t);
        if (e + 1 < n) {
          const ulonglong2 v = ld_stream128(p + e, pol);
          kk[2 * i] = v.x; kk[2 * i + 1] = v.y;
        } else {
          kk[2 * i] = e < n ? ld_stream64(p + e, pol) : 0ull;
          kk[2 * i + 1] = 0ull;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < KPT / 2; ++i) {
        const u32 e = 2 * (i * PTH + t);
        kk[2 * i] = e < n ? ld_stream64(p + e, pol) : 0ull;
        kk[2 * i + 1] = e + 1 < n ? ld_stream64(p + e + 1, pol) : 0ull;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < KPT / 2; ++i) {
      const u32 e = 2 * (i * PTH + t);
      kk[2 * i] = e < n ? ((u64)__ldcs(src + base + e) << 32) | __ldcs(dst + base + e) : 0ull;
      kk[2 * i + 1] = e + 1 < n ? ((u64)__ldcs(src + base + e + 1) << 32) | __ldcs(dst + base + e + 1) : 0ull;
    }
  }
  u32 zero = 0;  // weighted rows: bit i = row of element i has n_packets 0 (it adds nothing: dropped)
  if (WT) {
    u64 wsum = 0;
    for (u32 e = t; e < CH; e += PTH) {
      const u32 x = e < n ? __ldcs(g.wgt + base + e) : 0u;
      s.wraw[e] = x;
      wsum += x;
    }
    wsum = warp_sum64(wsum);
    if (lane == 0 && wsum) atomicAdd(&g.ws[w].wtot, (u32)min(wsum, (u64)WTOT_MAX));  // saturated per warp
    __syncthreads();
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const u32 e = 2 * ((i >> 1) * PTH + t) + (i & 1);
      zero |= (e < n && s.wraw[e] == 0u ? 1u : 0u) << i;
    }
  }
  __syncthreads();  // histogram cleared
  u32 bk[KPT], rk[KPT];
#pragma unroll
  for (int i = 0; i < KPT; ++i) bk[i] = link_bucket(kk[i], logB);
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    const u32 e = 2 * ((i >> 1) * PTH + t) + (i & 1);
    rk[i] = e < n && !(zero >> i & 1u) ? atomicAdd(&s.hist[bk[i]], 1u) : 0u;
  }
  __syncthreads();
  if (wid == 0) {
    u32* ko = g.koff + ((u64)wb * g.CP + c) * B;  // this item's own row
    warp_exscan(s.hist, s.offs, B, lane, [&](u32 i, u32 ex, u32 v) { ko[i] = (ex << 16) | v; });
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    const u32 e = 2 * ((i >> 1) * PTH + t) + (i & 1);
    if (e < n && !(zero >> i & 1u)) {
      s.stage[s.offs[bk[i]] + rk[i]] = kk[i];
      if (WT) s.wstage[s.offs[bk[i]] + rk[i]] = s.wraw[e];
    }
  }
  __syncthreads();
  const u32 nz = s.offs[B - 1] + s.hist[B - 1];  // rows kept (weighted rows of weight 0 are dropped)
  copy_out<PTH>(g.kscr + ((u64)wb * g.CP + c) * CH, s.stage, nz);
  if (WT) {
    u32* wd = g.wscr + ((u64)wb * g.CP + c) * CH;
    for (u32 e = t; e < nz; e += PTH) wd[e] = s.wstage[e];
  }
}

// ---------------------------------------------------------------------------------------------
// link(w, b)
// ---------------------------------------------------------------------------------------------
struct SmemL {
  u64 lkey[TL];
  u32 lcnt[TL];
  u32 hist[MAXB], offs[MAXB];      // per (side, node bucket): 2 * Bs <= MAXB
  uint16_t claim[FILL_L];          // the bucket's occupied slots, listed as they are claimed
  union {
    u32 segscr[LTH / 32][64];      // warp_segs (before the table is initialised)
    u32 agg[2][2][TA];             // then per side: node, packets | links << 20 of the heavy groups' nodes
  };
  u32 hmask[MAXB / 32];            // heavy groups (side * Bs + node bucket with >= AGG_T links)
  u32 ncl, esc, ovf, vbase;
};
static_assert(sizeof(u32) * 2 * 2 * TA <= sizeof(u32) * (LTH / 32) * 64, "aggregation tables fit the segment scratch");

// Shared-memory slot operations on 32-bit shared-window addresses, predicated (no branch, no reconvergence
// bookkeeping around each one): p ? op : keep the register's value.
__device__ __forceinline__ u32 smem_addr(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void sld_if(bool p, u32 a, u64& v) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q ld.volatile.shared.u64 %0, [%1]; }"
               : "+l"(v) : "r"(a), "r"((u32)p) : "memory");
}
__device__ __forceinline__ void sld_if(bool p, u32 a, u32& v) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q ld.volatile.shared.u32 %0, [%1]; }"
               : "+r"(v) : "r"(a), "r"((u32)p) : "memory");
}
__device__ __forceinline__ void scas_if(bool p, u32 a, u64 cmp, u64 val, u64& old) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %4, 0; @q atom.shared.cas.b64 %0, [%1], %2, %3; }"
               : "+l"(old) : "r"(a), "l"(cmp), "l"(val), "r"((u32)p) : "memory");
}
__device__ __forceinline__ void scas_if(bool p, u32 a, u32 cmp, u32 val, u32& old) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %4, 0; @q atom.shared.cas.b32 %0, [%1], %2, %3; }"
               : "+r"(old) : "r"(a), "r"(cmp), "r"(val), "r"((u32)p) : "memory");
}

// Lockstep probe of two keys per lane: every lane advances its unfinished keys by one slot per
// iteration (a found key, or a free slot claimed by CAS, finishes it), so the warp runs as many short
// iterations as its longest probe sequence and never serialises divergent probe loops.  Every slot
// operation is predicated on the lane's key still being unfinished.
// In: tab = shared address of slot 0, slot = home slot, cur = its content, act = key valid.
// Out: slot = the key's slot.  Returns which keys this lane inserted as new (bit 0: key a claimed a free
// slot, bit 1: key b).
template <class T, class Step>
__device__ __forceinline__ u32 probe2(u32 tab, u32 mask, T ka, T kb, u32& sa, u32& sb, T ca, T cb, bool aa, bool ab,
                                      u32* ovf, Step step) {
  constexpr T EMPTY = ~T(0);
  constexpr u32 SZ = sizeof(T);
  u32 claimed = 0;
  aa = aa && ca != ka;
  ab = ab && cb != kb;
  if (!__any_sync(0xffffffffu, aa || ab)) return 0;
  const u32 pa = step(ka), pb = step(kb);
  for (u32 it = 0;; ++it) {
    const bool xa = aa && ca == EMPTY, xb = ab && cb == EMPTY;  // a free slot: claim it
    T oa = ca, ob = cb;
    scas_if(xa, tab + sa * SZ, EMPTY, ka, oa);
    scas_if(xb, tab + sb * SZ, EMPTY, kb, ob);
    claimed |= (xa && oa == EMPTY ? 1u : 0u) | (xb && ob == EMPTY ? 2u : 0u);
    ca = oa == EMPTY ? ka : oa;  // (not claimed: oa = ca)
    cb = ob == EMPTY ? kb : ob;
    aa = aa && ca != ka;
    ab = ab && cb != kb;
    if (!__any_sync(0xffffffffu, aa || ab)) break;
    if (it >= mask) {  // table full (adversarial keys only)
      if (aa || ab) *ovf = 1;
      break;
    }
    sa = aa ? (sa + pa) & mask : sa;
    sb = ab ? (sb + pb) & mask : sb;
    sld_if(aa, tab + sa * SZ, ca);
    sld_if(ab, tab + sb * SZ, cb);
  }
  return claimed;
}

// The same lockstep probe with a branch around each slot operation (the link table's 64-bit keys: measured
// faster there than the predicated form, which the side table's 32-bit keys prefer).
template <class T, class Step>
__device__ __forceinline__ u32 probe2b(T* keys, u32 mask, T ka, T kb, u32& sa, u32& sb, T ca, T cb, bool aa, bool ab,
                                       u32* ovf, Step step) {
  constexpr T EMPTY = ~T(0);
  u32 claimed = 0;
  aa = aa && ca != ka;
  ab = ab && cb != kb;
  if (!__any_sync(0xffffffffu, aa || ab)) return 0;
  const u32 pa = step(ka), pb = step(kb);
  for (u32 it = 0;; ++it) {
    if (aa && ca == EMPTY) {
      const T o = atomicCAS(&keys[sa], EMPTY, ka);
      claimed |= o == EMPTY ? 1u : 0u;
      ca = o == EMPTY ? ka : o;
    }
    if (ab && cb == EMPTY) {
      const T o = atomicCAS(&keys[sb], EMPTY, kb);
      claimed |= o == EMPTY ? 2u : 0u;
      cb = o == EMPTY ? kb : o;
    }
    aa = aa && ca != ka;
    ab = ab && cb != kb;
    if (!__any_sync(0xffffffffu, aa || ab)) break;
    if (it >= mask) {  // table full (adversarial keys only)
      if (aa || ab) *ovf = 1;
      break;
    }
    if (aa) { sa = (sa + pa) & mask; ca = *reinterpret_cast<volatile T*>(&keys[sa]); }
    if (ab) { sb = (sb + pb) & mask; cb = *reinterpret_cast<volatile T*>(&keys[sb]); }
  }
  return claimed;
}

// A heavy group's link: add (packets | 1 << 20) to its node's entry in the side's aggregation table (probing at most
// 8 slots); false if the table has no room (the link then sends its own record).
__device__ __forceinline__ bool agg_add(u32 (*tab)[TA], u32 node, u32 pf) {
  if (node == EMPTY32) return false;  // the address ~0 is the empty marker (its records go as they are)
  u32 sl = (node * MUL_N) >> (32 - LOG_TA);
  for (int k = 0; k < 8; ++k, sl = (sl + 1) & (TA - 1)) {
    u32 cur = *reinterpret_cast<volatile u32*>(&tab[0][sl]);
    if (cur == EMPTY32) {
      cur = atomicCAS(&tab[0][sl], EMPTY32, node);
      if (cur == EMPTY32) cur = node;
    }
    if (cur == node) {
      atomicAdd(&tab[1][sl], pf);
      return true;
    }
  }
  return false;
}

#ifndef NSG_LINK_MINB
#define NSG_LINK_MINB 7  // link CTAs per SM (7 x 30 KB shared memory; 32 registers)
#endif
template <bool WT>
__global__ void __launch_bounds__(LTH, NSG_LINK_MINB)
link_kernel(const FGeo g) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SmemL& s = *reinterpret_cast<SmemL*>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  constexpr u32 NW = LTH / 32;
  const u32 wb = blockIdx.x / g.B, b = blockIdx.x % g.B;
  const u64 w = g.w0 + wb;
  const u32 CP = g.CP, B = g.B, Bs = g.Bs, logBs = g.logBs, logB = g.logB;
  if (t < MAXB / 32) s.hmask[t] = 0;
  if (t == 0) {
    s.ncl = 0; s.esc = 0;
    s.ovf = WT && ldcg32(&g.ws[w].wtot) >= WTOT_MAX ? 1u : 0u;  // weighted: packets past the 20-bit fields
  }
  // this warp's share of the bucket: its segment of chunks wid, wid + NW, ...; the table is initialised
  // while the segment descriptors load
  const u32* ko = g.koff + (u64)wb * CP * B + b;
  WarpSegs ws = warp_segs(CP, NW, s.segscr[wid], [&](u32 c) { return ldcg32(ko + (u64)c * B); }, [&](u32 c) { return c * (u32)CH; },
                          [&] {
                            for (u32 i = t; i < (u32)TL / 2; i += LTH)
                              reinterpret_cast<ulonglong2*>(s.lkey)[i] = make_ulonglong2(EMPTY64, EMPTY64);
                            for (u32 i = t; i < (u32)TL / 4; i += LTH) reinterpret_cast<uint4*>(s.lcnt)[i] = make_uint4(0u, 0u, 0u, 0u);
                            for (u32 i = t; i < 2 * Bs; i += LTH) s.hist[i] = 0;
                          });
  const u64* kb = g.kscr + (u64)wb * CP * CH;
  // the next step's keys are loaded while this step's are inserted (L2 latency off the chain); the first
  // step's load is issued before the barrier
  u64 nxa = EMPTY64, nxc = EMPTY64;
  u32 nwa = 1, nwc = 1;  // the keys' weights (weighted rows)
  const u32* wsb = WT ? g.wscr + (u64)wb * CP * CH : nullptr;
  auto fetch = [&](u32 e0) {
    u32 oa, ob;
    warp_seg_step(ws, e0, oa, ob);
    nxa = e0 + lane < ws.n ? __ldcg(reinterpret_cast<const unsigned long long*>(kb + oa)) : EMPTY64;
    nxc = e0 + 32 + lane < ws.n ? __ldcg(reinterpret_cast<const unsigned long long*>(kb + ob)) : EMPTY64;
    if (WT) {
      nwa = e0 + lane < ws.n ? ldcg32(wsb + oa) : 0u;
      nwc = e0 + 32 + lane < ws.n ? ldcg32(wsb + ob) : 0u;
    }
  };
  if (ws.n) fetch(0);
  __syncthreads();  // table initialised
  {
    u32 nesc = 0;
    for (u32 e0 = 0; e0 < ws.n; e0 += 64) {
      const bool va = e0 + lane < ws.n, vb = e0 + 32 + lane < ws.n;
      const u64 ka = nxa, kc = nxc;
      const u32 wa = nwa, wc = nwc;
      if (e0 + 64 < ws.n) fetch(e0 + 64);
      if (*reinterpret_cast<volatile u32*>(&s.ovf)) break;
      const bool aa = ka != EMPTY64, ab = kc != EMPTY64;  // the key ~0 is counted apart
      nesc += (va && !aa ? wa : 0u) + (vb && !ab ? wc : 0u);
      u32 sa = link_slot(ka, logB), sb = link_slot(kc, logB);
      const u64 ca = *reinterpret_cast<volatile u64*>(&s.lkey[sa]);
      const u64 cb = *reinterpret_cast<volatile u64*>(&s.lkey[sb]);
#if NSG_LINK_PTX_PROBE
      const u32 cl = probe2<u64>(smem_addr(s.lkey), TL - 1, ka, kc, sa, sb, ca, cb, aa, ab, &s.ovf,
                                 [](u64 k) { return link_step(k); });
#else
      const u32 cl = probe2b<unsigned long long>(reinterpret_cast<unsigned long long*>(s.lkey), TL - 1, ka, kc, sa, sb,
                                                 ca, cb, aa, ab, &s.ovf, [](u64 k) { return link_step(k); });
#endif
      if (WT) {
        if (aa) atomicAdd(&s.lcnt[sa], wa);
        if (ab) atomicAdd(&s.lcnt[sb], wc);
      } else {
        if (aa) atomicAdd(&s.lcnt[sa], 1u);
        if (ab) atomicAdd(&s.lcnt[sb], 1u);
      }
      // a new link: counted in its two node buckets' histograms and listed, when its slot is claimed
      if (cl & 1u) {
        atomicAdd(&s.hist[node_bucket((u32)(ka >> 32), logBs)], 1u);
        atomicAdd(&s.hist[Bs + node_bucket((u32)ka, logBs)], 1u);
      }
      if (cl & 2u) {
        atomicAdd(&s.hist[node_bucket((u32)(kc >> 32), logBs)], 1u);
        atomicAdd(&s.hist[Bs + node_bucket((u32)kc, logBs)], 1u);
      }
      const u32 ma = __ballot_sync(0xffffffffu, cl & 1u), mb = __ballot_sync(0xffffffffu, cl & 2u);
      if (ma | mb) {
        u32 p = 0;
        if (lane == 0) p = atomicAdd(&s.ncl, __popc(ma) + __popc(mb));
        p = __shfl_sync(0xffffffffu, p, 0);
        const u32 lt = (1u << lane) - 1u;
        const u32 pa = p + __popc(ma & lt), pb = p + __popc(ma) + __popc(mb & lt);
        if ((cl & 1u) && pa < FILL_L) s.claim[pa] = (uint16_t)sa;
        if ((cl & 2u) && pb < FILL_L) s.claim[pb] = (uint16_t)sb;
      }
    }
    nesc = __reduce_add_sync(0xffffffffu, nesc);
    if (lane == 0 && nesc) atomicAdd(&s.esc, nesc);
  }
  __syncthreads();  // every key of the bucket is counted, listed and histogrammed
  const u32 ncl = s.ncl, esc = s.esc;
  const u32 eb = node_bucket(EMPTY32, logBs);
  u32* ro = g.roff + ((u64)wb * B + b) * 2 * Bs;  // this item's own row
  if (s.ovf != 0 || ncl > FILL_L) {  // more links than the records take (or a full table): L2 path
    if (t == 0) g.ws[w].ovf = 1;
    for (u32 i = t; i < 2 * Bs; i += LTH) ro[i] = 0;
    return;
  }
  const u32 nl = ncl + (esc ? 1u : 0u);  // the key ~0 (kept out of the table) is one more link
  for (u32 i = t; i < 2 * TA; i += LTH) {  // the aggregation tables (the segment scratch is dead)
    s.agg[i / TA][0][i % TA] = EMPTY32;
    s.agg[i / TA][1][i % TA] = 0u;
  }
  if (wid < 2) {  // side-0 records first, then side 1 from nl (= the number of side-0 records)
    if (lane == 0 && esc) atomicAdd(&s.hist[wid * Bs + eb], 1u);
    __syncwarp();
    u32* r = ro + wid * Bs;
    const u32 o0 = wid ? nl : 0u;
    warp_exscan(s.hist + wid * Bs, s.offs + wid * Bs, Bs, lane, [&](u32 i, u32 ex, u32 v) {
      r[i] = ((o0 + ex) << 16) | v;
      s.offs[wid * Bs + i] = o0 + ex;
      if (v >= AGG_T) {  // a heavy group: its row descriptor is rewritten after the aggregation
        atomicOr(&s.hmask[(wid * Bs + i) >> 5], 1u << ((wid * Bs + i) & 31));
        s.hist[wid * Bs + i] = o0 + ex;  // its start
      }
    });
    if (t == 0) {
      atomicAdd(&g.ws[w].links, nl);
      if (g.v_lkey) s.vbase = atomicAdd(&g.ws[w].vfill[0], nl);  // this bucket's link-vector entries
    }
  }
  __syncthreads();
  // records (node << 32 | count) straight to the item's record row, placed by side bucket with a
  // cursor per bucket (side 0 first, then side 1 from nl); max / sum of the link counts on the way
  u64* rrow = g.rscr + ((u64)wb * B + b) * RCAP;
  const bool anyh = (s.hmask[0] | s.hmask[1] | s.hmask[2] | s.hmask[3]) != 0;  // some group is heavy
  u32 mx = 0, sm = 0;
  for (u32 e = t; e < ncl; e += LTH) {
    const u32 sl = s.claim[e];
    const u32 c = s.lcnt[sl];
    const u64 key = s.lkey[sl];
    mx = max(mx, c); sm += c;
    const u32 g0 = node_bucket((u32)(key >> 32), logBs), g1 = Bs + node_bucket((u32)key, logBs);
    const u32 pf = c | (1u << PFS);  // a record: packets | links << 20 (one link)
    if (!anyh || !(s.hmask[g0 >> 5] >> (g0 & 31) & 1u) || !agg_add(s.agg[0], (u32)(key >> 32), pf))
      __stcg(reinterpret_cast<unsigned long long*>(rrow + atomicAdd(&s.offs[g0], 1u)), (key & 0xFFFFFFFF00000000ull) | pf);
    if (!anyh || !(s.hmask[g1 >> 5] >> (g1 & 31) & 1u) || !agg_add(s.agg[1], (u32)key, pf))
      __stcg(reinterpret_cast<unsigned long long*>(rrow + atomicAdd(&s.offs[g1], 1u)), (key << 32) | pf);
    if (g.v_lkey) {  // A_t(i,j) of the link
      const u64 at = w * g.W + s.vbase + e;
      g.v_lkey[at] = key;
      g.v_lpk[at] = c;
    }
  }
  if (t == 0 && esc) {
    mx = max(mx, esc); sm += esc;
    rrow[atomicAdd(&s.offs[eb], 1u)] = ((u64)EMPTY32 << 32) | esc | (1u << PFS);
    rrow[atomicAdd(&s.offs[Bs + eb], 1u)] = ((u64)EMPTY32 << 32) | esc | (1u << PFS);
    if (g.v_lkey) {
      const u64 at = w * g.W + s.vbase + ncl;
      g.v_lkey[at] = EMPTY64;
      g.v_lpk[at] = esc;
    }
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  sm = __reduce_add_sync(0xffffffffu, sm);
  if (lane == 0 && sm) {
    atomicMax(&g.ws[w].maxc, mx);
    atomicAdd(&g.ws[w].sumc, sm);
  }
  if (anyh) {  // heavy groups: one record (node, packets | links << 20) per aggregated node, then their counts
    if (t == 0)
      atomicAdd(&g.diag[3], __popc(s.hmask[0]) + __popc(s.hmask[1]) + __popc(s.hmask[2]) + __popc(s.hmask[3]));
    __syncthreads();
    for (u32 i = t; i < 2 * TA; i += LTH) {
      const u32 side = i / TA, node = s.agg[side][0][i % TA];
      if (node != EMPTY32)
        __stcg(reinterpret_cast<unsigned long long*>(rrow + atomicAdd(&s.offs[side * Bs + node_bucket(node, logBs)], 1u)),
               ((u64)node << 32) | s.agg[side][1][i % TA]);
    }
    __syncthreads();
    for (u32 q = t; q < 2 * Bs; q += LTH)
      if (s.hmask[q >> 5] >> (q & 31) & 1u) ro[q] = (s.hist[q] << 16) | (s.offs[q] - s.hist[q]);
  }
}

// ---------------------------------------------------------------------------------------------
// side(w, s, q)
// ---------------------------------------------------------------------------------------------
struct SmemS {
  u32 nkey[TS];
  u32 npf[TS];                     // packets | fan << 20
  u32 wrap[WRAPCAP];
  u32 segscr[STH / 32][64];
  u32 red[3][STH / 32];
  u32 escP, escF, ovf, nwrap, last, vbase, n0;
};

// packets += c, fan += 1 for the node in slot `slot`.  An item with fewer than 4096 records cannot
// carry a fan past the 12-bit field: a fire-and-forget add.  Otherwise a fan field that passes 4095 is
// noted in the wrap list.
// Record (packets | links << 20) into the node's slot; a fan field that passes 4095 is noted in the wrap list
// (a record adds at most 1281 links, so at most one wrap).
__device__ __forceinline__ u32 node_add(SmemS& s, u32 slot, u32 a) {
  const u32 o = atomicAdd(&s.npf[slot], a);
  if ((o >> PFS) + (a >> PFS) > FMAX) {
    const u32 i = atomicAdd(&s.nwrap, 1u);
    if (i < (u32)WRAPCAP) s.wrap[i] = slot;
    else s.ovf = 1;
  }
  return o + a;  // the slot's packets | fan << 20 after this record (fan modulo 4096)
}

// One lane merges a cached node's totals (packets P, fan F, F possibly > 4095) into the table: probe to
// its slot, then add in steps of at most 4095 fan so that every wrap of the 12-bit field is recorded.
// Returns 1 if the node was new to the table; folds the slot's final packets / fan (mod 4096) into mp, mf.
__device__ __noinline__ u32 node_merge(SmemS& s, u32 node, u32 P, u32 F, u32 logBs, u32& mp, u32& mf) {
  u32 sl = node_slot(node, logBs);
  const u32 stp = node_step(node);
  u32 fresh = 0;
  for (u32 probe = 0;; ++probe) {
    const u32 cur = *reinterpret_cast<volatile u32*>(&s.nkey[sl]);
    if (cur == node) break;
    if (cur == EMPTY32) {
      const u32 o = atomicCAS(&s.nkey[sl], EMPTY32, node);
      if (o == EMPTY32) { fresh = 1; break; }
      if (o == node) break;
      continue;  // re-read this slot
    }
    if (probe >= (u32)TS) { s.ovf = 1; return 0; }
    sl = (sl + stp) & (TS - 1);
  }
  for (bool first = true; F; first = false) {
    const u32 a = min(F, FMAX);
    const u32 add = (first ? P : 0u) | (a << PFS);
    const u32 o = atomicAdd(&s.npf[sl], add);
    if ((o >> PFS) + a > FMAX) {
      const u32 i = atomicAdd(&s.nwrap, 1u);
      if (i < (u32)WRAPCAP) s.wrap[i] = sl;
      else s.ovf = 1;
    }
    mp = max(mp, (o + add) & PMASK);
    mf = max(mf, (o + add) >> PFS);
    F -= a;
  }
  return fresh;
}

// Is `node` in the (complete) node table?
__device__ __forceinline__ bool node_find(const SmemS& s, u32 node, u32 logBs) {
  u32 sl = node_slot(node, logBs);
  const u32 stp = node_step(node);
  for (u32 probe = 0; probe < (u32)TS; ++probe) {
    const u32 cur = s.nkey[sl];
    if (cur == node) return true;
    if (cur == EMPTY32) return false;
    sl = (sl + stp) & (TS - 1);
  }
  return false;
}

// fan of the node in slot sl, with the wraps of its 12-bit field recorded in the wrap list
__device__ __forceinline__ u32 node_fan(const SmemS& s, u32 sl, u32 pf, u32 nwrap) {
  u32 cnt = 0;
  for (u32 k = 0; k < nwrap; ++k) cnt += s.wrap[k] == sl;
  return (pf >> PFS) + (FMAX + 1) * cnt;
}

__device__ void finalize(const FGeo& g, u64 w, u64* out) {
  WinState* st = &g.ws[w];
  u32 ovf = ldcg32(&st->ovf);
  if ((g.inject & 1u) && (w & 1)) { st->ovf = 1; ovf = 1; }
  if (ovf) {  // recomputed by the L2 path; diag[0] counts the windows handed over
    atomicAdd(&g.diag[0], 1u);
    return;
  }
  const u64 len = g.wgt ? (u64)ldcg32(&st->wtot) : min(g.W, g.n - w * g.W);  // valid packets expected
  u64 row[NSG_NUM_STATS];
  row[0] = ldcg32(&st->sumc);
  row[1] = ldcg32(&st->links);
  row[2] = ldcg32(&st->maxc);
  row[3] = ldcg32(&st->nodes[0]);
  row[4] = ldcg32(&st->maxp[0]);
  row[5] = ldcg32(&st->maxf[0]);
  row[6] = ldcg32(&st->nodes[1]);
  row[7] = ldcg32(&st->maxp[1]);
  row[8] = ldcg32(&st->maxf[1]);
  if (row[0] != len || ((g.inject & 2u) && w == 0)) atomicAdd(&g.diag[1], 1u);  // self-check: the counts sum to the window's packets
  store_row(out + w * NSG_NUM_STATS, row);
  if (g.v_ipsets) {  // |S u D|, |S \ D|, |D \ S|, |S n D| (reading R13)
    const u64 b = ldcg32(&st->both);
    u64* ip = g.v_ipsets + w * 4;
    ip[0] = row[3] + row[6] - b; ip[1] = row[3] - b; ip[2] = row[6] - b; ip[3] = b;
  }
  for (u32 m = 0; m < g.n_mirror; ++m) store_row(g.mirror[m] + (g.mirror_row0 + w) * NSG_NUM_STATS, row);
}

__global__ void __launch_bounds__(STH, 1536 / STH)
side_kernel(const FGeo g, u64* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SmemS& s = *reinterpret_cast<SmemS*>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  constexpr u32 NW = STH / 32;
  const u32 Bs = g.Bs, B = g.B, logBs = g.logBs;
  const u32 wb = blockIdx.x / (2 * Bs), q = blockIdx.x % (2 * Bs);
  const u64 w = g.w0 + wb;
  if (t == 0) { s.escP = 0; s.escF = 0; s.ovf = 0; s.nwrap = 0; }
  const u32* ro = g.roff + (u64)wb * B * 2 * Bs + q;
  WarpSegs ws = warp_segs(B, NW, s.segscr[wid], [&](u32 b) { return ldcg32(ro + (u64)b * 2 * Bs); }, [&](u32 b) { return b * RCAP; },
                          [&] {  // the node table, while the descriptors load
                            for (u32 i = t; i < (u32)TS / 4; i += STH) {
                              reinterpret_cast<uint4*>(s.nkey)[i] = make_uint4(EMPTY32, EMPTY32, EMPTY32, EMPTY32);
                              reinterpret_cast<uint4*>(s.npf)[i] = make_uint4(0u, 0u, 0u, 0u);
                            }
                          });
  if (lane == 0) s.red[0][wid] = ws.n;
  const u64* rb = g.rscr + (u64)wb * B * RCAP;
  u64 nxa = ~0ull, nxc = ~0ull;  // the next step's records, loaded while this step's are merged (the first
  auto fetch = [&](u32 e0) {     // step's before the barrier)
    u32 oa, ob;
    warp_seg_step(ws, e0, oa, ob);
    nxa = e0 + lane < ws.n ? __ldcg(reinterpret_cast<const unsigned long long*>(rb + oa)) : ~0ull;
    nxc = e0 + 32 + lane < ws.n ? __ldcg(reinterpret_cast<const unsigned long long*>(rb + ob)) : ~0ull;
  };
  if (ws.n) fetch(0);
  __syncthreads();  // table initialised, per-warp counts visible
  u32 ntot = 0;
#pragma unroll
  for (u32 i = 0; i < NW; ++i) ntot += s.red[0][i];
  const bool heavy = ntot > HEAVY_S;
  // unique nodes (slots this thread claimed), max packets and max fan (mod 4096) of the table, taken from
  // the adds' return values (every slot's final value is the largest of its returns)
  u32 nn = 0, mp = 0, mf = 0;
  {
    u32 escP = 0, escF = 0;
    // A heavy item (a heavy hitter's bucket) caches one node per warp in lane registers: its records are
    // summed there instead of in one contended table slot, and merged once at the end.
    const u32 hot = heavy && ws.n ? __shfl_sync(0xffffffffu, (u32)(nxa >> 32), 0) : EMPTY32;
    u32 hP = 0, hF = 0;
    for (u32 e0 = 0; e0 < ws.n; e0 += 64) {
      const bool va = e0 + lane < ws.n, vb = e0 + 32 + lane < ws.n;
      const u64 ra = nxa, rc = nxc;
      if (e0 + 64 < ws.n) fetch(e0 + 64);
      if (*reinterpret_cast<volatile u32*>(&s.ovf)) break;
      const u32 na = (u32)(ra >> 32), nb = (u32)(rc >> 32);
      u32 sa = node_slot(na, logBs), sb = node_slot(nb, logBs);
      bool aa = na != EMPTY32, ab = nb != EMPTY32;  // the node ~0 is merged apart
      if (va && !aa) { escP += (u32)ra & PMASK; escF += (u32)ra >> PFS; }
      if (vb && !ab) { escP += (u32)rc & PMASK; escF += (u32)rc >> PFS; }
      if (aa && na == hot) { hP += (u32)ra & PMASK; hF += (u32)ra >> PFS; aa = false; }
      if (ab && nb == hot) { hP += (u32)rc & PMASK; hF += (u32)rc >> PFS; ab = false; }
      const u32 ca = aa ? *reinterpret_cast<volatile u32*>(&s.nkey[sa]) : 0u;
      const u32 cb = ab ? *reinterpret_cast<volatile u32*>(&s.nkey[sb]) : 0u;
      const u32 cl = probe2<u32>(smem_addr(s.nkey), TS - 1, na, nb, sa, sb, ca, cb, aa, ab, &s.ovf,
                                 [](u32 k) { return node_step(k); });
      nn += __popc(cl);
      if (aa) {
        const u32 v = node_add(s, sa, (u32)ra);
        mp = max(mp, v & PMASK); mf = max(mf, v >> PFS);
      }
      if (ab) {
        const u32 v = node_add(s, sb, (u32)rc);
        mp = max(mp, v & PMASK); mf = max(mf, v >> PFS);
      }
    }
    hP = __reduce_add_sync(0xffffffffu, hP);
    hF = __reduce_add_sync(0xffffffffu, hF);
    if (lane == 0 && hF) nn += node_merge(s, hot, hP, hF, logBs, mp, mf);
    escF = __reduce_add_sync(0xffffffffu, escF);
    escP = __reduce_add_sync(0xffffffffu, escP);
    if (lane == 0 && escF) { atomicAdd(&s.escP, escP); atomicAdd(&s.escF, escF); }
  }
  __syncthreads();
  // ---- final: the side bucket's nodes
  u32 wrapmax = 0;
  const u32 nwrap = min(s.nwrap, (u32)WRAPCAP);
  for (u32 i = lane; i < nwrap; i += 32) {  // exact fan of the nodes whose 12-bit field wrapped
    const u32 sl = s.wrap[i];
    u32 cnt = 0;
    for (u32 k = 0; k < nwrap; ++k) cnt += s.wrap[k] == sl;
    wrapmax = max(wrapmax, (s.npf[sl] >> PFS) + (FMAX + 1) * cnt);
  }
  const bool ovf = s.ovf != 0;
  constexpr int SPT = TS / STH;
  static_assert(SPT % 4 == 0, "slots are scanned 4 at a time");
  const u32 side = q >= Bs ? 1u : 0u;
  const bool emit = g.v_node[side] != nullptr || (g.v_ipsets && side == 0);
  u32 vpre = 0;  // vectors / IP sets: this thread's first entry among the item's table nodes
  if (emit) {  // the nodes are listed in slot order: this thread's slots [t * SPT, t * SPT + SPT)
    nn = 0;
#pragma unroll
    for (int j = 0; j < SPT; j += 4) {
      const uint4 p4 = *reinterpret_cast<const uint4*>(&s.npf[t * SPT + j]);
      nn += (p4.x ? 1u : 0u) + (p4.y ? 1u : 0u) + (p4.z ? 1u : 0u) + (p4.w ? 1u : 0u);
    }
    u32 x = nn;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, x, k);
      if (lane >= k) x += y;
    }
    vpre = x - nn;
  }
  mf = max(mf, wrapmax);
  const u32 escF = s.escF, escP = s.escP;
  if (t == 0 && escF) { nn += 1; mp = max(mp, escP); mf = max(mf, escF); }
  u32 z = 0;
  warp_reduce4(nn, mp, mf, z);
  if (lane == 0) { s.red[0][wid] = nn; s.red[1][wid] = mp; s.red[2][wid] = mf; }
  __syncthreads();
  if (emit) {  // the item's nodes (mirrors :173) and the side-0 node list
    u32 ntab = 0;  // table nodes (warp 0's count includes the address ~0, which goes last)
    for (u32 i = 0; i < NW; ++i) {
      if (i == (u32)wid) vpre += ntab;
      ntab += s.red[0][i] - (i == 0 && escF ? 1u : 0u);
    }
    const u32 tot = ntab + (escF ? 1u : 0u);
    if (t == 0 && g.v_node[side]) s.vbase = atomicAdd(&g.ws[w].vfill[1 + side], tot);
    __syncthreads();
    const u64 vb = w * g.W + s.vbase;
    u32* ipl = g.ipl + ((u64)wb * Bs + (q - side * Bs)) * TS;
    u32 pos = vpre;
    for (int j = 0; j < SPT; ++j) {
      const u32 sl = t * SPT + j;
      const u32 pf = s.npf[sl];
      if (!pf) continue;
      const u32 node = s.nkey[sl];
      if (g.v_node[side]) {
        g.v_node[side][vb + pos] = node;
        g.v_pk[side][vb + pos] = pf & PMASK;
        g.v_fan[side][vb + pos] = node_fan(s, sl, pf, nwrap);
      }
      if (g.v_ipsets && side == 0) ipl[pos] = node;
      ++pos;
    }
    if (t == 0 && escF && g.v_node[side]) {
      g.v_node[side][vb + ntab] = EMPTY32;
      g.v_pk[side][vb + ntab] = escP;
      g.v_fan[side][vb + ntab] = escF;
    }
    if (g.v_ipsets && side == 0) {  // publish the list for the side-1 item of the same node bucket
      __syncthreads();
      if (t == 0) {
        __threadfence();
        st_release32(&g.ipc[(u64)wb * Bs + q], (ntab + 1) | (escF ? 0x80000000u : 0u));
      }
    }
  }
  if (g.v_ipsets && side == 1) {  // |S n D| of this node bucket: the side-0 list probed in this table
    if (t == 0) {
      const u32* f = &g.ipc[(u64)wb * Bs + (q - Bs)];
      u32 v;
      while ((v = ld_acquire32(f)) == 0u) __nanosleep(64);  // side-0 items precede side-1 items in the grid
      s.n0 = v;
    }
    __syncthreads();
    const u32 n0 = (s.n0 & 0x7FFFFFFFu) - 1u;
    const u32* ipl = g.ipl + ((u64)wb * Bs + (q - Bs)) * TS;
    u32 both = 0;
    for (u32 e = t; e < n0; e += STH) both += node_find(s, ldcg32(&ipl[e]), logBs) ? 1u : 0u;
    if (t == 0 && (s.n0 >> 31) && escF) both += 1;  // the address ~0 is a source and a destination
    both = warp_sum(both);
    if (lane == 0 && both) {
      atomicAdd(&g.ws[w].both, both);
      __threadfence();  // before this item's count (below)
    }
    __syncthreads();
  }
  if (wid == 0) {
    nn = lane < (int)NW ? s.red[0][lane] : 0u;
    mp = lane < (int)NW ? s.red[1][lane] : 0u;
    mf = lane < (int)NW ? s.red[2][lane] : 0u;
    warp_reduce4(nn, mp, mf, z);
    if (lane == 0) {
      WinState* st = &g.ws[w];
      if (ovf) {
        st->ovf = 1;
      } else if (nn) {
        atomicAdd(&st->nodes[side], nn);
        atomicMax(&st->maxp[side], mp);
        atomicMax(&st->maxf[side], mf);
      }
      __threadfence();  // this item's accumulators before its count (the last item reads them)
      s.last = atomicAdd(&st->sdone, 1u) + 1 == 2 * Bs;
      if (s.last) {
        __threadfence();
        finalize(g, w, out);
      }
    }
  }
}

// After a call's last batch: its scratch (keys, records, descriptors) is dead; drop it from L2 so that the
// dirty lines are never written back to HBM (the earlier batches' scratch was overwritten in L2).
__global__ void __launch_bounds__(256)
discard_kernel(const unsigned char* base, u64 bytes) {
  for (u64 i = (u64)blockIdx.x * 256 + threadIdx.x; i < bytes / 128; i += (u64)gridDim.x * 256)
    discard_l2_line(base + i * 128);
}

}  // namespace flat
}  // namespace nsg
