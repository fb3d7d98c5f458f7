// nsg_flat.cuh — the per-window statistics kernels of libnsg (round 2), windows <= 2^18.
//
// What it computes: for every window of W consecutive packets, the nine Table 2 scalars of the
// traffic matrix A_t (destination mirrors, line 173): valid packets (:180),
// unique links (:181), max link packets (:183), unique sources (:184), max source packets (:186), max
// source fan-out (:188) and the three destination mirrors.  Readings: DESIGN.md §2.
//
// How: three flat kernels per batch of windows, one work item per CTA, several small
// CTAs resident per SM so that the latency chains of independent items overlap (a measured property
// of this work on B200: every item is a short chain of dependent shared-memory round trips, ~200-500
// cycles each under load, and one item in flight per SM leaves the SM idle most of the time):
//   part  (w, c)   4096 keys of window w (streaming 128-bit loads from HBM), counting-sorted by link
//                  bucket (top bits of key * phi64) into the batch's key scratch; one row of segment
//                  descriptors per item;
//   link  (w, b)   link bucket b: its segment of every chunk gathered into SMEM, group-by-count in an
//                  SMEM open-addressing table (A_t restricted to the bucket: unique links, max link,
//                  count sum -> window accumulators), then one record (node << 32 | count) per link and
//                  side, counting-sorted by side bucket into the record scratch;
//   side  (w,s,q)  side bucket q of side s: the records of every link bucket, merged per node in an
//                  SMEM table of (node, packets | fan << 20): unique nodes, max packets, max fan ->
//                  window accumulators; the last side item of a window writes its row.
// Tables are probed with a plain load first (a hot key's repeats cost a broadcast read and an
// aggregated increment, never a CAS); collisions probe on with double hashing; claimed slots are kept
// in a dense claim list so that the final scans visit entries only.
#pragma once
#include "nsg.h"
#include "nsg_common.cuh"

namespace nsg {
namespace flat {

constexpr int CH = 4096;                      // keys per partition item
constexpr int PTH = 256;                      // partition CTA threads
constexpr int LTH = 512;                      // link CTA threads
constexpr int STH = 512;                      // side CTA threads
constexpr u64 BK = 2048;                      // target keys per link bucket / nodes per side bucket
constexpr u64 MAX_W = 1ull << 18;             // windows this path takes (<= 128 link / side buckets)
constexpr int MAXB = 256;
constexpr int LOG_TL = 12, TL = 1 << LOG_TL;  // link-table slots (load <= 5/8)
constexpr int LOG_TS = 12, TS = 1 << LOG_TS;  // node-table slots
constexpr u32 FILL_L = 2560, FILL_S = 2560;   // distinct entries before the window goes to the L2 path
constexpr int LSK = 5124;                     // link stage (u64): keys per gather part, then the records
constexpr u32 RCAP = 2 * (FILL_L + 1);        // records per link bucket (both sides)
constexpr int SSK = 4096;                     // side stage (u64): records per gather part
constexpr int PFS = 20;                       // node packets: 20-bit field (W < 2^20)
constexpr u32 PMASK = (1u << PFS) - 1;
constexpr u32 FMAX = 0xFFFu;                  // fan field: 12 bits; items with >= 4096 records track wraps
constexpr int WRAPCAP = 64;
constexpr u64 MUL_L = 0x9E3779B97F4A7C15ull;  // link hash: top bits of key * phi64
constexpr u32 MUL_N = 0x9E3779B9u;            // node hash: top bits of node * phi32
static_assert(RCAP % 2 == 0, "record regions stay 16-B aligned");

// Per-window state (64 B), zeroed by the host before the launches.
struct WinState {
  u32 sdone, ovf, links, maxc, sumc, r0[3];
  u32 nodes[2], maxp[2], maxf[2], r1[2];
};
static_assert(sizeof(WinState) == 64, "WinState is 64 B");

struct FGeo {
  u64 n, W, nw;
  u64 w0;                          // first window of the batch
  u32 nbw;                         // windows in the batch
  u32 logB, B, logBs, Bs, CP;
  WinState* ws;                    // [nw]
  u64* kscr;                       // [nbw][CP][CH]
  u32* koff;                       // [nbw][CP][B]    start << 16 | count of bucket b in chunk c
  u64* rscr;                       // [nbw][B][RCAP]
  u32* roff;                       // [nbw][B][2Bs]   start << 16 | count of side bucket (s,q) in link bucket b
  u32* diag;                       // [0] windows handed to the L2 path, [1] self-check failures
  u64* const* mirror;
  u32 n_mirror;
  u64 mirror_row0;
  u32 inject;                      // NSG_FLAG_INJECT_OVERFLOW: odd windows are handed to the L2 path
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

__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((u32)__cvta_generic_to_shared(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ u64 ld_stream64(const u64* p) {
  u64 v;
  asm volatile("ld.global.cs.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ ulonglong2 ld_stream128(const u64* p) {
  ulonglong2 v;
  asm volatile("ld.global.cs.v2.u64 {%0,%1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
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

// Warp-wide reservation of n list entries (returns this thread's first position).
__device__ __forceinline__ u32 warp_reserve(u32 n, u32* ctr) {
  const int lane = threadIdx.x & 31;
  u32 x = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  const u32 tot = __shfl_sync(0xffffffffu, x, 31);
  u32 b = 0;
  if (lane == 31 && tot) b = atomicAdd(ctr, tot);
  return __shfl_sync(0xffffffffu, b, 31) + x - n;
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
// chunks / link buckets), enumerates their concatenation lane-parallel and loads the elements it
// processes straight from L2 into registers.  The inserts then need no CTA barrier: a warp inserts
// its own elements as soon as they arrive (slots only go from free to a key, so concurrent inserts
// from other warps are safe), and one barrier ends the whole insert phase.
// ---------------------------------------------------------------------------------------------
constexpr int WSEG = 16;  // segments per warp (>= segments / warps for W <= 2^18)

struct WarpSegs {
  u32 n;      // elements of the warp's concatenation
  u32 nseg;   // segments owned
};

// Load the warp's segment descriptors (desc(i) = start << 16 | count of segment i, i < nall) into
// pre[] / st[] (this warp's SMEM slice): pre[k] = first element of its k-th segment.
template <class D>
__device__ __forceinline__ WarpSegs warp_segs(u32 nall, u32 nwarps, u32* pre, u32* st, D desc) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpSegs r;
  r.nseg = nall > (u32)wid ? (nall - 1 - wid) / nwarps + 1 : 0u;
  const u32 i = wid + lane * nwarps;
  const u32 v = (u32)lane < r.nseg ? desc(i) : 0u;
  u32 x = v & 0xFFFFu;
#pragma unroll
  for (int k = 1; k < 32; k <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, x, k);
    if (lane >= k) x += y;
  }
  if ((u32)lane < r.nseg) { pre[lane] = x - (v & 0xFFFFu); st[lane] = v >> 16; }
  r.n = __shfl_sync(0xffffffffu, x, 31);
  __syncwarp();
  return r;
}

// element e (< n) of the warp's concatenation: its segment k and offset inside the segment
__device__ __forceinline__ void warp_seg_find(const u32* pre, u32 nseg, u32 e, u32& k, u32& off) {
  u32 j = 0;
  for (u32 q = 1; q < nseg; ++q) j = (e >= pre[q]) ? q : j;
  k = j;
  off = e - pre[j];
}

// ---------------------------------------------------------------------------------------------
// part(w, c): counting sort of one chunk by link bucket
// ---------------------------------------------------------------------------------------------
struct SmemP {
  u64 stage[CH];
  u32 hist[MAXB], offs[MAXB];
};

__global__ void __launch_bounds__(PTH, 4)
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
  if (keys) {
    const u64* p = keys + base;
    if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < KPT / 2; ++i) {
        const u32 e = 2 * (i * PTH + t);
        if (e + 1 < n) {
          const ulonglong2 v = ld_stream128(p + e);
          kk[2 * i] = v.x; kk[2 * i + 1] = v.y;
        } else {
          kk[2 * i] = e < n ? ld_stream64(p + e) : 0ull;
          kk[2 * i + 1] = 0ull;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < KPT / 2; ++i) {
        const u32 e = 2 * (i * PTH + t);
        kk[2 * i] = e < n ? ld_stream64(p + e) : 0ull;
        kk[2 * i + 1] = e + 1 < n ? ld_stream64(p + e + 1) : 0ull;
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
  __syncthreads();  // histogram cleared
  u32 bk[KPT], rk[KPT];
#pragma unroll
  for (int i = 0; i < KPT; ++i) bk[i] = link_bucket(kk[i], logB);
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    const u32 e = 2 * ((i >> 1) * PTH + t) + (i & 1);
    rk[i] = e < n ? atomicAdd(&s.hist[bk[i]], 1u) : 0u;
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
    if (e < n) s.stage[s.offs[bk[i]] + rk[i]] = kk[i];
  }
  __syncthreads();
  copy_out<PTH>(g.kscr + ((u64)wb * g.CP + c) * CH, s.stage, n);
}

// ---------------------------------------------------------------------------------------------
// link(w, b)
// ---------------------------------------------------------------------------------------------
struct SmemL {
  u64 stage[LSK];                  // 20 KB: the bucket's keys (part by part), then its records
  u64 lkey[TL];                    // 16 KB
  u32 lcnt[TL];                    // 8 KB
  uint16_t claim[TL];              // 4 KB
  u32 hist[2 * MAXB], offs[2 * MAXB];
  u32 wpre[LTH / 32][WSEG], wst[LTH / 32][WSEG];  // per-warp segment prefixes / starts
  u32 red[4][LTH / 32];
  u32 ncl, esc, ovf, L0;
};

// One slot for `key`: 1 = counted (found), 2 = claimed and counted, 0 = holds another key.
__device__ __forceinline__ u32 link_try(SmemL& s, u64 key, u32 sl, u64 cur) {
  if (cur == key) { atomicAdd(&s.lcnt[sl], 1u); return 1; }
  if (cur != EMPTY64) return 0;
  const u64 old = atomicCAS(reinterpret_cast<unsigned long long*>(&s.lkey[sl]), (unsigned long long)EMPTY64,
                            (unsigned long long)key);
  if (old == EMPTY64) { atomicAdd(&s.lcnt[sl], 1u); return 2; }
  if (old == key) { atomicAdd(&s.lcnt[sl], 1u); return 1; }
  return 0;
}

constexpr int KR = 4;  // keys / records per thread per insert round
// Insert up to KR keys per lane (bit i of vm: k[i] valid), all of the lane's loads / atomics in flight
// together; colliding keys probe on by double hashing, all together per step.  Claimed slots are
// appended to the claim list with one reservation per warp (ballot ranks).
__device__ __forceinline__ void link_insert_regs(SmemL& s, const u64 (&k)[KR], u32 vm, u32 logB) {
  const int lane = threadIdx.x & 31;
  u64 cur[KR];
  u32 sl[KR];
  u32 vmask = 0, nesc = 0;
#pragma unroll
  for (int i = 0; i < KR; ++i) {
    if ((vm >> i & 1u) && k[i] == EMPTY64) ++nesc;
    else if (vm >> i & 1u) vmask |= 1u << i;
    sl[i] = link_slot(k[i], logB);
  }
  if (*reinterpret_cast<volatile u32*>(&s.ovf)) vmask = 0;
#pragma unroll
  for (int i = 0; i < KR; ++i) cur[i] = (vmask >> i & 1u) ? *reinterpret_cast<volatile u64*>(&s.lkey[sl[i]]) : 0ull;
  u32 pmask = 0, wmask = 0;
#pragma unroll
  for (int i = 0; i < KR; ++i) {
    if (vmask >> i & 1u) {
      const u32 r = link_try(s, k[i], sl[i], cur[i]);
      if (r == 0) pmask |= 1u << i;
      if (r == 2) wmask |= 1u << i;
    }
  }
  if (nesc) atomicAdd(&s.esc, nesc);
  if (__any_sync(0xffffffffu, pmask != 0)) {
    u32 stp[KR];
#pragma unroll
    for (int i = 0; i < KR; ++i) stp[i] = link_step(k[i]);
    for (u32 step = 1; __any_sync(0xffffffffu, pmask != 0); ++step) {
      if (step >= (u32)TL) {  // table full (adversarial keys only)
        if (pmask) s.ovf = 1;
        break;
      }
#pragma unroll
      for (int i = 0; i < KR; ++i)
        if (pmask >> i & 1u) cur[i] = *reinterpret_cast<volatile u64*>(&s.lkey[(sl[i] + stp[i]) & (TL - 1)]);
#pragma unroll
      for (int i = 0; i < KR; ++i) {
        if (pmask >> i & 1u) {
          sl[i] = (sl[i] + stp[i]) & (TL - 1);
          const u32 r = link_try(s, k[i], sl[i], cur[i]);
          if (r) pmask &= ~(1u << i);
          if (r == 2) wmask |= 1u << i;
        }
      }
    }
  }
  // claim-list reservation: ballot ranks, one atomic per warp
  u32 m[KR], tot = 0;
#pragma unroll
  for (int i = 0; i < KR; ++i) { m[i] = __ballot_sync(0xffffffffu, wmask >> i & 1u); tot += __popc(m[i]); }
  if (tot) {
    u32 base = 0;
    if (lane == 0) {
      base = atomicAdd(&s.ncl, tot);
      if (base + tot > FILL_L) s.ovf = 1;  // more distinct links than the fast path takes
    }
    base = __shfl_sync(0xffffffffu, base, 0);
    const u32 lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < KR; ++i) {
      if (wmask >> i & 1u) {
        const u32 pos = base + __popc(m[i] & lt);
        if (pos < (u32)TL) s.claim[pos] = (uint16_t)sl[i];
      }
      base += __popc(m[i]);
    }
  }
}

__global__ void __launch_bounds__(LTH, 2)
link_kernel(const FGeo g) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SmemL& s = *reinterpret_cast<SmemL*>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  constexpr u32 NW = LTH / 32;
  const u32 wb = blockIdx.x / g.B, b = blockIdx.x % g.B;
  const u64 w = g.w0 + wb;
  const u32 CP = g.CP, B = g.B, Bs = g.Bs, logBs = g.logBs;
  for (u32 i = t; i < (u32)TL / 2; i += LTH) {  // table init (conflict-free wide stores)
    reinterpret_cast<ulonglong2*>(s.lkey)[i] = make_ulonglong2(EMPTY64, EMPTY64);
    reinterpret_cast<uint2*>(s.lcnt)[i] = make_uint2(0u, 0u);
  }
  if (t == 0) { s.ncl = 0; s.esc = 0; s.ovf = 0; }
  for (u32 i = t; i < 2 * Bs; i += LTH) s.hist[i] = 0;
  // this warp's share of the bucket: its segment of chunks wid, wid + NW, ...
  u32* pre = s.wpre[wid];
  u32* sst = s.wst[wid];
  const u32* ko = g.koff + (u64)wb * CP * B + b;
  const WarpSegs ws = warp_segs(CP, NW, pre, sst, [&](u32 c) { return ldcg32(ko + (u64)c * B); });
  const u64* kb = g.kscr + (u64)wb * CP * CH;
  __syncthreads();  // table initialised
  for (u32 r0 = 0; r0 < ws.n; r0 += 32 * KR) {
    u64 k[KR];
    u32 vm = 0;
#pragma unroll
    for (int i = 0; i < KR; ++i) {
      const u32 e = r0 + i * 32 + lane;
      k[i] = 0;
      if (e < ws.n) {
        u32 kk, off;
        warp_seg_find(pre, ws.nseg, e, kk, off);
        k[i] = __ldcg(reinterpret_cast<const unsigned long long*>(kb + (u64)(wid + kk * NW) * CH + sst[kk] + off));
        vm |= 1u << i;
      }
    }
    link_insert_regs(s, k, vm, g.logB);
  }
  __syncthreads();  // every key of the bucket is in the table
  // ---- final: the bucket's links (claim list), window statistics, records by side bucket
  const bool ovf = s.ovf != 0;
  const u32 ncl = min(s.ncl, (u32)TL);
  constexpr int SPT = TL / LTH;
  const int kmax = (int)((ncl + LTH - 1) / LTH);  // rounds with claims (warp-uniform bound)
  u64 lk[SPT];
  u32 lc[SPT], lb[SPT], r0[SPT], r1[SPT];
  u32 nl = 0, mx = 0, sm = 0;
#pragma unroll
  for (int k = 0; k < SPT; ++k) { lc[k] = 0; lk[k] = 0; lb[k] = 0; r0[k] = 0; r1[k] = 0; }
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    if (k >= kmax) break;
    const u32 e = k * LTH + t;
    const u32 sl = e < ncl ? s.claim[e] : 0u;
    lc[k] = e < ncl ? s.lcnt[sl] : 0u;
    lk[k] = e < ncl ? s.lkey[sl] : 0ull;
  }
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    if (k >= kmax) break;
    if (lc[k]) { nl += 1; mx = max(mx, lc[k]); sm += lc[k]; }
    lb[k] = node_bucket((u32)(lk[k] >> 32), logBs) | (node_bucket((u32)lk[k], logBs) << 16);
  }
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    if (k >= kmax) break;
    if (lc[k] && !ovf) {
      r0[k] = atomicAdd(&s.hist[lb[k] & 0xFFFFu], 1u);
      r1[k] = atomicAdd(&s.hist[Bs + (lb[k] >> 16)], 1u);
    }
  }
  const u32 esc = s.esc;
  u32 er0 = 0, er1 = 0;
  const u32 eb = node_bucket(EMPTY32, logBs);
  if (t == 0 && esc) {  // the key ~0 (kept out of the table) is one more link
    nl += 1; mx = max(mx, esc); sm += esc;
    if (!ovf) { er0 = atomicAdd(&s.hist[eb], 1u); er1 = atomicAdd(&s.hist[Bs + eb], 1u); }
  }
  {
    u32 z = 0;
    warp_reduce4(nl, mx, z, sm);
    if (lane == 0) { s.red[0][wid] = nl; s.red[1][wid] = mx; s.red[3][wid] = sm; }
  }
  __syncthreads();
  u32* ro = g.roff + ((u64)wb * B + b) * 2 * Bs;  // this item's own row
  if (ovf) {
    if (t == 0) g.ws[w].ovf = 1;
    for (u32 i = t; i < 2 * Bs; i += LTH) ro[i] = 0;
    return;
  }
  if (wid == 0) {
    u32 a = lane < LTH / 32 ? s.red[0][lane] : 0u, m2 = lane < LTH / 32 ? s.red[1][lane] : 0u, z = 0,
        d = lane < LTH / 32 ? s.red[3][lane] : 0u;
    warp_reduce4(a, m2, z, d);
    if (lane == 0 && a) {
      WinState* st = &g.ws[w];
      atomicAdd(&st->links, a);
      atomicMax(&st->maxc, m2);
      atomicAdd(&st->sumc, d);
    }
  }
  if (wid < 2) {  // side-0 records first, then side 1 from L0 = number of links (= sum of the side-0 counts)
    u32 L0 = 0;
    if (wid == 1)
      for (u32 i = lane; i < Bs; i += 32) L0 += s.hist[i];
    L0 = warp_sum(L0);
    u32* r = ro + wid * Bs;
    const u32 tot = warp_exscan(s.hist + wid * Bs, s.offs + wid * Bs, Bs, lane,
                                [&](u32 i, u32 ex, u32 v) { r[i] = ((L0 + ex) << 16) | v; });
    if (wid == 0 && lane == 0) s.L0 = tot;
  }
  __syncthreads();
  const u32 L0 = s.L0;
  u64* rdst = g.rscr + ((u64)wb * B + b) * RCAP;
  const bool one = 2 * L0 <= (u32)LSK;
  u32 p0[SPT], p1[SPT];
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    p0[k] = 0; p1[k] = 0;
    if (k >= kmax) break;
    p0[k] = lc[k] ? s.offs[lb[k] & 0xFFFFu] : 0u;
    p1[k] = lc[k] ? s.offs[Bs + (lb[k] >> 16)] : 0u;
  }
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    if (k >= kmax) break;
    if (lc[k]) {
      s.stage[p0[k] + r0[k]] = (lk[k] & 0xFFFFFFFF00000000ull) | lc[k];
      if (one) s.stage[L0 + p1[k] + r1[k]] = (lk[k] << 32) | lc[k];
    }
  }
  if (t == 0 && esc) {
    s.stage[s.offs[eb] + er0] = ((u64)EMPTY32 << 32) | esc;
    if (one) s.stage[L0 + s.offs[Bs + eb] + er1] = ((u64)EMPTY32 << 32) | esc;
  }
  __syncthreads();
  if (one) {
    copy_out<LTH>(rdst, s.stage, 2 * L0);
  } else {
    copy_out<LTH>(rdst, s.stage, L0);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      if (k >= kmax) break;
      if (lc[k]) s.stage[p1[k] + r1[k]] = (lk[k] << 32) | lc[k];
    }
    if (t == 0 && esc) s.stage[s.offs[Bs + eb] + er1] = ((u64)EMPTY32 << 32) | esc;
    __syncthreads();
    copy_out<LTH>(rdst + L0, s.stage, L0);
  }
}

// ---------------------------------------------------------------------------------------------
// side(w, s, q)
// ---------------------------------------------------------------------------------------------
struct SmemS {
  u32 nkey[TS];                    // 8 KB
  u32 npf[TS];                     // 8 KB   packets | fan << 20
  uint16_t claim[TS];              // 4 KB
  u32 wpre[STH / 32][WSEG], wst[STH / 32][WSEG];
  u32 wrap[WRAPCAP];
  u32 red[3][STH / 32];
  u32 ncl, escP, escF, ovf, nwrap, last;
};

// One slot for `node`: 1 = its slot, 2 = claimed now, 0 = holds another node.
__device__ __forceinline__ u32 node_try(SmemS& s, u32 node, u32 sl, u32 cur) {
  if (cur == node) return 1;
  if (cur != EMPTY32) return 0;
  const u32 old = atomicCAS(&s.nkey[sl], EMPTY32, node);
  if (old == EMPTY32) return 2;
  return old == node ? 1u : 0u;
}

// packets += c, fan += 1.  An item with fewer than 4096 records cannot carry a fan past the 12-bit
// field: a fire-and-forget add.  Otherwise a fan field that passes 4095 is noted in the wrap list.
__device__ __forceinline__ void node_add(SmemS& s, u32 slot, u32 c, bool wrapcheck) {
  if (!wrapcheck) { atomicAdd(&s.npf[slot], c | (1u << PFS)); return; }
  const u32 o = atomicAdd(&s.npf[slot], c | (1u << PFS));
  if ((o >> PFS) == FMAX) {
    const u32 i = atomicAdd(&s.nwrap, 1u);
    if (i < (u32)WRAPCAP) s.wrap[i] = slot;
    else s.ovf = 1;
  }
}

__device__ __forceinline__ void node_insert_regs(SmemS& s, const u32 (&nd)[KR], const u32 (&cc)[KR], u32 vm, u32 logBs,
                                                 bool wrapcheck) {
  const int lane = threadIdx.x & 31;
  u32 sl[KR], cur[KR];
  u32 vmask = 0, escP = 0, escF = 0;
#pragma unroll
  for (int i = 0; i < KR; ++i) {
    if ((vm >> i & 1u) && nd[i] == EMPTY32) { escP += cc[i]; ++escF; }
    else if (vm >> i & 1u) vmask |= 1u << i;
    sl[i] = node_slot(nd[i], logBs);
  }
  if (*reinterpret_cast<volatile u32*>(&s.ovf)) vmask = 0;
#pragma unroll
  for (int i = 0; i < KR; ++i) cur[i] = (vmask >> i & 1u) ? *reinterpret_cast<volatile u32*>(&s.nkey[sl[i]]) : 0u;
  u32 pmask = 0, wmask = 0;
#pragma unroll
  for (int i = 0; i < KR; ++i) {
    if (vmask >> i & 1u) {
      const u32 r = node_try(s, nd[i], sl[i], cur[i]);
      if (r == 0) pmask |= 1u << i;
      if (r == 2) wmask |= 1u << i;
    }
  }
  if (escF) { atomicAdd(&s.escP, escP); atomicAdd(&s.escF, escF); }
  if (__any_sync(0xffffffffu, pmask != 0)) {
    u32 stp[KR];
#pragma unroll
    for (int i = 0; i < KR; ++i) stp[i] = node_step(nd[i]);
    for (u32 step = 1; __any_sync(0xffffffffu, pmask != 0); ++step) {
      if (step >= (u32)TS) {
        if (pmask) { s.ovf = 1; vmask &= ~pmask; }
        break;
      }
#pragma unroll
      for (int i = 0; i < KR; ++i)
        if (pmask >> i & 1u) cur[i] = *reinterpret_cast<volatile u32*>(&s.nkey[(sl[i] + stp[i]) & (TS - 1)]);
#pragma unroll
      for (int i = 0; i < KR; ++i) {
        if (pmask >> i & 1u) {
          sl[i] = (sl[i] + stp[i]) & (TS - 1);
          const u32 r = node_try(s, nd[i], sl[i], cur[i]);
          if (r) pmask &= ~(1u << i);
          if (r == 2) wmask |= 1u << i;
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < KR; ++i)
    if (vmask >> i & 1u) node_add(s, sl[i], cc[i], wrapcheck);
  u32 m[KR], tot = 0;
#pragma unroll
  for (int i = 0; i < KR; ++i) { m[i] = __ballot_sync(0xffffffffu, wmask >> i & 1u); tot += __popc(m[i]); }
  if (tot) {
    u32 base = 0;
    if (lane == 0) {
      base = atomicAdd(&s.ncl, tot);
      if (base + tot > FILL_S) s.ovf = 1;
    }
    base = __shfl_sync(0xffffffffu, base, 0);
    const u32 lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < KR; ++i) {
      if (wmask >> i & 1u) {
        const u32 pos = base + __popc(m[i] & lt);
        if (pos < (u32)TS) s.claim[pos] = (uint16_t)sl[i];
      }
      base += __popc(m[i]);
    }
  }
}

__device__ void finalize(const FGeo& g, u64 w, u64* out) {
  WinState* st = &g.ws[w];
  u32 ovf = ldcg32(&st->ovf);
  if (g.inject && (w & 1)) { st->ovf = 1; ovf = 1; }
  if (ovf) {  // recomputed by the L2 path; diag[0] counts the windows handed over
    atomicAdd(&g.diag[0], 1u);
    return;
  }
  const u64 len = min(g.W, g.n - w * g.W);
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
  if (row[0] != len) atomicAdd(&g.diag[1], 1u);  // self-check: the counts sum to the window's packets
  store_row(out + w * NSG_NUM_STATS, row);
  for (u32 m = 0; m < g.n_mirror; ++m) store_row(g.mirror[m] + (g.mirror_row0 + w) * NSG_NUM_STATS, row);
}

__global__ void __launch_bounds__(STH, 3)
side_kernel(const FGeo g, u64* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SmemS& s = *reinterpret_cast<SmemS*>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const u32 Bs = g.Bs, B = g.B, logBs = g.logBs;
  const u32 wb = blockIdx.x / (2 * Bs), q = blockIdx.x % (2 * Bs);
  const u64 w = g.w0 + wb;
  for (u32 i = t; i < (u32)TS / 4; i += STH) {
    reinterpret_cast<uint4*>(s.nkey)[i] = make_uint4(EMPTY32, EMPTY32, EMPTY32, EMPTY32);
    reinterpret_cast<uint4*>(s.npf)[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (t == 0) { s.ncl = 0; s.escP = 0; s.escF = 0; s.ovf = 0; s.nwrap = 0; }
  constexpr u32 NW = STH / 32;
  u32* pre = s.wpre[wid];
  u32* sst = s.wst[wid];
  const u32* ro = g.roff + (u64)wb * B * 2 * Bs + q;
  const WarpSegs ws = warp_segs(B, NW, pre, sst, [&](u32 b) { return ldcg32(ro + (u64)b * 2 * Bs); });
  if (lane == 0) s.red[0][wid] = ws.n;
  __syncthreads();  // table initialised, per-warp counts visible
  u32 ntot = 0;
#pragma unroll
  for (u32 i = 0; i < NW; ++i) ntot += s.red[0][i];
  const bool wrapcheck = ntot > FMAX;
  const u64* rb = g.rscr + (u64)wb * B * RCAP;
  for (u32 r0 = 0; r0 < ws.n; r0 += 32 * KR) {
    u32 nd[KR], cc[KR];
    u32 vm = 0;
#pragma unroll
    for (int i = 0; i < KR; ++i) {
      const u32 e = r0 + i * 32 + lane;
      u64 rec = 0;
      if (e < ws.n) {
        u32 kk, off;
        warp_seg_find(pre, ws.nseg, e, kk, off);
        rec = __ldcg(reinterpret_cast<const unsigned long long*>(rb + (u64)(wid + kk * NW) * RCAP + sst[kk] + off));
        vm |= 1u << i;
      }
      nd[i] = (u32)(rec >> 32);
      cc[i] = (u32)rec;
    }
    node_insert_regs(s, nd, cc, vm, logBs, wrapcheck);
  }
  __syncthreads();
  // ---- final: the side bucket's nodes (claim list)
  u32 wrapmax = 0;
  const u32 nwrap = min(s.nwrap, (u32)WRAPCAP);
  for (u32 i = lane; i < nwrap; i += 32) {  // exact fan of the nodes whose 12-bit field wrapped
    const u32 sl = s.wrap[i];
    u32 cnt = 0;
    for (u32 k = 0; k < nwrap; ++k) cnt += s.wrap[k] == sl;
    wrapmax = max(wrapmax, (s.npf[sl] >> PFS) + (FMAX + 1) * cnt);
  }
  const bool ovf = s.ovf != 0;
  const u32 ncl = min(s.ncl, (u32)TS);
  constexpr int SPT = TS / STH;
  const int kmax = (int)((ncl + STH - 1) / STH);
  u32 nn = 0, mp = 0, mf = wrapmax;
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    if (k >= kmax) break;
    const u32 e = k * STH + t;
    const u32 pf = e < ncl ? s.npf[s.claim[e]] : 0u;
    if (pf) { nn += 1; mp = max(mp, pf & PMASK); mf = max(mf, pf >> PFS); }
  }
  if (t == 0 && s.escF) { nn += 1; mp = max(mp, s.escP); mf = max(mf, s.escF); }
  u32 z = 0;
  warp_reduce4(nn, mp, mf, z);
  if (lane == 0) { s.red[0][wid] = nn; s.red[1][wid] = mp; s.red[2][wid] = mf; }
  __syncthreads();
  if (wid == 0) {
    nn = lane < STH / 32 ? s.red[0][lane] : 0u;
    mp = lane < STH / 32 ? s.red[1][lane] : 0u;
    mf = lane < STH / 32 ? s.red[2][lane] : 0u;
    warp_reduce4(nn, mp, mf, z);
    if (lane == 0) {
      WinState* st = &g.ws[w];
      const u32 side = q >= Bs ? 1u : 0u;
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

}  // namespace flat
}  // namespace nsg
