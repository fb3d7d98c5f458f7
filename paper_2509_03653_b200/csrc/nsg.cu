// libnsg — per-window Network Sensing Graph Challenge statistics on B200 (sm_100a).
//
// PAPER.md (arXiv 2509.03653) Table 2 (lines 171-193) defines, for the traffic matrix A_t of a
// window, the scalars computed here: valid packets 1^T A_t 1 (:180), unique links 1^T|A_t|_0 1
// (:181), max link packets max(A_t) (:183), unique sources 1^T|A_t 1|_0 (:184), max source packets
// max(A_t 1) (:186), max source fan-out max(|A_t|_0 1) (:188), and the destination mirrors
// ("For reverse operations simply replace src and dst", :173; :241).  The paper computes them with
// cuDF group-by / value_counts / drop_duplicates (:213-239); this library computes the same
// quantities with its own sm_100a kernels (design: DESIGN.md "Kernels").
//
// Two device paths, one result:
//  * FAST path (window <= 2^20): one persistent kernel.  Per window three kinds of work item are
//    handed out by a global ticket counter, pipelined across windows:
//      P(w,c)  partition: a CH-key chunk of the window is read from HBM once (128-bit loads),
//              counting-sorted in SMEM by link bucket b = top bits of hash64(key), and written to an
//              L2-resident scratch slot (the window's group-by exchange).
//      L(w,b)  link bucket: all keys of bucket b are gathered and aggregated in an SMEM hash table
//              (A_t restricted to the bucket: key -> count).  Its scan gives the bucket's unique links,
//              max link packets and sum of counts, and pre-aggregates, per source and per destination,
//              (packets, fan) partials of the bucket; partials are emitted as u64 records
//              node<<32 | P<<16 | F, bucketed by side bucket hash32(node).
//      S(w,side,sb) side bucket: the records of side bucket sb from every link bucket are merged in
//              an SMEM table node -> (sum P, sum F): unique nodes, max packets, max fan.  The last
//              S item of a window reduces the per-bucket results into the nine outputs.
//    Items only wait on items with smaller tickets, so the schedule cannot deadlock.
//  * L2 path (any window up to 2^31; also the overflow hand-off): one CTA per window with global-
//    memory hash tables, same definitions.  The fast path falls back to it for a window whose SMEM
//    table would overflow (never for the generated workloads; forced in tests).
#include "nsg.h"
#include "nsg_common.cuh"

#include <cstdio>
#include <cstring>
#include <mutex>

namespace nsg {

// ------------------------------------------------------------------------------------------
// Fast-path geometry
// ------------------------------------------------------------------------------------------
constexpr int FT = 512;                      // threads per CTA (2 CTAs per SM)
constexpr int NWARP = FT / 32;
constexpr int KPT = 8;                       // keys per thread in a partition item
constexpr int CH = FT * KPT;                 // 4096 keys per chunk
constexpr int TBITS = 11;
constexpr int TCAP = 1 << TBITS;             // SMEM hash-table slots
constexpr int BUCKET_KEYS = TCAP / 2;        // target keys per link bucket (load <= 0.5)
constexpr int MAX_LOGB = 10;
constexpr int MAXB = 1 << MAX_LOGB;
constexpr u64 FAST_MAX_WINDOW = (u64)BUCKET_KEYS << MAX_LOGB;  // 2^20
constexpr int MAXCP = (int)(FAST_MAX_WINDOW / CH);
constexpr u32 REC_MAX = 0xFFFFu;             // per-record P/F field limit (16 bits)
constexpr int RCAP_MAX = TCAP + 2 + (int)(FAST_MAX_WINDOW / REC_MAX) + 1;
constexpr int LAG_L = 2, LAG_S = 4;          // pipeline lags (steps) of L and S items behind P
constexpr int RSLOTS = LAG_S + 4;            // scratch slots (windows in flight)

struct Geo {
  u64 n, W, nw;
  u32 logB, B, cp, cp_last, rcap, R;
  u64 total_items;
  u32 flags;
  u64* ticket;
  u32* diag;
  u32 *pdone, *ldone, *sdone, *fin, *ovf;
  u64* kscr;  // [R][cp*CH]
  u32* koff;  // [R][cp][B+1]
  u64* rscr;  // [R][B][2][rcap]
  u32* roff;  // [R][B][2][B+1]
  u32* lres;  // [R][B][4]
  u32* sres;  // [R][2][B][4]
};

struct SmemP { u64 stage[CH]; u32 hist[MAXB + 1]; };
struct SmemL {
  u64 lkey[TCAP];
  u32 lcnt[TCAP];
  u32 nkey[2][TCAP];
  u32 nP[2][TCAP];
  u32 nF[2][TCAP];
  u64 stage[RCAP_MAX];
  u32 seg[MAXCP + 1];
  u32 seglo[MAXCP];
  u32 hist[MAXB + 1];
};
struct SmemS { u32 key[TCAP]; u32 P[TCAP]; u32 F[TCAP]; u32 seg[MAXB + 1]; u32 seglo[MAXB]; };
struct SmemMisc {
  u32 wtmp[10 * NWARP];
  u32 esc[8];   // [0] link escape count; [1+2s] side s escape P; [2+2s] side s escape F
  u32 flag, last;
  u64 tk;
};
constexpr size_t cmax(size_t a, size_t b) { return a > b ? a : b; }
constexpr size_t MISC_BYTES = (sizeof(SmemMisc) + 15) & ~size_t(15);
constexpr size_t FAST_SMEM = MISC_BYTES + cmax(sizeof(SmemP), cmax(sizeof(SmemL), sizeof(SmemS)));

// ------------------------------------------------------------------------------------------
// Block helpers
// ------------------------------------------------------------------------------------------
// In-place exclusive scan of a[0..n) by the whole CTA; afterwards a[n] = total.
template <int NT>
__device__ void block_exclusive_scan(u32* a, int n, u32* wtmp) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int per = (n + NT - 1) / NT;
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
    u32 v = lane < NT / 32 ? wtmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    if (lane < NT / 32) wtmp[lane] = v;
  }
  __syncthreads();
  u32 run = x - s + (wid ? wtmp[wid - 1] : 0);
  for (int i = b; i < e; ++i) {
    const u32 v = a[i];
    a[i] = run;
    run += v;
  }
  if (t == 0) a[n] = wtmp[NT / 32 - 1];
  __syncthreads();
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
// SMEM hash tables (linear probing, CAS claim; a claimed slot never changes key)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ bool smem_link_insert(u64* lkey, u32* lcnt, u64 key) {
  u32 slot = (u32)hash64(key) & (TCAP - 1);
#pragma unroll 1
  for (int probe = 0; probe < TCAP; ++probe) {
    u64 k = reinterpret_cast<volatile u64*>(lkey)[slot];
    if (k == EMPTY64) {
      const u64 old = atomicCAS(reinterpret_cast<unsigned long long*>(&lkey[slot]), EMPTY64, key);
      k = (old == EMPTY64) ? key : old;
    }
    if (k == key) { atomicAdd(&lcnt[slot], 1u); return true; }
    slot = (slot + 1) & (TCAP - 1);
  }
  return false;
}

// node -> (P += p, F += f).  node == EMPTY32 goes to the escape accumulators.
__device__ __forceinline__ bool smem_node_upsert(u32* key, u32* P, u32* F, u32* escP, u32* escF, u32 node, u32 p,
                                                 u32 f) {
  if (node == EMPTY32) {
    atomicAdd(escP, p);
    if (f) atomicAdd(escF, f);
    return true;
  }
  u32 slot = hash32(node) & (TCAP - 1);
#pragma unroll 1
  for (int probe = 0; probe < TCAP; ++probe) {
    u32 k = reinterpret_cast<volatile u32*>(key)[slot];
    if (k == EMPTY32) {
      const u32 old = atomicCAS(&key[slot], EMPTY32, node);
      k = (old == EMPTY32) ? node : old;
    }
    if (k == node) {
      atomicAdd(&P[slot], p);
      if (f) atomicAdd(&F[slot], f);
      return true;
    }
    slot = (slot + 1) & (TCAP - 1);
  }
  return false;
}

__device__ __forceinline__ u32 side_bucket(u32 node, u32 logB) { return logB ? hash32(node) >> (32 - logB) : 0u; }
__device__ __forceinline__ u32 link_bucket(u64 key, u32 logB) { return logB ? (u32)(hash64(key) >> (64 - logB)) : 0u; }

__device__ __forceinline__ void mark_overflow(const Geo& g, u64 w) {
  if (atomicExch(&g.ovf[w], 1u) == 0u) atomicAdd(&g.diag[0], 1u);
}

__device__ __forceinline__ u32 chunks_of(const Geo& g, u64 w) { return w + 1 == g.nw ? g.cp_last : g.cp; }

__device__ __forceinline__ void wait_geq(const u32* p, u32 v) {
  while (ld_acquire32(p) < v) __nanosleep(100);
}

// ------------------------------------------------------------------------------------------
// P item: partition one chunk of window w by link bucket
// ------------------------------------------------------------------------------------------
__device__ void item_partition(const Geo& g, const u32* __restrict__ src, const u32* __restrict__ dst,
                               const u64* __restrict__ keys, u64 w, u32 c, SmemP& s, SmemMisc& m) {
  const int t = threadIdx.x;
  if (t == 0 && w >= g.R) { wait_geq(&g.fin[w - g.R], 1u); __threadfence(); }
  for (int i = t; i <= (int)g.B; i += FT) s.hist[i] = 0;
  const u64 wbase = w * g.W;
  const u64 wlen = min(g.W, g.n - wbase);
  const u64 base = wbase + (u64)c * CH;
  const u32 len = (u32)min((u64)CH, wlen - (u64)c * CH);
  const u32 slot = (u32)(w % g.R);

  u64 k[KPT];
  u32 idx[KPT];
  if (keys) {
    const u64* p = keys + base;
    if (len == CH && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
      const ulonglong2* p2 = reinterpret_cast<const ulonglong2*>(p);
#pragma unroll
      for (int j = 0; j < KPT / 2; ++j) {
        const ulonglong2 v = __ldcs(p2 + t + j * FT);
        k[2 * j] = v.x; k[2 * j + 1] = v.y;
        idx[2 * j] = 2 * (t + j * FT); idx[2 * j + 1] = idx[2 * j] + 1;
      }
    } else {
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        idx[j] = t + j * FT;
        k[j] = idx[j] < len ? __ldcs(p + idx[j]) : 0ull;
      }
    }
  } else {
    const u32* ps = src + base;
    const u32* pd = dst + base;
    if (len == CH && ((reinterpret_cast<uintptr_t>(ps) & 15) == 0) && ((reinterpret_cast<uintptr_t>(pd) & 15) == 0)) {
      const uint4* s4 = reinterpret_cast<const uint4*>(ps);
      const uint4* d4 = reinterpret_cast<const uint4*>(pd);
#pragma unroll
      for (int j = 0; j < KPT / 4; ++j) {
        const uint4 a = __ldcs(s4 + t + j * FT);
        const uint4 b = __ldcs(d4 + t + j * FT);
        const u32 i0 = 4 * (t + j * FT);
        k[4 * j + 0] = ((u64)a.x << 32) | b.x; idx[4 * j + 0] = i0;
        k[4 * j + 1] = ((u64)a.y << 32) | b.y; idx[4 * j + 1] = i0 + 1;
        k[4 * j + 2] = ((u64)a.z << 32) | b.z; idx[4 * j + 2] = i0 + 2;
        k[4 * j + 3] = ((u64)a.w << 32) | b.w; idx[4 * j + 3] = i0 + 3;
      }
    } else {
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        idx[j] = t + j * FT;
        k[j] = idx[j] < len ? (((u64)__ldcs(ps + idx[j]) << 32) | __ldcs(pd + idx[j])) : 0ull;
      }
    }
  }
  __syncthreads();  // hist cleared
  u32 bk[KPT];
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    bk[j] = link_bucket(k[j], g.logB);
    if (idx[j] < len) atomicAdd(&s.hist[bk[j]], 1u);
  }
  __syncthreads();
  block_exclusive_scan<FT>(s.hist, (int)g.B, m.wtmp);
  u32* off = g.koff + ((u64)slot * g.cp + c) * (g.B + 1);
  for (int i = t; i <= (int)g.B; i += FT) off[i] = s.hist[i];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    if (idx[j] < len) {
      const u32 pos = atomicAdd(&s.hist[bk[j]], 1u);
      s.stage[pos] = k[j];
    }
  }
  __syncthreads();
  u64* out = g.kscr + (u64)slot * g.cp * CH + (u64)c * CH;
  if (len == CH) {
    ulonglong2* o2 = reinterpret_cast<ulonglong2*>(out);
    const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(s.stage);
    for (int i = t; i < CH / 2; i += FT) o2[i] = s2[i];
  } else {
    for (u32 i = t; i < len; i += FT) out[i] = s.stage[i];
  }
  __syncthreads();
  if (t == 0) { __threadfence(); atomicAdd(&g.pdone[w], 1u); }
}

// ------------------------------------------------------------------------------------------
// L item helpers: emit one side's partial records of a link bucket
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void emit_records(u64* stage, u32* cursor, u32 node, u32 P, u32 F) {
  const u32 nrec = (P + REC_MAX - 1) / REC_MAX;
  u32 pos = atomicAdd(cursor, nrec);
  for (u32 r = 0; r < nrec; ++r) {
    const u32 p = min(P, REC_MAX), f = min(F, REC_MAX);
    stage[pos + r] = ((u64)node << 32) | ((u64)p << 16) | f;
    P -= p; F -= f;
  }
}

__device__ void emit_side(const Geo& g, SmemL& s, SmemMisc& m, u32 slot, u32 b, int side) {
  const int t = threadIdx.x;
  for (int i = t; i <= (int)g.B; i += FT) s.hist[i] = 0;
  __syncthreads();
  const u32* key = s.nkey[side];
  const u32* P = s.nP[side];
  const u32* F = s.nF[side];
  for (int i = t; i < TCAP; i += FT) {
    const u32 node = key[i];
    if (node != EMPTY32) atomicAdd(&s.hist[side_bucket(node, g.logB)], (P[i] + REC_MAX - 1) / REC_MAX);
  }
  if (t == 0 && m.esc[1 + 2 * side])
    atomicAdd(&s.hist[side_bucket(EMPTY32, g.logB)], (m.esc[1 + 2 * side] + REC_MAX - 1) / REC_MAX);
  __syncthreads();
  block_exclusive_scan<FT>(s.hist, (int)g.B, m.wtmp);
  u32* off = g.roff + (((u64)slot * g.B + b) * 2 + side) * (g.B + 1);
  for (int i = t; i <= (int)g.B; i += FT) off[i] = s.hist[i];
  const u32 total = s.hist[g.B];
  __syncthreads();
  for (int i = t; i < TCAP; i += FT) {
    const u32 node = key[i];
    if (node != EMPTY32) emit_records(s.stage, &s.hist[side_bucket(node, g.logB)], node, P[i], F[i]);
  }
  if (t == 0 && m.esc[1 + 2 * side])
    emit_records(s.stage, &s.hist[side_bucket(EMPTY32, g.logB)], EMPTY32, m.esc[1 + 2 * side], m.esc[2 + 2 * side]);
  __syncthreads();
  u64* out = g.rscr + (((u64)slot * g.B + b) * 2 + side) * g.rcap;
  for (u32 i = t; i < total; i += FT) out[i] = s.stage[i];
  __syncthreads();
}

// ------------------------------------------------------------------------------------------
// L item: aggregate link bucket b of window w
// ------------------------------------------------------------------------------------------
__device__ void item_link(const Geo& g, u64 w, u32 b, SmemL& s, SmemMisc& m) {
  const int t = threadIdx.x;
  const u32 ncp = chunks_of(g, w);
  if (t == 0) { wait_geq(&g.pdone[w], ncp); __threadfence(); }
  for (int i = t; i < TCAP; i += FT) {
    s.lkey[i] = EMPTY64; s.lcnt[i] = 0;
    s.nkey[0][i] = EMPTY32; s.nP[0][i] = 0; s.nF[0][i] = 0;
    s.nkey[1][i] = EMPTY32; s.nP[1][i] = 0; s.nF[1][i] = 0;
  }
  if (t < 8) m.esc[t] = 0;
  if (t == 0) m.flag = 0;
  __syncthreads();  // also publishes thread 0's acquire to the CTA
  const u32 slot = (u32)(w % g.R);
  const u32* koff = g.koff + (u64)slot * g.cp * (g.B + 1);
  for (u32 c = t; c < ncp; c += FT) {
    const u32 lo = ldcg32(koff + (u64)c * (g.B + 1) + b), hi = ldcg32(koff + (u64)c * (g.B + 1) + b + 1);
    s.seg[c] = hi - lo;
    s.seglo[c] = c * CH + lo;
  }
  __syncthreads();
  block_exclusive_scan<FT>(s.seg, (int)ncp, m.wtmp);
  const u32 nb = s.seg[ncp];
  const u64* ks = g.kscr + (u64)slot * g.cp * CH;
  bool ok = true;
  for (u32 i = t; i < nb; i += FT) {
    const u32 c = find_seg(s.seg, ncp, i);
    const u64 key = ldcg64(ks + s.seglo[c] + (i - s.seg[c]));
    if (key == EMPTY64) atomicAdd(&m.esc[0], 1u);
    else ok = smem_link_insert(s.lkey, s.lcnt, key) && ok;
  }
  if (!ok) m.flag = 1;
  __syncthreads();
  // Scan the bucket's part of A_t: unique links, max link packets, sum of counts; and
  // per-source / per-destination partials (row / column sums and nnz restricted to the bucket).
  u32 nl = 0, mx = 0, sm = 0;
  bool ok2 = true;
  for (int i = t; i < TCAP; i += FT) {
    const u64 key = s.lkey[i];
    if (key != EMPTY64) {
      const u32 c = s.lcnt[i];
      nl += 1; mx = max(mx, c); sm += c;
      ok2 = smem_node_upsert(s.nkey[0], s.nP[0], s.nF[0], &m.esc[1], &m.esc[2], (u32)(key >> 32), c, 1) && ok2;
      ok2 = smem_node_upsert(s.nkey[1], s.nP[1], s.nF[1], &m.esc[3], &m.esc[4], (u32)key, c, 1) && ok2;
    }
  }
  if (t == 0 && m.esc[0]) {  // the key ~0 (255.255.255.255 -> 255.255.255.255)
    const u32 c = m.esc[0];
    nl += 1; mx = max(mx, c); sm += c;
    atomicAdd(&m.esc[1], c); atomicAdd(&m.esc[2], 1u);
    atomicAdd(&m.esc[3], c); atomicAdd(&m.esc[4], 1u);
  }
  if (!ok2) m.flag = 1;
  nl = warp_sum(nl); mx = warp_max(mx); sm = warp_sum(sm);
  const int lane = t & 31, wid = t >> 5;
  if (lane == 0) { m.wtmp[wid] = nl; m.wtmp[NWARP + wid] = mx; m.wtmp[2 * NWARP + wid] = sm; }
  __syncthreads();
  if (t == 0) {
    u32 a = 0, bmx = 0, cs = 0;
    for (int i = 0; i < NWARP; ++i) { a += m.wtmp[i]; bmx = max(bmx, m.wtmp[NWARP + i]); cs += m.wtmp[2 * NWARP + i]; }
    u32* r = g.lres + ((u64)slot * g.B + b) * 4;
    r[0] = a; r[1] = bmx; r[2] = cs;
  }
  __syncthreads();
  emit_side(g, s, m, slot, b, 0);
  emit_side(g, s, m, slot, b, 1);
  if (t == 0) {
    if (m.flag) mark_overflow(g, w);
    __threadfence();
    atomicAdd(&g.ldone[w], 1u);
  }
}

// ------------------------------------------------------------------------------------------
// Window finalisation (run by the CTA that completes the window's last S item)
// ------------------------------------------------------------------------------------------
__device__ void finalize_window(const Geo& g, u64 w, SmemMisc& m, u64* __restrict__ out) {
  const int t = threadIdx.x;
  const u32 slot = (u32)(w % g.R);
  u32 v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};  // sums: 0 links, 1 sumc, 2 dsrc, 3 ddst; maxes: 4 maxc, 5 P0, 6 F0, 7 P1, 8 F1
  for (u32 i = t; i < g.B; i += FT) {
    const u32* r = g.lres + ((u64)slot * g.B + i) * 4;
    v[0] += ldcg32(r); v[4] = max(v[4], ldcg32(r + 1)); v[1] += ldcg32(r + 2);
    const u32* s0 = g.sres + (((u64)slot * 2 + 0) * g.B + i) * 4;
    const u32* s1 = g.sres + (((u64)slot * 2 + 1) * g.B + i) * 4;
    v[2] += ldcg32(s0); v[5] = max(v[5], ldcg32(s0 + 1)); v[6] = max(v[6], ldcg32(s0 + 2));
    v[3] += ldcg32(s1); v[7] = max(v[7], ldcg32(s1 + 1)); v[8] = max(v[8], ldcg32(s1 + 2));
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) v[j] = warp_sum(v[j]);
#pragma unroll
  for (int j = 4; j < 9; ++j) v[j] = warp_max(v[j]);
  const int lane = t & 31, wid = t >> 5;
  __syncthreads();
  if (lane == 0)
    for (int j = 0; j < 9; ++j) m.wtmp[j * NWARP + wid] = v[j];
  __syncthreads();
  if (t == 0) {
    u32 r[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < NWARP; ++i) {
      for (int j = 0; j < 4; ++j) r[j] += m.wtmp[j * NWARP + i];
      for (int j = 4; j < 9; ++j) r[j] = max(r[j], m.wtmp[j * NWARP + i]);
    }
    const u64 wlen = min(g.W, g.n - w * g.W);
    u64* o = out + w * NSG_NUM_STATS;
    o[NSG_VALID_PACKETS] = r[1];
    o[NSG_UNIQUE_LINKS] = r[0];
    o[NSG_MAX_LINK_PACKETS] = r[4];
    o[NSG_UNIQUE_SOURCES] = r[2];
    o[NSG_MAX_SOURCE_PACKETS] = r[5];
    o[NSG_MAX_SOURCE_FANOUT] = r[6];
    o[NSG_UNIQUE_DESTINATIONS] = r[3];
    o[NSG_MAX_DESTINATION_PACKETS] = r[7];
    o[NSG_MAX_DESTINATION_FANIN] = r[8];
    if ((u64)r[1] != wlen && ld_acquire32(&g.ovf[w]) == 0) atomicAdd(&g.diag[1], 1u);
    if ((g.flags & NSG_FLAG_INJECT_OVERFLOW) && (w & 1)) mark_overflow(g, w);
    __threadfence();
    st_release32(&g.fin[w], 1u);
  }
}

// ------------------------------------------------------------------------------------------
// S item: merge side bucket sb of one side of window w
// ------------------------------------------------------------------------------------------
__device__ void item_side(const Geo& g, u64 w, int side, u32 sb, SmemS& s, SmemMisc& m, u64* __restrict__ out) {
  const int t = threadIdx.x;
  if (t == 0) { wait_geq(&g.ldone[w], g.B); __threadfence(); }
  for (int i = t; i < TCAP; i += FT) { s.key[i] = EMPTY32; s.P[i] = 0; s.F[i] = 0; }
  if (t < 8) m.esc[t] = 0;
  if (t == 0) { m.flag = 0; m.last = 0; }
  __syncthreads();
  const u32 slot = (u32)(w % g.R);
  for (u32 b = t; b < g.B; b += FT) {
    const u32* off = g.roff + (((u64)slot * g.B + b) * 2 + side) * (g.B + 1);
    const u32 lo = ldcg32(off + sb), hi = ldcg32(off + sb + 1);
    s.seg[b] = hi - lo;
    s.seglo[b] = (b * 2 + side) * g.rcap + lo;
  }
  __syncthreads();
  block_exclusive_scan<FT>(s.seg, (int)g.B, m.wtmp);
  const u32 nr = s.seg[g.B];
  const u64* rs = g.rscr + (u64)slot * g.B * 2 * g.rcap;
  bool ok = true;
  for (u32 i = t; i < nr; i += FT) {
    const u32 b = find_seg(s.seg, g.B, i);
    const u64 rec = ldcg64(rs + s.seglo[b] + (i - s.seg[b]));
    ok = smem_node_upsert(s.key, s.P, s.F, &m.esc[1], &m.esc[2], (u32)(rec >> 32), (u32)(rec >> 16) & 0xFFFFu,
                          (u32)rec & 0xFFFFu) && ok;
  }
  if (!ok) m.flag = 1;
  __syncthreads();
  // unique nodes (1^T |A_t 1|_0 or its mirror), max packets (max A_t 1), max fan (max |A_t|_0 1)
  u32 d = 0, mp = 0, mf = 0;
  for (int i = t; i < TCAP; i += FT) {
    if (s.key[i] != EMPTY32) { d += 1; mp = max(mp, s.P[i]); mf = max(mf, s.F[i]); }
  }
  if (t == 0 && m.esc[1]) { d += 1; mp = max(mp, m.esc[1]); mf = max(mf, m.esc[2]); }
  d = warp_sum(d); mp = warp_max(mp); mf = warp_max(mf);
  const int lane = t & 31, wid = t >> 5;
  if (lane == 0) { m.wtmp[wid] = d; m.wtmp[NWARP + wid] = mp; m.wtmp[2 * NWARP + wid] = mf; }
  __syncthreads();
  if (t == 0) {
    u32 a = 0, bp = 0, cf = 0;
    for (int i = 0; i < NWARP; ++i) { a += m.wtmp[i]; bp = max(bp, m.wtmp[NWARP + i]); cf = max(cf, m.wtmp[2 * NWARP + i]); }
    u32* r = g.sres + (((u64)slot * 2 + side) * g.B + sb) * 4;
    r[0] = a; r[1] = bp; r[2] = cf;
    if (m.flag) mark_overflow(g, w);
    __threadfence();
    const u32 old = atomicAdd(&g.sdone[w], 1u);
    m.last = (old == 2 * g.B - 1) ? 1u : 0u;
    if (m.last) __threadfence();
  }
  __syncthreads();
  if (m.last) finalize_window(g, w, m, out);
}

// ------------------------------------------------------------------------------------------
// Ticket decoding: step k holds S(k-LAG_S), L(k-LAG_L), P(k) in that order.
// ------------------------------------------------------------------------------------------
__host__ __device__ __forceinline__ u64 step_prefix(const Geo& g, u64 k) {
  const u64 kp = k < g.nw ? k : g.nw;
  const u64 p = kp * g.cp - (kp == g.nw ? (u64)(g.cp - g.cp_last) : 0ull);
  const u64 kl = k > (u64)LAG_L ? (k - LAG_L < g.nw ? k - LAG_L : g.nw) : 0ull;
  const u64 ks = k > (u64)LAG_S ? (k - LAG_S < g.nw ? k - LAG_S : g.nw) : 0ull;
  return p + kl * g.B + ks * 2ull * g.B;
}

__global__ void __launch_bounds__(FT, 2)
fast_kernel(Geo g, const u32* __restrict__ src, const u32* __restrict__ dst, const u64* __restrict__ keys,
            u64* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SmemMisc& m = *reinterpret_cast<SmemMisc*>(smem_raw);
  unsigned char* u = smem_raw + MISC_BYTES;
  for (;;) {
    if (threadIdx.x == 0) m.tk = atomicAdd(reinterpret_cast<unsigned long long*>(g.ticket), 1ull);
    __syncthreads();
    const u64 tk = m.tk;
    __syncthreads();
    if (tk >= g.total_items) break;
    // binary search the step: largest k with step_prefix(k) <= tk
    u64 lo = 0, hi = g.nw + LAG_S;
    while (lo < hi) {
      const u64 mid = (lo + hi + 1) >> 1;
      if (step_prefix(g, mid) <= tk) lo = mid; else hi = mid - 1;
    }
    const u64 k = lo;
    u64 idx = tk - step_prefix(g, k);
    if (k >= (u64)LAG_S && k - LAG_S < g.nw) {
      if (idx < 2ull * g.B) {
        item_side(g, k - LAG_S, (int)(idx / g.B), (u32)(idx % g.B), *reinterpret_cast<SmemS*>(u), m, out);
        continue;
      }
      idx -= 2ull * g.B;
    }
    if (k >= (u64)LAG_L && k - LAG_L < g.nw) {
      if (idx < g.B) {
        item_link(g, k - LAG_L, (u32)idx, *reinterpret_cast<SmemL*>(u), m);
        continue;
      }
      idx -= g.B;
    }
    item_partition(g, src, dst, keys, k, (u32)idx, *reinterpret_cast<SmemP*>(u), m);
  }
}

// ------------------------------------------------------------------------------------------
// L2 path: one CTA per window, global-memory hash tables (also the overflow hand-off)
// ------------------------------------------------------------------------------------------
constexpr int GT = 512;

struct GGeo {
  u64 n, W, nw;
  u64 LC;       // slots per table (power of two >= 2*W)
  u32 G;        // table sets
  int only_overflowed;
  u64* lkey;    // [G][LC]
  u32* lcnt;    // [G][LC]
  u32* nkey;    // [G][2][LC]
  u32* nP;      // [G][2][LC]
  u32* nF;      // [G][2][LC]
  const u32* ovf;
  u32* diag;
};

__device__ __forceinline__ void glob_link_insert(u64* lkey, u32* lcnt, u64 LC, u64 key) {
  u64 slot = hash64(key) & (LC - 1);
  for (;;) {
    u64 k = ldcg64(&lkey[slot]);
    if (k == EMPTY64) {
      const u64 old = atomicCAS(reinterpret_cast<unsigned long long*>(&lkey[slot]), EMPTY64, key);
      k = (old == EMPTY64) ? key : old;
    }
    if (k == key) { atomicAdd(&lcnt[slot], 1u); return; }
    slot = (slot + 1) & (LC - 1);  // the table has >= 2x the window's slots: never full
  }
}

__device__ __forceinline__ void glob_node_upsert(u32* key, u32* P, u32* F, u64 LC, u32* escP, u32* escF, u32 node,
                                                 u32 p, u32 f) {
  if (node == EMPTY32) { atomicAdd(escP, p); atomicAdd(escF, f); return; }
  u64 slot = ((u64)hash32(node) * 0x9E3779B97F4A7C15ull >> 11) & (LC - 1);
  for (;;) {
    u32 k = ldcg32(&key[slot]);
    if (k == EMPTY32) {
      const u32 old = atomicCAS(&key[slot], EMPTY32, node);
      k = (old == EMPTY32) ? node : old;
    }
    if (k == node) { atomicAdd(&P[slot], p); atomicAdd(&F[slot], f); return; }
    slot = (slot + 1) & (LC - 1);
  }
}

__global__ void __launch_bounds__(GT)
global_kernel(GGeo g, const u32* __restrict__ src, const u32* __restrict__ dst, const u64* __restrict__ keys,
              u64* __restrict__ out) {
  __shared__ u32 esc[5];
  __shared__ u32 red[9 * (GT / 32)];
  if (g.only_overflowed && ldcg32(&g.diag[0]) == 0) return;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const u64 LC = g.LC;
  u64* lkey = g.lkey + (u64)blockIdx.x * LC;
  u32* lcnt = g.lcnt + (u64)blockIdx.x * LC;
  for (u64 w = blockIdx.x; w < g.nw; w += g.G) {
    if (g.only_overflowed && ldcg32(&g.ovf[w]) == 0) continue;
    const u64 base = w * g.W;
    const u64 len = min(g.W, g.n - base);
    for (u64 i = t; i < LC; i += GT) {
      lkey[i] = EMPTY64; lcnt[i] = 0;
      for (int sd = 0; sd < 2; ++sd) {
        const u64 o = ((u64)blockIdx.x * 2 + sd) * LC + i;
        g.nkey[o] = EMPTY32; g.nP[o] = 0; g.nF[o] = 0;
      }
    }
    if (t < 5) esc[t] = 0;
    __syncthreads();
    for (u64 i = t; i < len; i += GT) {
      const u64 key = keys ? keys[base + i] : (((u64)src[base + i] << 32) | dst[base + i]);
      if (key == EMPTY64) atomicAdd(&esc[0], 1u);
      else glob_link_insert(lkey, lcnt, LC, key);
    }
    __syncthreads();
    u32* k0 = g.nkey + ((u64)blockIdx.x * 2 + 0) * LC;
    u32* k1 = g.nkey + ((u64)blockIdx.x * 2 + 1) * LC;
    u32* P0 = g.nP + ((u64)blockIdx.x * 2 + 0) * LC;
    u32* P1 = g.nP + ((u64)blockIdx.x * 2 + 1) * LC;
    u32* F0 = g.nF + ((u64)blockIdx.x * 2 + 0) * LC;
    u32* F1 = g.nF + ((u64)blockIdx.x * 2 + 1) * LC;
    u32 nl = 0, mx = 0, sm = 0;
    for (u64 i = t; i < LC; i += GT) {
      const u64 key = ldcg64(&lkey[i]);
      if (key != EMPTY64) {
        const u32 c = ldcg32(&lcnt[i]);
        nl += 1; mx = max(mx, c); sm += c;
        glob_node_upsert(k0, P0, F0, LC, &esc[1], &esc[2], (u32)(key >> 32), c, 1);
        glob_node_upsert(k1, P1, F1, LC, &esc[3], &esc[4], (u32)key, c, 1);
      }
    }
    if (t == 0 && esc[0]) {
      const u32 c = esc[0];
      nl += 1; mx = max(mx, c); sm += c;
      atomicAdd(&esc[1], c); atomicAdd(&esc[2], 1u); atomicAdd(&esc[3], c); atomicAdd(&esc[4], 1u);
    }
    __syncthreads();
    u32 d0 = 0, p0 = 0, f0 = 0, d1 = 0, p1 = 0, f1 = 0;
    for (u64 i = t; i < LC; i += GT) {
      if (ldcg32(&k0[i]) != EMPTY32) { d0 += 1; p0 = max(p0, ldcg32(&P0[i])); f0 = max(f0, ldcg32(&F0[i])); }
      if (ldcg32(&k1[i]) != EMPTY32) { d1 += 1; p1 = max(p1, ldcg32(&P1[i])); f1 = max(f1, ldcg32(&F1[i])); }
    }
    if (t == 0 && esc[1]) { d0 += 1; p0 = max(p0, esc[1]); f0 = max(f0, esc[2]); }
    if (t == 0 && esc[3]) { d1 += 1; p1 = max(p1, esc[3]); f1 = max(f1, esc[4]); }
    u32 v[9] = {nl, sm, d0, d1, mx, p0, f0, p1, f1};
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = warp_sum(v[j]);
#pragma unroll
    for (int j = 4; j < 9; ++j) v[j] = warp_max(v[j]);
    if (lane == 0)
      for (int j = 0; j < 9; ++j) red[j * (GT / 32) + wid] = v[j];
    __syncthreads();
    if (t == 0) {
      u32 r[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int i = 0; i < GT / 32; ++i) {
        for (int j = 0; j < 4; ++j) r[j] += red[j * (GT / 32) + i];
        for (int j = 4; j < 9; ++j) r[j] = max(r[j], red[j * (GT / 32) + i]);
      }
      u64* o = out + w * NSG_NUM_STATS;
      o[NSG_VALID_PACKETS] = r[1];
      o[NSG_UNIQUE_LINKS] = r[0];
      o[NSG_MAX_LINK_PACKETS] = r[4];
      o[NSG_UNIQUE_SOURCES] = r[2];
      o[NSG_MAX_SOURCE_PACKETS] = r[5];
      o[NSG_MAX_SOURCE_FANOUT] = r[6];
      o[NSG_UNIQUE_DESTINATIONS] = r[3];
      o[NSG_MAX_DESTINATION_PACKETS] = r[7];
      o[NSG_MAX_DESTINATION_FANIN] = r[8];
      if ((u64)r[1] != len) atomicAdd(&g.diag[1], 1u);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------
// Host side: layout, device checks, launches
// ------------------------------------------------------------------------------------------
constexpr size_t DIAG_OFFSET = 64;
constexpr size_t CTRL_BYTES = 256;
constexpr u64 GLOBAL_BUDGET = 2ull << 30;  // cap on L2-path table memory

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
static u64 next_pow2(u64 x) { u64 p = 1; while (p < x) p <<= 1; return p; }
static u32 ilog2(u64 x) { u32 l = 0; while ((1ull << l) < x) ++l; return l; }

struct Layout {
  bool fast;
  u64 nw;
  // fast
  u32 logB, B, cp, cp_last, rcap, R;
  size_t o_pw, o_kscr, o_koff, o_rscr, o_roff, o_lres, o_sres;
  size_t memset_bytes;
  // global
  u64 LC;
  u32 G;
  size_t o_glk, o_glc, o_gnk, o_gnp, o_gnf;
  size_t total;
};

static Layout make_layout(u64 n, u64 W, int sms) {
  Layout L;
  memset(&L, 0, sizeof(L));
  L.nw = (n + W - 1) / W;
  L.fast = W <= FAST_MAX_WINDOW;
  size_t o = CTRL_BYTES;
  L.o_pw = o;
  o = align256(o + 5 * sizeof(u32) * L.nw);
  L.memset_bytes = o;
  if (L.fast) {
    const u64 want = (W + BUCKET_KEYS - 1) / BUCKET_KEYS;
    L.B = (u32)next_pow2(want < 1 ? 1 : want);
    L.logB = ilog2(L.B);
    L.cp = (u32)((W + CH - 1) / CH);
    const u64 last = n - (L.nw - 1) * W;
    L.cp_last = (u32)((last + CH - 1) / CH);
    L.rcap = (u32)(TCAP + 2 + W / REC_MAX + 1);
    L.R = (u32)(L.nw < (u64)RSLOTS ? L.nw : (u64)RSLOTS);
    L.o_kscr = o; o = align256(o + (size_t)L.R * L.cp * CH * sizeof(u64));
    L.o_koff = o; o = align256(o + (size_t)L.R * L.cp * (L.B + 1) * sizeof(u32));
    L.o_rscr = o; o = align256(o + (size_t)L.R * L.B * 2 * L.rcap * sizeof(u64));
    L.o_roff = o; o = align256(o + (size_t)L.R * L.B * 2 * (L.B + 1) * sizeof(u32));
    L.o_lres = o; o = align256(o + (size_t)L.R * L.B * 4 * sizeof(u32));
    L.o_sres = o; o = align256(o + (size_t)L.R * 2 * L.B * 4 * sizeof(u32));
  }
  // L2-path table sets: the full path for large windows, the overflow hand-off otherwise.
  L.LC = next_pow2(2 * W);
  const u64 set_bytes = L.LC * (8 + 4 + 2 * 12);
  u64 G = L.fast ? 8 : (u64)(2 * sms);
  const u64 by_budget = GLOBAL_BUDGET / set_bytes;
  if (G > by_budget) G = by_budget;
  if (G < 1) G = 1;
  if (G > L.nw) G = L.nw;
  L.G = (u32)G;
  L.o_glk = o; o = align256(o + (size_t)G * L.LC * 8);
  L.o_glc = o; o = align256(o + (size_t)G * L.LC * 4);
  L.o_gnk = o; o = align256(o + (size_t)G * 2 * L.LC * 4);
  L.o_gnp = o; o = align256(o + (size_t)G * 2 * L.LC * 4);
  L.o_gnf = o; o = align256(o + (size_t)G * 2 * L.LC * 4);
  L.total = o;
  return L;
}

struct DevInfo {
  bool init = false;
  bool supported = false;
  int sms = 0;
  int fast_blocks = 0;  // co-resident fast_kernel CTAs
};
static std::mutex g_mu;
static DevInfo g_dev[64];
static thread_local unsigned g_last_launches = 0;

static nsg_status dev_info(DevInfo& out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return NSG_ERR_CUDA;
  if (dev < 0 || dev >= 64) return NSG_ERR_UNSUPPORTED_DEVICE;
  std::lock_guard<std::mutex> lk(g_mu);
  DevInfo& d = g_dev[dev];
  if (!d.init) {
    int major = 0, minor = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return NSG_ERR_CUDA;
    if (cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) return NSG_ERR_CUDA;
    if (cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return NSG_ERR_CUDA;
    d.supported = (major == 10 && minor == 0);
    if (d.supported) {
      if (cudaFuncSetAttribute(fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FAST_SMEM) != cudaSuccess)
        return NSG_ERR_CUDA;
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fast_kernel, FT, FAST_SMEM) != cudaSuccess)
        return NSG_ERR_CUDA;
      if (per_sm < 1) return NSG_ERR_UNSUPPORTED_DEVICE;
      d.fast_blocks = per_sm * d.sms;
    }
    d.init = true;
  }
  out = d;
  return d.supported ? NSG_OK : NSG_ERR_UNSUPPORTED_DEVICE;
}

static int sms_for_layout() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 148;
  return sms;
}

static nsg_status run(const u32* src, const u32* dst, const u64* keys, u64 n, u64 W, u64* out, void* ws,
                      size_t ws_bytes, void* stream, u32 flags) {
  g_last_launches = 0;
  if (W == 0 || W > NSG_MAX_WINDOW) return NSG_ERR_INVALID_ARGUMENT;
  if (n == 0) return NSG_OK;
  if ((keys == nullptr) == (src == nullptr && dst == nullptr)) return NSG_ERR_INVALID_ARGUMENT;
  if (!keys && (!src || !dst)) return NSG_ERR_INVALID_ARGUMENT;
  if (!out || !ws) return NSG_ERR_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(ws) & 255) || (reinterpret_cast<uintptr_t>(out) & 7)) return NSG_ERR_INVALID_ARGUMENT;
  if (keys && (reinterpret_cast<uintptr_t>(keys) & 7)) return NSG_ERR_INVALID_ARGUMENT;
  if (src && ((reinterpret_cast<uintptr_t>(src) & 3) || (reinterpret_cast<uintptr_t>(dst) & 3)))
    return NSG_ERR_INVALID_ARGUMENT;
  DevInfo d;
  const nsg_status st = dev_info(d);
  if (st != NSG_OK) return st;
  const Layout L = make_layout(n, W, d.sms);
  if (ws_bytes < L.total) return NSG_ERR_WORKSPACE_TOO_SMALL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  unsigned char* base = reinterpret_cast<unsigned char*>(ws);
  if (cudaMemsetAsync(base, 0, L.memset_bytes, s) != cudaSuccess) return NSG_ERR_CUDA;

  u32* pw = reinterpret_cast<u32*>(base + L.o_pw);
  GGeo gg;
  gg.n = n; gg.W = W; gg.nw = L.nw; gg.LC = L.LC; gg.G = L.G;
  gg.lkey = reinterpret_cast<u64*>(base + L.o_glk);
  gg.lcnt = reinterpret_cast<u32*>(base + L.o_glc);
  gg.nkey = reinterpret_cast<u32*>(base + L.o_gnk);
  gg.nP = reinterpret_cast<u32*>(base + L.o_gnp);
  gg.nF = reinterpret_cast<u32*>(base + L.o_gnf);
  gg.ovf = pw + 4 * L.nw;
  gg.diag = reinterpret_cast<u32*>(base + DIAG_OFFSET);

  const bool use_fast = L.fast && !(flags & NSG_FLAG_FORCE_GLOBAL);
  if (use_fast) {
    Geo g;
    g.n = n; g.W = W; g.nw = L.nw;
    g.logB = L.logB; g.B = L.B; g.cp = L.cp; g.cp_last = L.cp_last; g.rcap = L.rcap; g.R = L.R;
    g.flags = flags;
    g.ticket = reinterpret_cast<u64*>(base);
    g.diag = reinterpret_cast<u32*>(base + DIAG_OFFSET);
    g.pdone = pw; g.ldone = pw + L.nw; g.sdone = pw + 2 * L.nw; g.fin = pw + 3 * L.nw; g.ovf = pw + 4 * L.nw;
    g.kscr = reinterpret_cast<u64*>(base + L.o_kscr);
    g.koff = reinterpret_cast<u32*>(base + L.o_koff);
    g.rscr = reinterpret_cast<u64*>(base + L.o_rscr);
    g.roff = reinterpret_cast<u32*>(base + L.o_roff);
    g.lres = reinterpret_cast<u32*>(base + L.o_lres);
    g.sres = reinterpret_cast<u32*>(base + L.o_sres);
    g.total_items = step_prefix(g, L.nw + LAG_S);
    u64 grid = (u64)d.fast_blocks;
    if (grid > g.total_items) grid = g.total_items;
    fast_kernel<<<(unsigned)grid, FT, FAST_SMEM, s>>>(g, src, dst, keys, out);
    g_last_launches++;
    if (cudaGetLastError() != cudaSuccess) return NSG_ERR_CUDA;
    if (!(flags & NSG_FLAG_NO_FALLBACK_CHECK)) {
      gg.only_overflowed = 1;
      global_kernel<<<L.G, GT, 0, s>>>(gg, src, dst, keys, out);
      g_last_launches++;
      if (cudaGetLastError() != cudaSuccess) return NSG_ERR_CUDA;
    }
  } else {
    gg.only_overflowed = 0;
    global_kernel<<<L.G, GT, 0, s>>>(gg, src, dst, keys, out);
    g_last_launches++;
    if (cudaGetLastError() != cudaSuccess) return NSG_ERR_CUDA;
  }
  return NSG_OK;
}

}  // namespace nsg

// ------------------------------------------------------------------------------------------
// C ABI
// ------------------------------------------------------------------------------------------
extern "C" {

uint64_t nsg_num_windows(uint64_t n_packets, uint64_t window) {
  if (n_packets == 0 || window == 0) return 0;
  return (n_packets + window - 1) / window;
}

size_t nsg_workspace_bytes(uint64_t n_packets, uint64_t window) {
  if (n_packets == 0 || window == 0 || window > NSG_MAX_WINDOW) return 0;
  return nsg::make_layout(n_packets, window, nsg::sms_for_layout()).total;
}

nsg_status nsg_window_stats(const uint32_t* src, const uint32_t* dst, uint64_t n_packets, uint64_t window,
                            uint64_t* out, void* workspace, size_t workspace_bytes, void* stream) {
  if (n_packets && (!src || !dst)) return NSG_ERR_INVALID_ARGUMENT;
  return nsg::run(src, dst, nullptr, n_packets, window, reinterpret_cast<nsg::u64*>(out), workspace, workspace_bytes,
                  stream, 0);
}

nsg_status nsg_window_stats_packed(const uint64_t* keys, uint64_t n_packets, uint64_t window, uint64_t* out,
                                   void* workspace, size_t workspace_bytes, void* stream) {
  if (n_packets && !keys) return NSG_ERR_INVALID_ARGUMENT;
  return nsg::run(nullptr, nullptr, reinterpret_cast<const nsg::u64*>(keys), n_packets, window,
                  reinterpret_cast<nsg::u64*>(out), workspace, workspace_bytes, stream, 0);
}

nsg_status nsg_window_stats_ex(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n_packets,
                               uint64_t window, uint64_t* out, void* workspace, size_t workspace_bytes,
                               void* stream, uint32_t flags) {
  return nsg::run(src, dst, reinterpret_cast<const nsg::u64*>(keys), n_packets, window,
                  reinterpret_cast<nsg::u64*>(out), workspace, workspace_bytes, stream, flags);
}

size_t nsg_diag_offset(void) { return nsg::DIAG_OFFSET; }

unsigned nsg_last_launches(void) { return nsg::g_last_launches; }

const char* nsg_status_string(nsg_status s) {
  switch (s) {
    case NSG_OK: return "NSG_OK";
    case NSG_ERR_INVALID_ARGUMENT: return "NSG_ERR_INVALID_ARGUMENT";
    case NSG_ERR_CUDA: return "NSG_ERR_CUDA";
    case NSG_ERR_WORKSPACE_TOO_SMALL: return "NSG_ERR_WORKSPACE_TOO_SMALL";
    case NSG_ERR_UNSUPPORTED_DEVICE: return "NSG_ERR_UNSUPPORTED_DEVICE";
    case NSG_ERR_INTERNAL: return "NSG_ERR_INTERNAL";
  }
  return "NSG_ERR_UNKNOWN";
}

const char* nsg_version(void) { return "libnsg sm_100a " __DATE__ " " __TIME__; }

}  // extern "C"
