// ARCHIVED EXPERIMENT (not built into libnsg): the persistent warp-specialised per-window kernel tried in
// round 2 (peaked at 13.7 Gpkt/s on C2, below the flat three-kernel path); kept for the phase
// microbenchmarks phases.cu / lpart.cu, see profiles/README.md.
// nsg_win.cuh — the per-window statistics kernel of libnsg (round 2 design), windows < 2^20.
//
// What it computes: for every window of W consecutive packets, the nine Table 2 scalars of the
// traffic matrix A_t (destination mirrors, line 173): valid packets (:180),
// unique links (:181), max link packets (:183), unique sources (:184), max source packets (:186), max
// source fan-out (:188) and the three destination mirrors.  Readings: DESIGN.md §2.
//
// How: one persistent CTA per SM pulls work items from a global ticket sequence.  Per
// window there are three item classes, exchanged through L2-resident scratch slots:
//   P(w,c)  partition: 4096 keys of the window (TMA bulk load from HBM) counting-sorted by link bucket
//           (top bits of key * phi64) and written to the window's key scratch;
//   L(w,b)  link bucket b: its segments of every chunk gathered (cp.async) into SMEM, group-by-count in
//           an SMEM open-addressing table (A_t restricted to the bucket: unique links, max link, sum of
//           counts), then one record (node<<32 | count) per link and side, counting-sorted by side bucket;
//   S(w,s,q) side bucket q of side s: the records of every link bucket, merged per node in an SMEM table
//           of (node, packets | fan << 20): unique nodes, max packets (row/column sums), max fan.
// The last S item of a window writes its row.  Window accumulators are global atomics.
//
// Inside a CTA the work is warp-specialised: K producer warps (one per SMEM stage) claim tickets in
// rounds of K, wait for the item's dependencies, and fill their stage with the item's input (bulk copies
// complete on an mbarrier); 16 consumer warps process the stages in ticket order; K signaler warps
// publish each finished item (release-add on the window counter) so the release latency is off the
// consumers' and producers' critical paths.  An item only waits on items with smaller tickets, and each
// CTA processes its items in ticket order, so the schedule is deadlock-free.
#pragma once
#include "nsg_internal.h"
#include "nsg_common.cuh"

namespace nsg {
namespace win {

constexpr int NCW = 16;                       // consumer warps
constexpr int NCT = NCW * 32;                 // consumer threads
constexpr int K = 4;                          // SMEM stages = producer warps
constexpr int NT = NCT + K * 32 + 32;         // + one signaler warp: 672 threads, one CTA per SM
constexpr int SK = 4096;                      // stage capacity in u64 (32 KB)
constexpr int CH = 4096;                      // keys per partition item
constexpr int LOG_TL = 12, TL = 1 << LOG_TL;  // link-table slots
constexpr int LOG_TS = 12, TS = 1 << LOG_TS;  // node-table slots
constexpr u32 FILL_L = 2560, FILL_S = 2560;   // distinct entries per item before the window is handed to the L2 path
constexpr u64 BKEYS = 2048;                   // target keys per link bucket and nodes per side bucket
constexpr u64 MAX_W = 1ull << 18;             // windows this kernel takes (<= 128 link / side buckets)
constexpr int PFS = 20;                       // node packets: 20-bit field (W < 2^20)
constexpr u32 PMASK = (1u << PFS) - 1;
constexpr u32 FMAX = 0xFFFu;                  // fan field: 12 bits, wraps counted in the wrap list
constexpr u32 RCAP = 5128;                    // records per link bucket (both sides) >= 2 * (FILL_L + 1)
constexpr int WRAPCAP = 64;
constexpr int LAG_L = 7, LAG_S = 14;          // steps between a window's P, L and S items
constexpr int RS = 18;                        // scratch slots (windows in flight) > LAG_S
constexpr int MAXB = 128;                     // link / side buckets
constexpr int PSEG = 64;                      // segment descriptors kept in SMEM per producer (more: read from L2)
constexpr int MAXREG = 8;
constexpr int RING = 32;                      // completed items awaiting their signal
constexpr u64 MUL_L = 0x9E3779B97F4A7C15ull;  // link hash: top bits of key * phi64
constexpr u32 MUL_N = 0x9E3779B9u;            // node hash: top bits of node * phi32
constexpr u64 TFREE = ~0ull, TPEND = ~0ull - 1;  // stage ticket states

enum : u32 { T_P = 0, T_L = 1, T_S = 2, T_END = 3 };

// Timing experiment only (-DNSG_WIN_PROF): per-CTA cycle counters, read by nsg_debug_win_prof.
#ifdef NSG_WIN_PROF
constexpr int PROF_N = 32;
__device__ unsigned long long g_win_prof[1024][PROF_N];
__device__ unsigned long long g_win_prof_pend;
#define WPROF_DECL unsigned long long _pt = clock64();
#define WPROF_MARK(slot) do { const unsigned long long _n = clock64(); atomicAdd(&g_win_prof[blockIdx.x][slot], _n - _pt); _pt = _n; } while (0)
#define WPROF_RESET() do { _pt = clock64(); } while (0)
#define WPROF_CNT(slot) atomicAdd(&g_win_prof[blockIdx.x][slot], 1ull)
#else
#define WPROF_DECL
#define WPROF_MARK(slot) do {} while (0)
#define WPROF_RESET() do {} while (0)
#define WPROF_CNT(slot) do {} while (0)
#endif
// Sub-phase marks for the phase microbenchmark (tools/microbench/phases.cu) only.
#ifdef NSG_PHASE_MARKS
__device__ long long g_pm[64];
#define PMARK(i) do { if (threadIdx.x == 0) { atomicAdd((unsigned long long*)&g_pm[i], (unsigned long long)clock64()); } } while (0)
#else
#define PMARK(i) do {} while (0)
#endif
#ifndef NSG_WIN_PROF
#define g_win_prof_pend g_win_prof_pend_unused
__device__ unsigned long long g_win_prof_pend_unused;
#endif
// counter slots: consumers 0 wait full, 1 P, 2 L part, 3 L final, 4 S part, 5 S final, 6 done arrive
//                producer (summed over j) 8 stage-free wait, 9 deps + offsets, 11 desc, 12 issue
//                signaler 16 idle, 18 signal; counts 24 P, 25 L, 26 S

// Per-window state (64 B), zeroed by the host before the launch.
struct WinState {
  u32 pdone, ldone, sdone, ovf;
  u32 links, maxc, sumc, r0;
  u32 nodes[2], maxp[2], maxf[2], r1[2];
};
static_assert(sizeof(WinState) == 64, "WinState is 64 B");

struct WGeo {
  u64 n, W, nw;
  u32 logB, B, logBs, Bs, CP;
  u32 nP, nL, nS;                  // items per window
  u32 nreg;
  u64 reg_k0[MAXREG], reg_t0[MAXREG + 1];
  u32 reg_f[MAXREG], reg_m[MAXREG];
  u64 total;                       // tickets
  u64* ticket;
  WinState* ws;                    // [nw]
  u64* kscr;                       // [RS][CP][CH]
  u32* koff;                       // [RS][CP][B]  (start << 16 | count) of bucket b in chunk c: a P item's row
  u64* rscr;                       // [RS][B][RCAP]
  u32* roff;                       // [RS][B][2Bs] (start << 16 | count) of side bucket (s,q) in link bucket b: an L item's row
  u32* diag;                       // [0] any window overflowed, [1] self-check failures
  const u32* arrived;              // streamed input: per chunk of chunk_w windows, set when copied
  u32 chunk_w;
  u64* const* mirror;
  u32 n_mirror;
  u64 mirror_row0;
  u32 inject;                      // NSG_FLAG_INJECT_OVERFLOW: odd windows are handed to the L2 path
};

struct Item { u32 type, idx; u64 w; };

struct Desc {
  u32 type, idx;
  u64 w;
  u32 n;      // elements in this stage fill
  u32 part, nparts;
  u32 ntot;   // elements of the whole item
  u32 len;    // window length (P items)
  u32 soa;    // P items: the stage holds src[0, CH) and dst[0, CH) as u32 (SoA input)
};

struct SigE { u32 type, idx; u64 w; };

// Shared memory (dynamic).  The stage buffers first (TMA destinations).
struct Smem {
  u64 stage[K][SK];                // 128 KB
  u64 lkey[TL];                    // 32 KB  link table keys (EMPTY64 = free)
  u32 lcnt[TL];                    // 16 KB  link counts (0 = free)
  u32 nkey[TS];                    // 16 KB  node table (EMPTY32 = free)
  u32 npf[TS];                     // 16 KB  packets | fan << 20
  uint16_t claim[TL];              // 8 KB   slots claimed by the current item, in claim order (dense final scans)
  u32 hist[2][2 * MAXB];           // 2 KB   counting-sort histograms, double-buffered by item parity
  u32 offs[2 * MAXB];              // 1 KB   exclusive offsets of the current item's histogram
  u32 pseg[K][PSEG];               // 1 KB   per-producer gathered segment descriptors
  u32 wrap[2][WRAPCAP];            // node slots whose fan field wrapped (per S-item parity)
  Desc desc[K];
  SigE ring[RING];                 // completed items, in completion (= ticket) order
  u64 tq[K][2];                    // per stage: ticket of the current item, ticket claimed next
  u64 full[K], done[K];            // mbarriers
  u32 red[4][NCW];                 // per-warp partials of an item's statistics
  u32 ring_head, ring_tail, sel, L0;
  u32 ncl[2][2];                   // claim-list lengths [L / S][item parity]
  // per-item scalars, double-buffered by item parity: an item resets its copy after its last barrier,
  // and the next item that uses that copy starts only after every thread passed the intermediate
  // item's first barrier
  u32 lesc[2], lfill[2], lovf[2];  // link item: escape-key count, claims, overflow
  u32 sescP[2], sescF[2], sfill[2], sovf[2], nwrap[2];
};

static_assert(sizeof(Smem) <= 232448, "Smem exceeds the 227 KB opt-in shared memory per CTA");

// ---------------------------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ u32 sa(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* b, u32 cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_arrive(u64* b) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(u64* b, u32 tx) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(sa(b)), "r"(tx)
               : "memory");
}
__device__ __forceinline__ bool mbar_try(u64* b, u32 par) {
  u32 ok;
  asm volatile(
      "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
      : "=r"(ok)
      : "r"(sa(b)), "r"(par), "r"(1000u)
      : "memory");
  return ok != 0;
}
// Waiting warps must not spin: they share the SM's issue slots with the consumers.
__device__ __forceinline__ void mbar_wait(u64* b, u32 par) {
  if (mbar_try(b, par)) return;
  u32 ns = 32;
  while (!mbar_try(b, par)) {
    __nanosleep(ns);
    ns = min(ns * 2, 256u);
  }
}
__device__ __forceinline__ void cp_async8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa(s)), "l"(g) : "memory");
}
// the mbarrier's pending count is raised now and lowered when this thread's cp.asyncs have landed
__device__ __forceinline__ void cp_async_arrive(u64* b) {
  asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void tma_load(void* s, const void* g, u32 bytes, u64* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(s)),
               "l"(g), "r"(bytes), "r"(sa(b))
               : "memory");
}
__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, %0;" ::"n"(NCT) : "memory"); }
__device__ __forceinline__ u32 atom_acq_rel_add32(u32* p, u32 v) {
  u32 old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void sm_release_add(u32* p, u32 v) {
  asm volatile("red.release.cta.shared::cta.add.u32 [%0], %1;" ::"r"(sa(p)), "r"(v) : "memory");
}
__device__ __forceinline__ u32 sm_acquire(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(sa(p)) : "memory");
  return v;
}
__device__ __forceinline__ u32 ld_relaxed32(const u32* p) {
  u32 v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Wait until *p >= target, then acquire (one acquire load: its L1 invalidation comes after the wait).
__device__ __forceinline__ void wait_geq(const u32* p, u32 target) {
#ifdef NSG_EXP_NOACQ  // timing experiment only: no acquire (unsafe)
  while (ld_relaxed32(p) < target) __nanosleep(64);
#else
  if (ld_acquire32(p) >= target) return;
  while (ld_relaxed32(p) < target) __nanosleep(64);
  (void)ld_acquire32(p);
#endif
}

__device__ __forceinline__ u32 link_bucket(u64 key, u32 logB) {
  return logB ? (u32)((key * MUL_L) >> (64 - logB)) : 0u;
}
__device__ __forceinline__ u32 link_slot(u64 key, u32 logB) {
  return (u32)((key * MUL_L) >> (64 - logB - LOG_TL)) & (TL - 1);
}
__device__ __forceinline__ u32 node_bucket(u32 node, u32 logBs) { return logBs ? (node * MUL_N) >> (32 - logBs) : 0u; }
__device__ __forceinline__ u32 node_slot(u32 node, u32 logBs) {
  return ((node * MUL_N) >> (32 - logBs - LOG_TS)) & (TS - 1);
}

__device__ Item decode(const WGeo& g, u64 t) {
  Item it;
  it.type = T_END; it.idx = 0; it.w = 0;
  if (t >= g.total) return it;
  u32 r = 0;
  while (r + 1 < g.nreg && t >= g.reg_t0[r + 1]) ++r;
  const u64 rel = t - g.reg_t0[r];
  const u32 f = g.reg_f[r];
  const u64 k = g.reg_k0[r] + rel / f;
  u32 off = (u32)(rel % f);
  const u32 m = g.reg_m[r];
  if (m & 1u) {
    if (off < g.nS) { it.type = T_S; it.idx = off; it.w = k - LAG_S; return it; }
    off -= g.nS;
  }
  if (m & 2u) {
    if (off < g.nL) { it.type = T_L; it.idx = off; it.w = k - LAG_L; return it; }
    off -= g.nL;
  }
  it.type = T_P; it.idx = off; it.w = k;
  return it;
}

// ---------------------------------------------------------------------------------------------
// Producer warp j: claims, dependencies, stage fills
// ---------------------------------------------------------------------------------------------
// Gather the concatenation of nseg segments (descriptor i = start << 16 | count, in pseg[i] for
// i < PSEG, else gseg[i]; segment i at base + i * stride + start) restricted to [lo, hi) into
// stage[0, hi - lo) with 8-byte cp.async.  The segments are short (tens of elements): each lane
// copies one segment, 32 segments at a time.
__device__ __forceinline__ void gather(const u32* pseg, const u32* gseg, u32 gst, u32 nseg, const u64* base, u64 stride,
                                       u32 lo, u32 hi, u64* stage, int lane) {
  u32 pre0 = 0;
  for (u32 c0 = 0; c0 < nseg && pre0 < hi; c0 += 32) {
    const u32 i = c0 + lane;
    const u32 v = i < nseg ? (i < (u32)PSEG ? pseg[i] : ldcg32(gseg + (u64)i * gst)) : 0u;
    const u32 st = v >> 16, cnt = v & 0xFFFFu;
    u32 x = cnt;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, x, k);
      if (lane >= k) x += y;
    }
    const u32 pre = pre0 + x - cnt;  // this segment's position in the concatenation
    const u32 a = lo > pre ? min(lo - pre, cnt) : 0u;
    const u32 z = hi > pre ? min(hi - pre, cnt) : 0u;
    const u64* src = base + i * stride + st;
    for (u32 e = a; e < z; ++e) cp_async8(stage + (pre + e - lo), src + e);
    pre0 += __shfl_sync(0xffffffffu, x, 31);
  }
}

__device__ __forceinline__ void st_vol64(u64* p, u64 v) { *reinterpret_cast<volatile u64*>(p) = v; }
__device__ __forceinline__ u64 ld_vol64(const u64* p) { return *reinterpret_cast<const volatile u64*>(p); }

// Producer warp j: claims a ticket ahead (tq[j][1]), and whenever stage j is free, makes it the stage's
// current item (tq[j][0]), waits for its dependencies and fills the stage with its input.
__device__ void producer(const WGeo& g, Smem& s, int j, const u32* __restrict__ src, const u32* __restrict__ dst,
                         const u64* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  u32 f = 0;  // fills issued into stage j
  u64* stage = s.stage[j];
  u32* pseg = s.pseg[j];
  const bool pr = lane == 0;
  WPROF_DECL
  u64 tnext = 0;
  if (lane == 0) {
    tnext = atomicAdd(reinterpret_cast<unsigned long long*>(g.ticket), 1ull);
    st_vol64(&s.tq[j][1], tnext);
  }
  for (;;) {
    // stage free: the consumers finished its previous fill
    if (f > 0) mbar_wait(&s.done[j], (f - 1) & 1u);
    u64 t = 0;
    if (lane == 0) {
      t = tnext;
      st_vol64(&s.tq[j][0], t);  // current first, then the claim in flight: never both free
      __threadfence_block();
      st_vol64(&s.tq[j][1], TPEND);
      tnext = atomicAdd(reinterpret_cast<unsigned long long*>(g.ticket), 1ull);  // used next round
    }
    t = __shfl_sync(0xffffffffu, t, 0);
    const Item it = decode(g, t);
    if (pr) WPROF_MARK(8);
    const u64 slot = it.w % RS;
    // ---- dependencies (items with smaller tickets) ----
    u32 nparts = 1, ntot = 0, len = 0, nseg = 0, sst = 1;
    const u32* segsrc = nullptr;
    if (it.type == T_P) {
      if (lane == 0) {
        if (it.w >= (u64)RS) wait_geq(&g.ws[it.w - RS].ldone, g.nL);  // key slot consumed
        if (g.arrived) {
          const u32* a = g.arrived + it.w / g.chunk_w;
          while (ld_acquire_sys32(a) == 0) __nanosleep(256);
        }
      }
      const u64 wl = min(g.W, g.n - it.w * g.W);
      const u64 c0 = (u64)it.idx * CH;
      len = (u32)wl;
      ntot = c0 < wl ? (u32)min((u64)CH, wl - c0) : 0u;
    } else if (it.type == T_L || it.type == T_S) {
      if (lane == 0) {
        if (it.type == T_L) {
          wait_geq(&g.ws[it.w].pdone, g.nP);
          if (it.w >= (u64)RS) wait_geq(&g.ws[it.w - RS].sdone, g.nS);  // record slot consumed
        } else {
          wait_geq(&g.ws[it.w].ldone, g.nL);
        }
      }
      __syncwarp();
      // segment i's descriptor at so[i * sst]: column it.idx of the producing items' rows
      const u32* so = (it.type == T_L) ? g.koff + slot * g.CP * g.B + it.idx : g.roff + slot * g.B * 2 * g.Bs + it.idx;
      sst = (it.type == T_L) ? g.B : 2 * g.Bs;
      nseg = (it.type == T_L) ? g.CP : g.B;
      u32 sum = 0;
      for (u32 i = lane; i < nseg; i += 32) {
        const u32 v = ldcg32(so + (u64)i * sst);
        if (i < (u32)PSEG) pseg[i] = v;
        sum += v & 0xFFFFu;
      }
      segsrc = so;
      ntot = warp_sum(sum);
      nparts = ntot ? (ntot + SK - 1) / SK : 1u;
    }
    if (pr) WPROF_MARK(9);
    __syncwarp();
    for (u32 p = 0; p < nparts; ++p, ++f) {
      if (p > 0) mbar_wait(&s.done[j], (f - 1) & 1u);  // the previous part is consumed
      if (lane == 0) {
        if (p == 0) WPROF_MARK(11);
        Desc d;
        d.type = it.type; d.idx = it.idx; d.w = it.w; d.part = p; d.nparts = nparts; d.ntot = ntot; d.len = len;
        d.soa = (it.type == T_P && !keys) ? 1u : 0u;
        d.n = (it.type == T_P) ? ntot : min((u32)SK, ntot - p * SK);
        if (it.type == T_END) d.n = 0;
        s.desc[j] = d;
        if (p == 0) st_vol64(&s.tq[j][1], tnext);  // the next claim has returned by now
      }
      __syncwarp();
      if (it.type == T_END) {
        if (lane == 0) mbar_arrive(&s.full[j]);
        return;
      }
      if (it.type == T_P) {
        const u64 base = it.w * g.W + (u64)it.idx * CH;
        const u32 n = ntot;
        if (keys) {
          const u64* gsrc = keys + base;
          if (n && ((reinterpret_cast<uintptr_t>(gsrc) & 15) == 0) && (n & 1u) == 0) {
            if (lane == 0) {
              mbar_arrive_tx(&s.full[j], n * 8u);
              tma_load(stage, gsrc, n * 8u, &s.full[j]);
            }
          } else {
            for (u32 e = lane; e < n; e += 32) cp_async8(stage + e, gsrc + e);
            cp_async_arrive(&s.full[j]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.full[j]);
          }
        } else {
          const u32* gs = src + base;
          const u32* gd = dst + base;
          u32* st32 = reinterpret_cast<u32*>(stage);
          if (n && ((reinterpret_cast<uintptr_t>(gs) & 15) == 0) && ((reinterpret_cast<uintptr_t>(gd) & 15) == 0) &&
              (n & 3u) == 0) {
            if (lane == 0) {
              mbar_arrive_tx(&s.full[j], n * 8u);
              tma_load(st32, gs, n * 4u, &s.full[j]);
              tma_load(st32 + CH, gd, n * 4u, &s.full[j]);
            }
          } else {
            for (u32 e = lane; e < n; e += 32) {
              cp_async4(st32 + e, gs + e);
              cp_async4(st32 + CH + e, gd + e);
            }
            cp_async_arrive(&s.full[j]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.full[j]);
          }
        }
      } else {
        const u32 lo = p * SK, hi = min(ntot, lo + SK);
        if (it.type == T_L)
          gather(pseg, segsrc, sst, nseg, g.kscr + slot * g.CP * CH, CH, lo, hi, stage, lane);
        else
          gather(pseg, segsrc, sst, nseg, g.rscr + slot * g.B * RCAP, RCAP, lo, hi, stage, lane);
        cp_async_arrive(&s.full[j]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&s.full[j]);
      }
      if (pr) WPROF_MARK(12);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Signaler warp: publish finished items (one fence per batch, then relaxed adds), finalize windows
// ---------------------------------------------------------------------------------------------
__device__ void finalize(const WGeo& g, u64 w, u64* out) {
  WinState* st = &g.ws[w];
  u32 ovf = ldcg32(&st->ovf);
  if (g.inject && (w & 1)) { st->ovf = 1; ovf = 1; }
  const u64 len = min(g.W, g.n - w * g.W);
  if (ovf) {  // recomputed by the L2 path; diag[0] counts the windows handed over
    atomicAdd(&g.diag[0], 1u);
    return;
  }
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

__device__ __forceinline__ void red_relaxed_add32(u32* p, u32 v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ void signaler(const WGeo& g, Smem& s, u64* out) {
  const int lane = threadIdx.x & 31;
  if (lane != 0) return;
  WPROF_DECL
  u32 tail = 0;
  for (;;) {
    u32 head;
    while ((head = sm_acquire(&s.ring_head)) == tail) __nanosleep(200);
    WPROF_MARK(16);
    // one fence makes every completed item's writes (ordered before ring_head by the consumers'
    // release) visible at gpu scope before the counter updates below
#ifndef NSG_EXP_NOACQ
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
    for (; tail != head; ++tail) {
      volatile SigE* ve = &s.ring[tail % RING];
      SigE e;
      e.type = ve->type; e.idx = ve->idx; e.w = ve->w;
      if (e.type == T_END) return;
      if (e.type == T_P) red_relaxed_add32(&g.ws[e.w].pdone, 1u);
      else if (e.type == T_L) red_relaxed_add32(&g.ws[e.w].ldone, 1u);
      else if (atom_acq_rel_add32(&g.ws[e.w].sdone, 1u) + 1 == g.nS) finalize(g, e.w, out);
    }
    *reinterpret_cast<volatile u32*>(&s.ring_tail) = tail;
    WPROF_MARK(18);
  }
}

// ---------------------------------------------------------------------------------------------
// Consumers (NCW warps, named barrier 1)
// ---------------------------------------------------------------------------------------------
// exclusive scan of h[0, n) by one warp into o[0, n); fn(i, excl, count) for every entry; returns the total
template <class F>
__device__ __forceinline__ u32 warp_exscan(const u32* h, u32* o, u32 n, int lane, F fn) {
  u32 carry = 0;
  for (u32 b0 = 0; b0 < n; b0 += 32) {
    const u32 i = b0 + lane;
    const u32 v = i < n ? h[i] : 0u;
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

// Warp reduction (sum a, max b, max c, sum d); the lane-0 values are the warp's totals.
__device__ __forceinline__ void warp_reduce4(u32& a, u32& b, u32& c, u32& d) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    c = max(c, __shfl_xor_sync(0xffffffffu, c, o));
    d += __shfl_xor_sync(0xffffffffu, d, o);
  }
}

// Combine the per-warp partials in s.red (written before the last consumer barrier) in warp 0:
// returns (sum a, max b, max c, sum d) in every lane of warp 0.
__device__ __forceinline__ void red_finish(const Smem& s, u32& a, u32& b, u32& c, u32& d) {
  const int lane = threadIdx.x & 31;
  a = lane < NCW ? s.red[0][lane] : 0u;
  b = lane < NCW ? s.red[1][lane] : 0u;
  c = lane < NCW ? s.red[2][lane] : 0u;
  d = lane < NCW ? s.red[3][lane] : 0u;
  warp_reduce4(a, b, c, d);
}

__device__ __forceinline__ void copy_out(u64* __restrict__ dstp, const u64* stage, u32 n) {
  const int t = threadIdx.x;
  if ((reinterpret_cast<uintptr_t>(dstp) & 15) == 0) {
    for (u32 e = 2 * t; e + 1 < n; e += 2 * NCT) {
      const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(stage + e);
      *reinterpret_cast<ulonglong2*>(dstp + e) = v;
    }
    if ((n & 1u) && t == 0) dstp[n - 1] = stage[n - 1];
  } else {
    for (u32 e = t; e < n; e += NCT) dstp[e] = stage[e];
  }
}

// ---- P(w, c): counting sort of one chunk by link bucket -------------------------------------
__device__ void cons_P(const WGeo& g, Smem& s, const Desc& d, u64* stage, u32 par) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const u32 n = d.n;
  u32* hist = s.hist[par];
  const u32 logB = g.logB, B = g.B;
  constexpr int KPT = CH / NCT;
  u64 kk[KPT];
  u32 br[KPT];
  const u32* s32 = reinterpret_cast<const u32*>(stage);
  PMARK(0);
  u32 bk[KPT];
#pragma unroll
  for (int i = 0; i < KPT; ++i) {  // all loads, then all hashes, then all atomics: independent, in flight together
    const u32 e = i * NCT + t;
    kk[i] = e < n ? (d.soa ? (((u64)s32[e] << 32) | s32[CH + e]) : stage[e]) : 0ull;
  }
#pragma unroll
  for (int i = 0; i < KPT; ++i) bk[i] = link_bucket(kk[i], logB);
#pragma unroll
  for (int i = 0; i < KPT; ++i) br[i] = (i * NCT + t < n) ? atomicAdd(&hist[bk[i]], 1u) : 0u;
#pragma unroll
  for (int i = 0; i < KPT; ++i) br[i] = bk[i] | (br[i] << 16);
  PMARK(1);
  cbar();
  PMARK(2);
  const u64 slot = d.w % RS;
  if (wid == 0) {
    u32* ko = g.koff + (slot * g.CP + d.idx) * B;  // this item's own row: no line shared with other items
    warp_exscan(hist, s.offs, B, lane, [&](u32 i, u32 ex, u32 v) { ko[i] = (ex << 16) | v; });
  }
  PMARK(3);
  cbar();
  PMARK(4);
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    const u32 e = i * NCT + t;
    if (e < n) stage[s.offs[br[i] & 0xFFFFu] + (br[i] >> 16)] = kk[i];
  }
  PMARK(5);
  cbar();
  PMARK(6);
  copy_out(g.kscr + (slot * g.CP + d.idx) * CH, stage, n);
  for (u32 b = t; b < B; b += NCT) hist[b] = 0;
  PMARK(7);
}

// ---- L(w, b): group-by-count of the bucket's keys --------------------------------------------
// Barrier-free vectorised insertion: each thread loads all its keys, reads all their home slots,
// then counts the keys found there (a hot link's repeats: broadcast read + aggregated increment,
// never a CAS) and CASes the free ones, every load / atomic of the thread in flight together.  A key
// whose home holds another key probes on by windows of WIN slots (one round trip each).  Every
// claimed slot is noted in a dense claim list, so the final scan visits the bucket's links only.
constexpr u32 WIN = 16;
constexpr int KW = SK / NCT;  // elements per thread in a full stage

// One slot for `key`: 1 = counted (found), 2 = claimed and counted, 0 = holds another key.
__device__ __forceinline__ u32 link_try(Smem& s, u64 key, u32 sl, u64 cur) {
  if (cur == key) { atomicAdd(&s.lcnt[sl], 1u); return 1; }
  if (cur != EMPTY64) return 0;
  const u64 old = atomicCAS(reinterpret_cast<unsigned long long*>(&s.lkey[sl]), (unsigned long long)EMPTY64,
                            (unsigned long long)key);
  if (old == EMPTY64) { atomicAdd(&s.lcnt[sl], 1u); return 2; }
  if (old == key) { atomicAdd(&s.lcnt[sl], 1u); return 1; }
  return 0;
}

// Probe on from home + 1, one slot per step (at load <= 5/8 almost always one or two steps);
// returns 1/2 as link_try (0 = table full: overflow).
__device__ __noinline__ u32 link_probe_on(Smem& s, u64 key, u32 home, u32* slot) {
  for (u32 off = 1; off < (u32)TL; ++off) {
    const u32 sl = (home + off) & (TL - 1);
    const u32 r = link_try(s, key, sl, *reinterpret_cast<volatile u64*>(&s.lkey[sl]));
    if (r) { *slot = sl; return r; }
  }
  return 0;
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

__device__ void cons_L_part(const WGeo& g, Smem& s, const Desc& d, const u64* stage, u32 par) {
  const int t = threadIdx.x, lane = t & 31;
  const u32 n = d.n;
  const bool guarded = d.ntot > FILL_L;
  const u32 logB = g.logB;
  u32* ncl = &s.ncl[0][par];
  PMARK(8);
  u64 k[KW], cur[KW];
  u32 sl[KW];
  u32 vmask = 0, nesc = 0;
#pragma unroll
  for (int i = 0; i < KW; ++i) {
    const u32 e = i * NCT + t;
    k[i] = e < n ? stage[e] : 0ull;
  }
#pragma unroll
  for (int i = 0; i < KW; ++i) {
    const bool v = i * NCT + t < n;
    if (v && k[i] == EMPTY64) ++nesc;
    else if (v) vmask |= 1u << i;
    sl[i] = link_slot(k[i], logB);
  }
  if (guarded && *reinterpret_cast<volatile u32*>(&s.lovf[par])) vmask = 0;
#pragma unroll
  for (int i = 0; i < KW; ++i) cur[i] = (vmask >> i & 1u) ? *reinterpret_cast<volatile u64*>(&s.lkey[sl[i]]) : 0ull;
  u32 pmask = 0, wmask = 0;
#pragma unroll
  for (int i = 0; i < KW; ++i) {
    if (vmask >> i & 1u) {
      const u32 r = link_try(s, k[i], sl[i], cur[i]);
      if (r == 0) pmask |= 1u << i;
      if (r == 2) wmask |= 1u << i;
    }
  }
  if (nesc) atomicAdd(&s.lesc[par], nesc);
  // keys whose home holds another key: probe on (per lane; few keys)
#pragma unroll 1
  for (u32 m = pmask; m; m &= m - 1) {
    const int i = __ffs(m) - 1;
    u32 slot = 0;
    u64 key = 0, home = 0;
#pragma unroll
    for (int q = 0; q < KW; ++q) if (q == i) { key = k[q]; home = sl[q]; }
    const u32 r = link_probe_on(s, key, (u32)home, &slot);
    if (r == 0) s.lovf[par] = 1;
#pragma unroll
    for (int q = 0; q < KW; ++q) if (q == i) sl[q] = slot;
    if (r == 2) wmask |= 1u << i;
  }
  u32 pw = warp_reserve(__popc(wmask), ncl);
#pragma unroll
  for (int i = 0; i < KW; ++i)
    if (wmask >> i & 1u) s.claim[pw++] = (uint16_t)sl[i];
  if (guarded) {
    const u32 c = __reduce_add_sync(0xffffffffu, (u32)__popc(wmask));
    if (lane == 0 && c && atomicAdd(&s.lfill[par], c) + c > FILL_L) s.lovf[par] = 1;
  }
  PMARK(9);
}

// Scan the bucket's links (claim list; cleaning the table), add its unique links / max count / count
// sum to the window, and emit one record per link and side (node << 32 | count) counting-sorted by
// side bucket.
__device__ void cons_L_final(const WGeo& g, Smem& s, const Desc& d, u64* stage, u32 par) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  PMARK(16);
  cbar();  // every insert of the bucket is done
  PMARK(17);
  const bool ovf = *reinterpret_cast<volatile u32*>(&s.lovf[par]) != 0;
  const u32 ncl = min(*reinterpret_cast<volatile u32*>(&s.ncl[0][par]), (u32)TL);
  const u32 Bs = g.Bs, logBs = g.logBs;
  u32* hist = s.hist[par];  // [0, Bs) side 0, [Bs, 2Bs) side 1
  constexpr int SPT = TL / NCT;
  u64 lk[SPT];
  u32 lc[SPT], lr[SPT], lb[SPT];
  u32 nl = 0, mx = 0, sm = 0;
  // the claimed slots first, then their keys and counts, then the hashes, then every histogram
  // atomic: independent, in flight together
  u32 cs[SPT];
#pragma unroll
  for (int k = 0; k < SPT; ++k) cs[k] = (k * NCT + t < ncl) ? s.claim[k * NCT + t] : 0xFFFFFFFFu;
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    lc[k] = cs[k] != 0xFFFFFFFFu ? s.lcnt[cs[k]] : 0u;
    lk[k] = cs[k] != 0xFFFFFFFFu ? s.lkey[cs[k]] : 0ull;
  }
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    if (lc[k]) {
      s.lkey[cs[k]] = EMPTY64;
      s.lcnt[cs[k]] = 0;
      nl += 1; mx = max(mx, lc[k]); sm += lc[k];
    }
    lb[k] = node_bucket((u32)(lk[k] >> 32), logBs) | (node_bucket((u32)lk[k], logBs) << 16);
  }
  u32 r0[SPT], r1[SPT];
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    r0[k] = 0; r1[k] = 0;
    if (lc[k] && !ovf) {
      r0[k] = atomicAdd(&hist[lb[k] & 0xFFFFu], 1u);
      r1[k] = atomicAdd(&hist[Bs + (lb[k] >> 16)], 1u);
    }
  }
#pragma unroll
  for (int k = 0; k < SPT; ++k) lr[k] = r0[k] | (r1[k] << 16);
  const u32 esc = s.lesc[par];
  u32 er = 0;
  if (t == 0 && esc) {
    nl += 1; mx = max(mx, esc); sm += esc;
    if (!ovf) {
      const u32 eb = node_bucket(EMPTY32, logBs);
      er = atomicAdd(&hist[eb], 1u) | (atomicAdd(&hist[Bs + eb], 1u) << 16);
    }
  }
  {  // per-warp partials of the bucket's link statistics
    u32 z = 0;
    warp_reduce4(nl, mx, z, sm);
    if (lane == 0) { s.red[0][wid] = nl; s.red[1][wid] = mx; s.red[3][wid] = sm; }
  }
  PMARK(18);
  cbar();  // the histograms and partials are complete
  PMARK(19);
  const u64 slot = d.w % RS;
  const u32 b = d.idx;
  u32* ro = g.roff + (slot * g.B + b) * 2 * Bs;  // this item's own row
  if (ovf) {
    if (t == 0) g.ws[d.w].ovf = 1;
    for (u32 i = t; i < 2 * Bs; i += NCT) ro[i] = 0;
  } else if (wid < 2) {
    if (wid == 0) {  // the bucket's unique links, max count and count sum go to the window accumulators
      u32 a, b2, c, dd;
      red_finish(s, a, b2, c, dd);
      if (lane == 0 && a) {
        WinState* st = &g.ws[d.w];
        atomicAdd(&st->links, a);
        atomicMax(&st->maxc, b2);
        atomicAdd(&st->sumc, dd);
      }
    }
    // side-0 records first, then side 1 from L0 = number of links (= sum of the side-0 counts)
    u32 L0 = 0;
    if (wid == 1)
      for (u32 i = lane; i < Bs; i += 32) L0 += hist[i];
    L0 = warp_sum(L0);
    const u32* h = hist + wid * Bs;
    u32* o = s.offs + wid * Bs;
    u32* r = ro + wid * Bs;
    const u32 tot = warp_exscan(h, o, Bs, lane, [&](u32 i, u32 ex, u32 v) { r[i] = ((L0 + ex) << 16) | v; });
    if (wid == 0 && lane == 0) s.L0 = tot;
  }
  PMARK(20);
  cbar();
  PMARK(21);
  if (!ovf) {
    const u32 L0 = s.L0;
    u64* rdst = g.rscr + (slot * g.B + b) * RCAP;
    const bool one = 2 * L0 <= (u32)SK;
    const u32* o0 = s.offs;
    const u32* o1 = s.offs + Bs;
    u32 p0[SPT], p1[SPT];
#pragma unroll
    for (int k = 0; k < SPT; ++k) {  // offsets first (all loads in flight), then the stores
      p0[k] = lc[k] ? o0[lb[k] & 0xFFFFu] : 0u;
      p1[k] = lc[k] ? o1[lb[k] >> 16] : 0u;
    }
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      if (lc[k]) {
        stage[p0[k] + (lr[k] & 0xFFFFu)] = (lk[k] & 0xFFFFFFFF00000000ull) | lc[k];
        if (one) stage[L0 + p1[k] + (lr[k] >> 16)] = (lk[k] << 32) | lc[k];
      }
    }
    if (t == 0 && esc) {
      const u32 eb = node_bucket(EMPTY32, logBs);
      stage[o0[eb] + (er & 0xFFFFu)] = ((u64)EMPTY32 << 32) | esc;
      if (one) stage[L0 + o1[eb] + (er >> 16)] = ((u64)EMPTY32 << 32) | esc;
    }
    PMARK(22);
    cbar();
    PMARK(23);
    if (one) {
      copy_out(rdst, stage, 2 * L0);
    } else {
      copy_out(rdst, stage, L0);
      cbar();
#pragma unroll
      for (int k = 0; k < SPT; ++k)
        if (lc[k]) stage[p1[k] + (lr[k] >> 16)] = (lk[k] << 32) | lc[k];
      if (t == 0 && esc) stage[o1[node_bucket(EMPTY32, logBs)] + (er >> 16)] = ((u64)EMPTY32 << 32) | esc;
      cbar();
      copy_out(rdst + L0, stage, L0);
    }
  }
  for (u32 i = t; i < 2 * Bs; i += NCT) hist[i] = 0;
  if (t == 0) { s.lesc[par] = 0; s.lfill[par] = 0; s.lovf[par] = 0; s.ncl[0][par] = 0; }
  PMARK(24);
}

// ---- S(w, side, q): merge the records of one side bucket per node ---------------------------
// packets += csum, fan += k for the node in `slot`.  An item with fewer than 4096 records cannot
// carry a fan past the 12-bit field: a fire-and-forget add.  Otherwise the old value is checked and
// a fan field that passes 4095 is noted in the wrap list.
__device__ __forceinline__ void node_add(Smem& s, u32 slot, u32 csum, u32 k, u32 par, bool wrapcheck) {
  if (!wrapcheck) { atomicAdd(&s.npf[slot], csum | (k << PFS)); return; }
  const u32 o = atomicAdd(&s.npf[slot], csum | (k << PFS));
  if ((o >> PFS) + k > FMAX) {
    const u32 i = atomicAdd(&s.nwrap[par], 1u);
    if (i < (u32)WRAPCAP) s.wrap[par][i] = slot;
    else s.sovf[par] = 1;
  }
}

// One slot for `node`: returns 1 = its slot, 2 = claimed now, 0 = holds another node.
__device__ __forceinline__ u32 node_try(Smem& s, u32 node, u32 sl, u32 cur) {
  if (cur == node) return 1;
  if (cur != EMPTY32) return 0;
  const u32 old = atomicCAS(&s.nkey[sl], EMPTY32, node);
  if (old == EMPTY32) return 2;
  return old == node ? 1u : 0u;
}

__device__ __noinline__ u32 node_probe_on(Smem& s, u32 node, u32 home, u32* slot) {
  for (u32 off = 1; off < (u32)TS; ++off) {
    const u32 q = (home + off) & (TS - 1);
    const u32 r = node_try(s, node, q, *reinterpret_cast<volatile u32*>(&s.nkey[q]));
    if (r) { *slot = q; return r; }
  }
  return 0;
}

__device__ void cons_S_part(const WGeo& g, Smem& s, const Desc& d, const u64* stage, u32 par) {
  const int t = threadIdx.x, lane = t & 31;
  const bool guarded = d.ntot > FILL_S;
  const bool wrapcheck = d.ntot > FMAX;
  const u32 n = d.n, logBs = g.logBs;
  u32* ncl = &s.ncl[1][par];
  u32 nd[KW], cc[KW], sl[KW], cur[KW];
  u32 vmask = 0, escP = 0, escF = 0;
#pragma unroll
  for (int i = 0; i < KW; ++i) {
    const u32 e = i * NCT + t;
    const u64 rec = e < n ? stage[e] : 0ull;
    nd[i] = (u32)(rec >> 32);
    cc[i] = (u32)rec;
  }
#pragma unroll
  for (int i = 0; i < KW; ++i) {
    const bool v = i * NCT + t < n;
    if (v && nd[i] == EMPTY32) { escP += cc[i]; ++escF; }
    else if (v) vmask |= 1u << i;
    sl[i] = node_slot(nd[i], logBs);
  }
  if (guarded && *reinterpret_cast<volatile u32*>(&s.sovf[par])) vmask = 0;
#pragma unroll
  for (int i = 0; i < KW; ++i) cur[i] = (vmask >> i & 1u) ? *reinterpret_cast<volatile u32*>(&s.nkey[sl[i]]) : 0u;
  u32 pmask = 0, wmask = 0;
#pragma unroll
  for (int i = 0; i < KW; ++i) {
    if (vmask >> i & 1u) {
      const u32 r = node_try(s, nd[i], sl[i], cur[i]);
      if (r == 0) pmask |= 1u << i;
      if (r == 2) wmask |= 1u << i;
    }
  }
  if (escF) { atomicAdd(&s.sescP[par], escP); atomicAdd(&s.sescF[par], escF); }
#pragma unroll 1
  for (u32 m = pmask; m; m &= m - 1) {
    const int i = __ffs(m) - 1;
    u32 node = 0, home = 0, slot = 0;
#pragma unroll
    for (int q = 0; q < KW; ++q) if (q == i) { node = nd[q]; home = sl[q]; }
    const u32 r = node_probe_on(s, node, home, &slot);
    if (r == 0) { s.sovf[par] = 1; vmask &= ~(1u << i); }
#pragma unroll
    for (int q = 0; q < KW; ++q) if (q == i) sl[q] = slot;
    if (r == 2) wmask |= 1u << i;
  }
#pragma unroll
  for (int i = 0; i < KW; ++i)
    if (vmask >> i & 1u) node_add(s, sl[i], cc[i], 1u, par, wrapcheck);
  u32 pw = warp_reserve(__popc(wmask), ncl);
#pragma unroll
  for (int i = 0; i < KW; ++i)
    if (wmask >> i & 1u) s.claim[pw++] = (uint16_t)sl[i];
  if (guarded) {
    const u32 c = __reduce_add_sync(0xffffffffu, (u32)__popc(wmask));
    if (lane == 0 && c && atomicAdd(&s.sfill[par], c) + c > FILL_S) s.sovf[par] = 1;
  }
}

__device__ void cons_S_final(const WGeo& g, Smem& s, const Desc& d, u32 par) {
  const int t = threadIdx.x, lane = t & 31;
  cbar();
  const u32 nwrap = *reinterpret_cast<volatile u32*>(&s.nwrap[par]);
  u32 wrapmax = 0;
  if (nwrap) {  // exact fan of the nodes whose 12-bit fan field wrapped (rare: fan >= 4096)
    const u32 nw = min(nwrap, (u32)WRAPCAP);
    for (u32 i = lane; i < nw; i += 32) {  // every consumer warp computes the same maximum
      const u32 sl = s.wrap[par][i];
      u32 cnt = 0;
      for (u32 k = 0; k < nw; ++k) cnt += s.wrap[par][k] == sl;
      wrapmax = max(wrapmax, (s.npf[sl] >> PFS) + (FMAX + 1) * cnt);
    }
    cbar();  // before the scan cleans the table
  }
  const bool ovf = *reinterpret_cast<volatile u32*>(&s.sovf[par]) != 0;
  const u32 ncl = min(*reinterpret_cast<volatile u32*>(&s.ncl[1][par]), (u32)TS);
  constexpr int SPT = TS / NCT;
  u32 nn = 0, mp = 0, mf = wrapmax;
  u32 cs[SPT], pf[SPT];
#pragma unroll
  for (int k = 0; k < SPT; ++k) cs[k] = (k * NCT + t < ncl) ? s.claim[k * NCT + t] : 0xFFFFFFFFu;
#pragma unroll
  for (int k = 0; k < SPT; ++k) pf[k] = cs[k] != 0xFFFFFFFFu ? s.npf[cs[k]] : 0u;
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    if (cs[k] != 0xFFFFFFFFu) {
      nn += 1;
      mp = max(mp, pf[k] & PMASK);
      mf = max(mf, pf[k] >> PFS);
      s.nkey[cs[k]] = EMPTY32;
      s.npf[cs[k]] = 0;
    }
  }
  if (t == 0 && s.sescF[par]) { nn += 1; mp = max(mp, s.sescP[par]); mf = max(mf, s.sescF[par]); }
  u32 z = 0;
  warp_reduce4(nn, mp, mf, z);
  if (lane == 0) { s.red[0][t >> 5] = nn; s.red[1][t >> 5] = mp; s.red[2][t >> 5] = mf; }
  cbar();
  if (t < 32) {
    red_finish(s, nn, mp, mf, z);
    const u32 side = d.idx >= g.Bs ? 1u : 0u;
    WinState* st = &g.ws[d.w];
    if (t == 0) {
      if (ovf) {
        st->ovf = 1;
      } else if (nn) {
        atomicAdd(&st->nodes[side], nn);
        atomicMax(&st->maxp[side], mp);
        atomicMax(&st->maxf[side], mf);
      }
      s.sescP[par] = 0; s.sescF[par] = 0; s.sfill[par] = 0; s.sovf[par] = 0; s.nwrap[par] = 0; s.ncl[1][par] = 0;
    }
  }
}

// The consumers take the stage holding the smallest ticket of the CTA (current or claimed next): a
// claim still in flight could be smaller than every stage's ticket, so it is waited for.  Items are
// therefore processed in ticket order within the CTA (deadlock freedom, see the file header).
__device__ __forceinline__ int pick_stage(const WGeo& g, Smem& s) {
  for (;;) {
    u64 best = TFREE;
    int bj = -1;
    bool blocked = false;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      u64 c = ld_vol64(&s.tq[j][0]);
      if (c == TFREE) {
        c = ld_vol64(&s.tq[j][1]);
        if (c == TPEND) { blocked = true; continue; }
      }
      if (c < best) { best = c; bj = j; }
    }
    if (!blocked && bj >= 0) return bj;
    __nanosleep(64);
  }
}

__device__ void consumer(const WGeo& g, Smem& s) {
  const int t = threadIdx.x, lane = t & 31;
  u32 fl[K];
#pragma unroll
  for (int j = 0; j < K; ++j) fl[j] = 0;
  u32 par = 0, spar = 0;
  const bool pr = t == 0;
  WPROF_DECL
  for (;;) {
    if (t == 0) s.sel = (u32)pick_stage(g, s);
    cbar();
    const int j = (int)s.sel;
    for (;;) {  // the parts of the item in stage j
      u32 f = 0;
#pragma unroll
      for (int q = 0; q < K; ++q) if (q == j) f = fl[q];
      mbar_wait(&s.full[j], f & 1u);
      if (pr) WPROF_MARK(0);
      const Desc d = s.desc[j];
      if (d.type == T_END) {
        if (t == 0) {
          s.ring[s.ring_head % RING].type = T_END;
          asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(sa(&s.ring_head)), "r"(s.ring_head + 1) : "memory");
        }
        return;
      }
      u64* stage = s.stage[j];
      if (d.type == T_P) {
        cons_P(g, s, d, stage, par);
        par ^= 1u;
        if (pr) { WPROF_MARK(1); WPROF_CNT(24); }
      } else if (d.type == T_L) {
        cons_L_part(g, s, d, stage, par);
        if (pr) WPROF_MARK(2);
        if (d.part + 1 == d.nparts) {
          cons_L_final(g, s, d, stage, par);
          par ^= 1u;
          if (pr) { WPROF_MARK(3); WPROF_CNT(25); }
        }
      } else {
        cons_S_part(g, s, d, stage, spar);
        if (pr) WPROF_MARK(4);
        if (d.part + 1 == d.nparts) {
          cons_S_final(g, s, d, spar);
          spar ^= 1u;
          if (pr) { WPROF_MARK(5); WPROF_CNT(26); }
        }
      }
#pragma unroll
      for (int q = 0; q < K; ++q) if (q == j) ++fl[q];
      const bool last = d.part + 1 == d.nparts;
      cbar();  // every consumer is done with the stage (and the item's writes)
      if (t == 0) {
        if (last) {
          // queue the item for its signal (release: the consumers' writes precede it via the barrier)
          while (s.ring_head - *reinterpret_cast<volatile u32*>(&s.ring_tail) >= (u32)RING) __nanosleep(32);
          SigE e;
          e.type = d.type; e.idx = d.idx; e.w = d.w;
          s.ring[s.ring_head % RING] = e;
          asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(sa(&s.ring_head)), "r"(s.ring_head + 1) : "memory");
          st_vol64(&s.tq[j][0], TFREE);
        }
        mbar_arrive(&s.done[j]);
      }
      if (pr) WPROF_MARK(6);
      if (last) break;
    }
  }
}

__global__ void __launch_bounds__(NT, 1)
win_kernel(const WGeo g, const u32* __restrict__ src, const u32* __restrict__ dst, const u64* __restrict__ keys,
           u64* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int t = threadIdx.x;
  for (u32 i = t; i < (u32)TL; i += NT) { s.lkey[i] = EMPTY64; s.lcnt[i] = 0; }
  for (u32 i = t; i < (u32)TS; i += NT) { s.nkey[i] = EMPTY32; s.npf[i] = 0; }
  for (u32 i = t; i < 4 * MAXB; i += NT) (&s.hist[0][0])[i] = 0;
  if (t < K) {
    mbar_init(&s.full[t], 1);
    mbar_init(&s.done[t], 1);
    s.tq[t][0] = TFREE;
    s.tq[t][1] = TPEND;
  }
  if (t < 2) {
    s.lesc[t] = 0; s.lfill[t] = 0; s.lovf[t] = 0;
    s.sescP[t] = 0; s.sescF[t] = 0; s.sfill[t] = 0; s.sovf[t] = 0; s.nwrap[t] = 0;
  }
  if (t == 0) { s.ring_head = 0; s.ring_tail = 0; }
  if (t < 4) (&s.ncl[0][0])[t] = 0;
  __syncthreads();
  const int wid = t >> 5;
  if (wid < NCW) {
    consumer(g, s);
  } else if (wid < NCW + K) {
    producer(g, s, wid - NCW, src, dst, keys);
  } else {
    signaler(g, s, out);
  }
}

}  // namespace win
}  // namespace nsg
