// nsg_global.cuh — the L2 path of libnsg: one CTA per window with global-memory hash tables.
// Used for windows larger than the fast path supports and as the fast path's overflow hand-off.
// Same definitions as the fast path (Table 2; mirrors line 173).
#pragma once
#include "nsg_internal.h"
#include "nsg_common.cuh"

namespace nsg {

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
  u32 ovf_stride;  // ovf of window w at ovf[w * ovf_stride]
  u32* diag;
  // optional vector outputs (as Geo): window w's entries at [w*W, w*W + count), hash order
  u64* v_lkey; u32* v_lpk;
  u32* v_node[2]; u32* v_pk[2]; u32* v_fan[2];
  u64* v_ipsets;
  const u32* wgt;  // weighted rows: n_packets per row (NULL: raw packets, weight 1)
  u64* const* mirror;  // result mirrors (as Geo)
  u32 n_mirror;
  u64 mirror_row0;
};

__device__ __forceinline__ void glob_link_insert(u64* lkey, u32* lcnt, u64 LC, u64 key, u32 add) {
  u64 slot = hash64(key) & (LC - 1);
  for (;;) {
    u64 k = ldcg64(&lkey[slot]);
    if (k == EMPTY64) {
      const u64 old = atomicCAS(reinterpret_cast<unsigned long long*>(&lkey[slot]), EMPTY64, key);
      k = (old == EMPTY64) ? key : old;
    }
    if (k == key) { atomicAdd(&lcnt[slot], add); return; }
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

__device__ __forceinline__ bool glob_node_present(const u32* key, u64 LC, u32 node) {
  u64 slot = ((u64)hash32(node) * 0x9E3779B97F4A7C15ull >> 11) & (LC - 1);
  for (;;) {
    const u32 k = ldcg32(&key[slot]);
    if (k == node) return true;
    if (k == EMPTY32) return false;
    slot = (slot + 1) & (LC - 1);
  }
}

__global__ void __launch_bounds__(GT)
global_kernel(GGeo g, const u32* __restrict__ src, const u32* __restrict__ dst, const u64* __restrict__ keys,
              u64* __restrict__ out) {
  __shared__ u32 esc[5];
  __shared__ u32 red[9 * (GT / 32)];
  __shared__ u32 vcnt[3], both_s;
  __shared__ unsigned long long wtot;
  if (g.only_overflowed && ldcg32(&g.diag[0]) == 0) return;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const u64 LC = g.LC;
  u64* lkey = g.lkey + (u64)blockIdx.x * LC;
  u32* lcnt = g.lcnt + (u64)blockIdx.x * LC;
  for (u64 w = blockIdx.x; w < g.nw; w += g.G) {
    if (g.only_overflowed && ldcg32(&g.ovf[w * g.ovf_stride]) == 0) continue;
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
    if (t < 3) vcnt[t] = 0;
    if (t == 0) { both_s = 0; wtot = 0; }
    __syncthreads();
    unsigned long long wl = 0;
    for (u64 i = t; i < len; i += GT) {
      const u32 a = g.wgt ? g.wgt[base + i] : 1u;  // A_t(i,j) += n_packets (1 for raw packets); 0 adds nothing
      if (a == 0) continue;
      wl += a;
      const u64 key = keys ? keys[base + i] : (((u64)src[base + i] << 32) | dst[base + i]);
      if (key == EMPTY64) atomicAdd(&esc[0], a);
      else glob_link_insert(lkey, lcnt, LC, key, a);
    }
    if (wl) atomicAdd(&wtot, wl);
    __syncthreads();
    u32* k0 = g.nkey + ((u64)blockIdx.x * 2 + 0) * LC;
    u32* k1 = g.nkey + ((u64)blockIdx.x * 2 + 1) * LC;
    u32* P0 = g.nP + ((u64)blockIdx.x * 2 + 0) * LC;
    u32* P1 = g.nP + ((u64)blockIdx.x * 2 + 1) * LC;
    u32* F0 = g.nF + ((u64)blockIdx.x * 2 + 0) * LC;
    u32* F1 = g.nF + ((u64)blockIdx.x * 2 + 1) * LC;
    u32 nl = 0, mx = 0, sm = 0;
    const u64 wb = w * g.W;  // the window's region of the vector outputs
    for (u64 i0 = 0; i0 < LC; i0 += GT) {  // warp-uniform trip count (vector appends are warp-collective)
      const u64 i = i0 + t;
      const u64 key = i < LC ? ldcg64(&lkey[i]) : EMPTY64;
      u32 c = 0;
      if (key != EMPTY64) {
        c = ldcg32(&lcnt[i]);
        nl += 1; mx = max(mx, c); sm += c;
        glob_node_upsert(k0, P0, F0, LC, &esc[1], &esc[2], (u32)(key >> 32), c, 1);
        glob_node_upsert(k1, P1, F1, LC, &esc[3], &esc[4], (u32)key, c, 1);
      }
      if (g.v_lkey) {
        const u32 r = warp_append(key != EMPTY64, &vcnt[0]);
        if (key != EMPTY64) { g.v_lkey[wb + r] = key; g.v_lpk[wb + r] = c; }
      }
    }
    if (t == 0 && esc[0]) {
      const u32 c = esc[0];
      nl += 1; mx = max(mx, c); sm += c;
      atomicAdd(&esc[1], c); atomicAdd(&esc[2], 1u); atomicAdd(&esc[3], c); atomicAdd(&esc[4], 1u);
      if (g.v_lkey) { const u32 r = atomicAdd(&vcnt[0], 1u); g.v_lkey[wb + r] = EMPTY64; g.v_lpk[wb + r] = c; }
    }
    __syncthreads();
    u32 d0 = 0, p0 = 0, f0 = 0, d1 = 0, p1 = 0, f1 = 0, both = 0;
    for (u64 i0 = 0; i0 < LC; i0 += GT) {
      const u64 i = i0 + t;
      const u32 n0 = i < LC ? ldcg32(&k0[i]) : EMPTY32, n1 = i < LC ? ldcg32(&k1[i]) : EMPTY32;
      u32 a0 = 0, b0 = 0, a1 = 0, b1 = 0;
      if (n0 != EMPTY32) {
        a0 = ldcg32(&P0[i]); b0 = ldcg32(&F0[i]);
        d0 += 1; p0 = max(p0, a0); f0 = max(f0, b0);
        if (g.v_ipsets) both += (u32)glob_node_present(k1, LC, n0);
      }
      if (n1 != EMPTY32) { a1 = ldcg32(&P1[i]); b1 = ldcg32(&F1[i]); d1 += 1; p1 = max(p1, a1); f1 = max(f1, b1); }
      if (g.v_node[0]) {
        const u32 r = warp_append(n0 != EMPTY32, &vcnt[1]);
        if (n0 != EMPTY32) { g.v_node[0][wb + r] = n0; g.v_pk[0][wb + r] = a0; g.v_fan[0][wb + r] = b0; }
      }
      if (g.v_node[1]) {
        const u32 r = warp_append(n1 != EMPTY32, &vcnt[2]);
        if (n1 != EMPTY32) { g.v_node[1][wb + r] = n1; g.v_pk[1][wb + r] = a1; g.v_fan[1][wb + r] = b1; }
      }
    }
    if (t == 0 && esc[1]) {
      d0 += 1; p0 = max(p0, esc[1]); f0 = max(f0, esc[2]);
      both += esc[3] != 0u;  // the address ~0 is a source; is it a destination too?
      if (g.v_node[0]) { const u32 r = atomicAdd(&vcnt[1], 1u); g.v_node[0][wb + r] = EMPTY32; g.v_pk[0][wb + r] = esc[1]; g.v_fan[0][wb + r] = esc[2]; }
    }
    if (t == 0 && esc[3]) {
      d1 += 1; p1 = max(p1, esc[3]); f1 = max(f1, esc[4]);
      if (g.v_node[1]) { const u32 r = atomicAdd(&vcnt[2], 1u); g.v_node[1][wb + r] = EMPTY32; g.v_pk[1][wb + r] = esc[3]; g.v_fan[1][wb + r] = esc[4]; }
    }
    if (g.v_ipsets) {
      both = warp_sum(both);
      if (lane == 0 && both) atomicAdd(&both_s, both);
    }
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
      const u64 row[NSG_NUM_STATS] = {r[1], r[0], r[4], r[2], r[5], r[6], r[3], r[7], r[8]};  // north_star order
      store_row(out + w * NSG_NUM_STATS, row);
      for (u32 j = 0; j < g.n_mirror; ++j) store_row(g.mirror[j] + (g.mirror_row0 + w) * NSG_NUM_STATS, row);
      // self-check: the counts sum to the window's packets (sum of n_packets for weighted rows, which the
      // 32-bit counters support up to 2^32 - 1 per window: beyond that the window is reported in diag[2])
      if (wtot >= (1ull << 32)) atomicAdd(&g.diag[2], 1u);
      else if ((u64)r[1] != wtot) atomicAdd(&g.diag[1], 1u);
      if (g.v_ipsets) {  // |S u D|, |S \ D|, |D \ S|, |S n D|
        const u32 b = both_s;
        u64* ip = g.v_ipsets + w * 4;
        ip[0] = (u64)r[2] + r[3] - b; ip[1] = r[2] - b; ip[2] = r[3] - b; ip[3] = b;
      }
    }
    __syncthreads();
  }
}

}  // namespace nsg
