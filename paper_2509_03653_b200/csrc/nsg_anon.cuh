// nsg_anon.cuh — IP address anonymisation.
//
// The paper: "Given an array of length N, we generate the sequence array with the values 0,1,..,N-1,
// followed by the use of the Python shuffle operation ... The shuffled array is then used to assign new
// values to the original source and destination IP addresses using gather instructions.  The size N ...
// [is] the number of unique value of src and dest ids"; several shuffle rounds may be
// applied.  This path computes, for the whole input:
//   U      = the distinct addresses of src and dst, in ascending order; N = |U|       ("unique")
//   rank(a)= the index of address a in U
//   pi     = a keyed pseudo-random permutation of [0, N) (reading R15: a 4-round Feistel network
//            on the smallest even-bit domain >= N with cycle walking, one network per shuffle round, in
//            place of the host shuffle; it is deterministic and needs no table, cf. the deterministic
//            HashGraph permutation the paper cites)
//   src'_p = pi(rank(src_p)), dst'_p = pi(rank(dst_p))                                 ("gather")
// U is never materialised: membership is a 2^32-bit bitmap (512 MiB) in the workspace and rank(a) is the
// number of set bits below a: an exclusive prefix per 128-bit group (128 MiB) plus the popcounts inside
// a's group (one 128-bit load).  When N <= ANON_TABLE_MAX the labels pi(rank(a)) are computed once per
// distinct address (a scan of the bitmap) into an address -> label hash table of next_pow2(2N) slots,
// small enough to stay in L2, and the gather is one table probe per address; otherwise every address
// is ranked and permuted directly.
#pragma once
#include "nsg_internal.h"
#include "nsg_common.cuh"

namespace nsg {

constexpr int AT = 512;                          // threads per CTA
constexpr u64 ANON_WORDS = 1ull << 27;           // u32 words of the 2^32-bit bitmap
constexpr u64 ANON_BLOCKS = ANON_WORDS / 4;      // 128-bit groups (2^25)
constexpr u32 ANON_SCAN_PER_CTA = 32768;         // groups per CTA in the prefix scan
constexpr u32 ANON_SCAN_CTAS = (u32)(ANON_BLOCKS / ANON_SCAN_PER_CTA);  // 1024
constexpr u64 ANON_TABLE_SLOTS = 1ull << 24;     // label table capacity (u64 slots: address << 32 | label)
constexpr u64 ANON_TABLE_MAX = ANON_TABLE_SLOTS / 2;  // largest N served by the table (load <= 1/2)
// workspace: bitmap | group prefix | CTA totals | label table | U (the distinct addresses in rank order)

__device__ __forceinline__ u64 anon_mix(u64 z) {  // splitmix64
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// One keyed Feistel permutation of [0, N) (N >= 1): 4 rounds on 2h-bit values (2^(2h) >= N, h >= 1),
// round function f_j(R) = low h bits of splitmix64(key ^ (j << 56) ^ R), cycle-walked into [0, N).
__device__ __forceinline__ u64 anon_feistel(u64 x, u64 N, u64 key) {
  u32 bits = 64 - __clzll((long long)(N - 1));  // ceil(log2 N) for N >= 2; 0 for N = 1
  if (bits < 2) bits = 2;
  const u32 h = (bits + 1) >> 1;
  const u64 mask = (1ull << h) - 1;
  do {
    u64 L = x >> h, R = x & mask;
#pragma unroll
    for (u32 j = 0; j < 4; ++j) {
      const u64 t = L ^ (anon_mix(key ^ ((u64)j << 56) ^ R) & mask);
      L = R;
      R = t;
    }
    x = (L << h) | R;
  } while (x >= N);
  return x;
}

__device__ __forceinline__ u64 anon_perm(u64 r, u64 N, u64 seed, u32 rounds) {
  for (u32 k = 0; k < rounds; ++k) r = anon_feistel(r, N, anon_mix(seed + k));
  return r;
}

__device__ __forceinline__ void anon_mark(u32* bitmap, u32 a) {
  u32* w = &bitmap[a >> 5];
  const u32 bit = 1u << (a & 31);
  if (!(ldcg32(w) & bit)) atomicOr(w, bit);  // read first: repeated addresses cost no atomic
}

__global__ void __launch_bounds__(AT) anon_mark_kernel(const u64* __restrict__ keys, const u32* __restrict__ src,
                                                       const u32* __restrict__ dst, u64 n, u32* __restrict__ bitmap) {
  for (u64 i = (u64)blockIdx.x * AT + threadIdx.x; i < n; i += (u64)gridDim.x * AT) {
    const u32 s = keys ? (u32)(keys[i] >> 32) : src[i];
    const u32 d = keys ? (u32)keys[i] : dst[i];
    anon_mark(bitmap, s);
    anon_mark(bitmap, d);
  }
}

// Set bits per 128-bit group, then the exclusive prefix over groups: per-CTA totals, a one-CTA scan of
// the totals (N = their sum), per-CTA downsweep.
__global__ void __launch_bounds__(AT) anon_block_count(const u32* __restrict__ bitmap, u32* __restrict__ bcnt,
                                                       u32* __restrict__ ctot) {
  __shared__ u32 red[AT / 32];
  const u64 b0 = (u64)blockIdx.x * ANON_SCAN_PER_CTA;
  const uint4* p = reinterpret_cast<const uint4*>(bitmap);
  u32 mine = 0;
  for (u32 j = threadIdx.x; j < ANON_SCAN_PER_CTA; j += AT) {
    const uint4 v = __ldcg(p + b0 + j);  // kept in L2 for the relabel kernel
    const u32 c = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
    bcnt[b0 + j] = c;
    mine += c;
  }
  mine = warp_sum(mine);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mine;
  __syncthreads();
  if (threadIdx.x < 32) {
    u32 v = threadIdx.x < AT / 32 ? red[threadIdx.x] : 0u;
    v = warp_sum(v);
    if (threadIdx.x == 0) ctot[blockIdx.x] = v;
  }
}

__global__ void __launch_bounds__(1024) anon_scan_totals(u32* __restrict__ ctot, u64* __restrict__ n_unique) {
  __shared__ u32 wsum[32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const u32 v = ctot[t];  // ANON_SCAN_CTAS == 1024 == blockDim.x
  u32 x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    u32 s = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    wsum[lane] = s;
  }
  __syncthreads();
  const u32 incl = x + (wid ? wsum[wid - 1] : 0u);
  ctot[t] = incl - v;  // exclusive
  if (t == 1023) *n_unique = (u64)(incl - v) + v;  // the exclusive prefix fits 32 bits even when N = 2^32
}

__global__ void __launch_bounds__(AT) anon_block_prefix(u32* __restrict__ bcnt, const u32* __restrict__ ctot) {
  // in-CTA exclusive scan of this CTA's group counts (PER contiguous per thread), offset by the CTA prefix
  __shared__ u32 wsum[AT / 32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  constexpr int PER = ANON_SCAN_PER_CTA / AT;
  u32* b = bcnt + (u64)blockIdx.x * ANON_SCAN_PER_CTA + t * PER;
  u32 s = 0;
  for (int q = 0; q < PER; q += 4) {
    const uint4 v = *reinterpret_cast<const uint4*>(b + q);
    s += v.x + v.y + v.z + v.w;
  }
  u32 x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    u32 w = lane < AT / 32 ? wsum[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < AT / 32) wsum[lane] = w;
  }
  __syncthreads();
  u32 run = ctot[blockIdx.x] + (x - s) + (wid ? wsum[wid - 1] : 0u);
  for (int q = 0; q < PER; q += 4) {
    uint4 v = *reinterpret_cast<const uint4*>(b + q);
    uint4 o;
    o.x = run; run += v.x;
    o.y = run; run += v.y;
    o.z = run; run += v.z;
    o.w = run; run += v.w;
    *reinterpret_cast<uint4*>(b + q) = o;
  }
}

// rank(a) = set bits of the bitmap below a: the group prefix + the bits of a's group below a
__device__ __forceinline__ u64 anon_rank(const u32* __restrict__ bitmap, const u32* __restrict__ bpre, u32 a) {
  const uint4 g = __ldcg(reinterpret_cast<const uint4*>(bitmap) + (a >> 7));
  const u32 q = (a >> 5) & 3u, below = (1u << (a & 31)) - 1u;
  u32 r = bpre[a >> 7];
  r += q > 0 ? __popc(g.x) : __popc(g.x & below);
  if (q >= 1) r += q > 1 ? __popc(g.y) : __popc(g.y & below);
  if (q >= 2) r += q > 2 ? __popc(g.z) : __popc(g.z & below);
  if (q == 3) r += __popc(g.w & below);
  return r;
}

// ---- label table (N <= ANON_TABLE_MAX): slot = entry (address << 32 | label), EMPTY64 = free.  A real
// entry never equals EMPTY64 because labels are < N <= 2^23.
__device__ __forceinline__ u64 anon_table_cap(u64 N) {
  u64 c = 1;
  while (c < 2 * N) c <<= 1;
  return c;
}
__device__ __forceinline__ u64 anon_slot(u32 a, u64 cap) { return ((u64)hash32(a) * 0x9E3779B97F4A7C15ull >> 17) & (cap - 1); }

__global__ void __launch_bounds__(AT) anon_table_fill(u64* __restrict__ table, const u64* __restrict__ n_unique) {
  const u64 N = *n_unique;
  if (N > ANON_TABLE_MAX) return;
  const u64 cap = anon_table_cap(N);
  for (u64 i = (u64)blockIdx.x * AT + threadIdx.x; i < cap; i += (u64)gridDim.x * AT) table[i] = EMPTY64;
}

// Enumerate the distinct addresses in ascending order, U[rank] = a (one thread per 128-bit group of the
// bitmap, the granularity of the rank prefix; the work per set bit is one store), then label them densely
// (anon_table_label: full warps for the permutation arithmetic).
__global__ void __launch_bounds__(AT) anon_enumerate(const u32* __restrict__ bitmap, const u32* __restrict__ bpre,
                                                     const u64* __restrict__ n_unique, u32* __restrict__ U) {
  if (*n_unique > ANON_TABLE_MAX) return;
  const uint4* g4 = reinterpret_cast<const uint4*>(bitmap);
  for (u64 gi = (u64)blockIdx.x * AT + threadIdx.x; gi < ANON_BLOCKS; gi += (u64)gridDim.x * AT) {
    const uint4 g = __ldcs(g4 + gi);
    if ((g.x | g.y | g.z | g.w) == 0) continue;
    u32 r = bpre[gi];
    const u32 wv[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      u32 bits = wv[q];
      while (bits) {
        const u32 b = __ffs(bits) - 1;
        bits &= bits - 1;
        U[r++] = (u32)(gi * 128 + q * 32 + b);
      }
    }
  }
}

__global__ void __launch_bounds__(AT) anon_table_label(const u32* __restrict__ U, const u64* __restrict__ n_unique,
                                                       u64 seed, u32 rounds, u64* __restrict__ table) {
  const u64 N = *n_unique;
  if (N > ANON_TABLE_MAX) return;
  const u64 cap = anon_table_cap(N);
  for (u64 r = (u64)blockIdx.x * AT + threadIdx.x; r < N; r += (u64)gridDim.x * AT) {
    const u32 a = U[r];
    const u64 e = ((u64)a << 32) | (u32)anon_perm(r, N, seed, rounds);
    u64 slot = anon_slot(a, cap);
    while (atomicCAS(reinterpret_cast<unsigned long long*>(&table[slot]), EMPTY64, e) != EMPTY64)
      slot = (slot + 1) & (cap - 1);  // each address is inserted once: a taken slot holds another address
  }
}

__device__ __forceinline__ u32 anon_lookup(const u64* __restrict__ table, u64 cap, u32 a) {
  u64 slot = anon_slot(a, cap);
  for (;;) {
    const u64 e = __ldcg(reinterpret_cast<const unsigned long long*>(&table[slot]));
    if ((u32)(e >> 32) == a && e != EMPTY64) return (u32)e;
    slot = (slot + 1) & (cap - 1);  // every looked-up address is present
  }
}

__global__ void __launch_bounds__(AT) anon_relabel_kernel(const u64* __restrict__ keys, const u32* __restrict__ src,
                                                          const u32* __restrict__ dst, u64 n,
                                                          const u32* __restrict__ bitmap, const u32* __restrict__ bpre,
                                                          const u64* __restrict__ table,
                                                          const u64* __restrict__ n_unique, u64 seed, u32 rounds,
                                                          u32* __restrict__ src_out, u32* __restrict__ dst_out) {
  const u64 N = *n_unique;
  const bool tab = N <= ANON_TABLE_MAX;
  const u64 cap = tab ? anon_table_cap(N) : 0;
  for (u64 i = (u64)blockIdx.x * AT + threadIdx.x; i < n; i += (u64)gridDim.x * AT) {
    const u32 s = keys ? (u32)(keys[i] >> 32) : src[i];
    const u32 d = keys ? (u32)keys[i] : dst[i];
    if (tab) {
      src_out[i] = anon_lookup(table, cap, s);
      dst_out[i] = anon_lookup(table, cap, d);
    } else {
      src_out[i] = (u32)anon_perm(anon_rank(bitmap, bpre, s), N, seed, rounds);
      dst_out[i] = (u32)anon_perm(anon_rank(bitmap, bpre, d), N, seed, rounds);
    }
  }
}

}  // namespace nsg
