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
// Membership is a 2^32-bit bitmap (512 MiB) in the workspace, of which only the 128-bit groups that hold
// an address of the input are ever touched: a summary bitmap (one bit per group, 4 MiB, zeroed per call)
// is marked first, the marked groups are zeroed, then the addresses' bits are set.  Counting, ranking and
// enumeration visit the marked groups only (the 4 MiB summary drives them), so a call moves
// O(input + marked groups) bytes instead of scanning 512 MiB three times.  rank(a) = the number of set
// bits below a: an exclusive prefix per marked 128-bit group plus the popcounts inside a's group.  When N <= ANON_TABLE_MAX the labels pi(rank(a)) are computed once per
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
constexpr u64 ANON_SWORDS = ANON_BLOCKS / 32;     // u32 words of the summary bitmap (one bit per group)
constexpr u32 ANON_SCAN_PER_CTA = 2 * AT;        // summary words per CTA in the count / prefix (2 per thread)
constexpr u32 ANON_SCAN_CTAS = (u32)(ANON_SWORDS / ANON_SCAN_PER_CTA);  // 1024
static_assert(ANON_SCAN_CTAS == 1024, "anon_scan_totals scans one total per thread of one 1024-thread CTA");
constexpr u64 ANON_TABLE_SLOTS = 1ull << 24;     // label table capacity (u64 slots: address << 32 | label)
constexpr u64 ANON_TABLE_MAX = ANON_TABLE_SLOTS / 2;  // largest N served by the table (load <= 1/2)
// workspace: bitmap | group prefix | CTA totals | label table | U (the distinct addresses in rank order) |
// summary bitmap | set bits per summary word

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

__device__ __forceinline__ void anon_set(u32* bits, u32 i) {
  u32* w = &bits[i >> 5];
  const u32 bit = 1u << (i & 31);
  if (!(ldcg32(w) & bit)) atomicOr(w, bit);  // read first: repeated addresses cost no atomic
}

// Pass 1: mark the summary bit of every address's 128-bit group.
__global__ void __launch_bounds__(AT) anon_touch_kernel(const u64* __restrict__ keys, const u32* __restrict__ src,
                                                        const u32* __restrict__ dst, u64 n, u32* __restrict__ summ) {
  for (u64 i = (u64)blockIdx.x * AT + threadIdx.x; i < n; i += (u64)gridDim.x * AT) {
    const u32 s = keys ? (u32)(keys[i] >> 32) : src[i];
    const u32 d = keys ? (u32)keys[i] : dst[i];
    anon_set(summ, s >> 7);
    anon_set(summ, d >> 7);
  }
}

// Pass 2: zero the marked groups (the rest of the bitmap is never read).
__global__ void __launch_bounds__(AT) anon_clear_groups(const u32* __restrict__ summ, u32* __restrict__ bitmap) {
  uint4* g4 = reinterpret_cast<uint4*>(bitmap);
  for (u64 w = (u64)blockIdx.x * AT + threadIdx.x; w < ANON_SWORDS; w += (u64)gridDim.x * AT) {
    u32 bits = summ[w];
    while (bits) {
      const u32 b = __ffs(bits) - 1;
      bits &= bits - 1;
      g4[w * 32 + b] = make_uint4(0u, 0u, 0u, 0u);
    }
  }
}

// Pass 3: set every address's bit.
__global__ void __launch_bounds__(AT) anon_mark_kernel(const u64* __restrict__ keys, const u32* __restrict__ src,
                                                       const u32* __restrict__ dst, u64 n, u32* __restrict__ bitmap) {
  for (u64 i = (u64)blockIdx.x * AT + threadIdx.x; i < n; i += (u64)gridDim.x * AT) {
    const u32 s = keys ? (u32)(keys[i] >> 32) : src[i];
    const u32 d = keys ? (u32)keys[i] : dst[i];
    anon_set(bitmap, s);
    anon_set(bitmap, d);
  }
}

__device__ __forceinline__ u32 popc4(const uint4 v) { return __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w); }

// Set bits per summary word (its marked groups' popcounts; 2 words per thread), and per CTA.
__global__ void __launch_bounds__(AT) anon_word_count(const u32* __restrict__ summ, const u32* __restrict__ bitmap,
                                                      u32* __restrict__ wcnt, u32* __restrict__ ctot) {
  __shared__ u32 red[AT / 32];
  const u64 w0 = (u64)blockIdx.x * ANON_SCAN_PER_CTA + 2 * threadIdx.x;
  const uint4* g4 = reinterpret_cast<const uint4*>(bitmap);
  const uint2 sw = *reinterpret_cast<const uint2*>(summ + w0);
  u32 c[2] = {0u, 0u};
  const u32 sv[2] = {sw.x, sw.y};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    u32 bits = sv[k];
    while (bits) {
      const u32 b = __ffs(bits) - 1;
      bits &= bits - 1;
      c[k] += popc4(__ldcg(g4 + (w0 + k) * 32 + b));
    }
  }
  *reinterpret_cast<uint2*>(wcnt + w0) = make_uint2(c[0], c[1]);
  u32 mine = warp_sum(c[0] + c[1]);
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

// The rank of each marked group's first address (CTA prefix + in-CTA exclusive scan of the words' counts +
// the groups before it in its word): stored per group (bpre, read by anon_rank) when N is above the table
// range; with the table (N <= ANON_TABLE_MAX) the distinct addresses are enumerated instead, U[rank] = a.
__global__ void __launch_bounds__(AT) anon_enumerate(const u32* __restrict__ summ, const u32* __restrict__ bitmap,
                                                     const u32* __restrict__ wcnt, const u32* __restrict__ ctot,
                                                     const u64* __restrict__ n_unique, u32* __restrict__ bpre,
                                                     u32* __restrict__ U) {
  __shared__ u32 wsum[AT / 32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const bool tab = *n_unique <= ANON_TABLE_MAX;
  const u64 w0 = (u64)blockIdx.x * ANON_SCAN_PER_CTA + 2 * t;
  const uint2 cc = *reinterpret_cast<const uint2*>(wcnt + w0);
  const u32 s = cc.x + cc.y;
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
  u32 r = ctot[blockIdx.x] + (x - s) + (wid ? wsum[wid - 1] : 0u);
  const uint4* g4 = reinterpret_cast<const uint4*>(bitmap);
  const uint2 sw = *reinterpret_cast<const uint2*>(summ + w0);
  const u32 sv[2] = {sw.x, sw.y};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    u32 gb = sv[k];
    while (gb) {
      const u32 gi = (u32)((w0 + k) * 32) + (__ffs(gb) - 1);
      gb &= gb - 1;
      const uint4 g = __ldcg(g4 + gi);
      if (!tab) {
        bpre[gi] = r;
        r += popc4(g);
        continue;
      }
      const u32 wv[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        u32 bits = wv[q];
        while (bits) {
          const u32 b = __ffs(bits) - 1;
          bits &= bits - 1;
          U[r++] = gi * 128 + q * 32 + b;
        }
      }
    }
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
