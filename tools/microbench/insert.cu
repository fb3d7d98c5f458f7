// Design microbenchmark: cost of "gather 4096 keys + insert into an 8192-slot SMEM hash table" per CTA
// (the link-bucket item's hot phase), isolating the gather, the segment search and the insert.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o insert insert.cu
#include <cstdio>
#include <cstdint>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
typedef unsigned long long u64; typedef uint32_t u32;
constexpr int FT = 512, KPT = 8, TCAP = 8192;

__device__ __forceinline__ u64 hash64(u64 h) {
  h ^= h >> 33; h *= 0xff51afd7ed558ccdull; h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ull; h ^= h >> 33; return h;
}
__device__ __forceinline__ bool ins(u64* lkey, u32* lcnt, u64 key, u32 add) {
  u32 slot = (u32)hash64(key) & (TCAP - 1);
#pragma unroll 1
  for (int probe = 0; probe < TCAP; ++probe) {
    u64 k = reinterpret_cast<volatile u64*>(lkey)[slot];
    if (k == ~0ull) { const u64 old = atomicCAS(&lkey[slot], ~0ull, key); k = (old == ~0ull) ? key : old; }
    if (k == key) { atomicAdd(&lcnt[slot], add); return true; }
    slot = (slot + 1) & (TCAP - 1);
  }
  return false;
}
// batched: the N probes of a thread proceed together (independent LDS, then independent CAS)
template <int N>
__device__ __forceinline__ void ins_batch(u64* lkey, u32* lcnt, const u64 (&k)[N], u32 pending) {
  u32 slot[N];
#pragma unroll
  for (int j = 0; j < N; ++j) slot[j] = (u32)hash64(k[j]) & (TCAP - 1);
  while (pending) {
    u64 cur[N];
#pragma unroll
    for (int j = 0; j < N; ++j) cur[j] = (pending >> j & 1) ? reinterpret_cast<volatile u64*>(lkey)[slot[j]] : 0ull;
#pragma unroll
    for (int j = 0; j < N; ++j)
      if ((pending >> j & 1) && cur[j] == ~0ull) { const u64 old = atomicCAS(&lkey[slot[j]], ~0ull, k[j]); cur[j] = old == ~0ull ? k[j] : old; }
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if (!(pending >> j & 1)) continue;
      if (cur[j] == k[j]) { atomicAdd(&lcnt[slot[j]], 1u); pending &= ~(1u << j); }
      else slot[j] = (slot[j] + 1) & (TCAP - 1);
    }
  }
}
__device__ __forceinline__ void ins_nopre(u64* lkey, u32* lcnt, u64 key) {  // CAS first, no plain read
  u32 slot = (u32)hash64(key) & (TCAP - 1);
  for (;;) {
    const u64 old = atomicCAS(&lkey[slot], ~0ull, key);
    if (old == ~0ull || old == key) { atomicAdd(&lcnt[slot], 1u); return; }
    slot = (slot + 1) & (TCAP - 1);
  }
}
__device__ __forceinline__ void ins32(u32* key32, u32* lcnt, u32 key) {
  u32 slot = (key * 0x9E3779B1u) >> 19;
  for (;;) {
    u32 k = reinterpret_cast<volatile u32*>(key32)[slot];
    if (k == ~0u) { const u32 old = atomicCAS(&key32[slot], ~0u, key); k = old == ~0u ? key : old; }
    if (k == key) { atomicAdd(&lcnt[slot], 1u); return; }
    slot = (slot + 1) & (TCAP - 1);
  }
}
// per-lane work queue: a lane that finishes a key moves on to its next one, so the warp waits for
// the max over lanes of the SUM of probes, not the sum over keys of the max.  INFL probes in flight.
template <int N, int INFL>
__device__ __forceinline__ void ins_queue(u64* lkey, u32* lcnt, u64 (&q)[N], int nq) {
  u64 cur[INFL]; u32 slot[INFL]; bool act[INFL];
#pragma unroll
  for (int f = 0; f < INFL; ++f) { act[f] = false; }
  for (;;) {
#pragma unroll
    for (int f = 0; f < INFL; ++f) {
      if (!act[f] && nq > 0) {
        cur[f] = q[0];
#pragma unroll
        for (int j = 0; j + 1 < N; ++j) q[j] = q[j + 1];
        --nq; act[f] = true; slot[f] = (u32)hash64(cur[f]) & (TCAP - 1);
      }
    }
    bool any = false;
#pragma unroll
    for (int f = 0; f < INFL; ++f) any |= act[f];
    if (!__any_sync(0xffffffffu, any)) break;
    u64 v[INFL];
#pragma unroll
    for (int f = 0; f < INFL; ++f) v[f] = act[f] ? reinterpret_cast<volatile u64*>(lkey)[slot[f]] : 0ull;
#pragma unroll
    for (int f = 0; f < INFL; ++f)
      if (act[f] && v[f] == ~0ull) { const u64 old = atomicCAS(&lkey[slot[f]], ~0ull, cur[f]); v[f] = old == ~0ull ? cur[f] : old; }
#pragma unroll
    for (int f = 0; f < INFL; ++f) {
      if (!act[f]) continue;
      if (v[f] == cur[f]) { atomicAdd(&lcnt[slot[f]], 1u); act[f] = false; }
      else slot[f] = (slot[f] + 1) & (TCAP - 1);
    }
  }
}
__device__ __forceinline__ void ins_dh(u64* lkey, u32* lcnt, u64 key) {  // double hashing
  const u64 h = hash64(key);
  u32 slot = (u32)h & (TCAP - 1);
  const u32 step = ((u32)(h >> 32) << 1) | 1u;
  for (;;) {
    u64 k = reinterpret_cast<volatile u64*>(lkey)[slot];
    if (k == ~0ull) { const u64 old = atomicCAS(&lkey[slot], ~0ull, key); k = (old == ~0ull) ? key : old; }
    if (k == key) { atomicAdd(&lcnt[slot], 1u); return; }
    slot = (slot + step) & (TCAP - 1);
  }
}
__device__ unsigned long long g_probes;
__device__ __forceinline__ void ins_count(u64* lkey, u32* lcnt, u64 key, u32& probes) {
  u32 slot = (u32)hash64(key) & (TCAP - 1);
  for (;;) {
    ++probes;
    u64 k = reinterpret_cast<volatile u64*>(lkey)[slot];
    if (k == ~0ull) { const u64 old = atomicCAS(&lkey[slot], ~0ull, key); k = (old == ~0ull) ? key : old; }
    if (k == key) { atomicAdd(&lcnt[slot], 1u); return; }
    slot = (slot + 1) & (TCAP - 1);
  }
}
// queue insert without pre-read: every active lane issues one CAS per iteration (full warp-instrs)
template <int N, int INFL>
__device__ __forceinline__ void ins_queue2(u64* lkey, u32* lcnt, u64 (&q)[N], int nq) {
  u64 cur[INFL]; u32 slot[INFL]; bool act[INFL];
#pragma unroll
  for (int f = 0; f < INFL; ++f) act[f] = false;
  for (;;) {
#pragma unroll
    for (int f = 0; f < INFL; ++f) {
      if (!act[f] && nq > 0) {
        cur[f] = q[0];
#pragma unroll
        for (int j = 0; j + 1 < N; ++j) q[j] = q[j + 1];
        --nq; act[f] = true; slot[f] = (u32)hash64(cur[f]) & (TCAP - 1);
      }
    }
    bool any = false;
#pragma unroll
    for (int f = 0; f < INFL; ++f) any |= act[f];
    if (!__any_sync(0xffffffffu, any)) break;
    u64 v[INFL];
#pragma unroll
    for (int f = 0; f < INFL; ++f) v[f] = act[f] ? atomicCAS(&lkey[slot[f]], ~0ull, cur[f]) : 0ull;
#pragma unroll
    for (int f = 0; f < INFL; ++f) {
      if (!act[f]) continue;
      if (v[f] == ~0ull || v[f] == cur[f]) { atomicAdd(&lcnt[slot[f]], 1u); act[f] = false; }
      else slot[f] = (slot[f] + 1) & (TCAP - 1);
    }
  }
}
__device__ __forceinline__ u32 find_seg(const u32* pre, u32 n, u32 i) {
  u32 lo = 0, hi = n - 1;
  while (lo < hi) { const u32 mid = (lo + hi + 1) >> 1; if (pre[mid] <= i) lo = mid; else hi = mid - 1; }
  return lo;
}

// MODE 0: keys from registers (no gather), plain insert
// MODE 1: contiguous gather (ldcg) + insert
// MODE 2: segmented gather with find_seg (32 segments) + insert
// MODE 3: segmented gather only (sum keys), no insert
// MODE 4: MODE 2 + warp-leader aggregation (as in nsg_fast)
// MODE 5: table init + MODE 2 (one full item phase 0..2)
template <int MODE>
__global__ void __launch_bounds__(FT, 2) k_ins(const u64* __restrict__ src, int items, unsigned long long* cyc, u64* sink) {
  extern __shared__ __align__(16) unsigned char sm[];
  u64* lkey = (u64*)sm; u32* lcnt = (u32*)(sm + TCAP * 8); u32* seg = lcnt + TCAP; u32* seglo = seg + 64;
  const int t = threadIdx.x, lane = t & 31;
  u64 acc = 0; long long tot = 0;
  for (int it = 0; it < items; ++it) {
    const u64* base = src + ((u64)(blockIdx.x * items + it) % 512) * 4096;
    if (MODE != 5) for (int i = t; i < TCAP; i += FT) { lkey[i] = ~0ull; lcnt[i] = 0; }
    if (t < 32) { seg[t] = t * 128; seglo[t] = t * 128; }
    if (t == 0) seg[32] = 4096;
    __syncthreads();
    long long t0 = clock64();
    if (MODE == 5) { for (int i = t; i < TCAP; i += FT) { lkey[i] = ~0ull; lcnt[i] = 0; } __syncthreads(); }
    u64 k[KPT];
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      const u32 i = t + j * FT;
      if (MODE == 0 || MODE == 6 || MODE >= 8) k[j] = hash64(i + 4096ull * (blockIdx.x * items + it));
      else if (MODE == 1) k[j] = __ldcg(base + i);
      else { const u32 c = find_seg(seg, 32, i); k[j] = __ldcg(base + seglo[c] + (i - seg[c])); }
    }
    if (MODE == 3) {
#pragma unroll
      for (int j = 0; j < KPT; ++j) acc += k[j];
    } else if (MODE == 4) {
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        const u64 lead = __shfl_sync(0xffffffffu, k[j], 0);
        const u32 same = __ballot_sync(0xffffffffu, k[j] == lead);
        if (k[j] == lead) { if (lane == __ffs(same) - 1) ins(lkey, lcnt, lead, __popc(same)); }
        else ins(lkey, lcnt, k[j], 1);
      }
    } else if (MODE == 8) {   // CAS only, no add, no probing (slot from hash)
#pragma unroll
      for (int j = 0; j < KPT; ++j) atomicCAS(&lkey[(u32)hash64(k[j]) & (TCAP - 1)], ~0ull, k[j]);
    } else if (MODE == 9) {   // random u32 adds only
#pragma unroll
      for (int j = 0; j < KPT; ++j) atomicAdd(&lcnt[(u32)hash64(k[j]) & (TCAP - 1)], 1u);
    } else if (MODE == 10) {  // u32 keys
#pragma unroll
      for (int j = 0; j < KPT; ++j) ins32((u32*)lkey, lcnt, (u32)(k[j] >> 32) | 1u);
    } else if (MODE == 11) {
#pragma unroll
      for (int j = 0; j < KPT; ++j) ins_nopre(lkey, lcnt, k[j]);
    } else if (MODE == 13) {
      ins_queue<KPT, 1>(lkey, lcnt, k, KPT);
    } else if (MODE == 14) {
      ins_queue<KPT, 2>(lkey, lcnt, k, KPT);
    } else if (MODE == 15) {
      ins_queue<KPT, 4>(lkey, lcnt, k, KPT);
    } else if (MODE == 16) {  // CAS with result used
#pragma unroll
      for (int j = 0; j < KPT; ++j) acc += atomicCAS(&lkey[(u32)hash64(k[j]) & (TCAP - 1)], ~0ull, k[j]);
    } else if (MODE == 17) {  // ADD with result used
#pragma unroll
      for (int j = 0; j < KPT; ++j) acc += atomicAdd(&lcnt[(u32)hash64(k[j]) & (TCAP - 1)], 1u);
    } else if (MODE == 18) {  // random volatile LDS.64
#pragma unroll
      for (int j = 0; j < KPT; ++j) acc += reinterpret_cast<volatile u64*>(lkey)[(u32)hash64(k[j]) & (TCAP - 1)];
    } else if (MODE == 19) {  // CAS with result used, then dependent add
#pragma unroll
      for (int j = 0; j < KPT; ++j) { const u32 sl = (u32)hash64(k[j]) & (TCAP - 1); u64 o = atomicCAS(&lkey[sl], ~0ull, k[j]); if (o == ~0ull || o == k[j]) atomicAdd(&lcnt[sl], 1u); }
    } else if (MODE == 20) {  // u32 CAS with result used
#pragma unroll
      for (int j = 0; j < KPT; ++j) acc += atomicCAS(&lcnt[(u32)hash64(k[j]) & (TCAP - 1)], ~0u, (u32)k[j]);
    } else if (MODE == 21) {
#pragma unroll
      for (int j = 0; j < KPT; ++j) ins_dh(lkey, lcnt, k[j]);
    } else if (MODE == 22) {
      u32 pr = 0;
#pragma unroll
      for (int j = 0; j < KPT; ++j) ins_count(lkey, lcnt, k[j], pr);
      atomicAdd(&g_probes, (unsigned long long)pr);
    } else if (MODE == 23) {
      ins_queue2<KPT, 1>(lkey, lcnt, k, KPT);
    } else if (MODE == 24) {
      ins_queue2<KPT, 2>(lkey, lcnt, k, KPT);
    } else if (MODE == 12) {  // hash only
#pragma unroll
      for (int j = 0; j < KPT; ++j) acc += hash64(k[j]);
    } else if (MODE == 6 || MODE == 7) {
      ins_batch<KPT>(lkey, lcnt, k, 0xFFu);
    } else {
#pragma unroll
      for (int j = 0; j < KPT; ++j) ins(lkey, lcnt, k[j], 1);
    }
    __syncthreads();
    tot += clock64() - t0;
  }
  if (t == 0) cyc[blockIdx.x] = tot / items;
  if (acc == 42) sink[0] = acc;
}

template <int MODE>
void run(const char* name, const u64* src, unsigned long long* cyc, u64* sink, int sms) {
  auto k = k_ins<MODE>;
  int smem = TCAP * 12 + 1024;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int grid = 2 * sms, items = 64;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<<<grid, FT, smem>>>(src, items, cyc, sink);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  k<<<grid, FT, smem>>>(src, items, cyc, sink);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  static unsigned long long h[1024]; CK(cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost));
  double avg = 0; for (int i = 0; i < grid; ++i) avg += h[i]; avg /= grid;
  printf("%-44s: %8.0f cycles/item (4096 keys), chip %.1f Gkeys/s\n", name, avg, (double)grid * items * 4096 / ms / 1e6);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  u64* src; CK(cudaMalloc(&src, 512 * 4096 * 8));
  // distinct random keys
  u64* h = (u64*)malloc(512 * 4096 * 8);
  u64 x = 88172645463325252ull;
  for (int i = 0; i < 512 * 4096; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = x; }
  CK(cudaMemcpy(src, h, 512 * 4096 * 8, cudaMemcpyHostToDevice));
  unsigned long long* cyc; CK(cudaMalloc(&cyc, 8192)); u64* sink; CK(cudaMalloc(&sink, 64));
  run<0>("registers -> insert", src, cyc, sink, sms);
  run<1>("contiguous ldcg gather -> insert", src, cyc, sink, sms);
  run<2>("segmented gather (find_seg) -> insert", src, cyc, sink, sms);
  run<3>("segmented gather only", src, cyc, sink, sms);
  run<4>("segmented gather -> leader-agg insert", src, cyc, sink, sms);
  run<5>("init + segmented gather -> insert", src, cyc, sink, sms);
  run<6>("registers -> batched insert", src, cyc, sink, sms);
  run<7>("segmented gather -> batched insert", src, cyc, sink, sms);
  run<8>("CAS.64 only (no probe, no add)", src, cyc, sink, sms);
  run<9>("ATOMS.ADD.32 only", src, cyc, sink, sms);
  run<10>("u32-key table insert", src, cyc, sink, sms);
  run<11>("insert, CAS without pre-read", src, cyc, sink, sms);
  run<12>("hash64 only", src, cyc, sink, sms);
  run<13>("queue insert, 1 in flight", src, cyc, sink, sms);
  run<14>("queue insert, 2 in flight", src, cyc, sink, sms);
  run<15>("queue insert, 4 in flight", src, cyc, sink, sms);
  run<16>("CAS.64, result used", src, cyc, sink, sms);
  run<17>("ATOMS.ADD.32, result used", src, cyc, sink, sms);
  run<18>("random volatile LDS.64", src, cyc, sink, sms);
  run<19>("CAS.64 then dependent ADD (1 probe)", src, cyc, sink, sms);
  run<20>("CAS.32, result used", src, cyc, sink, sms);
  run<21>("double-hashing insert", src, cyc, sink, sms);
  run<23>("queue insert no pre-read, 1 in flight", src, cyc, sink, sms);
  run<24>("queue insert no pre-read, 2 in flight", src, cyc, sink, sms);
  unsigned long long z = 0; cudaMemcpyToSymbol(g_probes, &z, 8);
  run<22>("linear insert counting probes", src, cyc, sink, sms);
  cudaMemcpyFromSymbol(&z, g_probes, 8);
  printf("avg probes per insert: %.3f\n", (double)z / (2.0 * 2 * sms * 64 * 4096));
  printf("done\n");
}
