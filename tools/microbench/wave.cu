// Design microbenchmark: cost of the ingredients of the link item's first insertion wave
// (2048 keys per CTA, 2 CTAs per SM, 6144-slot table), one ingredient added at a time.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o wave wave.cu
#include <cstdio>
#include <cstdint>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
typedef unsigned long long u64; typedef uint32_t u32;
constexpr int FT = 512, KPT = 4, TCAP = 6144, B = 64, PCAP = 512;
struct Pend { u64 a; u32 b; u32 probe; };

__device__ __forceinline__ u64 hash64(u64 h) {
  h ^= h >> 33; h *= 0xff51afd7ed558ccdull; h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ull; h ^= h >> 33; return h;
}
__device__ __forceinline__ u32 hash32(u32 x) { x ^= x >> 16; x *= 0x85ebca6bu; x ^= x >> 13; x *= 0xc2b2ae35u; x ^= x >> 16; return x; }
__device__ __forceinline__ u32 home_slot(u32 h) { return (u32)(((u64)h * (u64)TCAP) >> 32); }
__device__ __forceinline__ u32 sb(u32 node) { return hash32(node) >> 26; }

template <int MODE>
__global__ void __launch_bounds__(FT, 2) k_wave(int items, unsigned long long* cyc, u64* sink) {
  extern __shared__ __align__(16) unsigned char sm[];
  u64* lkey = (u64*)sm; u32* lcnt = (u32*)(lkey + TCAP); u32* hist = lcnt + TCAP; Pend* pend = (Pend*)(hist + 2 * B + 4);
  __shared__ u32 pcnt;
  const int t = threadIdx.x, lane = t & 31;
  long long tot = 0; u64 acc = 0;
  for (int it = 0; it < items; ++it) {
    for (int i = t; i < TCAP; i += FT) { lkey[i] = ~0ull; lcnt[i] = 0; }
    for (int i = t; i < 2 * B; i += FT) hist[i] = 0;
    if (t == 0) pcnt = 0;
    u64 k[KPT];
#pragma unroll
    for (int j = 0; j < KPT; ++j) k[j] = hash64(t + j * FT + 4096ull * (blockIdx.x * items + it) + 1);
    __syncthreads();
    const long long t0 = clock64();
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      u64 key = k[j];
      u32 add = 1;
      bool entry = true;
      if (MODE >= 1) {  // leader aggregation
        const u64 lead = __shfl_sync(0xffffffffu, key, 0);
        const u32 same = __ballot_sync(0xffffffffu, key == lead);
        if (key == lead) { entry = lane == __ffs(same) - 1; add = __popc(same); }
      }
      bool placed = true;
      u32 home = 0;
      if (entry) {
        home = home_slot((u32)hash64(key));
        const u64 old = atomicCAS(&lkey[home], ~0ull, key);
        if (MODE >= 2 && old == ~0ull) {  // claim-time side-bucket histogram
          atomicAdd(&hist[sb((u32)(key >> 32))], 1u);
          atomicAdd(&hist[B + sb((u32)key)], 1u);
        }
        placed = old == ~0ull || old == key;
        if (placed) atomicAdd(&lcnt[home], add);
      }
      if (MODE >= 3 && !placed) {  // second probe
        const u32 s2 = home + 1 == TCAP ? 0 : home + 1;
        const u64 old = atomicCAS(&lkey[s2], ~0ull, key);
        if (MODE >= 2 && old == ~0ull) { atomicAdd(&hist[sb((u32)(key >> 32))], 1u); atomicAdd(&hist[B + sb((u32)key)], 1u); }
        placed = old == ~0ull || old == key;
        if (placed) atomicAdd(&lcnt[s2], add);
      }
      if (MODE >= 4) {  // pending push
        const bool want = !placed;
        const u32 mask = __ballot_sync(0xffffffffu, want);
        if (mask) {
          const int leader = __ffs(mask) - 1;
          u32 base = 0;
          if (lane == leader) base = atomicAdd(&pcnt, (u32)__popc(mask));
          base = __shfl_sync(0xffffffffu, base, leader);
          if (want) { const u32 pos = base + __popc(mask & ((1u << lane) - 1u)); if (pos < PCAP) pend[pos] = Pend{key, add, 2u}; }
        }
      } else {
        acc += placed;
      }
    }
    __syncthreads();
    tot += clock64() - t0;
  }
  if (t == 0) cyc[blockIdx.x] = tot / items;
  if (acc == 12345) sink[0] = acc;
}

// Counting-sort dedup: histogram of 13 slot bits (8192 bins), block scan, scatter, per-bin dedup by
// a thread owning 16 consecutive bins.  Produces the distinct count (checked against 2048).
constexpr int NBIN = 8192;
__global__ void __launch_bounds__(FT, 2) k_sort(int items, unsigned long long* cyc, u64* sink, int dup) {
  extern __shared__ __align__(16) unsigned char sm[];
  u32* bins = (u32*)sm;                      // NBIN + 1
  u64* sorted = (u64*)(bins + NBIN + 8);     // 4096
  u32* wsum = (u32*)(sorted + 4096);         // 16
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  long long tot = 0; u64 acc = 0;
  for (int it = 0; it < items; ++it) {
    {
      uint4* b4 = (uint4*)bins;
      for (int i = t; i < NBIN / 4; i += FT) b4[i] = make_uint4(0, 0, 0, 0);
    }
    u64 k[KPT];
#pragma unroll
    for (int j = 0; j < KPT; ++j) k[j] = hash64(((t + j * FT) % dup) + 4096ull * (blockIdx.x * items + it) + 1);
    __syncthreads();
    const long long t0 = clock64();
    u32 bn[KPT];
#pragma unroll
    for (int j = 0; j < KPT; ++j) { bn[j] = (u32)hash64(k[j]) & (NBIN - 1); atomicAdd(&bins[bn[j]], 1u); }
    __syncthreads();
    // block scan of NBIN bins: thread t owns bins [16t, 16t+16)
    u32 v[16]; u32 s = 0;
    {
      const uint4* b4 = (const uint4*)(bins + 16 * t);
#pragma unroll
      for (int q = 0; q < 4; ++q) { uint4 x = b4[q]; v[4*q] = x.x; v[4*q+1] = x.y; v[4*q+2] = x.z; v[4*q+3] = x.w; }
#pragma unroll
      for (int q = 0; q < 16; ++q) s += v[q];
    }
    u32 x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const u32 y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    u32 wbase = 0;
    for (int w = 0; w < wid; ++w) wbase += wsum[w];
    u32 run = wbase + x - s;
    u32 start[16];
    {
      uint4* b4 = (uint4*)(bins + 16 * t);
#pragma unroll
      for (int q = 0; q < 16; ++q) { start[q] = run; run += v[q]; }
#pragma unroll
      for (int q = 0; q < 4; ++q) b4[q] = make_uint4(start[4*q], start[4*q+1], start[4*q+2], start[4*q+3]);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < KPT; ++j) sorted[atomicAdd(&bins[bn[j]], 1u)] = k[j];
    __syncthreads();
    // dedup: bins[b] now = end of bin b; start[q] kept in registers
    u32 distinct = 0;
#pragma unroll 1
    for (int q = 0; q < 16; ++q) {
      const u32 lo = start[q], hi = lo + v[q];
      for (u32 i = lo; i < hi; ++i) {
        const u64 a = sorted[i];
        bool first = true;
        for (u32 j2 = lo; j2 < i; ++j2) if (sorted[j2] == a) { first = false; break; }
        distinct += first;
      }
    }
    __syncthreads();
    tot += clock64() - t0;
    acc += distinct;
  }
  if (t == 0) cyc[blockIdx.x] = tot / items;
  if (acc == 12345) sink[0] = acc;
}

template <int MODE>
void run(const char* name, unsigned long long* cyc, u64* sink, int sms) {
  auto k = k_wave<MODE>;
  int smem = TCAP * 12 + (2 * B + 4) * 4 + PCAP * 16;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int grid = 2 * sms, items = 64;
  k<<<grid, FT, smem>>>(items, cyc, sink);
  CK(cudaDeviceSynchronize());
  k<<<grid, FT, smem>>>(items, cyc, sink);
  CK(cudaDeviceSynchronize());
  static unsigned long long h[1024]; CK(cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost));
  double avg = 0; for (int i = 0; i < grid; ++i) avg += h[i]; avg /= grid;
  printf("%-48s: %8.0f cycles per 2048-key wave\n", name, avg);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* cyc; CK(cudaMalloc(&cyc, 8192)); u64* sink; CK(cudaMalloc(&sink, 64));
  run<0>("CAS home + ADD", cyc, sink, sms);
  run<1>("+ leader aggregation", cyc, sink, sms);
  run<2>("+ claim-time side histogram (2 x 64 bins)", cyc, sink, sms);
  run<3>("+ second probe", cyc, sink, sms);
  run<4>("+ pending push", cyc, sink, sms);
  {
    int smem = (NBIN + 8) * 4 + 4096 * 8 + 64;
    CK(cudaFuncSetAttribute(k_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int dup : {1 << 30, 1024, 64}) {
      int grid = 2 * sms, items = 64;
      k_sort<<<grid, FT, smem>>>(items, cyc, sink, dup);
      CK(cudaDeviceSynchronize());
      k_sort<<<grid, FT, smem>>>(items, cyc, sink, dup);
      CK(cudaDeviceSynchronize());
      static unsigned long long h[1024]; CK(cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost));
      double avg = 0; for (int i = 0; i < grid; ++i) avg += h[i]; avg /= grid;
      printf("counting-sort dedup (hist+scan+scatter+dedup), %4d distinct-ish: %8.0f cycles per 2048 keys\n", dup > 4096 ? 2048 : dup, avg);
    }
  }
  printf("done\n");
}
