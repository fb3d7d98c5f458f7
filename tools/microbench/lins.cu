// Design microbenchmark (not product code): cycles of one link-bucket insert + scan phase in SMEM,
// isolated from the persistent kernel's scheduling.  Keys = one real C2 link bucket (file keys.bin,
// u64[n]).  Variants: 0 CAS-first, 1 load-first, 2 load-first with two keys per lane in flight.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lins lins.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
typedef unsigned long long u64;
typedef uint32_t u32;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
constexpr u64 EMPTY = ~0ull;
constexpr u64 MUL = 0x9E3779B97F4A7C15ull;

template <int V, int TL, int NT>
__global__ void __launch_bounds__(NT) k(const u64* keys, int n, int reps, u64* cyc, u32* sink, int logB) {
  extern __shared__ __align__(16) unsigned char sm[];
  u64* stage = (u64*)sm;
  u64* lkey = stage + 4096;
  u32* lcnt = (u32*)(lkey + TL);
  for (int i = threadIdx.x; i < n; i += NT) stage[i] = keys[i];
  for (int i = threadIdx.x; i < TL; i += NT) { lkey[i] = EMPTY; lcnt[i] = 0; }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long tins = 0, tscan = 0;
  u32 acc = 0;
  for (int r = 0; r < reps; ++r) {
    long long t0 = clock64();
    if (V >= 7 && V <= 10) {
      for (int b0 = wid * 32; b0 < n; b0 += NT) {
        int e = b0 + lane;
        if (e < n) {
          u64 key = stage[e];
          u32 s = (u32)((key * MUL) >> (64 - logB - 12)) & (TL - 1);
          if (V == 7) { u64 o = atomicCAS(&lkey[s], EMPTY, key); acc += (u32)o; }
          if (V == 8) { u64 o = atomicCAS(&lkey[s], EMPTY, key); if (o == EMPTY || o == key) atomicAdd(&lcnt[s], 1u); }
          if (V == 9) { lkey[s] = key; }
          if (V == 10) { u64 o = atomicCAS(&lkey[s], EMPTY, key); if (o == EMPTY || o == key) atomicAdd(&lcnt[s], (u32)(key >> 60) | 1u); }
        }
      }
    } else if (V == 3 || V == 4) {
      // vectorized: each thread owns KT keys (keys t, t+NT, ...); every round issues one probe for each
      // of its unfinished keys before looking at any result
      constexpr int KT = 4096 / NT;
      u64 kk[KT]; u32 ss[KT]; bool dn[KT];
#pragma unroll
      for (int i = 0; i < KT; ++i) {
        int e = i * NT + threadIdx.x;
        dn[i] = e >= n;
        kk[i] = dn[i] ? 0 : stage[e];
        ss[i] = (u32)((kk[i] * MUL) >> (64 - logB - 12)) & (TL - 1);
      }
      for (;;) {
        bool any = false;
        u64 cur[KT];
#pragma unroll
        for (int i = 0; i < KT; ++i) {
          if (!dn[i]) {
            if (V == 4) cur[i] = ((volatile u64*)lkey)[ss[i]];
            else cur[i] = atomicCAS(&lkey[ss[i]], EMPTY, kk[i]);
          }
        }
        if (V == 4) {
#pragma unroll
          for (int i = 0; i < KT; ++i)
            if (!dn[i] && cur[i] == EMPTY) cur[i] = atomicCAS(&lkey[ss[i]], EMPTY, kk[i]);
        }
#pragma unroll
        for (int i = 0; i < KT; ++i) {
          if (!dn[i]) {
            if (cur[i] == EMPTY || cur[i] == kk[i]) { atomicAdd(&lcnt[ss[i]], 1u); dn[i] = true; }
            else { ss[i] = (ss[i] + 1) & (TL - 1); any = true; }
          }
        }
        if (!__syncthreads_or(any)) break;
      }
    } else if (V == 2) {
      for (int b0 = wid * 64; b0 < n; b0 += NT * 2) {
        int e0 = b0 + lane, e1 = b0 + 32 + lane;
        u64 k0 = e0 < n ? stage[e0] : EMPTY, k1 = e1 < n ? stage[e1] : EMPTY;
        u32 s0 = (u32)((k0 * MUL) >> (64 - logB - 12)) & (TL - 1), s1 = (u32)((k1 * MUL) >> (64 - logB - 12)) & (TL - 1);
        u64 c0 = ((volatile u64*)lkey)[s0], c1 = ((volatile u64*)lkey)[s1];
        bool d0 = k0 == EMPTY, d1 = k1 == EMPTY;
        if (!d0 && c0 == k0) { atomicAdd(&lcnt[s0], 1u); d0 = true; }
        if (!d1 && c1 == k1) { atomicAdd(&lcnt[s1], 1u); d1 = true; }
        while (!d0) {
          u64 cur = ((volatile u64*)lkey)[s0];
          if (cur == k0) { atomicAdd(&lcnt[s0], 1u); break; }
          if (cur == EMPTY) { u64 o = atomicCAS(&lkey[s0], EMPTY, k0); if (o == EMPTY || o == k0) { atomicAdd(&lcnt[s0], 1u); break; } }
          s0 = (s0 + 1) & (TL - 1);
        }
        while (!d1) {
          u64 cur = ((volatile u64*)lkey)[s1];
          if (cur == k1) { atomicAdd(&lcnt[s1], 1u); break; }
          if (cur == EMPTY) { u64 o = atomicCAS(&lkey[s1], EMPTY, k1); if (o == EMPTY || o == k1) { atomicAdd(&lcnt[s1], 1u); break; } }
          s1 = (s1 + 1) & (TL - 1);
        }
      }
    } else {
      for (int b0 = wid * 32; b0 < n; b0 += NT) {
        int e = b0 + lane;
        if (e < n) {
          u64 key = stage[e];
          u32 s = (u32)((key * MUL) >> (64 - logB - 12)) & (TL - 1);
          for (;;) {
            if (V == 1) {
              u64 cur = ((volatile u64*)lkey)[s];
              if (cur == key) { atomicAdd(&lcnt[s], 1u); break; }
              if (cur != EMPTY) { s = (s + 1) & (TL - 1); continue; }
            }
            u64 o = atomicCAS(&lkey[s], EMPTY, key);
            if (o == EMPTY || o == key) { atomicAdd(&lcnt[s], 1u); break; }
            s = (s + 1) & (TL - 1);
          }
        }
      }
    }
    __syncthreads();
    long long t1 = clock64();
    for (int i = threadIdx.x; i < TL; i += NT) {
      u32 c = lcnt[i];
      if (c) { acc += c + (u32)lkey[i]; lkey[i] = EMPTY; lcnt[i] = 0; }
    }
    __syncthreads();
    long long t2 = clock64();
    tins += t1 - t0; tscan += t2 - t1;
  }
  if (threadIdx.x == 0) { cyc[blockIdx.x * 2] = tins; cyc[blockIdx.x * 2 + 1] = tscan; }
  if (acc == 12345) sink[0] = acc;
}

template <int V, int TL, int NT>
void run(const u64* dk, int n, int blocks, const char* name) {
  const int reps = 200;
  size_t smem = 4096 * 8 + TL * 12;
  CK(cudaFuncSetAttribute(k<V, TL, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  u64* cyc; u32* sink;
  CK(cudaMalloc(&cyc, blocks * 16)); CK(cudaMalloc(&sink, 4));
  k<V, TL, NT><<<blocks, NT, smem>>>(dk, n, reps, cyc, sink, 6);
  CK(cudaDeviceSynchronize());
  std::vector<u64> h(blocks * 2);
  CK(cudaMemcpy(h.data(), cyc, blocks * 16, cudaMemcpyDeviceToHost));
  double a = 0, b = 0;
  for (int i = 0; i < blocks; ++i) { a += h[2 * i]; b += h[2 * i + 1]; }
  a /= blocks * (double)reps; b /= blocks * (double)reps;
  printf("%-28s TL=%5d NT=%4d blocks=%4d: insert %7.0f cyc (%.2f cyc/key), scan %6.0f cyc\n", name, TL, NT, blocks, a, a / n, b);
  cudaFree(cyc); cudaFree(sink);
}

int main(int argc, char** argv) {
  FILE* f = fopen(argc > 1 ? argv[1] : "keys.bin", "rb");
  std::vector<u64> keys(1 << 16);
  int n = (int)fread(keys.data(), 8, keys.size(), f);
  fclose(f);
  printf("%d keys\n", n);
  u64* dk;
  CK(cudaMalloc(&dk, n * 8));
  CK(cudaMemcpy(dk, keys.data(), n * 8, cudaMemcpyHostToDevice));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<7, 4096, 512>(dk, n, sms, "single CAS only");
  run<8, 4096, 512>(dk, n, sms, "single CAS + INC");
  run<10, 4096, 512>(dk, n, sms, "single CAS + ADD(var)");
  run<9, 4096, 512>(dk, n, sms, "STS only");
  run<7, 4096, 1024>(dk, n, sms, "single CAS only 1024t");
  run<8, 4096, 1024>(dk, n, sms, "single CAS + INC 1024t");
  run<3, 4096, 512>(dk, n, sms, "vec CAS-first");
  run<4, 4096, 512>(dk, n, sms, "vec load-first");
  run<3, 4096, 256>(dk, n, sms, "vec CAS-first 256t");
  run<4, 4096, 256>(dk, n, sms, "vec load-first 256t");
  run<3, 4096, 256>(dk, n, 2 * sms, "vec CAS-first 256t 2cta");
  run<4, 4096, 256>(dk, n, 2 * sms, "vec load-first 256t 2cta");
  run<3, 4096, 1024>(dk, n, sms, "vec CAS-first 1024t");
  run<0, 4096, 512>(dk, n, sms, "CAS-first");
  run<1, 4096, 512>(dk, n, sms, "load-first");
  run<2, 4096, 512>(dk, n, sms, "load-first x2");
  run<0, 4096, 512>(dk, n, 2 * sms, "CAS-first 2cta");
  run<1, 4096, 512>(dk, n, 2 * sms, "load-first 2cta");
  run<0, 4096, 1024>(dk, n, sms, "CAS-first 1024t");
  run<1, 4096, 1024>(dk, n, sms, "load-first 1024t");
  run<0, 4096, 256>(dk, n, sms, "CAS-first 256t");
  run<1, 4096, 256>(dk, n, sms, "load-first 256t");
  return 0;
}
