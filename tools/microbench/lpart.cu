// Design microbenchmark (not product code): the link-bucket insert of nsg_win.cuh built up piece by
// piece, to attribute its cycles.  One real C2 bucket per CTA (keys file), 512 threads, 1 CTA per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include -I../../paper_2509_03653_b200/csrc -o lpart lpart.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "nsg_win.cuh"
using namespace nsg;
using namespace nsg::win;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int V>
__device__ __forceinline__ void lpart(Smem& s, const u64* stage, u32 n, u32 logB, u32* ncl, u32* sink) {
  const int t = threadIdx.x;
  u64 k[KW], cur[KW];
  u32 sl[KW];
  u32 vmask = 0;
#pragma unroll
  for (int i = 0; i < KW; ++i) { const u32 e = i * NCT + t; k[i] = e < n ? stage[e] : 0ull; }
#pragma unroll
  for (int i = 0; i < KW; ++i) { if (i * NCT + t < n) vmask |= 1u << i; sl[i] = link_slot(k[i], logB); }
  if (V == 0) {  // loads of the home slots only
#pragma unroll
    for (int i = 0; i < KW; ++i) cur[i] = (vmask >> i & 1u) ? *reinterpret_cast<volatile u64*>(&s.lkey[sl[i]]) : 0ull;
    u32 x = 0;
#pragma unroll
    for (int i = 0; i < KW; ++i) x += (u32)cur[i];
    if (x == 0x12345) *sink = x;
    return;
  }
  if (V == 5) {  // CAS-first, no load
    u32 wmask = 0;
#pragma unroll
    for (int i = 0; i < KW; ++i)
      if (vmask >> i & 1u) cur[i] = atomicCAS(reinterpret_cast<unsigned long long*>(&s.lkey[sl[i]]), (unsigned long long)EMPTY64, (unsigned long long)k[i]);
#pragma unroll
    for (int i = 0; i < KW; ++i)
      if ((vmask >> i & 1u) && (cur[i] == EMPTY64 || cur[i] == k[i])) { atomicAdd(&s.lcnt[sl[i]], 1u); wmask |= (cur[i] == EMPTY64) << i; }
    u32 pw = warp_reserve(__popc(wmask), ncl);
#pragma unroll
    for (int i = 0; i < KW; ++i) if (wmask >> i & 1u) s.claim[pw++] = (uint16_t)sl[i];
    return;
  }
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
  if (V == 6) {  // vectorised probe steps, double hashing: step = odd, from other hash bits
    u32 st[KW];
#pragma unroll
    for (int i = 0; i < KW; ++i) st[i] = ((u32)(k[i] * MUL_L) >> 7) | 1u;
    for (u32 step = 1; __any_sync(0xffffffffu, pmask != 0); ++step) {
#pragma unroll
      for (int i = 0; i < KW; ++i) if (pmask >> i & 1u) cur[i] = *reinterpret_cast<volatile u64*>(&s.lkey[(sl[i] + step * st[i]) & (TL - 1)]);
#pragma unroll
      for (int i = 0; i < KW; ++i) {
        if (pmask >> i & 1u) {
          const u32 q = (sl[i] + step * st[i]) & (TL - 1);
          const u32 r = link_try(s, k[i], q, cur[i]);
          if (r) { pmask &= ~(1u << i); if (r == 2) wmask |= 1u << i; }
        }
      }
      if (step > 64) break;
    }
  }
  if (V == 4) {  // vectorised probe steps for the failed keys
    for (u32 step = 1; __any_sync(0xffffffffu, pmask != 0); ++step) {
#pragma unroll
      for (int i = 0; i < KW; ++i) if (pmask >> i & 1u) cur[i] = *reinterpret_cast<volatile u64*>(&s.lkey[(sl[i] + step) & (TL - 1)]);
#pragma unroll
      for (int i = 0; i < KW; ++i) {
        if (pmask >> i & 1u) {
          const u32 q = (sl[i] + step) & (TL - 1);
          const u32 r = link_try(s, k[i], q, cur[i]);
          if (r) { pmask &= ~(1u << i); sl[i] = q - step; if (r == 2) wmask |= 1u << i; }
        }
      }
      if (step > 64) break;
    }
  }
  if (V == 3) {
#pragma unroll 1
    for (u32 m = pmask; m; m &= m - 1) {
      const int i = __ffs(m) - 1;
      u32 slot = 0; u64 key = 0, home = 0;
#pragma unroll
      for (int q = 0; q < KW; ++q) if (q == i) { key = k[q]; home = sl[q]; }
      const u32 r = link_probe_on(s, key, (u32)home, &slot);
#pragma unroll
      for (int q = 0; q < KW; ++q) if (q == i) sl[q] = slot;
      if (r == 2) wmask |= 1u << i;
    }
  }
  if (V >= 2) {
    u32 pw = warp_reserve(__popc(wmask), ncl);
#pragma unroll
    for (int i = 0; i < KW; ++i) if (wmask >> i & 1u) s.claim[pw++] = (uint16_t)sl[i];
  }
}

__device__ unsigned long long g_w[8][3];
template <int V>
__global__ void __launch_bounds__(NCT, 1) kl(const u64* keys, int n, int reps, unsigned long long* cyc) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int t = threadIdx.x;
  __shared__ u32 sink;
  for (u32 i = t; i < (u32)TL; i += NCT) { s.lkey[i] = EMPTY64; s.lcnt[i] = 0; }
  for (int i = t; i < n; i += NCT) s.stage[0][i] = keys[i];
  if (t == 0) s.ncl[0][0] = 0;
  __syncthreads();
  unsigned long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    cbar();
    long long t0 = clock64();
    lpart<V>(s, s.stage[0], n, 6, &s.ncl[0][0], &sink);
    long long tw = clock64() - t0;
    if ((t & 31) == 0) { atomicAdd(&g_w[V][0], (unsigned long long)tw); atomicMax(&g_w[V][1], (unsigned long long)tw); }
    cbar();
    tot += clock64() - t0;
    // clean the table for the next rep (not timed)
    for (u32 i = t; i < (u32)TL; i += NCT) { s.lkey[i] = EMPTY64; s.lcnt[i] = 0; }
    if (t == 0) s.ncl[0][0] = 0;
    cbar();
  }
  if (t == 0) cyc[blockIdx.x] = tot;
}

template <int V>
void run(const u64* dk, int n, int sms, const char* nm) {
  unsigned long long* cyc; CK(cudaMalloc(&cyc, sms * 8));
  CK(cudaFuncSetAttribute(kl<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem)));
  const int reps = 50;
  kl<V><<<sms, NCT, sizeof(Smem)>>>(dk, n, reps, cyc);
  CK(cudaDeviceSynchronize());
  std::vector<unsigned long long> h(sms); CK(cudaMemcpy(h.data(), cyc, sms * 8, cudaMemcpyDeviceToHost));
  unsigned long long w[8][3]; CK(cudaMemcpyFromSymbol(w, g_w, sizeof(w)));
  double a = 0; for (auto x : h) a += x; a /= sms * (double)reps;
  printf("%-34s %7.0f cyc (warp mean %.0f, max %llu)\n", nm, a, (double)w[V][0] / ((double)sms * reps * NCW), w[V][1]);
  cudaFree(cyc);
}

int main(int argc, char** argv) {
  FILE* f = fopen(argc > 1 ? argv[1] : "keys_med.bin", "rb");
  std::vector<u64> keys(1 << 16);
  int n = (int)fread(keys.data(), 8, keys.size(), f); fclose(f);
  if (n > SK) n = SK;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  u64* dk; CK(cudaMalloc(&dk, n * 8)); CK(cudaMemcpy(dk, keys.data(), n * 8, cudaMemcpyHostToDevice));
  printf("n = %d\n", n);
  run<0>(dk, n, sms, "V0 home loads only");
  run<1>(dk, n, sms, "V1 + INC / CAS (no collisions)");
  run<2>(dk, n, sms, "V2 + claim list");
  run<3>(dk, n, sms, "V3 + collision probing (full)");
  run<5>(dk, n, sms, "V5 CAS-first + claim (no coll.)");
  run<4>(dk, n, sms, "V4 vectorised probe steps");
  run<6>(dk, n, sms, "V6 vectorised double hashing");
  return 0;
}
