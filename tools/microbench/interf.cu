// Design microbenchmark (not product code): does a concurrent global->SMEM gather (cp.async 8 B, as
// the producer warps issue) or a TMA bulk copy slow down an SMEM CAS insert wave of other warps?
// 16 "consumer" warps run the single-CAS insert wave on a 2048-key stage; 4 "producer" warps either
// idle, issue cp.async.ca 8-byte gathers, or issue cp.async.bulk copies, from an L2-resident buffer.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o interf interf.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
typedef unsigned long long u64;
typedef uint32_t u32;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
constexpr u64 EMPTY = ~0ull;
constexpr u64 MUL = 0x9E3779B97F4A7C15ull;
__device__ __forceinline__ u32 sa(const void* p) { return (u32)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(640) k(const u64* keys, int n, const u64* gbuf, int reps, u64* cyc, volatile int* stop) {
  extern __shared__ __align__(128) unsigned char sm[];
  u64* stage = (u64*)sm;                 // 32 KB
  u64* lkey = stage + 4096;              // 32 KB
  u32* lcnt = (u32*)(lkey + 4096);       // 16 KB
  u64* pbuf = (u64*)(lcnt + 4096);       // 4 x 16 KB producer buffers
  __shared__ __align__(8) u64 mb[4];
  __shared__ int done_flag;
  const int t = threadIdx.x, wid = t >> 5, lane = t & 31;
  for (int i = t; i < n; i += 640) stage[i] = keys[i];
  for (int i = t; i < 4096; i += 640) { lkey[i] = EMPTY; lcnt[i] = 0; }
  if (t < 4) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&mb[t])));
  if (t == 0) done_flag = 0;
  __syncthreads();
  if (wid < 16) {
    long long tot = 0;
    for (int r = 0; r < reps; ++r) {
      asm volatile("bar.sync 1, 512;");
      long long t0 = clock64();
      for (int b0 = wid * 32; b0 < n; b0 += 512) {
        int e = b0 + lane;
        if (e < n) {
          u64 key = stage[e];
          u32 s = (u32)((key * MUL) >> 46) & 4095;
          u64 o = atomicCAS(&lkey[s], EMPTY, key);
          if (o == EMPTY || o == key) atomicAdd(&lcnt[s], 1u);
        }
      }
      asm volatile("bar.sync 1, 512;");
      tot += clock64() - t0;
      for (int i = t; i < 4096; i += 512) if (lcnt[i]) { lkey[i] = EMPTY; lcnt[i] = 0; }
    }
    if (t == 0) { cyc[blockIdx.x] = tot; done_flag = 1; }
  } else if (MODE != 0) {
    const int j = wid - 16;
    u64* dst = pbuf + j * 2048;
    u32 ph = 0;
    const u64* src = gbuf + (size_t)(blockIdx.x * 4 + j) * 65536;
    int it = 0;
    while (!*(volatile int*)&done_flag) {
      const u64* s0 = src + ((it * 2048) & 65535);
      if (MODE == 1) {  // cp.async 8 B, lane-parallel, 2048 elements
        for (int e = lane; e < 2048; e += 32)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa(dst + e)), "l"(s0 + e) : "memory");
        asm volatile("cp.async.wait_all;" ::: "memory");
      } else {  // one bulk copy of 16 KB
        if (lane == 0) {
          asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(sa(&mb[j])), "r"(16384) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)), "l"(s0), "r"(16384), "r"(sa(&mb[j])) : "memory");
          u32 ok = 0;
          while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(sa(&mb[j])), "r"(ph) : "memory");
          ph ^= 1;
        }
        __syncwarp();
      }
      ++it;
    }
  }
}

template <int MODE>
void run(const u64* dk, int n, const u64* gb, int sms, const char* name) {
  u64* cyc; CK(cudaMalloc(&cyc, sms * 8));
  const int smem = 32768 + 32768 + 16384 + 65536;
  CK(cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int reps = 100;
  k<MODE><<<sms, 640, smem>>>(dk, n, gb, reps, cyc, nullptr);
  CK(cudaDeviceSynchronize());
  std::vector<u64> h(sms); CK(cudaMemcpy(h.data(), cyc, sms * 8, cudaMemcpyDeviceToHost));
  double a = 0; for (auto x : h) a += x; a /= sms * (double)reps;
  printf("%-40s insert wave %7.0f cyc (%.2f cyc/key)\n", name, a, a / n);
  cudaFree(cyc);
}

int main(int argc, char** argv) {
  FILE* f = fopen(argc > 1 ? argv[1] : "keys_med.bin", "rb");
  std::vector<u64> keys(1 << 16);
  int n = (int)fread(keys.data(), 8, keys.size(), f); fclose(f);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  u64 *dk, *gb;
  CK(cudaMalloc(&dk, n * 8)); CK(cudaMemcpy(dk, keys.data(), n * 8, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&gb, (size_t)sms * 4 * 65536 * 8));  // 8 B x 64 Ki per producer: 296 MB... L2-resident per SM slice: no
  CK(cudaMemset(gb, 1, (size_t)sms * 4 * 65536 * 8));
  run<0>(dk, n, gb, sms, "producers idle");
  run<1>(dk, n, gb, sms, "producers cp.async 8B gathers");
  run<2>(dk, n, gb, sms, "producers bulk copies 16KB");
  return 0;
}
