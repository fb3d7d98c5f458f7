// Design microbenchmark (not product code): latency of k independent SMEM atomics issued back to back
// by one warp (k = 1, 2, 4, 8), conflict-free addresses.  Tells whether a warp pipelines its
// outstanding ATOMS / LDS or serialises them.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mlp mlp.cu
#include <cstdio>
#include <cstdint>
typedef unsigned long long u64;
typedef uint32_t u32;
__device__ u64 g_sink;
template <int K, int OP>
__global__ void k(int iters, u64* out) {
  __shared__ u64 tab[4096];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) tab[i] = ~0ull;
  __syncthreads();
  u64 acc = 0;
  u32 base = lane;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    u64 r[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      u32 idx = (base + j * 32 * 7 + (u32)acc * 0) & 4095;
      if (OP == 0) r[j] = atomicCAS(&tab[idx], 5ull, 6ull);          // fails: value unchanged
      if (OP == 1) r[j] = atomicAdd((u32*)&tab[idx], 0u);
      if (OP == 2) r[j] = ((volatile u64*)tab)[idx];
    }
#pragma unroll
    for (int j = 0; j < K; ++j) acc += r[j];
    base = (base + 32 * 13 + (u32)(acc & 1)) & 4095;                  // next batch depends on the results
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 42) g_sink = acc;
}
template <int K, int OP> void run(const char* nm) {
  u64* o; cudaMalloc(&o, 8);
  k<K, OP><<<1, 32>>>(1000, o); cudaDeviceSynchronize();
  u64 h; cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
  printf("%-6s K=%d: %6.1f cycles per batch (%5.1f per op)\n", nm, K, h / 1000.0, h / 1000.0 / K);
  cudaFree(o);
}
int main() {
  run<1, 0>("CAS64"); run<2, 0>("CAS64"); run<4, 0>("CAS64"); run<8, 0>("CAS64");
  run<1, 1>("ADD32"); run<2, 1>("ADD32"); run<4, 1>("ADD32"); run<8, 1>("ADD32");
  run<1, 2>("LDS64"); run<2, 2>("LDS64"); run<4, 2>("LDS64"); run<8, 2>("LDS64");
  return 0;
}
