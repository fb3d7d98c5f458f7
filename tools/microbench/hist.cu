// Design microbenchmark (not product code): per-warp "multisplit" positions for a small number of
// buckets (the side-bucket record layout of the L item) on B200 (sm_100a).
//   OP 0: atomicAdd(&h[b], 1) per lane (return value used: the record position)
//   OP 1: ballot peer masks over the bucket bits, one atomicAdd per distinct bucket (leader), shfl base
//   OP 2: like 0, but per-warp private counters
//   OP 3: __match_any_sync peers, leader atomicAdd, shfl
// Grid: 2 CTAs x 512 threads per SM (the product's shape).  Prints lane-ops per clock per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hist hist.cu
#include <cstdio>
#include <cstdint>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)
__device__ __forceinline__ uint32_t mixr(uint32_t x) { x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x; }
__device__ unsigned long long g_sink;

template <int OP>
__global__ void __launch_bounds__(512, 2) k(int iters, int logb, unsigned long long* cyc) {
  __shared__ uint32_t h[16 * 256];
  for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t acc = 0;
  uint32_t s = mixr(blockIdx.x * 512 + threadIdx.x + 1);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    s = mixr(s + it);
    const uint32_t b = s >> (32 - logb);
    uint32_t pos;
    if (OP == 0) pos = atomicAdd(&h[b], 1u);
    if (OP == 2) pos = atomicAdd(&h[wid * 256 + b], 1u);
    if (OP == 1 || OP == 3) {
      uint32_t peers;
      if (OP == 1) {
        peers = 0xffffffffu;
        for (int q = 0; q < logb; ++q) {
          const uint32_t bal = __ballot_sync(0xffffffffu, (b >> q) & 1u);
          peers &= ((b >> q) & 1u) ? bal : ~bal;
        }
      } else {
        peers = __match_any_sync(0xffffffffu, b);
      }
      const int leader = __ffs(peers) - 1;
      const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
      uint32_t base = 0;
      if (lane == leader) base = atomicAdd(&h[b], (uint32_t)__popc(peers));
      pos = __shfl_sync(0xffffffffu, base, leader) + rank;
    }
    acc += pos;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  if (acc == 0x12345) g_sink = acc;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  unsigned long long* cyc; CK(cudaMalloc(&cyc, 8));
  const int iters = 4096;
  for (int logb : {5, 6, 8}) {
    for (int op = 0; op < 4; ++op) {
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaMemset(cyc, 0, 8));
        if (op == 0) k<0><<<2 * sms, 512>>>(iters, logb, cyc);
        if (op == 1) k<1><<<2 * sms, 512>>>(iters, logb, cyc);
        if (op == 2) k<2><<<2 * sms, 512>>>(iters, logb, cyc);
        if (op == 3) k<3><<<2 * sms, 512>>>(iters, logb, cyc);
        CK(cudaDeviceSynchronize());
        unsigned long long c; CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
        const double cyc_per_cta = (double)c / (2 * sms);
        if (rep) printf("logb %d op %d: %.2f lane-ops/clk/SM (%.0f cyc per CTA)\n", logb, op, 2.0 * 512 * iters / cyc_per_cta, cyc_per_cta);
      }
    }
  }
  return 0;
}
