// Design microbenchmark (not product code): SMEM operation costs on B200 per warp-instruction, with
// the success/failure and address patterns a hash insert actually produces.
//   cycles per warp-instruction = total cycles / (warps x iterations), 32 lanes, random slots in a
//   table of 4096 entries unless noted.  1 CTA per SM, NW warps.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atoms atoms.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
typedef unsigned long long u64;
typedef uint32_t u32;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ u32 mix(u32 x) { x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x; }
__device__ u64 g_sink;

// OP: 0 CAS64 success (fresh table each iteration region), 1 CAS64 fail, 2 CAS32 success, 3 CAS32 fail,
//     4 ADD32 ret, 5 ADD32 red, 6 INC32 (+1, unused ret), 7 LDS64, 8 STS64, 9 ADD64 red, 10 EXCH64,
//     11 CAS64 success same-bank-free (lane-distinct columns), 12 LDS64+CAS64 (load-first on fresh)
template <int OP>
__global__ void k(int iters, int nw_active, u64* out) {
  extern __shared__ __align__(16) u64 tab[];  // 8192 u64 (64 KB)
  const int NS = 8192;
  for (int i = threadIdx.x; i < NS; i += blockDim.x) tab[i] = (OP == 1 || OP == 3) ? 0x5555ull : ~0ull;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  u64 acc = 0;
  long long t0 = clock64();
  if (wid < nw_active) {
    u32 s = mix(blockIdx.x * 4096 + threadIdx.x * 7 + 1);
    for (int it = 0; it < iters; ++it) {
      s = mix(s + it);
      u32 idx = s & (NS - 1);
      if (OP == 11) idx = ((s >> 5) & (NS / 32 - 1)) * 32 + lane;  // column = lane: conflict-free
      u64 key = ((u64)s << 32) | (u32)(it * 977 + threadIdx.x);
      if (OP == 0 || OP == 11) { u64 o = atomicCAS(&tab[idx], ~0ull, key); acc += o; tab[idx] = ~0ull; }
      if (OP == 1) acc += atomicCAS(&tab[idx], ~0ull, key);
      if (OP == 2) { u32* t = (u32*)tab; u32 o = atomicCAS(&t[idx], ~0u, (u32)key); acc += o; t[idx] = ~0u; }
      if (OP == 3) { u32* t = (u32*)tab; acc += atomicCAS(&t[idx], ~0u, (u32)key); }
      if (OP == 4) { u32* t = (u32*)tab; acc += atomicAdd(&t[idx], 1u + (s & 3)); }
      if (OP == 5) { u32* t = (u32*)tab; atomicAdd(&t[idx], 1u + (s & 3)); }
      if (OP == 6) { u32* t = (u32*)tab; atomicAdd(&t[idx], 1u); }
      if (OP == 7) acc += ((volatile u64*)tab)[idx];
      if (OP == 8) ((volatile u64*)tab)[idx] = key;
      if (OP == 9) atomicAdd(&tab[idx], (u64)(1 + (s & 3)));
      if (OP == 10) acc += atomicExch(&tab[idx], key);
      if (OP == 12) { u64 c = ((volatile u64*)tab)[idx]; if (c == ~0ull) { u64 o = atomicCAS(&tab[idx], ~0ull, key); acc += o; } tab[idx] = ~0ull; }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 42) g_sink = acc;
}

template <int OP>
void run(const char* name, int nw, int sms) {
  const int iters = 256;
  u64* out; CK(cudaMalloc(&out, sms * 8));
  CK(cudaFuncSetAttribute(k<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  k<OP><<<sms, nw * 32, 65536>>>(iters, nw, out);
  CK(cudaDeviceSynchronize());
  u64 h[1024]; CK(cudaMemcpy(h, out, sms * 8, cudaMemcpyDeviceToHost));
  double a = 0; for (int i = 0; i < sms; ++i) a += h[i];
  a /= sms;
  printf("%-34s warps=%2d: %7.1f cyc per warp-instr (SM throughput), %6.2f lanes/clk\n", name, nw, a / iters / nw * 1.0 * 1, 32.0 * nw * iters / a);
  cudaFree(out);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int nw : {1, 16, 32}) {
    run<0>("CAS64 success (+STS reset)", nw, sms);
    run<1>("CAS64 fail", nw, sms);
    run<11>("CAS64 success, lane columns", nw, sms);
    run<12>("LDS64 then CAS64 success (+STS)", nw, sms);
    run<2>("CAS32 success (+STS reset)", nw, sms);
    run<3>("CAS32 fail", nw, sms);
    run<4>("ADD32 with return", nw, sms);
    run<5>("ADD32 no return (RED)", nw, sms);
    run<6>("INC32 (+1, no return)", nw, sms);
    run<7>("LDS64 random", nw, sms);
    run<8>("STS64 random", nw, sms);
    run<9>("ADD64 RED", nw, sms);
    run<10>("EXCH64", nw, sms);
  }
  return 0;
}
