// Design microbenchmark (not product code): throughput of the memory operations a
// per-window hash group-by can be built from on B200 (sm_100a).
//   SMEM atomics (local), DSMEM atomics/stores (cluster remote), L2 atomics, HBM stream read,
//   __match_any_sync on u64.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomics atomics.cu
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t lcg(uint32_t& s) { s = s * 1664525u + 1013904223u; return s; }
__device__ __forceinline__ uint32_t mixr(uint32_t x) { x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x; }

__device__ unsigned long long g_sink;

// ---------------- SMEM local ----------------
template <int OP>
__global__ void __launch_bounds__(1024) k_smem(int iters, unsigned long long* cyc) {
  extern __shared__ unsigned long long tab[];
  const int NS = 16384;  // 128 KB of u64
  for (int i = threadIdx.x; i < NS; i += blockDim.x) tab[i] = 0x1234567800000000ull + i;
  __syncthreads();
  uint32_t s = mixr(blockIdx.x * 1024 + threadIdx.x + 1);
  unsigned long long acc = 0;
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < iters; ++it) {
    uint32_t r = lcg(s);
    int idx = (r >> 8) & (NS - 1);
    if (OP == 0) acc += atomicCAS(&tab[idx], 0ull, (unsigned long long)r);
    if (OP == 1) atomicAdd(((unsigned int*)tab) + 2 * idx, 1u);
    if (OP == 2) atomicAdd(&tab[idx], 1ull);
    if (OP == 3) acc += atomicAdd(((unsigned int*)tab) + 2 * idx, 1u);
    if (OP == 4) { tab[idx] += 1; }
    if (OP == 5) acc += tab[idx];
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 42) g_sink = acc;
  if (threadIdx.x == 0) g_sink += tab[threadIdx.x];
}

// ---------------- DSMEM remote ----------------
template <int OP>
__global__ void __launch_bounds__(1024) k_dsmem(int iters, unsigned long long* cyc) {
  extern __shared__ unsigned long long tab[];
  cg::cluster_group cl = cg::this_cluster();
  const int NS = 16384;
  for (int i = threadIdx.x; i < NS; i += blockDim.x) tab[i] = 0x1234567800000000ull + i;
  cl.sync();
  const unsigned C = cl.num_blocks();
  unsigned long long* rt[16];
  for (unsigned r = 0; r < C; ++r) rt[r] = cl.map_shared_rank(tab, r);
  uint32_t s = mixr(blockIdx.x * 1024 + threadIdx.x + 1);
  unsigned long long acc = 0;
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < iters; ++it) {
    uint32_t r = lcg(s);
    int idx = (r >> 8) & (NS - 1);
    unsigned long long* t = rt[(r >> 24) % C];
    if (OP == 0) acc += atomicCAS(&t[idx], 0ull, (unsigned long long)r);
    if (OP == 1) atomicAdd(((unsigned int*)t) + 2 * idx, 1u);
    if (OP == 2) t[idx] = r;
    if (OP == 3) acc += atomicAdd(((unsigned int*)t) + 2 * idx, 1u);
  }
  long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 42) g_sink = acc;
}

// ---------------- global / L2 ----------------
template <int OP>
__global__ void __launch_bounds__(512) k_gmem(unsigned long long* tab, int mask, int iters) {
  uint32_t s = mixr(blockIdx.x * 1024 + threadIdx.x + 7);
  unsigned long long acc = 0;
#pragma unroll 4
  for (int it = 0; it < iters; ++it) {
    uint32_t r = lcg(s);
    uint32_t r2 = mixr(r);
    int idx = r2 & mask;
    if (OP == 0) acc += atomicCAS(&tab[idx], 0ull, (unsigned long long)r);
    if (OP == 1) atomicAdd(((unsigned int*)tab) + 2 * idx, 1u);
    if (OP == 2) acc += atomicAdd(&tab[idx], 1ull);
    if (OP == 3) acc += tab[idx];
  }
  if (acc == 42) g_sink = acc;
}

// ---------------- HBM stream read ----------------
__global__ void __launch_bounds__(512) k_read(const uint4* __restrict__ p, size_t n16, unsigned long long* out) {
  uint32_t x = 0;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
#pragma unroll 8
  for (; i < n16; i += stride) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
    x ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (x == 0x12345678) out[0] = x;
}

// ---------------- match_any u64 ----------------
__global__ void __launch_bounds__(1024) k_match(int iters, unsigned long long* cyc) {
  uint32_t s = mixr(blockIdx.x * 1024 + threadIdx.x + 3);
  unsigned acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r = lcg(s);
    unsigned long long k = (unsigned long long)(r & 0xF0) << 32 | (r & 0x7);
    acc += __match_any_sync(0xffffffffu, k);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 42) g_sink = acc;
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) { float ms; CK(cudaEventElapsedTime(&ms, a, b)); return ms; }

template <typename F>
static float bench(F f, int reps = 5) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) { CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); float t = time_ms(a, b); if (t < best) best = t; }
  CK(cudaGetLastError());
  return best;
}

static double avg_cyc(unsigned long long* d, int n) {
  static unsigned long long h[4096]; CK(cudaMemcpy(h, d, n * 8, cudaMemcpyDeviceToHost));
  double s = 0; for (int i = 0; i < n; ++i) s += h[i]; return s / n;
}

template <int OP>
static void run_dsmem(int C, int nsm, unsigned long long* cyc, const char* name) {
  auto kern = k_dsmem<OP>;
  int smem = 16384 * 8;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  if (C > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = smem;
  int maxc = 0;
  cfg.gridDim = dim3(C * 64);
  CK(cudaOccupancyMaxActiveClusters(&maxc, kern, &cfg));
  int grid = maxc * C;
  cfg.gridDim = dim3(grid);
  int iters = 2048;
  float ms = bench([&] { CK(cudaLaunchKernelEx(&cfg, kern, iters, cyc)); });
  double ops = (double)grid * 1024 * iters;
  double c = avg_cyc(cyc, grid);
  printf("DSMEM C=%2d %-22s maxActiveClusters=%3d (SMs used %3d): %8.1f Gop/s chip, %6.2f lane-ops/clk/SM (cycles/CTA %.0f)\n",
         C, name, maxc, grid, ops / ms / 1e6, (1024.0 * iters) / c, c);
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int nsm = p.multiProcessorCount;
  int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  int smemOptin; CK(cudaDeviceGetAttribute(&smemOptin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  printf("device %s SMs=%d clockRate=%d kHz smemOptin=%d L2=%d\n", p.name, nsm, clk, smemOptin, p.l2CacheSize);
  unsigned long long* cyc; CK(cudaMalloc(&cyc, 4096 * 8));

  // SMEM local
  {
    int iters = 4096, smem = 16384 * 8;
    const char* names[] = {"atomicCAS u64", "atomicAdd u32 (RED)", "atomicAdd u64 (RED)", "atomicAdd u32 (ret)", "ld+st u64 (nonatomic)", "ld u64"};
#define SM1(OP) { auto k = k_smem<OP>; CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
      float ms = bench([&]{ k<<<nsm, 1024, smem>>>(iters, cyc); }); double ops = (double)nsm * 1024 * iters; double c = avg_cyc(cyc, nsm); \
      printf("SMEM  %-24s: %8.1f Gop/s chip, %6.2f lane-ops/clk/SM (cycles/CTA %.0f)\n", names[OP], ops / ms / 1e6, 1024.0 * iters / c, c); }
    SM1(0) SM1(1) SM1(2) SM1(3) SM1(4) SM1(5)
  }
  // DSMEM
  for (int C : {2, 4, 8, 16}) {
    run_dsmem<0>(C, nsm, cyc, "atomicCAS u64");
    run_dsmem<1>(C, nsm, cyc, "atomicAdd u32 (RED)");
    run_dsmem<2>(C, nsm, cyc, "st u64");
    run_dsmem<3>(C, nsm, cyc, "atomicAdd u32 (ret)");
  }
  // global
  {
    size_t slots = 1 << 24;  // 128 MB table, and a 8 MB one
    unsigned long long* tab; CK(cudaMalloc(&tab, slots * 8)); CK(cudaMemset(tab, 0x11, slots * 8));
    for (int lg : {20, 24}) {
      int mask = (1 << lg) - 1; int iters = 256; int grid = nsm * 4;
      const char* names[] = {"atomicCAS u64", "atomicAdd u32 (RED)", "atomicAdd u64 (ret)", "ld u64"};
#define G1(OP) { float ms = bench([&]{ k_gmem<OP><<<grid, 512>>>(tab, mask, iters); }); double ops = (double)grid * 512 * iters; \
      printf("GMEM table 2^%d x8B %-22s: %8.1f Gop/s chip\n", lg, names[OP], ops / ms / 1e6); }
      G1(0) G1(1) G1(2) G1(3)
    }
    CK(cudaFree(tab));
  }
  // HBM read
  {
    size_t bytes = 4ull << 30;
    uint4* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
    for (int bpsm : {2, 4, 8}) {
      int grid = nsm * bpsm;
      float ms = bench([&]{ k_read<<<grid, 512>>>(buf, bytes / 16, cyc); });
      printf("HBM read 4 GiB grid=%d x512: %.1f GB/s\n", grid, bytes / ms / 1e6);
    }
    CK(cudaFree(buf));
  }
  // match_any
  {
    int iters = 4096;
    float ms = bench([&]{ k_match<<<nsm, 1024>>>(iters, cyc); });
    double c = avg_cyc(cyc, nsm);
    printf("match_any u64: %.1f Gwarp-op/s chip, %.3f warp-ops/clk/SM\n", (double)nsm * 32 * iters / ms / 1e6, 32.0 * iters / c);
  }
  printf("done\n");
  return 0;
}
