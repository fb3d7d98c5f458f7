// Design microbenchmark (not product code): bulk-copy bandwidth of the exchange options a
// cluster-based per-window design could use instead of the L2 scratch round trip:
//   (a) SMEM -> peer SMEM in the cluster  (cp.async.bulk.shared::cluster.shared::cta, mbarrier complete_tx)
//   (b) SMEM -> global (L2-resident)       (cp.async.bulk.global.shared::cta, bulk_group)
//   (c) global (L2-resident) -> SMEM       (cp.async.bulk.shared::cluster.global, mbarrier complete_tx)
// One CTA per SM; each round moves ROUND_BYTES per CTA in CHUNK-byte copies, rounds separated by a
// cluster barrier (a) or a bulk wait / mbarrier wait (b, c).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk bulk.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int BUF = 64 * 1024;      // source and destination buffers per CTA
constexpr int CHUNK = 8 * 1024;
constexpr int ROUND_BYTES = 128 * 1024;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// (a) every CTA sends ROUND_BYTES per round to the next rank of its cluster
__global__ void k_dsmem_bulk(int rounds, unsigned long long* cyc) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* src = sm;
  unsigned char* dst = sm + BUF;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 2 * BUF);
  cg::cluster_group cl = cg::this_cluster();
  const unsigned C = cl.num_blocks(), r = cl.block_rank(), peer = (r + 1) % C;
  for (int i = threadIdx.x; i < BUF; i += blockDim.x) src[i] = (unsigned char)i;
  if (threadIdx.x == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  cl.sync();
  uint32_t rdst, rbar;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(smem_u32(dst)), "r"(peer));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(bar)), "r"(peer));
  long long t0 = clock64();
  for (int it = 0; it < rounds; ++it) {
    if (threadIdx.x == 0) mbar_expect(bar, ROUND_BYTES);  // what the previous rank will send here
    cl.sync();                                             // every receiver is armed
    if (threadIdx.x == 0) {
      for (int off = 0; off < ROUND_BYTES; off += CHUNK)
        asm volatile(
            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                rdst + (off % BUF)),
            "r"(smem_u32(src + (off % BUF))), "r"(CHUNK), "r"(rbar)
            : "memory");
    }
    if (threadIdx.x == 0) mbar_wait(bar, it & 1);
    __syncthreads();
  }
  cl.sync();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

// (b) SMEM -> global, (c) global -> SMEM, each CTA on its own 128 KB region of an L2-resident buffer
__global__ void k_global_bulk(int rounds, int dir, unsigned char* g, unsigned long long* cyc) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 2 * BUF);
  unsigned char* mine = g + (size_t)blockIdx.x * ROUND_BYTES;
  for (int i = threadIdx.x; i < 2 * BUF; i += blockDim.x) sm[i] = (unsigned char)i;
  if (threadIdx.x == 0) { mbar_init(bar, 1); asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < rounds; ++it) {
    if (threadIdx.x == 0) {
      if (dir == 0) {
        for (int off = 0; off < ROUND_BYTES; off += CHUNK)
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(mine + off),
                       "r"(smem_u32(sm + (off % (2 * BUF)))), "r"(CHUNK)
                       : "memory");
        asm volatile("cp.async.bulk.commit_group;\n cp.async.bulk.wait_group 0;" ::: "memory");
      } else {
        mbar_expect(bar, ROUND_BYTES);
        for (int off = 0; off < ROUND_BYTES; off += CHUNK)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(sm + (off % (2 * BUF)))),
              "l"(mine + off), "r"(CHUNK), "r"(smem_u32(bar))
              : "memory");
        mbar_wait(bar, it & 1);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  int sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  const size_t smem = 2 * BUF + 64;
  CK(cudaFuncSetAttribute(k_dsmem_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_dsmem_bulk, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(k_global_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  unsigned long long* cyc;
  CK(cudaMalloc(&cyc, 1024 * sizeof(unsigned long long)));
  unsigned long long hc[1024];
  const int rounds = 2000;
  for (int C : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem; cfg.attrs = attr; cfg.numAttrs = 1;
    int nclusters = 0;
    cfg.gridDim = dim3(C);
    CK(cudaOccupancyMaxActiveClusters(&nclusters, k_dsmem_bulk, &cfg));
    cfg.gridDim = dim3(nclusters * C);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    CK(cudaLaunchKernelEx(&cfg, k_dsmem_bulk, 10, cyc));
    CK(cudaEventRecord(a));
    CK(cudaLaunchKernelEx(&cfg, k_dsmem_bulk, rounds, cyc));
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0; CK(cudaEventElapsedTime(&ms, a, b));
    const double bytes = (double)nclusters * C * rounds * ROUND_BYTES;
    CK(cudaMemcpy(hc, cyc, sizeof(unsigned long long) * nclusters * C, cudaMemcpyDeviceToHost));
    printf("DSMEM bulk C=%2d: %3d clusters (%3d SMs)  %8.1f GB/s chip  %6.1f B/clk/SM  (cycles/CTA %llu)\n", C,
           nclusters, nclusters * C, bytes / ms / 1e6, bytes / (nclusters * C) / ((double)ms * 1e-3 * clk * 1e3), hc[0]);
  }
  unsigned char* g;
  CK(cudaMalloc(&g, (size_t)sms * ROUND_BYTES));
  for (int dir = 0; dir < 2; ++dir) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    k_global_bulk<<<sms, 128, smem>>>(10, dir, g, cyc);
    CK(cudaEventRecord(a));
    k_global_bulk<<<sms, 128, smem>>>(rounds, dir, g, cyc);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0; CK(cudaEventElapsedTime(&ms, a, b));
    const double bytes = (double)sms * rounds * ROUND_BYTES;
    printf("%s: %8.1f GB/s chip  %6.1f B/clk/SM (L2-resident %d x 128 KB)\n",
           dir == 0 ? "SMEM->global bulk" : "global->SMEM bulk", bytes / ms / 1e6,
           bytes / sms / ((double)ms * 1e-3 * clk * 1e3), sms);
  }
  printf("done\n");
  return 0;
}
