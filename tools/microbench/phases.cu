// Design microbenchmark (not product code): cycles of the per-window kernel's consumer phases
// (nsg_win.cuh cons_P / cons_L_part / cons_L_final / cons_S_part / cons_S_final), run in isolation on one
// real C2 link bucket per CTA (keys file), one CTA per SM, consumer threads only.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include -I../../paper_2509_03653_b200/csrc -o phases phases.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "nsg_win.cuh"
using namespace nsg;
using namespace nsg::win;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ unsigned g_leaks;
__device__ unsigned long long g_wsum, g_wmax, g_wmin = ~0ull;
__global__ void __launch_bounds__(NCT, 1) kph(WGeo g, const u64* keys, int n, const u64* chunk, int reps, unsigned long long* cyc) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int t = threadIdx.x;
  for (u32 i = t; i < (u32)TL; i += NCT) { s.lkey[i] = EMPTY64; s.lcnt[i] = 0; }
  for (u32 i = t; i < (u32)TS; i += NCT) { s.nkey[i] = EMPTY32; s.npf[i] = 0; }
  for (u32 i = t; i < 4 * MAXB; i += NCT) (&s.hist[0][0])[i] = 0;
  if (t < 4) (&s.ncl[0][0])[t] = 0;
  if (t < 2) { s.lesc[t] = 0; s.lfill[t] = 0; s.lovf[t] = 0; s.sescP[t] = 0; s.sescF[t] = 0; s.sfill[t] = 0; s.sovf[t] = 0; s.nwrap[t] = 0; }
  __syncthreads();
  unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
  u32 par = 0, spar = 0;
  for (int r = 0; r < reps; ++r) {
    // P on the keys
    for (int i = t; i < CH; i += NCT) s.stage[0][i] = chunk[i];
    cbar();
    Desc d; d.type = T_P; d.idx = blockIdx.x % g.CP; d.w = blockIdx.x / g.CP; d.n = CH; d.part = 0; d.nparts = 1; d.ntot = CH; d.len = CH; d.soa = 0;
    long long t0 = clock64();
    cons_P(g, s, d, s.stage[0], par); par ^= 1;
    cbar();
    long long t1 = clock64();
    // L on the keys
    for (int i = t; i < n; i += NCT) s.stage[1][i] = keys[i];
    cbar();
    d.type = T_L; d.idx = blockIdx.x % g.B; d.n = n; d.ntot = n;
    long long t2 = clock64();
    cons_L_part(g, s, d, s.stage[1], par);
    {
      long long tw = clock64() - t2;
      if ((t & 31) == 0) { atomicAdd(&g_wsum, (unsigned long long)tw); atomicMax(&g_wmax, (unsigned long long)tw); atomicMin(&g_wmin, (unsigned long long)tw); }
    }
    cbar();
    long long t3 = clock64();
    cons_L_final(g, s, d, s.stage[1], par); par ^= 1;
    cbar();
    long long t4 = clock64();
    // S on the side-0 records the link item just wrote (region of its bucket)
    const u32* ro = g.roff + (u64)d.idx * 2 * g.Bs;
    u32 nr = 0;
    for (u32 i = 0; i < g.Bs; ++i) nr += ro[i] & 0xFFFF;  // all side-0 records (several side buckets)
    const u64* rsrc = g.rscr + (u64)d.idx * RCAP;
    for (u32 i = t; i < nr && i < (u32)SK; i += NCT) s.stage[2][i] = rsrc[i];
    cbar();
    d.type = T_S; d.idx = 0; d.n = min(nr, (u32)SK); d.ntot = d.n;
    long long t5 = clock64();
    cons_S_part(g, s, d, s.stage[2], spar);
    cbar();
    long long t6 = clock64();
    cons_S_final(g, s, d, spar); spar ^= 1;
    cbar();
    long long t7 = clock64();
    c[0] += t1 - t0; c[1] += t3 - t2; c[2] += t4 - t3; c[3] += t6 - t5; c[4] += t7 - t6; c[5] += d.n;
    {  // leak check: both tables must be clean after every item
      u32 bad = 0;
      for (u32 i = t; i < (u32)TL; i += NCT) bad += (s.lkey[i] != EMPTY64) + (s.lcnt[i] != 0);
      for (u32 i = t; i < (u32)TS; i += NCT) bad += (s.nkey[i] != EMPTY32) + (s.npf[i] != 0);
      if (bad) atomicAdd(&g_leaks, bad);
      cbar();
    }
  }
  if (t == 0) for (int i = 0; i < 6; ++i) cyc[blockIdx.x * 6 + i] = c[i];
}

int main(int argc, char** argv) {
  FILE* f = fopen(argc > 1 ? argv[1] : "keys_med.bin", "rb");
  std::vector<u64> keys(1 << 16);
  int n = (int)fread(keys.data(), 8, keys.size(), f); fclose(f);
  if (n > SK) n = SK;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  WGeo g; memset(&g, 0, sizeof(g));
  g.W = 1 << 17; g.n = g.W; g.nw = 1; g.logB = 6; g.B = 64; g.logBs = 6; g.Bs = 64; g.CP = 32;
  g.nP = 32; g.nL = 64; g.nS = 128;
  u64 *dk, *kscr, *rscr, *dch;
  {
    FILE* fc = fopen("keys_chunk.bin", "rb");
    std::vector<u64> ch(CH);
    fread(ch.data(), 8, CH, fc); fclose(fc);
    CK(cudaMalloc(&dch, CH * 8)); CK(cudaMemcpy(dch, ch.data(), CH * 8, cudaMemcpyHostToDevice));
  } u32 *koff, *roff; WinState* ws; unsigned long long* cyc;
  CK(cudaMalloc(&dk, n * 8)); CK(cudaMemcpy(dk, keys.data(), n * 8, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&kscr, (size_t)RS * g.CP * CH * 8)); CK(cudaMalloc(&koff, (size_t)RS * g.B * g.CP * 4));
  CK(cudaMalloc(&rscr, (size_t)RS * g.B * RCAP * 8)); CK(cudaMalloc(&roff, (size_t)RS * 2 * g.Bs * g.B * 4));
  CK(cudaMalloc(&ws, 64 * 256)); CK(cudaMemset(ws, 0, 64 * 256));
  CK(cudaMalloc(&cyc, sms * 6 * 8));
  g.kscr = kscr; g.koff = koff; g.rscr = rscr; g.roff = roff; g.ws = ws;
  CK(cudaFuncSetAttribute(kph, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem)));
  const int reps = argc > 2 ? atoi(argv[2]) : 50;
  kph<<<sms, NCT, sizeof(Smem)>>>(g, dk, n, dch, reps, cyc);
  CK(cudaDeviceSynchronize());
  std::vector<unsigned long long> h(sms * 6);
  CK(cudaMemcpy(h.data(), cyc, h.size() * 8, cudaMemcpyDeviceToHost));
  double a[6] = {0};
  for (int b = 0; b < sms; ++b) for (int i = 0; i < 6; ++i) a[i] += h[b * 6 + i];
  for (int i = 0; i < 6; ++i) a[i] /= (double)sms * reps;
#ifdef NSG_PHASE_MARKS
  {
    long long pm[64];
    CK(cudaMemcpyFromSymbol(pm, g_pm, sizeof(pm)));
    printf("P sub-phases (cycles, thread 0 mean):");
    for (int i = 1; i < 8; ++i) printf(" %d:%.0f", i, (double)(pm[i] - pm[i - 1]) / ((double)sms * reps));
    printf("\nL part: wave %.0f bar %.0f rounds %.0f\n", (double)(pm[9] - pm[8]) / ((double)sms * reps),
           (double)(pm[10] - pm[9]) / ((double)sms * reps), (double)(pm[11] - pm[10]) / ((double)sms * reps));
    printf("L final:");
    for (int i = 17; i < 25; ++i) printf(" %d:%.0f", i, (double)(pm[i] - pm[i - 1]) / ((double)sms * reps));
    printf("\n");
  }
#endif
  unsigned leaks = 0; CK(cudaMemcpyFromSymbol(&leaks, g_leaks, 4)); printf("leaks %u\n", leaks);
  unsigned long long wsum_h, wx, wn;
  CK(cudaMemcpyFromSymbol(&wsum_h, g_wsum, 8)); CK(cudaMemcpyFromSymbol(&wx, g_wmax, 8)); CK(cudaMemcpyFromSymbol(&wn, g_wmin, 8));
  printf("L part per-warp time: mean %.0f min %llu max %llu\n", (double)wsum_h / ((double)sms * reps * NCW), wn, wx);
  printf("n=%d: P %.0f  L part %.0f  L final %.0f  S part %.0f (%.0f records)  S final %.0f  cycles\n", n, a[0], a[1], a[2],
         a[3], a[5], a[4]);
  return 0;
}
