// gen/nsggen.cu — seeded, counter-based synthetic packet generator (test + bench input).
//
// NOT part of the method: it holds none of the network-quantity arithmetic.  It is the one
// module both the oracle side (tests) and the CUDA side (bench, parity tests) draw inputs
// from.  Packet i of a stream depends only on (distribution, seed, i), so a host call and a
// device call over the same index range give bit-identical packets, and any window of a
// 2^32-packet stream can be regenerated on the host by itself.
//
// Recipe:
//   u(seed, c)   = mix64(seed + (c+1) * 0x9E3779B97F4A7C15)   (splitmix64 finalizer)
//   lowbias32(x) = x^=x>>16; x*=0x7feb352d; x^=x>>15; x*=0x846ca68b; x^=x>>16  (bijective)
//   uniform      : k = u(seed, i); src = k>>32; dst = (u32)k
//   zipf(s, K)   : r_s = min{r : u(seed,2i) <= T[r]}, r_d = min{r : u(seed,2i+1) <= T[r]}
//                  src = lowbias32(r_s ^ 0x0A000000), dst = lowbias32(r_d ^ 0xC0A80000)
//                  T[r] = floor(2^64 * F(r)), F(r) = sum_{k<=r+1} k^-s / H_{K,s}; T[K-1] = 2^64-1
//   heavy        : x = u(seed,2i), y = u(seed,2i+1); src = (x>>63) ? 0x0A000001 : (u32)x; dst = (u32)y
// Addresses are IPv4 in host integer order (a.b.c.d <-> a<<24|b<<16|c<<8|d).
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "nsggen.h"

namespace {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27; z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}
__host__ __device__ __forceinline__ uint64_t u64_at(uint64_t seed, uint64_t c) {
  return mix64(seed + (c + 1) * 0x9E3779B97F4A7C15ull);
}
__host__ __device__ __forceinline__ uint32_t lowbias32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}
// smallest r in [0, K) with v <= T[r]; T nondecreasing and T[K-1] = 2^64-1
__host__ __device__ __forceinline__ uint32_t cdf_search(const uint64_t* T, uint32_t K, uint64_t v) {
  uint32_t lo = 0, hi = K - 1;
  while (lo < hi) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    if (v <= T[mid]) hi = mid; else lo = mid + 1;
  }
  return lo;
}
__host__ __device__ __forceinline__ void packet_at(int dist, uint64_t seed, uint64_t i, const uint64_t* T, uint32_t K,
                                                   uint32_t& s, uint32_t& d) {
  if (dist == NSG_GEN_UNIFORM) {
    const uint64_t k = u64_at(seed, i);
    s = uint32_t(k >> 32); d = uint32_t(k);
  } else if (dist == NSG_GEN_ZIPF) {
    const uint32_t rs = cdf_search(T, K, u64_at(seed, 2 * i));
    const uint32_t rd = cdf_search(T, K, u64_at(seed, 2 * i + 1));
    s = lowbias32(rs ^ 0x0A000000u); d = lowbias32(rd ^ 0xC0A80000u);
  } else {  // NSG_GEN_HEAVY
    const uint64_t x = u64_at(seed, 2 * i), y = u64_at(seed, 2 * i + 1);
    s = (x >> 63) ? 0x0A000001u : uint32_t(x); d = uint32_t(y);
  }
}

__global__ void gen_kernel(int dist, uint64_t seed, uint64_t first, uint64_t count, const uint64_t* __restrict__ T,
                           uint32_t K, uint32_t* __restrict__ src, uint32_t* __restrict__ dst, uint64_t* __restrict__ keys) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < count; j += stride) {
    uint32_t s, d;
    packet_at(dist, seed, first + j, T, K, s, d);
    if (keys) keys[j] = (uint64_t(s) << 32) | d;
    if (src) src[j] = s;
    if (dst) dst[j] = d;
  }
}

bool dist_ok(int dist) { return dist == NSG_GEN_UNIFORM || dist == NSG_GEN_ZIPF || dist == NSG_GEN_HEAVY; }

}  // namespace

extern "C" {

int nsg_gen_zipf_table(double s, uint32_t K, uint64_t* T) {
  if (!T || K == 0 || !(s > 0.0)) return 1;
  // H_{K,s}, small terms first (k = K down to 1), in long double.
  long double H = 0.0L;
  for (uint64_t k = K; k >= 1; --k) H += powl((long double)k, -(long double)s);
  long double c = 0.0L;
  const long double two64 = 18446744073709551616.0L;
  for (uint32_t r = 0; r < K; ++r) {
    c += powl((long double)(r + 1), -(long double)s);
    long double f = c / H * two64;
    uint64_t t;
    if (f >= two64) t = ~0ull;
    else t = (uint64_t)floorl(f);
    if (r > 0 && t < T[r - 1]) t = T[r - 1];  // keep the table monotone under rounding
    T[r] = t;
  }
  T[K - 1] = ~0ull;
  return 0;
}

int nsg_gen_host(int dist, uint64_t seed, uint64_t first, uint64_t count, const uint64_t* T, uint32_t K,
                 uint32_t* src, uint32_t* dst, uint64_t* keys, int n_threads) {
  if (!dist_ok(dist) || (dist == NSG_GEN_ZIPF && (!T || K == 0))) return 1;
  if (count == 0) return 0;
  if (!src && !dst && !keys) return 1;
  unsigned nt = n_threads > 0 ? unsigned(n_threads) : std::max(1u, std::thread::hardware_concurrency());
  if (uint64_t(nt) > count / 4096 + 1) nt = unsigned(count / 4096 + 1);
  auto work = [&](unsigned t) {
    const uint64_t b = count * t / nt, e = count * (t + 1) / nt;
    for (uint64_t j = b; j < e; ++j) {
      uint32_t s, d;
      packet_at(dist, seed, first + j, T, K, s, d);
      if (keys) keys[j] = (uint64_t(s) << 32) | d;
      if (src) src[j] = s;
      if (dst) dst[j] = d;
    }
  };
  if (nt <= 1) { work(0); return 0; }
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < nt; ++t) pool.emplace_back(work, t);
  for (auto& th : pool) th.join();
  return 0;
}

int nsg_gen_device(int dist, uint64_t seed, uint64_t first, uint64_t count, const uint64_t* T_dev, uint32_t K,
                   uint32_t* src, uint32_t* dst, uint64_t* keys, void* stream) {
  if (!dist_ok(dist) || (dist == NSG_GEN_ZIPF && (!T_dev || K == 0))) return 1;
  if (count == 0) return 0;
  if (!src && !dst && !keys) return 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t blocks = (count + 255) / 256;
  if (blocks > uint64_t(sms) * 64) blocks = uint64_t(sms) * 64;
  gen_kernel<<<unsigned(blocks), 256, 0, (cudaStream_t)stream>>>(dist, seed, first, count, T_dev, K, src, dst, keys);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // extern "C"
