// nsg_common.cuh — shared device helpers of libnsg (the CUDA path).  Nothing here is shared
// with oracle/ or gen/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace nsg {

typedef unsigned long long u64;
typedef uint32_t u32;
typedef uint16_t u16;

// Empty-slot sentinels.  Every 64-bit key and every 32-bit address is a legal value (DESIGN.md
// reading R6), so the one key equal to a sentinel is never stored in a table: it is counted in a
// per-table "escape" accumulator instead and folded back in when the table is scanned.
constexpr u64 EMPTY64 = ~0ull;
constexpr u32 EMPTY32 = ~0u;

// Bijective mixers (murmur3 finalizers) used to spread keys over buckets and slots.  Bucket index
// = top bits, slot index = low bits, so the two are independent.
__host__ __device__ __forceinline__ u64 hash64(u64 h) {
  h ^= h >> 33; h *= 0xff51afd7ed558ccdull;
  h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ull;
  h ^= h >> 33;
  return h;
}
__host__ __device__ __forceinline__ u32 hash32(u32 x) {
  x ^= x >> 16; x *= 0x85ebca6bu;
  x ^= x >> 13; x *= 0xc2b2ae35u;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ u64 ldcg64(const u64* p) { return __ldcg(reinterpret_cast<const unsigned long long*>(p)); }
__device__ __forceinline__ u32 ldcg32(const u32* p) { return __ldcg(reinterpret_cast<const unsigned int*>(p)); }

// acquire at system scope: a flag written by a stream memory operation (cuStreamWriteValue32)
__device__ __forceinline__ u32 ld_acquire_sys32(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u32 ld_acquire32(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release32(u32* p, u32 v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Semaphore signal without a return value: after a __syncthreads(), one thread's release-RMW
// publishes every write the CTA made before the barrier (PTX causality order is cumulative through
// bar.sync; the same pattern as CUTLASS's GenericBarrier).
__device__ __forceinline__ void red_release_add32(u32* p, u32 v) {
#ifndef NSG_EXP_RELAXED_RELEASE
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#else  // timing experiment only: no ordering
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#endif
}

// Drop a 128-byte L2 line without writing it back (its contents become undefined).
__device__ __forceinline__ void discard_l2_line(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

__device__ __forceinline__ u32 warp_sum(u32 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ u32 warp_max(u32 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Rank of this lane among the lanes of its warp with `want`, offset by a CTA-shared counter that the
// warp advances once (warp-aggregated append).  All lanes of the warp must call it.
__device__ __forceinline__ u32 warp_append(bool want, u32* ctr) {
  const u32 mask = __ballot_sync(0xffffffffu, want);
  const int lane = threadIdx.x & 31;
  u32 base = 0;
  if (mask && lane == 0) base = atomicAdd(ctr, (u32)__popc(mask));
  base = __shfl_sync(0xffffffffu, base, 0);
  return base + (u32)__popc(mask & ((1u << lane) - 1u));
}

// One result row (nine u64, column order of include/nsg.h: valid, links, max link, sources, max source
// packets, max fan-out, destinations, max destination packets, max fan-in).
__device__ __forceinline__ void store_row(u64* o, const u64* row) {
#pragma unroll
  for (int j = 0; j < 9; ++j) o[j] = row[j];
}

}  // namespace nsg
