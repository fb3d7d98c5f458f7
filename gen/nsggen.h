/* gen/nsggen.h — seeded counter-based synthetic packet generator (inputs only; not the method).
 * Recipe: gen/nsggen.cu header and DESIGN.md "Input recipe". Returns 0 ok, 1 bad argument, 2 CUDA error. */
#ifndef NSGGEN_H
#define NSGGEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { NSG_GEN_UNIFORM = 0, NSG_GEN_ZIPF = 1, NSG_GEN_HEAVY = 2 };

/* Zipf CDF table T[K] (host): T[r] = floor(2^64 * sum_{k<=r+1} k^-s / H_{K,s}), T[K-1] = 2^64-1. */
int nsg_gen_zipf_table(double s, uint32_t K, uint64_t* T);

/* Packets [first, first+count) of stream (dist, seed) into host buffers; any of src/dst/keys may be
 * NULL (keys[j] = src<<32 | dst). T/K are only read for NSG_GEN_ZIPF. n_threads<=0: all cores. */
int nsg_gen_host(int dist, uint64_t seed, uint64_t first, uint64_t count, const uint64_t* T, uint32_t K,
                 uint32_t* src, uint32_t* dst, uint64_t* keys, int n_threads);

/* Same packets into device buffers, asynchronously on `stream` (a cudaStream_t); T_dev is a device copy
 * of the table. */
int nsg_gen_device(int dist, uint64_t seed, uint64_t first, uint64_t count, const uint64_t* T_dev, uint32_t K,
                   uint32_t* src, uint32_t* dst, uint64_t* keys, void* stream);

#ifdef __cplusplus
}
#endif
#endif
