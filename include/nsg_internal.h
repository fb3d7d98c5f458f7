/* include/nsg_internal.h — development and measurement hooks of libnsg; NOT part of the product
 * interface (include/nsg.h).  Used by bench.py (kernel timing), the tests (fault injection, A/B of the
 * round-1 kernel) and tools/.  Everything here may change without notice.
 *
 * Conventions as in nsg.h (asynchronous on `stream`, caller-owned buffers, synchronous argument errors).
 */
#ifndef NSG_INTERNAL_H
#define NSG_INTERNAL_H

#include "nsg.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Further flags for nsg_window_stats_ex / nsg_window_stats_timed (bits above nsg.h's). */
enum {
  NSG_FLAG_NO_FALLBACK_CHECK = 1u << 2, /* skip the L2-path fallback launch: results of an overflowed window
                                           are then undefined (measurement of the shared-memory kernels only) */
  NSG_FLAG_PROFILE = 1u << 3,           /* round-1 kernel, profile build only (-DNSG_PROFILE_BUILD): per-item-type
                                           SM cycles, u64[112] at nsg_diag_offset()+64 */
  NSG_FLAG_LEGACY_FAST = 1u << 4,       /* run the round-1 persistent kernel (nsg_fast.cuh) instead of the
                                           round-2 kernels (nsg_flat.cuh) for windows <= 2^17 (A/B measurement) */
  NSG_FLAG_INJECT_SELF_CHECK = 1u << 5  /* the round-2 kernels count a self-check failure for window 0 (tests the
                                           diagnostics / NSG_ERR_INTERNAL readback; results are unaffected) */
};

/* nsg_window_stats_ex plus measurement hooks: ev_before / ev_after (cudaEvent_t as void*, may be NULL) are
 * recorded on `stream` immediately before and after the main kernels (the per-window kernels, or the
 * L2-path kernel), excluding the workspace reset and the overflow-check launch, so a caller can time them
 * with CUDA events without changing the work. */
nsg_status nsg_window_stats_timed(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n_packets,
                                  uint64_t window, uint64_t* out, void* workspace, size_t workspace_bytes,
                                  void* stream, uint32_t flags, void* ev_before, void* ev_after);

/* Whole-trace tables of at least `slots` slots probe by CAS (the CAS returns the occupant) instead of a load
 * first; 0 restores the default (2^26 slots: DRAM-resident tables).  Process-wide, for tests that run the
 * CAS-as-probe inserts on small inputs; not thread safe against concurrent trace calls. */
nsg_status nsg_debug_trace_cas_first_slots(uint64_t slots);

#ifdef __cplusplus
}
#endif

#endif /* NSG_INTERNAL_H */
