// libnsg — per-window Network Sensing Graph Challenge statistics on B200 (sm_100a).
//
// PAPER.md (arXiv 2509.03653) Table 2 (lines 171-193) defines, for the traffic matrix A_t of a
// window, the scalars computed here: valid packets 1^T A_t 1 (:180), unique links 1^T|A_t|_0 1
// (:181), max link packets max(A_t) (:183), unique sources 1^T|A_t 1|_0 (:184), max source packets
// max(A_t 1) (:186), max source fan-out max(|A_t|_0 1) (:188), and the destination mirrors
// ("For reverse operations simply replace src and dst", :173; :241).  The paper computes them with
// cuDF group-by / value_counts / drop_duplicates (:213-239); this library computes the same
// quantities with its own sm_100a kernels:
//   nsg_fast.cuh   — window <= 2^20: one persistent kernel (partition -> link buckets -> side buckets,
//                    SMEM hash tables, exchange through L2-resident scratch).
//   nsg_global.cuh — any window <= 2^31 and the fast path's overflow hand-off: one CTA per window
//                    with global-memory hash tables.
//   nsg_anon.cuh   — IP address anonymisation (bitmap unique + rank, keyed permutation, gather).
//   nsg_trace.cuh  — the whole-trace path (A = sum of the A_t): HBM-resident tables filled by every SM,
//                    in steps a multi-GPU driver interleaves with all-to-all exchanges.
// This file holds the C ABI: argument checks, workspace layout, launches.
#include <algorithm>
#include <mutex>
#include <utility>
#include <vector>
#include <cuda.h>  // driver types for cuStreamWriteValue32 (resolved at run time: no libcuda link)
#include "nsg_internal.h"
#include "nsg_common.cuh"
#include "nsg_fast.cuh"
#include "nsg_flat.cuh"
#include "nsg_global.cuh"
#include "nsg_trace.cuh"
#include "nsg_anon.cuh"

#include <cstdio>
#include <cstring>
#include <mutex>

namespace nsg {


// ------------------------------------------------------------------------------------------
// Host side: layout, device checks, launches
// ------------------------------------------------------------------------------------------
constexpr size_t DIAG_OFFSET = 64;
constexpr size_t PROF_OFFSET = 128;  // u64[16], NSG_FLAG_PROFILE
constexpr size_t CTRL_BYTES = 4096;  // ticket, diag (64), prof u64[256] (128)
constexpr u64 GLOBAL_BUDGET = 2ull << 30;  // cap on L2-path table memory
#ifndef NSG_FLAT_BATCH
#define NSG_FLAT_BATCH 32
#endif
constexpr u64 FLAT_BATCH = NSG_FLAT_BATCH;  // windows per batch of the round-2 kernels (scratch ~3.6 MB per window)
#ifndef NSG_FLAT_BATCH_SMALL
#define NSG_FLAT_BATCH_SMALL 8
#endif
#ifndef NSG_SMALL_CALL
#define NSG_SMALL_CALL 64
#endif
// Calls of at most NSG_SMALL_CALL windows (C2: 64) use batches of NSG_FLAT_BATCH_SMALL windows: their
// scratch (~29 MB per batch) stays in L2 until the scratch discard, so the call moves little more than its
// input (C2: 85 MB of DRAM traffic per call instead of 184 MB), and their batches run on two lanes.  Larger
// calls keep FLAT_BATCH-window batches: the host enqueues ~4 operations per batch, and with 8-window batches
// a long call is bound by that enqueue rate (C5 2^30: 33.7 instead of 39.3 Gpkt/s).
constexpr u64 FLAT_BATCH_SMALL = NSG_FLAT_BATCH_SMALL;
constexpr u64 SMALL_CALL = NSG_SMALL_CALL;

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
static u64 next_pow2(u64 x) { u64 p = 1; while (p < x) p <<= 1; return p; }
static u32 ilog2(u64 x) { u32 l = 0; while ((1ull << l) < x) ++l; return l; }

struct Layout {
  bool fast;
  u64 nw;
  // fast
  u32 logB, B, logB2, B2, cp, cp_last, R;
  size_t o_pw, o_s0win, o_kscr, o_koff, o_rscr, o_roff, o_rend, o_lres, o_sres, o_s0list, o_wscr;
  size_t memset_bytes;
  // round-2 per-window kernels (nsg_flat.cuh), overlaid on the fast-path scratch
  bool flat;
  u32 flogB, fB, flogBs, fBs, fCP, fNB;  // fNB: windows per batch
  size_t o_fws, o_fkscr, o_fkoff, o_frscr, o_froff, o_fwscr, o_fend, o_fipl, o_fipc;
  u32 fLanes;        // scratch sets [o_fkscr, o_fend): one per lane of the call's batches
  size_t o_fset[3];  // set l starts at o_fset[l] (its offsets = the first's + o_fset[l] - o_fkscr)
  // global
  u64 LC;
  u32 G;
  size_t o_glk, o_glc, o_gnk, o_gnp, o_gnf;
  size_t total;
};

static Layout make_layout(u64 n, u64 W, int sms) {
  Layout L;
  memset(&L, 0, sizeof(L));
  L.nw = (n + W - 1) / W;
  L.fast = W <= FAST_MAX_WINDOW;
  if (L.fast) {
    const u64 want = (W + BUCKET_KEYS - 1) / BUCKET_KEYS;
    L.B = (u32)next_pow2(want < 1 ? 1 : want);
    L.logB = ilog2(L.B);
    const u64 want2 = (W + NODE_BUCKET - 1) / NODE_BUCKET;
    L.B2 = (u32)next_pow2(want2 < 1 ? 1 : want2);
    L.logB2 = ilog2(L.B2);
    L.cp = (u32)((W + CH - 1) / CH);
    const u64 last = n - (L.nw - 1) * W;
    L.cp_last = (u32)((last + CH - 1) / CH);
    L.R = (u32)(L.nw < (u64)RSLOTS ? next_pow2(L.nw) : (u64)RSLOTS);
  }
  size_t o = CTRL_BYTES;
  // zeroed at every call: per window pdone, ldone, sdone, fin, ovf, arrived (streamed input) and the
  // three vector fill counters; per (slot, side bucket) the published-window word and list length of
  // the side-0 node lists (IP sets)
  L.o_pw = o;
  o = align256(o + 9 * sizeof(u32) * L.nw);
  L.o_s0win = o;
  o = align256(o + 2 * sizeof(u32) * (size_t)L.R * L.B2);
  L.memset_bytes = o;
  if (L.fast) {
    L.o_kscr = o; o = align256(o + (size_t)L.R * L.cp * CH * sizeof(u64));
    L.o_koff = o; o = align256(o + (size_t)L.R * L.cp * (L.B + 1) * sizeof(u32));
    L.o_rscr = o; o = align256(o + (size_t)L.R * L.B * RCAP * sizeof(u64));
    L.o_roff = o; o = align256(o + (size_t)L.R * L.B * (2 * L.B2 + 1) * sizeof(u32));
    L.o_rend = o; o = align256(o + (size_t)L.R * L.B * (2 * L.B2) * sizeof(u32));
    L.o_lres = o; o = align256(o + (size_t)L.R * L.B * 4 * sizeof(u32));
    L.o_sres = o; o = align256(o + (size_t)L.R * 2 * L.B2 * 4 * sizeof(u32));
    L.o_s0list = o; o = align256(o + (size_t)L.R * L.B2 * S0LIST * sizeof(u32));
    L.o_wscr = o; o = align256(o + (size_t)L.R * L.cp * CH * sizeof(u32));
  }
  L.flat = W <= flat::MAX_W;
  if (L.flat) {  // overlaid on the fast path's scratch (one path or the other runs per call)
    size_t q = L.memset_bytes;
    const u64 want = (W + flat::BK - 1) / flat::BK;
    L.fB = (u32)next_pow2(want < 1 ? 1 : want);
    L.flogB = ilog2(L.fB);
    L.fBs = L.fB > 1 ? L.fB / 2 : 1;  // side buckets: ~2x the records of a link bucket per item
    L.flogBs = L.flogB > 0 ? L.flogB - 1 : 0;
    L.fCP = (u32)((W + flat::CH - 1) / flat::CH);
    const u64 fb = L.nw <= SMALL_CALL ? FLAT_BATCH_SMALL : FLAT_BATCH;
    L.fNB = (u32)(L.nw < fb ? L.nw : fb);
    L.o_fws = q; q = align256(q + (size_t)L.nw * sizeof(flat::WinState));
    L.o_fkscr = q; q = align256(q + (size_t)L.fNB * L.fCP * flat::CH * sizeof(u64));
    L.o_fkoff = q; q = align256(q + (size_t)L.fNB * L.fCP * L.fB * sizeof(u32));
    L.o_frscr = q; q = align256(q + (size_t)L.fNB * L.fB * flat::RCAP * sizeof(u64));
    L.o_froff = q; q = align256(q + (size_t)L.fNB * L.fB * 2 * L.fBs * sizeof(u32));
    L.o_fwscr = q; q = align256(q + (size_t)L.fNB * L.fCP * flat::CH * sizeof(u32));   // weighted rows
    L.o_fipc = q; q = align256(q + (size_t)L.fNB * L.fBs * sizeof(u32));                 // IP sets (vectors)
    L.o_fipl = q; q = align256(q + (size_t)L.fNB * L.fBs * flat::TS * sizeof(u32));
    L.o_fend = q;
    // A call of more than two batches runs them on two lanes (each its own scratch set and stream pair), so
    // that one lane's batch fills the SMs while the other's drains (the kernels' tails, part's low
    // occupancy); calls of one or two batches keep one set (its write-back is the DRAM traffic of C2).
#ifndef NSG_LANES_FROM_BATCHES
#define NSG_LANES_FROM_BATCHES 3  // calls of at least this many batches run on NSG_LANES lanes
#endif
#ifndef NSG_LANES
#define NSG_LANES 2
#endif
    static_assert(NSG_LANES >= 1 && NSG_LANES <= 3, "1..3 lanes");
    const u64 nbat = (L.nw + L.fNB - 1) / L.fNB;
    L.fLanes = nbat >= (u64)NSG_LANES_FROM_BATCHES ? (u32)std::min<u64>(NSG_LANES, nbat) : 1u;
    L.o_fset[0] = L.o_fkscr;
    for (u32 l = 1; l < 3; ++l) {
      L.o_fset[l] = q;
      if (l < L.fLanes) q = align256(q + (L.o_fend - L.o_fkscr));
    }
    if (q > o) o = q;
  }
  // L2-path table sets: the full path for large windows, the overflow hand-off otherwise.
  L.LC = next_pow2(2 * W);
  const u64 set_bytes = L.LC * (8 + 4 + 2 * 12);
  u64 G = L.fast ? 8 : (u64)(2 * sms);
  const u64 by_budget = GLOBAL_BUDGET / set_bytes;
  if (G > by_budget) G = by_budget;
  if (G < 1) G = 1;
  if (G > L.nw) G = L.nw;
  L.G = (u32)G;
  L.o_glk = o; o = align256(o + (size_t)G * L.LC * 8);
  L.o_glc = o; o = align256(o + (size_t)G * L.LC * 4);
  L.o_gnk = o; o = align256(o + (size_t)G * 2 * L.LC * 4);
  L.o_gnp = o; o = align256(o + (size_t)G * 2 * L.LC * 4);
  L.o_gnf = o; o = align256(o + (size_t)G * 2 * L.LC * 4);
  L.total = o;
  return L;
}

struct DevInfo {
  bool init = false;
  bool supported = false;
  int sms = 0;
  int fast_blocks = 0;    // co-resident fast_kernel<false> CTAs
  int fast_blocks_w = 0;  // co-resident fast_kernel<true> CTAs (weighted rows)
};
static std::mutex g_mu;
static DevInfo g_dev[64];
static thread_local unsigned g_last_launches = 0;

static nsg_status dev_info(DevInfo& out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return NSG_ERR_CUDA;
  if (dev < 0 || dev >= 64) return NSG_ERR_UNSUPPORTED_DEVICE;
  std::lock_guard<std::mutex> lk(g_mu);
  DevInfo& d = g_dev[dev];
  if (!d.init) {
    int major = 0, minor = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return NSG_ERR_CUDA;
    if (cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) return NSG_ERR_CUDA;
    if (cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return NSG_ERR_CUDA;
    d.supported = (major == 10 && minor == 0);
    if (d.supported) {
      if (cudaFuncSetAttribute(fast_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FAST_SMEM) != cudaSuccess ||
          cudaFuncSetAttribute(fast_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FAST_SMEM) != cudaSuccess)
        return NSG_ERR_CUDA;
      int per_sm = 0, per_sm_w = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fast_kernel<false>, FT, FAST_SMEM) != cudaSuccess ||
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_w, fast_kernel<true>, FT, FAST_SMEM) != cudaSuccess)
        return NSG_ERR_CUDA;
      if (per_sm < 1 || per_sm_w < 1) return NSG_ERR_UNSUPPORTED_DEVICE;
      d.fast_blocks = per_sm * d.sms;
      d.fast_blocks_w = per_sm_w * d.sms;
      if (cudaFuncSetAttribute(flat::part_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(flat::SmemP)) != cudaSuccess ||
          cudaFuncSetAttribute(flat::part_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(flat::SmemP)) != cudaSuccess ||
          cudaFuncSetAttribute(flat::link_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(flat::SmemL)) != cudaSuccess ||
          cudaFuncSetAttribute(flat::link_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(flat::SmemL)) != cudaSuccess ||
          cudaFuncSetAttribute(flat::side_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(flat::SmemS)) != cudaSuccess)
        return NSG_ERR_CUDA;
    }
    d.init = true;
  }
  out = d;
  return d.supported ? NSG_OK : NSG_ERR_UNSUPPORTED_DEVICE;
}

static int sms_for_layout() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 148;
  return sms;
}

// Streamed input (nsg_window_stats_from_host): the host keys are copied to `keys` (device) in chunks
// of chunk_w windows on copy_stream, each chunk followed by a stream write of its arrival flag, while
// the kernel already runs on the main stream; its partition items wait for their chunk's flag.
struct StreamIn {
  const u64* host;
  cudaStream_t cs;
  u32 chunk_w;
};
typedef CUresult (*WriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static WriteValue32Fn write_value32() {
  static WriteValue32Fn fn = nullptr;
  static bool tried = false;
  std::lock_guard<std::mutex> lk(g_mu);
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WriteValue32Fn>(p);
  }
  return fn;
}

// Side stream and events of the round-2 batch pipeline, one set per caller stream (created on first use,
// kept for the process; calls on one caller stream are ordered, so they can share it).
struct Aux {
  cudaStream_t a;
  cudaEvent_t part_done, link_done, copied;
  cudaStream_t la[3], ls[3];                     // lanes 1, 2 of a call's batches: part stream, link/side stream
  cudaEvent_t lpart[3], llink[3], start, ldone[3];
};
static Aux* aux_for(cudaStream_t s) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, cudaStream_t>, Aux*>> tab;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : tab)
    if (e.first.first == dev && e.first.second == s) return e.second;
  Aux* x = new Aux();
  if (cudaStreamCreateWithFlags(&x->a, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&x->part_done, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&x->link_done, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&x->copied, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&x->start, cudaEventDisableTiming) != cudaSuccess) {
    delete x;
    return nullptr;
  }
  bool ok = true;
  for (int l = 1; l < 3; ++l)
    ok = ok && cudaStreamCreateWithFlags(&x->la[l], cudaStreamNonBlocking) == cudaSuccess &&
         cudaStreamCreateWithFlags(&x->ls[l], cudaStreamNonBlocking) == cudaSuccess &&
         cudaEventCreateWithFlags(&x->lpart[l], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&x->llink[l], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&x->ldone[l], cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    delete x;
    return nullptr;
  }
  tab.push_back({{dev, s}, x});
  return x;
}

static nsg_status run_impl(const u32* src, const u32* dst, const u64* keys, u64 n, u64 W, u64* out, void* ws,
                      size_t ws_bytes, void* stream, u32 flags, void* ev_before = nullptr, void* ev_after = nullptr,
                      const StreamIn* sin = nullptr, const nsg_vectors* vec = nullptr, const u32* wgt = nullptr,
                      u64* const* mirror = nullptr, u32 n_mirror = 0, u64 mirror_row0 = 0) {
  g_last_launches = 0;
  if (W == 0 || W > NSG_MAX_WINDOW) return NSG_ERR_INVALID_ARGUMENT;
  if (n == 0) return NSG_OK;
  if ((keys == nullptr) == (src == nullptr && dst == nullptr)) return NSG_ERR_INVALID_ARGUMENT;
  if (!keys && (!src || !dst)) return NSG_ERR_INVALID_ARGUMENT;
  if (!out || !ws) return NSG_ERR_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(ws) & 255) || (reinterpret_cast<uintptr_t>(out) & 7)) return NSG_ERR_INVALID_ARGUMENT;
  if (keys && (reinterpret_cast<uintptr_t>(keys) & 7)) return NSG_ERR_INVALID_ARGUMENT;
  if (wgt && (reinterpret_cast<uintptr_t>(wgt) & 3)) return NSG_ERR_INVALID_ARGUMENT;
  if (n_mirror && (!mirror || (reinterpret_cast<uintptr_t>(mirror) & 7))) return NSG_ERR_INVALID_ARGUMENT;
  nsg_vectors V;
  memset(&V, 0, sizeof(V));
  if (vec) {
    V = *vec;
    // a vector is requested only as a whole: its arrays are all NULL or all non-NULL, naturally aligned
    if (!V.link_key != !V.link_packets) return NSG_ERR_INVALID_ARGUMENT;
    if (!V.src_node != !V.src_packets || !V.src_node != !V.src_fanout) return NSG_ERR_INVALID_ARGUMENT;
    if (!V.dst_node != !V.dst_packets || !V.dst_node != !V.dst_fanin) return NSG_ERR_INVALID_ARGUMENT;
    const void* a8[] = {V.link_key, V.ip_sets};
    const void* a4[] = {V.link_packets, V.src_node, V.src_packets, V.src_fanout, V.dst_node, V.dst_packets, V.dst_fanin};
    for (const void* p : a8) if (reinterpret_cast<uintptr_t>(p) & 7) return NSG_ERR_INVALID_ARGUMENT;
    for (const void* p : a4) if (reinterpret_cast<uintptr_t>(p) & 3) return NSG_ERR_INVALID_ARGUMENT;
  }
  if (src && ((reinterpret_cast<uintptr_t>(src) & 3) || (reinterpret_cast<uintptr_t>(dst) & 3)))
    return NSG_ERR_INVALID_ARGUMENT;
  DevInfo d;
  const nsg_status st = dev_info(d);
  if (st != NSG_OK) return st;
  const Layout L = make_layout(n, W, d.sms);
  if (ws_bytes < L.total) return NSG_ERR_WORKSPACE_TOO_SMALL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  unsigned char* base = reinterpret_cast<unsigned char*>(ws);
  if (cudaMemsetAsync(base, 0, L.memset_bytes, s) != cudaSuccess) return NSG_ERR_CUDA;
  u32* arrived = reinterpret_cast<u32*>(base + L.o_pw) + 5 * L.nw;
  cudaEvent_t ev_copied = nullptr;
  const bool flat_path = L.flat && !(flags & (NSG_FLAG_FORCE_GLOBAL | NSG_FLAG_LEGACY_FAST));
  if (sin && flat_path) {  // the round-2 path copies per batch (below), after the work already on `s`
    cudaEvent_t ev0 = nullptr;
    if (cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming) != cudaSuccess) return NSG_ERR_CUDA;
    const bool ok = cudaEventRecord(ev0, s) == cudaSuccess && cudaStreamWaitEvent(sin->cs, ev0, 0) == cudaSuccess;
    cudaEventDestroy(ev0);
    if (!ok) return NSG_ERR_CUDA;
  }
  if (sin && !flat_path) {  // chunked H2D on the copy stream, after the workspace reset (which clears the flags)
    WriteValue32Fn wv = write_value32();
    if (!wv) return NSG_ERR_CUDA;
    cudaEvent_t ev_reset = nullptr;
    if (cudaEventCreateWithFlags(&ev_reset, cudaEventDisableTiming) != cudaSuccess) return NSG_ERR_CUDA;
    if (cudaEventCreateWithFlags(&ev_copied, cudaEventDisableTiming) != cudaSuccess) {
      cudaEventDestroy(ev_reset);
      return NSG_ERR_CUDA;
    }
    bool okc = cudaEventRecord(ev_reset, s) == cudaSuccess && cudaStreamWaitEvent(sin->cs, ev_reset, 0) == cudaSuccess;
    const u64 per = (u64)sin->chunk_w * W;
    u64* kd = const_cast<u64*>(keys);
    for (u64 c = 0, p0 = 0; okc && p0 < n; ++c, p0 += per) {
      const u64 len = per < n - p0 ? per : n - p0;
      okc = cudaMemcpyAsync(kd + p0, sin->host + p0, len * sizeof(u64), cudaMemcpyHostToDevice, sin->cs) == cudaSuccess &&
            wv(sin->cs, reinterpret_cast<CUdeviceptr>(arrived + c), 1u, 0) == CUDA_SUCCESS;
    }
    okc = okc && cudaEventRecord(ev_copied, sin->cs) == cudaSuccess;
    cudaEventDestroy(ev_reset);
    if (!okc) { cudaEventDestroy(ev_copied); return NSG_ERR_CUDA; }
  }
  // every exit below joins the copy stream back into `s` (the input buffer is complete after the call)
  struct Join {
    cudaEvent_t ev; cudaStream_t s;
    ~Join() { if (ev) { cudaStreamWaitEvent(s, ev, 0); cudaEventDestroy(ev); } }
  } join{ev_copied, s};

  u32* pw = reinterpret_cast<u32*>(base + L.o_pw);
  GGeo gg;
  gg.n = n; gg.W = W; gg.nw = L.nw; gg.LC = L.LC; gg.G = L.G;
  gg.lkey = reinterpret_cast<u64*>(base + L.o_glk);
  gg.lcnt = reinterpret_cast<u32*>(base + L.o_glc);
  gg.nkey = reinterpret_cast<u32*>(base + L.o_gnk);
  gg.nP = reinterpret_cast<u32*>(base + L.o_gnp);
  gg.nF = reinterpret_cast<u32*>(base + L.o_gnf);
  gg.ovf = pw + 4 * L.nw;
  gg.diag = reinterpret_cast<u32*>(base + DIAG_OFFSET);
  gg.v_lkey = reinterpret_cast<u64*>(V.link_key); gg.v_lpk = V.link_packets;
  gg.v_node[0] = V.src_node; gg.v_pk[0] = V.src_packets; gg.v_fan[0] = V.src_fanout;
  gg.v_node[1] = V.dst_node; gg.v_pk[1] = V.dst_packets; gg.v_fan[1] = V.dst_fanin;
  gg.v_ipsets = reinterpret_cast<u64*>(V.ip_sets);
  gg.wgt = wgt;
  gg.mirror = mirror; gg.n_mirror = n_mirror; gg.mirror_row0 = mirror_row0;

  gg.ovf_stride = 1;
  const bool use_flat = flat_path;
  const bool use_fast = !use_flat && L.fast && !(flags & NSG_FLAG_FORCE_GLOBAL);
  if (use_flat) {
    flat::FGeo g;
    memset(&g, 0, sizeof(g));
    g.n = n; g.W = W; g.nw = L.nw;
    g.logB = L.flogB; g.B = L.fB; g.logBs = L.flogBs; g.Bs = L.fBs; g.CP = L.fCP;
    g.ws = reinterpret_cast<flat::WinState*>(base + L.o_fws);
    g.kscr = reinterpret_cast<u64*>(base + L.o_fkscr);
    g.koff = reinterpret_cast<u32*>(base + L.o_fkoff);
    g.rscr = reinterpret_cast<u64*>(base + L.o_frscr);
    g.roff = reinterpret_cast<u32*>(base + L.o_froff);
    g.diag = reinterpret_cast<u32*>(base + DIAG_OFFSET);
    g.mirror = mirror; g.n_mirror = n_mirror; g.mirror_row0 = mirror_row0;
    g.inject = ((flags & NSG_FLAG_INJECT_OVERFLOW) ? 1u : 0u) | ((flags & NSG_FLAG_INJECT_SELF_CHECK) ? 2u : 0u);
    g.v_lkey = reinterpret_cast<u64*>(V.link_key); g.v_lpk = V.link_packets;
    g.v_node[0] = V.src_node; g.v_pk[0] = V.src_packets; g.v_fan[0] = V.src_fanout;
    g.v_node[1] = V.dst_node; g.v_pk[1] = V.dst_packets; g.v_fan[1] = V.dst_fanin;
    g.v_ipsets = reinterpret_cast<u64*>(V.ip_sets);
    g.ipl = reinterpret_cast<u32*>(base + L.o_fipl);
    g.wgt = wgt;
    g.wscr = reinterpret_cast<u32*>(base + L.o_fwscr);
    g.ipc = reinterpret_cast<u32*>(base + L.o_fipc);
    if (cudaMemsetAsync(base + L.o_fws, 0, (size_t)L.nw * sizeof(flat::WinState), s) != cudaSuccess) return NSG_ERR_CUDA;
    if (ev_before && cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev_before), s) != cudaSuccess) return NSG_ERR_CUDA;
    // Batches pipeline over two streams per lane: part(i) runs on the lane's side stream as soon as the lane's
    // previous link has read the key scratch (so it overlaps that batch's side kernel); link(i) waits for
    // part(i) and follows the lane's previous side kernel (the record scratch).  One scratch set of
    // FLAT_BATCH windows per lane stays L2-resident.  Calls of NSG_LANES_FROM_BATCHES or more batches run
    // on L.fLanes lanes, batch i on lane i mod lanes (each lane's set includes its own side-0 node lists for the
    // IP sets); the lanes join the caller's stream at the end.
    Aux* ax = aux_for(s);
    if (!ax) return NSG_ERR_CUDA;
    const u32 lanes = L.fLanes;
    ax->la[0] = ax->a; ax->ls[0] = s; ax->lpart[0] = ax->part_done; ax->llink[0] = ax->link_done;
    if (cudaEventRecord(ax->link_done, s) != cudaSuccess) return NSG_ERR_CUDA;  // the reset above
    if (lanes > 1 && cudaEventRecord(ax->start, s) != cudaSuccess) return NSG_ERR_CUDA;
    for (u32 l = 1; l < lanes; ++l)
      if (cudaStreamWaitEvent(ax->ls[l], ax->start, 0) != cudaSuccess || cudaEventRecord(ax->llink[l], ax->ls[l]) != cudaSuccess)
        return NSG_ERR_CUDA;
    const flat::FGeo g0 = g;
    u64 bi = 0;
    for (u64 w0 = 0; w0 < L.nw; w0 += L.fNB, ++bi) {
      const u32 l = (u32)(bi % lanes);
      cudaStream_t sa = ax->la[l], ss = ax->ls[l];
      cudaEvent_t pd = ax->lpart[l], ld = ax->llink[l];
      const ptrdiff_t d = (ptrdiff_t)L.o_fset[l] - (ptrdiff_t)L.o_fkscr;  // this lane's scratch set
      g.kscr = reinterpret_cast<u64*>(reinterpret_cast<unsigned char*>(g0.kscr) + d);
      g.koff = reinterpret_cast<u32*>(reinterpret_cast<unsigned char*>(g0.koff) + d);
      g.rscr = reinterpret_cast<u64*>(reinterpret_cast<unsigned char*>(g0.rscr) + d);
      g.roff = reinterpret_cast<u32*>(reinterpret_cast<unsigned char*>(g0.roff) + d);
      g.wscr = reinterpret_cast<u32*>(reinterpret_cast<unsigned char*>(g0.wscr) + d);
      g.ipl = reinterpret_cast<u32*>(reinterpret_cast<unsigned char*>(g0.ipl) + d);
      g.ipc = reinterpret_cast<u32*>(reinterpret_cast<unsigned char*>(g0.ipc) + d);
      g.w0 = w0;
      g.nbw = (u32)(L.nw - w0 < (u64)L.fNB ? L.nw - w0 : (u64)L.fNB);
      if (cudaStreamWaitEvent(sa, ld, 0) != cudaSuccess) return NSG_ERR_CUDA;
      if (sin) {  // this batch's keys arrive on the copy stream
        const u64 p0 = w0 * W, p1 = (w0 + g.nbw) * W < n ? (w0 + g.nbw) * W : n;
        const bool ok = cudaMemcpyAsync(const_cast<u64*>(keys) + p0, sin->host + p0, (p1 - p0) * sizeof(u64),
                                        cudaMemcpyHostToDevice, sin->cs) == cudaSuccess &&
                        cudaEventRecord(ax->copied, sin->cs) == cudaSuccess &&
                        cudaStreamWaitEvent(sa, ax->copied, 0) == cudaSuccess;
        if (!ok) return NSG_ERR_CUDA;
      }
      if (wgt) flat::part_kernel<true><<<g.nbw * g.CP, flat::PTH, flat::part_smem(true), sa>>>(g, src, dst, keys);
      else flat::part_kernel<false><<<g.nbw * g.CP, flat::PTH, flat::part_smem(false), sa>>>(g, src, dst, keys);
      if (cudaEventRecord(pd, sa) != cudaSuccess || cudaStreamWaitEvent(ss, pd, 0) != cudaSuccess)
        return NSG_ERR_CUDA;
      if (wgt) flat::link_kernel<true><<<g.nbw * g.B, flat::LTH, sizeof(flat::SmemL), ss>>>(g);
      else flat::link_kernel<false><<<g.nbw * g.B, flat::LTH, sizeof(flat::SmemL), ss>>>(g);
      if (cudaEventRecord(ld, ss) != cudaSuccess) return NSG_ERR_CUDA;
      if (g.v_ipsets && cudaMemsetAsync(g.ipc, 0, (size_t)g.nbw * g.Bs * sizeof(u32), ss) != cudaSuccess)
        return NSG_ERR_CUDA;
      flat::side_kernel<<<g.nbw * 2 * g.Bs, flat::STH, sizeof(flat::SmemS), ss>>>(g, out);
      g_last_launches += 3;
      if (cudaGetLastError() != cudaSuccess) return NSG_ERR_CUDA;
    }
    for (u32 l = 1; l < lanes; ++l)  // the lanes join the caller's stream
      if (cudaEventRecord(ax->ldone[l], ax->ls[l]) != cudaSuccess || cudaStreamWaitEvent(s, ax->ldone[l], 0) != cudaSuccess)
        return NSG_ERR_CUDA;
#ifndef NSG_NO_DISCARD
    for (u32 l = 0; l < lanes; ++l) {  // the scratch is dead: drop it from L2 (no write-back of dirty scratch lines to HBM)
      const u64 bytes = (u64)((g.v_ipsets ? L.o_fend : L.o_fipc) - L.o_fkscr);  // the IP-set lists only when used
      const u32 blocks = (u32)std::min<u64>((bytes / 128 + 255) / 256, (u64)4 * 148);
      flat::discard_kernel<<<blocks, 256, 0, s>>>(base + L.o_fset[l], bytes);
      g_last_launches++;
    }
#endif
    if (ev_after && cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev_after), s) != cudaSuccess) return NSG_ERR_CUDA;
    if (ev_copied && cudaStreamWaitEvent(s, ev_copied, 0) != cudaSuccess) return NSG_ERR_CUDA;
    if (!(flags & NSG_FLAG_NO_FALLBACK_CHECK)) {
      gg.only_overflowed = 1;
      gg.ovf = &g.ws[0].ovf;
      gg.ovf_stride = sizeof(flat::WinState) / sizeof(u32);
      global_kernel<<<L.G, GT, 0, s>>>(gg, src, dst, keys, out);
      g_last_launches++;
      if (cudaGetLastError() != cudaSuccess) return NSG_ERR_CUDA;
    }
  } else if (use_fast) {
    Geo g;
    g.n = n; g.W = W; g.nw = L.nw;
    g.logB = L.logB; g.B = L.B; g.logB2 = L.logB2; g.B2 = L.B2; g.cp = L.cp; g.cp_last = L.cp_last; g.R = L.R;
    g.flags = flags;
    g.ticket = reinterpret_cast<u64*>(base);
    g.diag = reinterpret_cast<u32*>(base + DIAG_OFFSET);
    g.prof = reinterpret_cast<u64*>(base + PROF_OFFSET);
    g.pdone = pw; g.ldone = pw + L.nw; g.sdone = pw + 2 * L.nw; g.fin = pw + 3 * L.nw; g.ovf = pw + 4 * L.nw;
    g.arrived = sin ? arrived : nullptr;
    g.chunk_w = sin ? sin->chunk_w : 1u;
    g.kscr = reinterpret_cast<u64*>(base + L.o_kscr);
    g.koff = reinterpret_cast<u32*>(base + L.o_koff);
    g.rscr = reinterpret_cast<u64*>(base + L.o_rscr);
    g.roff = reinterpret_cast<u32*>(base + L.o_roff);
    g.rend = reinterpret_cast<u32*>(base + L.o_rend);
    g.lres = reinterpret_cast<u32*>(base + L.o_lres);
    g.sres = reinterpret_cast<u32*>(base + L.o_sres);
    g.v_lkey = gg.v_lkey; g.v_lpk = gg.v_lpk;
    for (int sd = 0; sd < 2; ++sd) { g.v_node[sd] = gg.v_node[sd]; g.v_pk[sd] = gg.v_pk[sd]; g.v_fan[sd] = gg.v_fan[sd]; }
    g.v_ipsets = gg.v_ipsets;
    g.vfill = pw + 6 * L.nw;
    g.s0win = reinterpret_cast<u32*>(base + L.o_s0win);
    g.s0cnt = g.s0win + (size_t)L.R * L.B2;
    g.s0list = reinterpret_cast<u32*>(base + L.o_s0list);
    g.wgt = wgt;
    g.wscr = reinterpret_cast<u32*>(base + L.o_wscr);
    g.mirror = mirror; g.n_mirror = n_mirror; g.mirror_row0 = mirror_row0;
    {  // ticket regions (see Geo): breakpoints where an item class enters or leaves the schedule
      u64 pts[8] = {0, (u64)LAG_L, (u64)LAG_S, (u64)LAG_F, L.nw, L.nw + LAG_L, L.nw + LAG_S, L.nw + LAG_F};
      std::sort(pts, pts + 8);
      u64 t = 0;
      bool bad = false;
      g.nreg = 0;
      auto add = [&](u64 a, u64 b, u32 keep) {  // steps [a, b), the classes in `keep` only
        u32 mask = 0, ips = 0;
        if (a >= (u64)LAG_F && a < L.nw + LAG_F) { mask |= 1u; ips += 1; }
        if (a >= (u64)LAG_S && a < L.nw + LAG_S) { mask |= 2u; ips += 2 * g.B2; }
        if (a >= (u64)LAG_L && a < L.nw + LAG_L) { mask |= 4u; ips += g.B; }
        if (a < L.nw) { mask |= 8u; ips += g.cp; }
        if (!(mask & keep)) return;
        if ((mask & keep) != mask) {  // recount for the kept classes
          mask &= keep;
          ips = ((mask & 1u) ? 1 : 0) + ((mask & 2u) ? 2 * g.B2 : 0) + ((mask & 4u) ? g.B : 0) + ((mask & 8u) ? g.cp : 0);
        }
        if (g.nreg >= (u32)MAX_REG) { bad = true; return; }
        g.reg_k0[g.nreg] = a; g.reg_t0[g.nreg] = t; g.reg_ips[g.nreg] = ips; g.reg_mask[g.nreg] = mask;
        t += (b - a) * ips;
        ++g.nreg;
      };
      for (int i = 0; i + 1 < 8; ++i) {
        const u64 a = pts[i], b = pts[i + 1];
        if (a == b) continue;
        if (a >= L.nw && a < L.nw + LAG_L) {
          // drain: once the last partition items are out, every remaining link item goes first (they
          // head the longest remaining chains), then the side and final items of those steps
          add(a, b, 4u);
          add(a, b, 3u);
        } else {
          add(a, b, 15u);
        }
      }
      if (bad) return NSG_ERR_INTERNAL;
      g.reg_t0[g.nreg] = t;
      g.total_items = t;
    }
    u64 grid = (u64)(wgt ? d.fast_blocks_w : d.fast_blocks);
    if (grid > g.total_items) grid = g.total_items;
    if (ev_before && cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev_before), s) != cudaSuccess) return NSG_ERR_CUDA;
    if (wgt) fast_kernel<true><<<(unsigned)grid, FT, FAST_SMEM, s>>>(g, src, dst, keys, out);
    else fast_kernel<false><<<(unsigned)grid, FT, FAST_SMEM, s>>>(g, src, dst, keys, out);
    g_last_launches++;
    if (cudaGetLastError() != cudaSuccess) return NSG_ERR_CUDA;
    if (ev_after && cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev_after), s) != cudaSuccess) return NSG_ERR_CUDA;
    if (ev_copied && cudaStreamWaitEvent(s, ev_copied, 0) != cudaSuccess) return NSG_ERR_CUDA;
    if (!(flags & NSG_FLAG_NO_FALLBACK_CHECK)) {
      gg.only_overflowed = 1;
      global_kernel<<<L.G, GT, 0, s>>>(gg, src, dst, keys, out);
      g_last_launches++;
      if (cudaGetLastError() != cudaSuccess) return NSG_ERR_CUDA;
    }
  } else {
    if (ev_copied && cudaStreamWaitEvent(s, ev_copied, 0) != cudaSuccess) return NSG_ERR_CUDA;
    gg.only_overflowed = 0;
    if (ev_before && cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev_before), s) != cudaSuccess) return NSG_ERR_CUDA;
    global_kernel<<<L.G, GT, 0, s>>>(gg, src, dst, keys, out);
    g_last_launches++;
    if (cudaGetLastError() != cudaSuccess) return NSG_ERR_CUDA;
    if (ev_after && cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev_after), s) != cudaSuccess) return NSG_ERR_CUDA;
  }
  return NSG_OK;
}

// The nsg_window_stats* entry points.  A debug build (-DNSG_DEBUG_CHECKS) reads the device self-check
// back (nsg.h "Errors"): it synchronises the stream and returns NSG_ERR_INTERNAL if any window failed it.
static nsg_status run(const u32* src, const u32* dst, const u64* keys, u64 n, u64 W, u64* out, void* ws,
                      size_t ws_bytes, void* stream, u32 flags, void* ev_before = nullptr, void* ev_after = nullptr,
                      const StreamIn* sin = nullptr, const nsg_vectors* vec = nullptr, const u32* wgt = nullptr,
                      u64* const* mirror = nullptr, u32 n_mirror = 0, u64 mirror_row0 = 0) {
  const nsg_status st = run_impl(src, dst, keys, n, W, out, ws, ws_bytes, stream, flags, ev_before, ev_after, sin, vec,
                                 wgt, mirror, n_mirror, mirror_row0);
#ifdef NSG_DEBUG_CHECKS
  if (st == NSG_OK && n) {
    u32 dg[4];
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (cudaMemcpyAsync(dg, reinterpret_cast<unsigned char*>(ws) + DIAG_OFFSET, sizeof(dg), cudaMemcpyDeviceToHost, s) !=
            cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return NSG_ERR_CUDA;
    if (dg[1] != 0) return NSG_ERR_INTERNAL;
  }
#endif
  return st;
}

// ------------------------------------------------------------------------------------------
// Whole-trace path (nsg_trace.cuh): workspace layout and step launches
// ------------------------------------------------------------------------------------------
struct TLayout {
  u64 LC, NC;
  u32 grid, world;
  size_t o_acc, o_ccount, o_coff, o_lt, o_nt, total;
};

static TLayout trace_layout(u64 key_cap, u64 rec_cap, u32 world, int sms) {
  TLayout T;
  memset(&T, 0, sizeof(T));
  T.LC = next_pow2(2 * (key_cap ? key_cap : 1));
  T.NC = next_pow2(2 * (rec_cap ? rec_cap : 1));
  T.grid = (u32)(sms * (2048 / TT));
  T.world = world;
  size_t o = 0;
  T.o_acc = o; o = align256(o + 64 * sizeof(u64));  // u32 esc[0] (link key ~0), esc[2..3] (node ~0 P, F)
  T.o_ccount = o; o = align256(o + (size_t)T.grid * 2 * world * sizeof(u32));
  T.o_coff = o; o = align256(o + (size_t)T.grid * 2 * world * sizeof(u64));
  T.o_lt = o; o = align256(o + (size_t)T.LC * sizeof(LSlot));
  T.o_nt = o; o = align256(o + (size_t)T.NC * sizeof(NSlot));
  T.total = o;
  return T;
}

struct TraceCall {
  TLayout T;
  unsigned char* base;
  cudaStream_t s;
};

static nsg_status trace_begin(void* ws, size_t ws_bytes, u64 key_cap, u64 rec_cap, u32 world, void* stream,
                              TraceCall& c) {
  if (!ws || (reinterpret_cast<uintptr_t>(ws) & 255)) return NSG_ERR_INVALID_ARGUMENT;
  if (world < 1 || world > (u32)TRACE_MAX_WORLD) return NSG_ERR_INVALID_ARGUMENT;
  DevInfo d;
  const nsg_status st = dev_info(d);
  if (st != NSG_OK) return st;
  c.T = trace_layout(key_cap, rec_cap, world, d.sms);
  if (ws_bytes < c.T.total) return NSG_ERR_WORKSPACE_TOO_SMALL;
  c.base = reinterpret_cast<unsigned char*>(ws);
  c.s = reinterpret_cast<cudaStream_t>(stream);
  return NSG_OK;
}

static bool input_ok(const u32* src, const u32* dst, const u64* keys) {
  if ((keys == nullptr) == (src == nullptr && dst == nullptr)) return false;
  if (!keys && (!src || !dst)) return false;
  if (keys && (reinterpret_cast<uintptr_t>(keys) & 7)) return false;
  if (src && ((reinterpret_cast<uintptr_t>(src) & 3) || (reinterpret_cast<uintptr_t>(dst) & 3))) return false;
  return true;
}

static nsg_status trace_links_impl(const u32* src, const u32* dst, const u64* keys, u64 n, u32 world, u64* link_stats,
                                   u64* rec_src, u64* rec_dst, u64* rec_counts, TraceCall& c,
                                   const u32* wgt = nullptr) {
  const TLayout& T = c.T;
  u32* esc = reinterpret_cast<u32*>(c.base + T.o_acc);
  LSlot* lt = reinterpret_cast<LSlot*>(c.base + T.o_lt);
  u32* ccount = reinterpret_cast<u32*>(c.base + T.o_ccount);
  u64* coff = reinterpret_cast<u64*>(c.base + T.o_coff);
  if (cudaMemsetAsync(esc, 0, 16, c.s) != cudaSuccess || cudaMemsetAsync(link_stats, 0, 24, c.s) != cudaSuccess)
    return NSG_ERR_CUDA;
  trace_fill<<<T.grid, TT, 0, c.s>>>(lt, T.LC, nullptr, 0);
  if (n) {
    trace_link_insert<<<T.grid, TT, 0, c.s>>>(keys, src, dst, n, lt, T.LC, esc, wgt);
    g_last_launches++;
  }
  trace_link_count<<<T.grid, TT, 0, c.s>>>(lt, T.LC, esc, world, ccount, reinterpret_cast<unsigned long long*>(link_stats));
  trace_scan<<<1, TRACE_MAX_WORLD, 0, c.s>>>(ccount, T.grid, 2, world, coff, rec_counts);
  trace_link_emit<<<T.grid, TT, 0, c.s>>>(lt, T.LC, esc, world, coff, rec_src, rec_dst, nullptr, nullptr, nullptr,
                                          nullptr);
  g_last_launches += 4;
  return cudaGetLastError() == cudaSuccess ? NSG_OK : NSG_ERR_CUDA;
}

static nsg_status trace_nodes_counted(const u64* rec, const u64* m_dev, u64* node_stats, TraceCall& c) {
  const TLayout& T = c.T;
  u32* esc = reinterpret_cast<u32*>(c.base + T.o_acc) + 2;
  NSlot* nt = reinterpret_cast<NSlot*>(c.base + T.o_nt);
  if (cudaMemsetAsync(esc, 0, 8, c.s) != cudaSuccess || cudaMemsetAsync(node_stats, 0, 24, c.s) != cudaSuccess)
    return NSG_ERR_CUDA;
  trace_fill<<<T.grid, TT, 0, c.s>>>(nullptr, 0, nt, T.NC, m_dev);  // tables sized by the device record count
  g_last_launches++;
  trace_node_insert_dev<<<T.grid, TT, 0, c.s>>>(rec, m_dev, nt, T.NC, esc);
  trace_node_scan<<<T.grid, TT, 0, c.s>>>(nt, T.NC, esc, reinterpret_cast<unsigned long long*>(node_stats), m_dev);
  g_last_launches += 2;
  return cudaGetLastError() == cudaSuccess ? NSG_OK : NSG_ERR_CUDA;
}

static nsg_status trace_nodes_impl(const u64* rec, u64 m, u64* node_stats, TraceCall& c) {
  const TLayout& T = c.T;
  u32* esc = reinterpret_cast<u32*>(c.base + T.o_acc) + 2;
  NSlot* nt = reinterpret_cast<NSlot*>(c.base + T.o_nt);
  if (cudaMemsetAsync(esc, 0, 8, c.s) != cudaSuccess || cudaMemsetAsync(node_stats, 0, 24, c.s) != cudaSuccess)
    return NSG_ERR_CUDA;
  trace_fill<<<T.grid, TT, 0, c.s>>>(nullptr, 0, nt, T.NC);
  g_last_launches++;
  if (m) {
    trace_node_insert<<<T.grid, TT, 0, c.s>>>(rec, m, nt, T.NC, esc);
    g_last_launches++;
  }
  trace_node_scan<<<T.grid, TT, 0, c.s>>>(nt, T.NC, esc, reinterpret_cast<unsigned long long*>(node_stats));
  g_last_launches++;
  return cudaGetLastError() == cudaSuccess ? NSG_OK : NSG_ERR_CUDA;
}

}  // namespace nsg

// ------------------------------------------------------------------------------------------
// C ABI
// ------------------------------------------------------------------------------------------
extern "C" {

uint64_t nsg_num_windows(uint64_t n_packets, uint64_t window) {
  if (n_packets == 0 || window == 0) return 0;
  return (n_packets + window - 1) / window;
}

size_t nsg_workspace_bytes(uint64_t n_packets, uint64_t window) {
  if (n_packets == 0 || window == 0 || window > NSG_MAX_WINDOW) return 0;
  return nsg::make_layout(n_packets, window, nsg::sms_for_layout()).total;
}

nsg_status nsg_window_stats(const uint32_t* src, const uint32_t* dst, uint64_t n_packets, uint64_t window,
                            uint64_t* out, void* workspace, size_t workspace_bytes, void* stream) {
  if (n_packets && (!src || !dst)) return NSG_ERR_INVALID_ARGUMENT;
  return nsg::run(src, dst, nullptr, n_packets, window, reinterpret_cast<nsg::u64*>(out), workspace, workspace_bytes,
                  stream, 0);
}

nsg_status nsg_window_stats_packed(const uint64_t* keys, uint64_t n_packets, uint64_t window, uint64_t* out,
                                   void* workspace, size_t workspace_bytes, void* stream) {
  if (n_packets && !keys) return NSG_ERR_INVALID_ARGUMENT;
  return nsg::run(nullptr, nullptr, reinterpret_cast<const nsg::u64*>(keys), n_packets, window,
                  reinterpret_cast<nsg::u64*>(out), workspace, workspace_bytes, stream, 0);
}

nsg_status nsg_window_stats_ex(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n_packets,
                               uint64_t window, uint64_t* out, void* workspace, size_t workspace_bytes,
                               void* stream, uint32_t flags) {
  return nsg::run(src, dst, reinterpret_cast<const nsg::u64*>(keys), n_packets, window,
                  reinterpret_cast<nsg::u64*>(out), workspace, workspace_bytes, stream, flags);
}

nsg_status nsg_window_stats_timed(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n_packets,
                                  uint64_t window, uint64_t* out, void* workspace, size_t workspace_bytes, void* stream,
                                  uint32_t flags, void* ev_before, void* ev_after) {
  return nsg::run(src, dst, reinterpret_cast<const nsg::u64*>(keys), n_packets, window,
                  reinterpret_cast<nsg::u64*>(out), workspace, workspace_bytes, stream, flags, ev_before, ev_after);
}

nsg_status nsg_window_stats_from_host(const uint64_t* keys_host, uint64_t n_packets, uint64_t window,
                                      uint64_t* keys_dev, uint64_t* out, uint64_t* out_host, void* workspace,
                                      size_t workspace_bytes, void* stream, void* copy_stream, uint32_t chunk_windows) {
  nsg::g_last_launches = 0;
  if (window == 0 || window > NSG_MAX_WINDOW) return NSG_ERR_INVALID_ARGUMENT;
  if (n_packets == 0) return NSG_OK;
  if (!keys_host || !keys_dev || !out || !copy_stream || copy_stream == stream) return NSG_ERR_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(keys_host) & 7) || (reinterpret_cast<uintptr_t>(out_host) & 7))
    return NSG_ERR_INVALID_ARGUMENT;
  const nsg::StreamIn sin{reinterpret_cast<const nsg::u64*>(keys_host), reinterpret_cast<cudaStream_t>(copy_stream),
                          chunk_windows ? chunk_windows : 8u};
  const nsg_status st = nsg::run(nullptr, nullptr, reinterpret_cast<const nsg::u64*>(keys_dev), n_packets, window,
                                 reinterpret_cast<nsg::u64*>(out), workspace, workspace_bytes, stream, 0, nullptr,
                                 nullptr, &sin);
  if (st != NSG_OK || !out_host) return st;
  const size_t bytes = (size_t)nsg_num_windows(n_packets, window) * NSG_NUM_STATS * sizeof(uint64_t);
  if (cudaMemcpyAsync(out_host, out, bytes, cudaMemcpyDeviceToHost, reinterpret_cast<cudaStream_t>(stream)) != cudaSuccess)
    return NSG_ERR_CUDA;
  return NSG_OK;
}

nsg_status nsg_window_vectors(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n_packets,
                              uint64_t window, uint64_t* out, const nsg_vectors* vectors, void* workspace,
                              size_t workspace_bytes, void* stream, uint32_t flags) {
  if (!vectors) return NSG_ERR_INVALID_ARGUMENT;
  return nsg::run(src, dst, reinterpret_cast<const nsg::u64*>(keys), n_packets, window,
                  reinterpret_cast<nsg::u64*>(out), workspace, workspace_bytes, stream, flags, nullptr, nullptr,
                  nullptr, vectors);
}

nsg_status nsg_window_stats_mirrored(const uint32_t* src, const uint32_t* dst, const uint64_t* keys,
                                     uint64_t n_packets, uint64_t window, uint64_t* out, void* workspace,
                                     size_t workspace_bytes, void* stream, uint32_t flags, uint64_t* const* mirrors,
                                     uint32_t n_mirrors, uint64_t mirror_row0) {
  if (n_mirrors == 0 || !mirrors) return NSG_ERR_INVALID_ARGUMENT;
  return nsg::run(src, dst, reinterpret_cast<const nsg::u64*>(keys), n_packets, window, reinterpret_cast<nsg::u64*>(out),
                  workspace, workspace_bytes, stream, flags, nullptr, nullptr, nullptr, nullptr, nullptr,
                  reinterpret_cast<nsg::u64* const*>(mirrors), n_mirrors, mirror_row0);
}

nsg_status nsg_window_stats_weighted(const uint32_t* src, const uint32_t* dst, const uint64_t* keys,
                                     const uint32_t* n_packets, uint64_t n_rows, uint64_t window, uint64_t* out,
                                     void* workspace, size_t workspace_bytes, void* stream, uint32_t flags) {
  if (n_rows && !n_packets) return NSG_ERR_INVALID_ARGUMENT;
  return nsg::run(src, dst, reinterpret_cast<const nsg::u64*>(keys), n_rows, window, reinterpret_cast<nsg::u64*>(out),
                  workspace, workspace_bytes, stream, flags, nullptr, nullptr, nullptr, nullptr, n_packets);
}

size_t nsg_trace_workspace_bytes(uint64_t key_capacity, uint64_t record_capacity, uint32_t world) {
  if (world < 1 || world > (uint32_t)nsg::TRACE_MAX_WORLD) return 0;
  return nsg::trace_layout(key_capacity, record_capacity, world, nsg::sms_for_layout()).total;
}

size_t nsg_trace_stats_workspace_bytes(uint64_t n_packets) {
  const size_t t = nsg::align256(nsg_trace_workspace_bytes(n_packets, n_packets, 1));
  return t + 2 * nsg::align256((size_t)(n_packets ? n_packets : 1) * 8) + 256;
}

nsg_status nsg_trace_partition(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n,
                               uint32_t world, uint64_t* send_keys, uint64_t* send_counts, void* workspace,
                               size_t workspace_bytes, uint64_t key_capacity, uint64_t record_capacity, void* stream) {
  nsg::g_last_launches = 0;
  if (n && !nsg::input_ok(src, dst, reinterpret_cast<const nsg::u64*>(keys))) return NSG_ERR_INVALID_ARGUMENT;
  if (!send_keys || !send_counts || (reinterpret_cast<uintptr_t>(send_keys) & 7) ||
      (reinterpret_cast<uintptr_t>(send_counts) & 7))
    return NSG_ERR_INVALID_ARGUMENT;
  nsg::TraceCall c;
  nsg_status st = nsg::trace_begin(workspace, workspace_bytes, key_capacity, record_capacity, world, stream, c);
  if (st != NSG_OK) return st;
  nsg::u32* ccount = reinterpret_cast<nsg::u32*>(c.base + c.T.o_ccount);
  nsg::u64* coff = reinterpret_cast<nsg::u64*>(c.base + c.T.o_coff);
  const nsg::u64* k = reinterpret_cast<const nsg::u64*>(keys);
  nsg::trace_part_count<<<c.T.grid, nsg::TT, 0, c.s>>>(k, src, dst, n, world, ccount);
  nsg::trace_scan<<<1, nsg::TRACE_MAX_WORLD, 0, c.s>>>(ccount, c.T.grid, 1, world, coff,
                                                        reinterpret_cast<nsg::u64*>(send_counts));
  nsg::trace_part_scatter<<<c.T.grid, nsg::TT, 0, c.s>>>(k, src, dst, n, world, coff,
                                                         reinterpret_cast<nsg::u64*>(send_keys), nullptr, nullptr);
  nsg::g_last_launches = 3;
  return cudaGetLastError() == cudaSuccess ? NSG_OK : NSG_ERR_CUDA;
}

nsg_status nsg_trace_links(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n, uint32_t world,
                           uint64_t* link_stats, uint64_t* rec_src, uint64_t* rec_dst, uint64_t* rec_counts,
                           void* workspace, size_t workspace_bytes, uint64_t key_capacity, uint64_t record_capacity,
                           void* stream) {
  nsg::g_last_launches = 0;
  if (n > key_capacity || n >= (1ull << 32)) return NSG_ERR_INVALID_ARGUMENT;  // 32-bit link sums
  if (n && !nsg::input_ok(src, dst, reinterpret_cast<const nsg::u64*>(keys))) return NSG_ERR_INVALID_ARGUMENT;
  const void* p8[] = {link_stats, rec_src, rec_dst, rec_counts};
  for (const void* p : p8)
    if (!p || (reinterpret_cast<uintptr_t>(p) & 7)) return NSG_ERR_INVALID_ARGUMENT;
  nsg::TraceCall c;
  nsg_status st = nsg::trace_begin(workspace, workspace_bytes, key_capacity, record_capacity, world, stream, c);
  if (st != NSG_OK) return st;
  return nsg::trace_links_impl(src, dst, reinterpret_cast<const nsg::u64*>(keys), n, world,
                               reinterpret_cast<nsg::u64*>(link_stats), reinterpret_cast<nsg::u64*>(rec_src),
                               reinterpret_cast<nsg::u64*>(rec_dst), reinterpret_cast<nsg::u64*>(rec_counts), c);
}

nsg_status nsg_trace_nodes(const uint64_t* records, uint64_t m, uint64_t* node_stats, void* workspace,
                           size_t workspace_bytes, uint64_t key_capacity, uint64_t record_capacity, void* stream) {
  nsg::g_last_launches = 0;
  if (m > record_capacity || (m && !records) || (reinterpret_cast<uintptr_t>(records) & 7)) return NSG_ERR_INVALID_ARGUMENT;
  if (!node_stats || (reinterpret_cast<uintptr_t>(node_stats) & 7)) return NSG_ERR_INVALID_ARGUMENT;
  nsg::TraceCall c;
  nsg_status st = nsg::trace_begin(workspace, workspace_bytes, key_capacity, record_capacity, 1, stream, c);
  if (st != NSG_OK) return st;
  return nsg::trace_nodes_impl(reinterpret_cast<const nsg::u64*>(records), m, reinterpret_cast<nsg::u64*>(node_stats), c);
}

// ---- fused exchange over peer memory (CUDA IPC): the scatters write straight into the owners' buffers
size_t nsg_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

nsg_status nsg_ipc_alloc(size_t bytes, void** dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out || bytes == 0) return NSG_ERR_INVALID_ARGUMENT;
  nsg::DevInfo d;
  const nsg_status st = nsg::dev_info(d);
  if (st != NSG_OK) return st;
  if (cudaMalloc(dev_ptr, bytes) != cudaSuccess) return NSG_ERR_CUDA;
  if (cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle_out), *dev_ptr) != cudaSuccess) {
    cudaFree(*dev_ptr);
    *dev_ptr = nullptr;
    return NSG_ERR_CUDA;
  }
  return NSG_OK;
}

nsg_status nsg_ipc_open(const void* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return NSG_ERR_INVALID_ARGUMENT;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess ? NSG_OK : NSG_ERR_CUDA;
}

nsg_status nsg_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return NSG_ERR_INVALID_ARGUMENT;
  return cudaIpcCloseMemHandle(dev_ptr) == cudaSuccess ? NSG_OK : NSG_ERR_CUDA;
}

nsg_status nsg_ipc_free(void* dev_ptr) {
  if (!dev_ptr) return NSG_ERR_INVALID_ARGUMENT;
  return cudaFree(dev_ptr) == cudaSuccess ? NSG_OK : NSG_ERR_CUDA;
}

nsg_status nsg_trace_owner_counts(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n,
                                  uint32_t world, uint64_t* counts, void* workspace, size_t workspace_bytes,
                                  uint64_t key_capacity, uint64_t record_capacity, void* stream) {
  nsg::g_last_launches = 0;
  if (n && !nsg::input_ok(src, dst, reinterpret_cast<const nsg::u64*>(keys))) return NSG_ERR_INVALID_ARGUMENT;
  if (!counts || (reinterpret_cast<uintptr_t>(counts) & 7)) return NSG_ERR_INVALID_ARGUMENT;
  nsg::TraceCall c;
  nsg_status st = nsg::trace_begin(workspace, workspace_bytes, key_capacity, record_capacity, world, stream, c);
  if (st != NSG_OK) return st;
  nsg::u32* ccount = reinterpret_cast<nsg::u32*>(c.base + c.T.o_ccount);
  nsg::u64* coff = reinterpret_cast<nsg::u64*>(c.base + c.T.o_coff);
  nsg::trace_part_count<<<c.T.grid, nsg::TT, 0, c.s>>>(reinterpret_cast<const nsg::u64*>(keys), src, dst, n, world, ccount);
  nsg::trace_scan<<<1, nsg::TRACE_MAX_WORLD, 0, c.s>>>(ccount, c.T.grid, 1, world, coff, reinterpret_cast<nsg::u64*>(counts));
  nsg::g_last_launches = 2;
  return cudaGetLastError() == cudaSuccess ? NSG_OK : NSG_ERR_CUDA;
}

nsg_status nsg_trace_partition_peers(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n,
                                     uint32_t world, uint64_t* const* peers, const uint64_t* peer_base,
                                     void* workspace, size_t workspace_bytes, uint64_t key_capacity,
                                     uint64_t record_capacity, void* stream) {
  nsg::g_last_launches = 0;
  if (n && !nsg::input_ok(src, dst, reinterpret_cast<const nsg::u64*>(keys))) return NSG_ERR_INVALID_ARGUMENT;
  if (!peers || !peer_base || (reinterpret_cast<uintptr_t>(peers) & 7) || (reinterpret_cast<uintptr_t>(peer_base) & 7))
    return NSG_ERR_INVALID_ARGUMENT;
  nsg::TraceCall c;
  nsg_status st = nsg::trace_begin(workspace, workspace_bytes, key_capacity, record_capacity, world, stream, c);
  if (st != NSG_OK) return st;
  nsg::u32* ccount = reinterpret_cast<nsg::u32*>(c.base + c.T.o_ccount);
  nsg::u64* coff = reinterpret_cast<nsg::u64*>(c.base + c.T.o_coff);
  const nsg::u64* k = reinterpret_cast<const nsg::u64*>(keys);
  nsg::trace_part_count<<<c.T.grid, nsg::TT, 0, c.s>>>(k, src, dst, n, world, ccount);
  nsg::trace_scan<<<1, nsg::TRACE_MAX_WORLD, 0, c.s>>>(ccount, c.T.grid, 1, world, coff, nullptr);
  nsg::trace_part_scatter<<<c.T.grid, nsg::TT, 0, c.s>>>(k, src, dst, n, world, coff, nullptr,
                                                         reinterpret_cast<nsg::u64* const*>(peers),
                                                         reinterpret_cast<const nsg::u64*>(peer_base));
  nsg::g_last_launches = 3;
  return cudaGetLastError() == cudaSuccess ? NSG_OK : NSG_ERR_CUDA;
}

nsg_status nsg_trace_links_count(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n,
                                 uint32_t world, uint64_t* link_stats, uint64_t* rec_counts, void* workspace,
                                 size_t workspace_bytes, uint64_t key_capacity, uint64_t record_capacity, void* stream) {
  nsg::g_last_launches = 0;
  if (n > key_capacity || n >= (1ull << 32)) return NSG_ERR_INVALID_ARGUMENT;  // 32-bit link sums
  if (n && !nsg::input_ok(src, dst, reinterpret_cast<const nsg::u64*>(keys))) return NSG_ERR_INVALID_ARGUMENT;
  if (!link_stats || !rec_counts || (reinterpret_cast<uintptr_t>(link_stats) & 7) ||
      (reinterpret_cast<uintptr_t>(rec_counts) & 7))
    return NSG_ERR_INVALID_ARGUMENT;
  nsg::TraceCall c;
  nsg_status st = nsg::trace_begin(workspace, workspace_bytes, key_capacity, record_capacity, world, stream, c);
  if (st != NSG_OK) return st;
  const nsg::TLayout& T = c.T;
  nsg::u32* esc = reinterpret_cast<nsg::u32*>(c.base + T.o_acc);
  nsg::LSlot* lt = reinterpret_cast<nsg::LSlot*>(c.base + T.o_lt);
  nsg::u32* ccount = reinterpret_cast<nsg::u32*>(c.base + T.o_ccount);
  nsg::u64* coff = reinterpret_cast<nsg::u64*>(c.base + T.o_coff);
  if (cudaMemsetAsync(esc, 0, 16, c.s) != cudaSuccess || cudaMemsetAsync(link_stats, 0, 24, c.s) != cudaSuccess)
    return NSG_ERR_CUDA;
  nsg::trace_fill<<<T.grid, nsg::TT, 0, c.s>>>(lt, T.LC, nullptr, 0);
  if (n)
    nsg::trace_link_insert<<<T.grid, nsg::TT, 0, c.s>>>(reinterpret_cast<const nsg::u64*>(keys), src, dst, n, lt, T.LC, esc);
  nsg::trace_link_count<<<T.grid, nsg::TT, 0, c.s>>>(lt, T.LC, esc, world, ccount,
                                                     reinterpret_cast<unsigned long long*>(link_stats));
  nsg::trace_scan<<<1, nsg::TRACE_MAX_WORLD, 0, c.s>>>(ccount, T.grid, 2, world, coff,
                                                       reinterpret_cast<nsg::u64*>(rec_counts));
  nsg::g_last_launches = n ? 4 : 3;
  return cudaGetLastError() == cudaSuccess ? NSG_OK : NSG_ERR_CUDA;
}

nsg_status nsg_trace_links_emit_peers(uint32_t world, uint64_t* const* peers_src, uint64_t* const* peers_dst,
                                      const uint64_t* base_src, const uint64_t* base_dst, void* workspace,
                                      size_t workspace_bytes, uint64_t key_capacity, uint64_t record_capacity,
                                      void* stream) {
  nsg::g_last_launches = 0;
  const void* p8[] = {peers_src, peers_dst, base_src, base_dst};
  for (const void* p : p8)
    if (!p || (reinterpret_cast<uintptr_t>(p) & 7)) return NSG_ERR_INVALID_ARGUMENT;
  nsg::TraceCall c;
  nsg_status st = nsg::trace_begin(workspace, workspace_bytes, key_capacity, record_capacity, world, stream, c);
  if (st != NSG_OK) return st;
  const nsg::TLayout& T = c.T;
  nsg::trace_link_emit<<<T.grid, nsg::TT, 0, c.s>>>(
      reinterpret_cast<const nsg::LSlot*>(c.base + T.o_lt), T.LC, reinterpret_cast<const nsg::u32*>(c.base + T.o_acc),
      world, reinterpret_cast<const nsg::u64*>(c.base + T.o_coff), nullptr, nullptr,
      reinterpret_cast<nsg::u64* const*>(peers_src), reinterpret_cast<nsg::u64* const*>(peers_dst),
      reinterpret_cast<const nsg::u64*>(base_src), reinterpret_cast<const nsg::u64*>(base_dst));
  nsg::g_last_launches = 1;
  return cudaGetLastError() == cudaSuccess ? NSG_OK : NSG_ERR_CUDA;
}

static nsg_status trace_stats_impl(const uint32_t* src, const uint32_t* dst, const uint64_t* keys,
                                   const uint32_t* wgt, uint64_t n_packets, uint64_t* out, void* workspace,
                                   size_t workspace_bytes, void* stream);

nsg_status nsg_trace_stats(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n_packets,
                           uint64_t* out, void* workspace, size_t workspace_bytes, void* stream) {
  return trace_stats_impl(src, dst, keys, nullptr, n_packets, out, workspace, workspace_bytes, stream);
}

nsg_status nsg_trace_stats_weighted(const uint32_t* src, const uint32_t* dst, const uint64_t* keys,
                                    const uint32_t* n_packets, uint64_t n_rows, uint64_t* out, void* workspace,
                                    size_t workspace_bytes, void* stream) {
  if (n_rows && (!n_packets || (reinterpret_cast<uintptr_t>(n_packets) & 3))) return NSG_ERR_INVALID_ARGUMENT;
  return trace_stats_impl(src, dst, keys, n_packets, n_rows, out, workspace, workspace_bytes, stream);
}

static nsg_status trace_stats_impl(const uint32_t* src, const uint32_t* dst, const uint64_t* keys,
                                   const uint32_t* wgt, uint64_t n_packets, uint64_t* out, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  nsg::g_last_launches = 0;
  if (n_packets == 0) return NSG_OK;
  if (n_packets >= (1ull << 32)) return NSG_ERR_INVALID_ARGUMENT;  // per-link / per-node sums are 32-bit
  if (!nsg::input_ok(src, dst, reinterpret_cast<const nsg::u64*>(keys))) return NSG_ERR_INVALID_ARGUMENT;
  if (!out || (reinterpret_cast<uintptr_t>(out) & 7)) return NSG_ERR_INVALID_ARGUMENT;
  if (workspace_bytes < nsg_trace_stats_workspace_bytes(n_packets)) return NSG_ERR_WORKSPACE_TOO_SMALL;
  nsg::TraceCall c;
  const size_t tb = nsg::align256(nsg_trace_workspace_bytes(n_packets, n_packets, 1));
  nsg_status st = nsg::trace_begin(workspace, tb, n_packets, n_packets, 1, stream, c);
  if (st != NSG_OK) return st;
  unsigned char* extra = c.base + tb;
  nsg::u64* rec_src = reinterpret_cast<nsg::u64*>(extra);
  nsg::u64* rec_dst = reinterpret_cast<nsg::u64*>(extra + nsg::align256((size_t)n_packets * 8));
  nsg::u64* part = reinterpret_cast<nsg::u64*>(extra + 2 * nsg::align256((size_t)n_packets * 8));  // [12] + [2] counts
  // 256 B tail: link [0..2], src [4..6], dst [8..10], record counts [12..13]
  {  // links: one pass gives the statistics and both sides' records (same positions on both sides)
    const nsg::TLayout& T = c.T;
    nsg::u32* esc = reinterpret_cast<nsg::u32*>(c.base + T.o_acc);
    nsg::LSlot* lt = reinterpret_cast<nsg::LSlot*>(c.base + T.o_lt);
    if (cudaMemsetAsync(esc, 0, 16, c.s) != cudaSuccess || cudaMemsetAsync(part, 0, 16 * sizeof(nsg::u64), c.s) != cudaSuccess)
      return NSG_ERR_CUDA;
    nsg::trace_fill<<<T.grid, nsg::TT, 0, c.s>>>(lt, T.LC, nullptr, 0);
    nsg::trace_link_insert<<<T.grid, nsg::TT, 0, c.s>>>(reinterpret_cast<const nsg::u64*>(keys), src, dst, n_packets,
                                                        lt, T.LC, esc, wgt);
    nsg::trace_link_emit1<<<T.grid, nsg::TT, 0, c.s>>>(lt, T.LC, esc, rec_src, rec_dst,
                                                       reinterpret_cast<unsigned long long*>(part + 12),
                                                       reinterpret_cast<unsigned long long*>(part));
    nsg::g_last_launches += 3;
  }
  // with one rank every record stays here; the node steps read the record count from device memory, so
  // the whole call is asynchronous (no host sync for the counts)
  st = nsg::trace_nodes_counted(rec_src, part + 12, part + 4, c);
  if (st != NSG_OK) return st;
  st = nsg::trace_nodes_counted(rec_dst, part + 12, part + 8, c);
  if (st != NSG_OK) return st;
  nsg::trace_finish<<<1, 32, 0, c.s>>>(reinterpret_cast<unsigned long long*>(part),
                                       reinterpret_cast<unsigned long long*>(part + 4),
                                       reinterpret_cast<unsigned long long*>(part + 8), reinterpret_cast<nsg::u64*>(out));
  nsg::g_last_launches += 1;
  return cudaGetLastError() == cudaSuccess ? NSG_OK : NSG_ERR_CUDA;
}

size_t nsg_anonymize_workspace_bytes(void) {
  return nsg::ANON_WORDS * 4 + nsg::ANON_BLOCKS * 4 + nsg::ANON_SCAN_CTAS * 4 + nsg::ANON_TABLE_SLOTS * 8 +
         nsg::ANON_TABLE_MAX * 4 + nsg::ANON_SWORDS * 4 * 2;
}

nsg_status nsg_anonymize(const uint32_t* src, const uint32_t* dst, const uint64_t* keys, uint64_t n_packets,
                         uint64_t seed, uint32_t rounds, uint32_t* src_out, uint32_t* dst_out, uint64_t* n_unique,
                         void* workspace, size_t workspace_bytes, void* stream) {
  nsg::g_last_launches = 0;
  if (!n_unique || (reinterpret_cast<uintptr_t>(n_unique) & 7)) return NSG_ERR_INVALID_ARGUMENT;
  if (n_packets && !nsg::input_ok(src, dst, reinterpret_cast<const nsg::u64*>(keys))) return NSG_ERR_INVALID_ARGUMENT;
  if (n_packets && (!src_out || !dst_out || (reinterpret_cast<uintptr_t>(src_out) & 3) ||
                    (reinterpret_cast<uintptr_t>(dst_out) & 3)))
    return NSG_ERR_INVALID_ARGUMENT;
  if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 255)) return NSG_ERR_INVALID_ARGUMENT;
  if (workspace_bytes < nsg_anonymize_workspace_bytes()) return NSG_ERR_WORKSPACE_TOO_SMALL;
  nsg::DevInfo d;
  const nsg_status st = nsg::dev_info(d);
  if (st != NSG_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  unsigned char* base = reinterpret_cast<unsigned char*>(workspace);
  nsg::u32* bitmap = reinterpret_cast<nsg::u32*>(base);
  nsg::u32* bpre = reinterpret_cast<nsg::u32*>(base + nsg::ANON_WORDS * 4);
  nsg::u32* ctot = bpre + nsg::ANON_BLOCKS;
  nsg::u64* table = reinterpret_cast<nsg::u64*>(ctot + nsg::ANON_SCAN_CTAS);  // 8 B aligned: offsets are multiples of 4 KiB
  nsg::u32* U = reinterpret_cast<nsg::u32*>(table + nsg::ANON_TABLE_SLOTS);
  nsg::u32* summ = U + nsg::ANON_TABLE_MAX;
  nsg::u32* wcnt = summ + nsg::ANON_SWORDS;
  nsg::u64* nu = reinterpret_cast<nsg::u64*>(n_unique);
  const nsg::u64* k = reinterpret_cast<const nsg::u64*>(keys);
  if (cudaMemsetAsync(summ, 0, nsg::ANON_SWORDS * 4, s) != cudaSuccess) return NSG_ERR_CUDA;
  const unsigned grid = (unsigned)(d.sms * (2048 / nsg::AT));
  if (n_packets) {
    nsg::anon_touch_kernel<<<grid, nsg::AT, 0, s>>>(k, src, dst, n_packets, summ);
    nsg::anon_clear_groups<<<grid, nsg::AT, 0, s>>>(summ, bitmap);
    nsg::anon_mark_kernel<<<grid, nsg::AT, 0, s>>>(k, src, dst, n_packets, bitmap);
  }
  nsg::anon_word_count<<<nsg::ANON_SCAN_CTAS, nsg::AT, 0, s>>>(summ, bitmap, wcnt, ctot);
  nsg::anon_scan_totals<<<1, 1024, 0, s>>>(ctot, nu);
  if (n_packets) {
    nsg::anon_enumerate<<<nsg::ANON_SCAN_CTAS, nsg::AT, 0, s>>>(summ, bitmap, wcnt, ctot, nu, bpre, U);
    nsg::anon_table_fill<<<grid, nsg::AT, 0, s>>>(table, nu);
    nsg::anon_table_label<<<grid, nsg::AT, 0, s>>>(U, nu, seed, rounds, table);
    nsg::anon_relabel_kernel<<<grid, nsg::AT, 0, s>>>(k, src, dst, n_packets, bitmap, bpre, table, nu, seed, rounds,
                                                      src_out, dst_out);
  }
  nsg::g_last_launches = n_packets ? 9 : 2;
  return cudaGetLastError() == cudaSuccess ? NSG_OK : NSG_ERR_CUDA;
}

nsg_status nsg_window_vectors_weighted(const uint32_t* src, const uint32_t* dst, const uint64_t* keys,
                                       const uint32_t* n_packets, uint64_t n_rows, uint64_t window, uint64_t* out,
                                       const nsg_vectors* vectors, void* workspace, size_t workspace_bytes,
                                       void* stream, uint32_t flags) {
  if (!vectors || (n_rows && !n_packets)) return NSG_ERR_INVALID_ARGUMENT;
  return nsg::run(src, dst, reinterpret_cast<const nsg::u64*>(keys), n_rows, window, reinterpret_cast<nsg::u64*>(out),
                  workspace, workspace_bytes, stream, flags, nullptr, nullptr, nullptr, vectors, n_packets);
}

size_t nsg_diag_offset(void) { return nsg::DIAG_OFFSET; }

nsg_status nsg_debug_trace_cas_first_slots(uint64_t slots) {
  const nsg::u64 v = slots ? slots : nsg::TRACE_CAS_FIRST_SLOTS;
  return cudaMemcpyToSymbol(nsg::g_trace_cas_first_slots, &v, sizeof(v)) == cudaSuccess ? NSG_OK : NSG_ERR_CUDA;
}

unsigned nsg_last_launches(void) { return nsg::g_last_launches; }


#ifdef NSG_EXP_TRACE
// timing experiment only: copy the item trace of the last launches to `host` (u64[cap][4]) and reset
unsigned nsg_debug_trace(void* host, unsigned cap) {
  unsigned n = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&n, nsg::g_trace_n, sizeof(n));
  n = n < cap ? n : cap;
  if (n > nsg::TRACE_CAP) n = nsg::TRACE_CAP;
  cudaMemcpyFromSymbol(host, nsg::g_trace, (size_t)n * 32);
  const unsigned z = 0;
  cudaMemcpyToSymbol(nsg::g_trace_n, &z, sizeof(z));
  return n;
}
#endif

const char* nsg_status_string(nsg_status s) {
  switch (s) {
    case NSG_OK: return "NSG_OK";
    case NSG_ERR_INVALID_ARGUMENT: return "NSG_ERR_INVALID_ARGUMENT";
    case NSG_ERR_CUDA: return "NSG_ERR_CUDA";
    case NSG_ERR_WORKSPACE_TOO_SMALL: return "NSG_ERR_WORKSPACE_TOO_SMALL";
    case NSG_ERR_UNSUPPORTED_DEVICE: return "NSG_ERR_UNSUPPORTED_DEVICE";
    case NSG_ERR_INTERNAL: return "NSG_ERR_INTERNAL";
  }
  return "NSG_ERR_UNKNOWN";
}

const char* nsg_version(void) { return "libnsg sm_100a " __DATE__ " " __TIME__; }

}  // extern "C"
