// oracle/oracle.cpp — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously-correct CPU implementation of the nine per-window network
// quantities of the Anonymized Network Sensing Graph Challenge, as restated by
// arXiv 2509.03653 ("Combining Performance and Productivity ...").  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load
// this library.  It shares no code, header, table or helper with the CUDA path under
// paper_2509_03653_b200/ and must never be reached from it.
//
// Citations: "P:n" = /root/reference/PAPER.md line n (Table 2 "tab:graph_operations",
// lines 171-193; caption line 173 defines A_t as the traffic matrix and the destination
// mirrors: "For reverse operations simply replace `src` and `dst`").
//
// Definition (readings R1-R6): for window w the packet multiset M_w holds the
// packets [w*W, min((w+1)*W, n)).  A_t(i,j) = #{p in M_w : src_p = i, dst_p = j}, i.e.
// raw packets of weight 1 (reading R2), directed (R5), self-loops ordinary entries (R4).
// Output row, nine u64 in north_star order:
//   0 valid packets            1^T A_t 1
//   1 unique links             1^T |A_t|_0 1
//   2 max link packets         max(A_t)
//   3 unique sources           1^T |A_t 1|_0
//   4 max source packets       max(A_t 1)
//   5 max source fan-out       max(|A_t|_0 1)
//   6 unique destinations      mirror of 3
//   7 max destination packets  mirror of 4, max(1^T A_t)
//   8 max destination fan-in   mirror of 5, max(1^T|A_t|_0)
// Any max over an empty set is 0 (reading R7).
//
// Procedures:
//   O1 (nsg_oracle_window_stats_map): the literal definition with std::map, step by step
//      in Table 2's order: build A_t as a map (i,j) -> count ("Link packets from i
//      to j"), then the whole-matrix rows, then row sums / row nnz and the
//      column mirrors.
//   O2 (nsg_oracle_window_stats_sort): the same definition reached through a library sort
//      (std::sort) and run-length scans; a thread pool over windows.  Windows are
//      independent, so the thread count cannot change any result.
//   O1w (nsg_oracle_window_stats_weighted): O1 on weighted rows (src, dst, n_packets), the paper's
//      three-column frame; SURVEY §8(f) row f4a.
//   O1d (nsg_oracle_window_distributions): the vector-valued rows of Table 2 (link packets,
//      row sums / nnz and their column mirrors) and the four globally-unique-IP set counts, from
//      the same std::map definition.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <thread>
#include <utility>
#include <vector>

namespace {

constexpr int kStats = 9;

uint64_t num_windows(uint64_t n, uint64_t window) { return n == 0 ? 0 : (n + window - 1) / window; }

// ---- O1: literal definition over std::map --------------------------------------------
void window_map(const uint32_t* src, const uint32_t* dst, uint64_t len, uint64_t* out) {
  // A_t(i,j): "Link packets from i to j" = A_t(i,j); raw rows have weight 1.
  std::map<std::pair<uint32_t, uint32_t>, uint64_t> A;
  for (uint64_t p = 0; p < len; ++p) A[{src[p], dst[p]}] += 1;

  uint64_t valid = 0, max_link = 0;
  for (const auto& e : A) {
    valid += e.second;                                   // P:180  sum_i sum_j A_t(i,j)
    max_link = std::max(max_link, e.second);             // P:183  max_ij A_t(i,j)
  }
  const uint64_t unique_links = A.size();                // P:181  sum_ij |A_t(i,j)|_0

  // Row sums A_t 1 and row nnz |A_t|_0 1; column mirrors.
  std::map<uint32_t, uint64_t> row_sum, row_nnz, col_sum, col_nnz;
  for (const auto& e : A) {
    row_sum[e.first.first] += e.second;
    row_nnz[e.first.first] += 1;
    col_sum[e.first.second] += e.second;
    col_nnz[e.first.second] += 1;
  }
  auto max_of = [](const std::map<uint32_t, uint64_t>& m) {
    uint64_t r = 0;
    for (const auto& e : m) r = std::max(r, e.second);
    return r;
  };
  out[0] = valid;
  out[1] = unique_links;
  out[2] = max_link;
  out[3] = row_sum.size();      // P:184 1^T |A_t 1|_0 : rows whose sum is nonzero
  out[4] = max_of(row_sum);     // P:186 max(A_t 1)
  out[5] = max_of(row_nnz);     // P:188 max(|A_t|_0 1)
  out[6] = col_sum.size();      // mirror of P:184
  out[7] = max_of(col_sum);     // mirror of P:186
  out[8] = max_of(col_nnz);     // mirror of P:188
}

// ---- O2: sort + run-length scan ------------------------------------------------------
// Sorting the keys (major, minor) makes every distinct (major, minor) pair a run (a
// nonzero of A_t, run length = its value) and every distinct major a run of runs (a
// nonzero row: its length is the row sum, its number of sub-runs the row nnz).
struct Side { uint64_t total, distinct_pairs, max_pair, distinct_major, max_major_sum, max_major_nnz; };

Side scan_sorted(std::vector<uint64_t>& keys) {
  std::sort(keys.begin(), keys.end());
  Side s{0, 0, 0, 0, 0, 0};
  const size_t n = keys.size();
  size_t i = 0;
  while (i < n) {
    const uint32_t major = uint32_t(keys[i] >> 32);
    uint64_t sum = 0, nnz = 0;
    while (i < n && uint32_t(keys[i] >> 32) == major) {
      size_t j = i;
      while (j < n && keys[j] == keys[i]) ++j;
      const uint64_t c = j - i;                           // A_t(i,j) for this pair
      s.total += c;
      s.distinct_pairs += 1;
      s.max_pair = std::max(s.max_pair, c);
      sum += c;
      nnz += 1;
      i = j;
    }
    s.distinct_major += 1;
    s.max_major_sum = std::max(s.max_major_sum, sum);
    s.max_major_nnz = std::max(s.max_major_nnz, nnz);
  }
  return s;
}

void window_sort(const uint32_t* src, const uint32_t* dst, uint64_t len, uint64_t* out) {
  std::vector<uint64_t> keys(len);
  for (uint64_t p = 0; p < len; ++p) keys[p] = (uint64_t(src[p]) << 32) | dst[p];
  const Side s = scan_sorted(keys);                      // rows of A_t (sources)
  for (uint64_t p = 0; p < len; ++p) keys[p] = (uint64_t(dst[p]) << 32) | src[p];
  const Side d = scan_sorted(keys);                      // columns of A_t (P:173 mirror)
  out[0] = s.total;        // 1^T A_t 1: the sum of all run lengths
  out[1] = s.distinct_pairs;
  out[2] = s.max_pair;
  out[3] = s.distinct_major;
  out[4] = s.max_major_sum;
  out[5] = s.max_major_nnz;
  out[6] = d.distinct_major;
  out[7] = d.max_major_sum;
  out[8] = d.max_major_nnz;
  // Self-check: the transposed scan sees the same nonzeros.
  if (d.total != s.total || d.distinct_pairs != s.distinct_pairs || d.max_pair != s.max_pair) out[0] = ~0ull;
}

// ---- O1w: weighted (aggregated) input rows ----------------------------
// The paper's frame has three columns src, dst, n_packets and sums n_packets for the valid
// packets.  With row p carrying weight n_p, A_t(i,j) = sum of n_p over the window's rows with
// src = i, dst = j; a link is a nonzero of A_t (|A_t|_0), so a row of weight 0 adds nothing
// (reading R14).  Everything else is Table 2 on this A_t, as O1.  Raw packets are the
// special case n_p = 1 (reading R2); SPEC S:142 states the raw / aggregated equivalence.
void window_map_weighted(const uint32_t* src, const uint32_t* dst, const uint32_t* wgt, uint64_t len, uint64_t* out) {
  std::map<std::pair<uint32_t, uint32_t>, uint64_t> A;
  for (uint64_t p = 0; p < len; ++p)
    if (wgt[p] != 0) A[{src[p], dst[p]}] += wgt[p];
  uint64_t valid = 0, max_link = 0;
  for (const auto& e : A) {
    valid += e.second;
    max_link = std::max(max_link, e.second);
  }
  std::map<uint32_t, uint64_t> row_sum, row_nnz, col_sum, col_nnz;
  for (const auto& e : A) {
    row_sum[e.first.first] += e.second;
    row_nnz[e.first.first] += 1;
    col_sum[e.first.second] += e.second;
    col_nnz[e.first.second] += 1;
  }
  auto max_of = [](const std::map<uint32_t, uint64_t>& m) {
    uint64_t r = 0;
    for (const auto& e : m) r = std::max(r, e.second);
    return r;
  };
  out[0] = valid;             // P:180 df['n_packets'].sum()
  out[1] = A.size();
  out[2] = max_link;
  out[3] = row_sum.size();
  out[4] = max_of(row_sum);
  out[5] = max_of(row_nnz);
  out[6] = col_sum.size();    // mirrors
  out[7] = max_of(col_sum);
  out[8] = max_of(col_nnz);
}

// ---- O1d: the vector-valued rows of Table 2 and the globally unique IPs ----
// For window w, literally from the definition, in the same std::map form as O1:
//   links       the nonzeros of A_t: (key = i<<32 | j, A_t(i,j))    P:182 "Link packets from i to j"
//   sources     per nonzero row i: (i, (A_t 1)_i, (|A_t|_0 1)_i)     P:185 "Packets from source i",
//                                                                    P:187 "Source fan-out from i"
//   destinations the column mirrors (1^T A_t)_j, (1^T |A_t|_0)_j     P:173 "replace src and dst"
//   ip sets     {|S u D|, |S \ D|, |D \ S|, |S n D|} with S = sources, D = destinations of the window:
//               P:209 "Globally unique IP addresses ... unique() ... on each column and subsequently
//               removing common values across the two unique sets"; all four counts (SPEC S:239-245,
//               S:272), reading R13.
// Every vector is written in ascending key order (std::map order) at offset w*window of
// its array; cnt[w] = {links, sources, destinations}.
struct DistOut {
  uint64_t* link_key; uint64_t* link_packets;
  uint32_t* src_node; uint64_t* src_packets; uint64_t* src_fan;
  uint32_t* dst_node; uint64_t* dst_packets; uint64_t* dst_fan;
  uint64_t* cnt;      // [nw][3]
  uint64_t* ip_sets;  // [nw][4]
};

// wgt: NULL for raw packets (weight 1), else the rows' n_packets (O1w's reading: a row of weight 0 adds
// nothing, so it creates no link and no node).
void window_dist(const uint32_t* src, const uint32_t* dst, const uint32_t* wgt, uint64_t len, uint64_t w,
                 uint64_t window, const DistOut& o) {
  std::map<std::pair<uint32_t, uint32_t>, uint64_t> A;             // A_t(i,j)
  for (uint64_t p = 0; p < len; ++p)
    if (!wgt || wgt[p] != 0) A[{src[p], dst[p]}] += wgt ? wgt[p] : 1;
  std::map<uint32_t, std::pair<uint64_t, uint64_t>> row, col;       // (sum, nnz) per row / column
  for (const auto& e : A) {
    row[e.first.first].first += e.second;   // (A_t 1)_i
    row[e.first.first].second += 1;         // (|A_t|_0 1)_i
    col[e.first.second].first += e.second;  // mirror
    col[e.first.second].second += 1;
  }
  const uint64_t b = w * window;
  uint64_t k = 0;
  for (const auto& e : A) {
    o.link_key[b + k] = (uint64_t(e.first.first) << 32) | e.first.second;
    o.link_packets[b + k] = e.second;
    ++k;
  }
  k = 0;
  for (const auto& e : row) { o.src_node[b + k] = e.first; o.src_packets[b + k] = e.second.first; o.src_fan[b + k] = e.second.second; ++k; }
  k = 0;
  for (const auto& e : col) { o.dst_node[b + k] = e.first; o.dst_packets[b + k] = e.second.first; o.dst_fan[b + k] = e.second.second; ++k; }
  o.cnt[w * 3 + 0] = A.size();
  o.cnt[w * 3 + 1] = row.size();
  o.cnt[w * 3 + 2] = col.size();
  // The two unique sets and their common values.
  uint64_t both = 0;
  for (const auto& e : row) both += col.count(e.first);
  o.ip_sets[w * 4 + 0] = row.size() + col.size() - both;  // |S u D|
  o.ip_sets[w * 4 + 1] = row.size() - both;               // |S \ D|
  o.ip_sets[w * 4 + 2] = col.size() - both;               // |D \ S|
  o.ip_sets[w * 4 + 3] = both;                            // |S n D|
}

using WindowFn = void (*)(const uint32_t*, const uint32_t*, uint64_t, uint64_t*);

int run_windows(WindowFn fn, const uint32_t* src, const uint32_t* dst, uint64_t n, uint64_t window,
                uint64_t* out, int n_threads) {
  if (window == 0) return 1;
  if (n == 0) return 0;
  if (!src || !dst || !out) return 1;
  const uint64_t nw = num_windows(n, window);
  unsigned T = n_threads > 0 ? unsigned(n_threads) : std::max(1u, std::thread::hardware_concurrency());
  if (T > nw) T = unsigned(nw);
  auto worker = [&](unsigned t) {
    for (uint64_t w = t; w < nw; w += T) {
      const uint64_t b = w * window;
      const uint64_t len = std::min(window, n - b);
      fn(src + b, dst + b, len, out + w * kStats);
    }
  };
  if (T <= 1) {
    worker(0);
  } else {
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t) pool.emplace_back(worker, t);
    for (auto& th : pool) th.join();
  }
  return 0;
}

}  // namespace

extern "C" {

// Returns 0 on success, 1 on invalid arguments.  out is host [ceil(n/window)][9] u64.
int nsg_oracle_window_stats_map(const uint32_t* src, const uint32_t* dst, uint64_t n, uint64_t window,
                                uint64_t* out, int n_threads) {
  return run_windows(window_map, src, dst, n, window, out, n_threads);
}

int nsg_oracle_window_stats_sort(const uint32_t* src, const uint32_t* dst, uint64_t n, uint64_t window,
                                 uint64_t* out, int n_threads) {
  return run_windows(window_sort, src, dst, n, window, out, n_threads);
}

// Weighted rows: wgt[n] u32 weights (n_packets).  Returns 0 on success, 1 on invalid arguments.
int nsg_oracle_window_stats_weighted(const uint32_t* src, const uint32_t* dst, const uint32_t* wgt, uint64_t n,
                                     uint64_t window, uint64_t* out, int n_threads) {
  if (window == 0) return 1;
  if (n == 0) return 0;
  if (!src || !dst || !wgt || !out) return 1;
  const uint64_t nw = num_windows(n, window);
  unsigned T = n_threads > 0 ? unsigned(n_threads) : std::max(1u, std::thread::hardware_concurrency());
  if (T > nw) T = unsigned(nw);
  auto worker = [&](unsigned t) {
    for (uint64_t w = t; w < nw; w += T) {
      const uint64_t b = w * window;
      window_map_weighted(src + b, dst + b, wgt + b, std::min(window, n - b), out + w * kStats);
    }
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < T; ++t) pool.emplace_back(worker, t);
  worker(0);
  for (auto& th : pool) th.join();
  return 0;
}

// Returns 0 on success, 1 on invalid arguments.  Every vector array is host [n] (window w's entries at
// [w*window, w*window + cnt)); cnt is host [nw][3], ip_sets host [nw][4]; wgt host [n] or NULL (raw packets).
int nsg_oracle_window_distributions(const uint32_t* src, const uint32_t* dst, const uint32_t* wgt, uint64_t n,
                                    uint64_t window, uint64_t* link_key, uint64_t* link_packets, uint32_t* src_node,
                                    uint64_t* src_packets, uint64_t* src_fan, uint32_t* dst_node,
                                    uint64_t* dst_packets, uint64_t* dst_fan, uint64_t* cnt, uint64_t* ip_sets,
                                    int n_threads) {
  if (window == 0) return 1;
  if (n == 0) return 0;
  if (!src || !dst || !link_key || !link_packets || !src_node || !src_packets || !src_fan || !dst_node ||
      !dst_packets || !dst_fan || !cnt || !ip_sets)
    return 1;
  const DistOut o{link_key, link_packets, src_node, src_packets, src_fan, dst_node, dst_packets, dst_fan, cnt, ip_sets};
  const uint64_t nw = num_windows(n, window);
  unsigned T = n_threads > 0 ? unsigned(n_threads) : std::max(1u, std::thread::hardware_concurrency());
  if (T > nw) T = unsigned(nw);
  auto worker = [&](unsigned t) {
    for (uint64_t w = t; w < nw; w += T) {
      const uint64_t b = w * window;
      window_dist(src + b, dst + b, wgt ? wgt + b : nullptr, std::min(window, n - b), w, window, o);
    }
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < T; ++t) pool.emplace_back(worker, t);
  worker(0);
  for (auto& th : pool) th.join();
  return 0;
}

unsigned nsg_oracle_hardware_threads(void) { return std::max(1u, std::thread::hardware_concurrency()); }

}  // extern "C"
