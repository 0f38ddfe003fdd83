// Host-side types and algorithms of the B200 CBM library (C++20).
//
// The reference keeps everything on the CPU (proj/src/*.cpp). Here only the
// construction (builder) and the device-layout planning stay on the host; the
// multiply runs in paper_2409_02208_b200/csrc/cbm_kernels.cu.
#pragma once

#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "errors.hpp"

namespace cbmb {

inline constexpr uint32_t kVirtual = 0xFFFFFFFFu;  // kVirtualParent (types.hpp:19)

// Pattern CSR (CsrBinaryMatrix, csr.hpp:14-40).
struct Csr {
  uint32_t n_rows = 0;
  uint32_t n_cols = 0;
  std::vector<uint64_t> row_ptr{0};
  std::vector<uint32_t> col_idx;

  uint64_t nnz() const { return row_ptr.back(); }
  uint64_t row_nnz(uint32_t r) const { return row_ptr[r + 1] - row_ptr[r]; }
  const uint32_t* row(uint32_t r) const { return col_idx.data() + row_ptr[r]; }
};

// Structural check of csr.cpp:12-33 (sizes, monotone offsets, strictly
// increasing in-range columns). Throws cbmb::invalid_argument.
void validate_csr(uint32_t n_rows, uint32_t n_cols, const uint64_t* row_ptr,
                  const uint32_t* col_idx);

// Built CBM (CbmMatrix + CompressionChain, builder.hpp:26-74), f32 values.
struct HostCbm {
  uint32_t n_rows = 0;
  uint32_t n_cols = 0;
  uint64_t alpha = 0;
  bool normalized = false;
  std::vector<uint32_t> parent;
  std::vector<uint32_t> topo_order;
  std::vector<uint32_t> root_children;
  std::vector<uint64_t> branch_ptr;
  std::vector<uint64_t> row_ptr{0};
  std::vector<uint32_t> col_idx;
  std::vector<float> values;
  std::vector<float> row_scale;
  // build statistics
  double t_edges = 0, t_arb = 0, t_deltas = 0, t_total = 0;
  uint64_t candidate_edges = 0;
  uint32_t rounds = 0;
};

// DFS-preorder chain from parent links (CompressionChain::from_parents,
// builder.cpp:16-64): children visited in ascending row id, every root branch
// a contiguous topo segment. Throws cbmb::invalid_argument on bad links/cycles.
void chain_from_parents(HostCbm& c);

// Full construction (build_cbm / build_cbm_normalized, builder.cpp:394-429).
// algo 0: heap-based Edmonds (default), 1: round-synchronous restatement.
HostCbm build_cbm(const Csr& a, uint64_t alpha, int threads, int algo = 0);
HostCbm build_cbm_normalized(const Csr& a, uint64_t alpha, int threads,
                             bool degrees_from_original, int algo = 0);

// CBM1 container (io.hpp:44-57, io.cpp:198-382); throws format_error.
void save_cbm1(const HostCbm& c, const std::string& path);
HostCbm load_cbm1(const std::string& path);

// ---- internals exposed for tests ------------------------------------------

// Candidate edges in dst-major CSR: for destination row x, entries
// [ptr[x], ptr[x+1]) hold (src node, weight), src ascending, the virtual edge
// (src 0, weight nnz(a_x)) first. Node ids: 0 = virtual root, row r = r + 1.
struct EdgeLists {
  std::vector<uint64_t> ptr;
  std::vector<uint32_t> src;
  std::vector<uint32_t> w;
};
EdgeLists candidate_edges(const Csr& a, uint64_t alpha, int threads);

// Chu-Liu/Edmonds with the reference's deterministic tie rules; returns
// parent[m] (kVirtual for roots). `rounds` receives the contraction count.
std::vector<uint32_t> min_arborescence(const EdgeLists& e, uint32_t m, int threads,
                                       uint32_t* rounds);
// Same arborescence with mergeable heaps, O(E log E) (arborescence.cpp).
std::vector<uint32_t> min_arborescence_heap(const EdgeLists& e, uint32_t m, uint32_t* rounds,
                                            int threads = 1);

// ---- parallel helper (the reference's parallel_chunks, parallel.hpp:13-32)
template <typename Fn>
void parallel_for_chunks(size_t n, int threads, Fn&& fn);

// ---- workload generators (UniformRng semantics, prng.hpp:11-28) -----------
class Rng {
 public:
  explicit Rng(uint64_t seed) : g_(seed) {}
  uint64_t bits() { return g_(); }
  double unit() { return double(g_() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t n) { return n ? g_() % n : 0; }

 private:
  std::mt19937_64 g_;
};

Csr gen_graph(const std::string& kind, const std::vector<double>& p, uint64_t seed);
Csr csr_from_pairs(uint32_t rows, uint32_t cols,
                   std::vector<std::pair<uint32_t, uint32_t>>& pairs);

}  // namespace cbmb

#include <thread>

namespace cbmb {
template <typename Fn>
void parallel_for_chunks(size_t n, int threads, Fn&& fn) {
  if (n == 0) return;
  size_t parts = threads <= 1 ? 1 : size_t(threads);
  if (parts > n) parts = n;
  if (parts == 1) {
    fn(size_t(0), n, 0);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(parts - 1);
  for (size_t t = 1; t < parts; ++t)
    pool.emplace_back([&fn, n, parts, t] { fn(n * t / parts, n * (t + 1) / parts, int(t)); });
  fn(0, n / parts, 0);
  for (auto& th : pool) th.join();
}
}  // namespace cbmb
