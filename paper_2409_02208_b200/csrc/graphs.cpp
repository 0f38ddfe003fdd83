// Seeded synthetic graphs standing in for the datasets of BASELINE.json's
// configs (no dataset is available offline; DESIGN.md §Workloads gives the
// exact definitions). Every stream is UniformRng (prng.hpp:11-28).
#include <algorithm>
#include <cmath>
#include <numeric>

#include "cbm_host.hpp"

namespace cbmb {

Csr csr_from_pairs(uint32_t rows, uint32_t cols,
                   std::vector<std::pair<uint32_t, uint32_t>>& pairs) {
  // counting sort by row, then sort + dedup each row (CsrBinaryMatrix::from_coo,
  // csr.cpp:44-66, without its O(nnz log nnz) global sort)
  Csr a;
  a.n_rows = rows;
  a.n_cols = cols;
  std::vector<uint64_t> cnt(size_t(rows) + 1, 0);
  for (auto& p : pairs) {
    if (p.first >= rows || p.second >= cols)
      throw invalid_argument("from_coo: entry (" + std::to_string(p.first) + ", " +
                             std::to_string(p.second) + ") out of range");
    ++cnt[p.first + 1];
  }
  std::partial_sum(cnt.begin(), cnt.end(), cnt.begin());
  std::vector<uint32_t> cols_tmp(pairs.size());
  {
    std::vector<uint64_t> cur(cnt.begin(), cnt.end() - 1);
    for (auto& p : pairs) cols_tmp[cur[p.first]++] = p.second;
  }
  std::vector<std::pair<uint32_t, uint32_t>>().swap(pairs);
  a.row_ptr.assign(size_t(rows) + 1, 0);
  std::vector<uint64_t> keep(rows, 0);
  parallel_for_chunks(rows, int(std::max(1u, std::thread::hardware_concurrency())),
                      [&](size_t lo, size_t hi, int) {
                        for (size_t r = lo; r < hi; ++r) {
                          auto b = cols_tmp.begin() + cnt[r], e = cols_tmp.begin() + cnt[r + 1];
                          std::sort(b, e);
                          keep[r] = uint64_t(std::unique(b, e) - b);
                        }
                      });
  for (uint32_t r = 0; r < rows; ++r) a.row_ptr[r + 1] = a.row_ptr[r] + keep[r];
  a.col_idx.resize(a.row_ptr.back());
  for (uint32_t r = 0; r < rows; ++r)
    std::copy(cols_tmp.begin() + cnt[r], cols_tmp.begin() + cnt[r] + keep[r],
              a.col_idx.begin() + a.row_ptr[r]);
  return a;
}

namespace {

void add_undirected(std::vector<std::pair<uint32_t, uint32_t>>& e, uint32_t u, uint32_t v) {
  e.emplace_back(u, v);
  e.emplace_back(v, u);
}

// Planted communities (cfg[0]: n=4096, size 64, 0.5 / 0.001; cfg[3]:
// n=132,534, size 500, 0.8 / 1e-4). Intra-community pairs are Bernoulli draws
// in order (community, i < j); inter-community pairs are drawn by geometric
// skipping over the row-major sequence of all pairs i < j, ignoring landings
// inside a community. Symmetric, no self-loops.
Csr community(const std::vector<double>& p, uint64_t seed) {
  const uint32_t n = uint32_t(p.at(0)), size = uint32_t(p.at(1));
  const double p_in = p.at(2), p_out = p.at(3);
  Rng rng(seed);
  std::vector<std::pair<uint32_t, uint32_t>> e;
  for (uint32_t c0 = 0; c0 < n; c0 += size) {
    const uint32_t c1 = std::min(n, c0 + size);
    for (uint32_t i = c0; i < c1; ++i)
      for (uint32_t j = i + 1; j < c1; ++j)
        if (rng.unit() < p_in) add_undirected(e, i, j);
  }
  if (p_out > 0 && n > 1) {
    const double lq = std::log1p(-p_out);
    uint64_t i = 0, j = 0;  // current pair (i, j), j > i; start before (0,1)
    bool first = true;
    for (;;) {
      const double u = rng.unit();
      const uint64_t gap = uint64_t(std::floor(std::log1p(-u) / lq));  // failures before success
      uint64_t step = gap + (first ? 1 : 1);
      first = false;
      // advance `step` positions along the pair sequence
      while (i < n - 1) {
        const uint64_t room = (n - 1) - j;  // positions left in row i after j
        if (step <= room) {
          j += step;
          break;
        }
        step -= room;
        ++i;
        j = i;  // next row starts at (i, i+1) after one more step
      }
      if (i >= n - 1) break;
      if (i / size != j / size) add_undirected(e, uint32_t(i), uint32_t(j));
    }
  }
  return csr_from_pairs(n, n, e);
}

// Preferential attachment with triangle closing (cfg[1]: n=19,717, m=2,
// p=0.3). Seed: a triangle on nodes 0..m. Node v then makes m edges to
// distinct earlier nodes drawn from the endpoint pool (probability ~ degree);
// after each such edge (v, t), with probability p_t it also links to a random
// neighbour of t not yet adjacent to v (Holme–Kim triad formation).
Csr pa_triangle(const std::vector<double>& p, uint64_t seed) {
  const uint32_t n = uint32_t(p.at(0)), m = uint32_t(p.at(1));
  const double pt = p.at(2);
  Rng rng(seed);
  std::vector<std::vector<uint32_t>> adj(n);
  std::vector<uint32_t> pool;
  auto linked = [&](uint32_t u, uint32_t v) {
    const auto& a = adj[u].size() < adj[v].size() ? adj[u] : adj[v];
    const uint32_t w = adj[u].size() < adj[v].size() ? v : u;
    return std::find(a.begin(), a.end(), w) != a.end();
  };
  auto link = [&](uint32_t u, uint32_t v) {
    adj[u].push_back(v);
    adj[v].push_back(u);
    pool.push_back(u);
    pool.push_back(v);
  };
  const uint32_t s = std::min(n, m + 1);
  for (uint32_t i = 0; i < s; ++i)
    for (uint32_t j = i + 1; j < s; ++j) link(i, j);
  for (uint32_t v = s; v < n; ++v) {
    uint32_t made = 0, guard = 0;
    while (made < m && guard++ < 64 * m) {
      const uint32_t t = pool[rng.below(pool.size())];
      if (t == v || linked(v, t)) continue;
      link(v, t);
      ++made;
      if (rng.unit() < pt) {
        const auto& nb = adj[t];
        for (int tries = 0; tries < 8; ++tries) {
          const uint32_t u = nb[rng.below(nb.size())];
          if (u != v && !linked(v, u)) {
            link(v, u);
            break;
          }
        }
      }
    }
  }
  std::vector<std::pair<uint32_t, uint32_t>> e;
  for (uint32_t u = 0; u < n; ++u)
    for (uint32_t v : adj[u]) e.emplace_back(u, v);
  return csr_from_pairs(n, n, e);
}

// Clique overlay (cfg[2]: n=235,868, 1.2M groups of 2..10; cfg[4]:
// n=2,449,029, 4M groups of 2..16; Zipf s=1.1). Popularity rank r (1-based)
// has weight r^-s; ranks map to node ids through a seeded Fisher–Yates
// permutation. Each group draws its size k uniformly, then k distinct members
// by inverse-CDF sampling (duplicates redrawn), and adds the k-clique.
Csr clique_overlay(const std::vector<double>& p, uint64_t seed) {
  const uint32_t n = uint32_t(p.at(0));
  const uint64_t groups = uint64_t(p.at(1));
  const uint32_t kmin = uint32_t(p.at(2)), kmax = uint32_t(p.at(3));
  const double s = p.at(4);
  Rng rng(seed);
  std::vector<uint32_t> perm(n);
  std::iota(perm.begin(), perm.end(), 0u);
  for (uint32_t i = n; i > 1; --i) std::swap(perm[i - 1], perm[rng.below(i)]);
  std::vector<double> cdf(n);
  double acc = 0;
  for (uint32_t r = 0; r < n; ++r) {
    acc += std::pow(double(r + 1), -s);
    cdf[r] = acc;
  }
  for (auto& c : cdf) c /= acc;
  std::vector<std::pair<uint32_t, uint32_t>> e;
  e.reserve(size_t(groups) * 40);
  std::vector<uint32_t> mem;
  for (uint64_t g = 0; g < groups; ++g) {
    const uint32_t k = kmin + uint32_t(rng.below(kmax - kmin + 1));
    mem.clear();
    while (mem.size() < k) {
      const double u = rng.unit();
      uint32_t r = uint32_t(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
      if (r >= n) r = n - 1;
      const uint32_t node = perm[r];
      if (std::find(mem.begin(), mem.end(), node) == mem.end()) mem.push_back(node);
    }
    for (uint32_t a = 0; a < k; ++a)
      for (uint32_t b = a + 1; b < k; ++b) add_undirected(e, mem[a], mem[b]);
  }
  return csr_from_pairs(n, n, e);
}

// random_binary (oracles.hpp:167-175): row-major Bernoulli sweep.
Csr random_binary(const std::vector<double>& p, uint64_t seed) {
  const uint32_t rows = uint32_t(p.at(0)), cols = uint32_t(p.at(1));
  const double density = p.at(2);
  Rng rng(seed);
  Csr a;
  a.n_rows = rows;
  a.n_cols = cols;
  a.row_ptr.assign(size_t(rows) + 1, 0);
  for (uint32_t i = 0; i < rows; ++i) {
    for (uint32_t j = 0; j < cols; ++j)
      if (rng.unit() < density) a.col_idx.push_back(j);
    a.row_ptr[i + 1] = a.col_idx.size();
  }
  return a;
}

}  // namespace

Csr gen_graph(const std::string& kind, const std::vector<double>& p, uint64_t seed) {
  if (kind == "community") return community(p, seed);
  if (kind == "pa_triangle") return pa_triangle(p, seed);
  if (kind == "clique_overlay") return clique_overlay(p, seed);
  if (kind == "random_binary") return random_binary(p, seed);
  throw invalid_argument("gen_graph: unknown kind '" + kind + "'");
}

}  // namespace cbmb
