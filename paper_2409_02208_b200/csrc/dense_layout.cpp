// Dense-block layout planner (dense_layout.hpp).
#include "dense_layout.hpp"

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <thread>

#include "cbm_host.hpp"
#include "layout.hpp"

namespace cbmb {

namespace {

struct TilePlan {
  std::vector<uint32_t> cols;     // kDenseK per chunk
  std::vector<uint32_t> masks;    // kDenseRows per chunk
  std::vector<uint32_t> cold_cnt; // per tile row
  std::vector<uint32_t> cold;     // cold columns, row by row
  uint64_t dense = 0;
};

// Row ranges of the tiles (ascending, bounds[0] = 0, bounds.back() = m).
std::vector<uint32_t> tile_bounds(uint32_t m, uint32_t n, const std::vector<uint64_t>& fptr,
                                  const std::vector<uint32_t>& fcol) {
  std::vector<uint32_t> fixed;
  for (uint32_t r = 0; r < m; r += kDenseRows) fixed.push_back(r);
  fixed.push_back(m);
  if (const char* e = std::getenv("CBM_B200_DENSE_FIXED_TILES"))  // dev A/B
    if (std::atoi(e)) return fixed;
  std::vector<uint32_t> b{0};
  std::vector<uint8_t> in_tile(n, 0);
  uint32_t r0 = 0;
  for (uint32_t r = 0; r < m; ++r) {
    const uint64_t len = fptr[r + 1] - fptr[r];
    bool cut = r - r0 >= kDenseRows;
    if (!cut && r > r0 && len >= 8) {
      uint64_t hit = 0;
      for (uint64_t k = fptr[r]; k < fptr[r + 1]; ++k) hit += in_tile[fcol[k]];
      cut = 2 * hit < len;
    }
    if (cut) {
      for (uint32_t q = r0; q < r; ++q)
        for (uint64_t k = fptr[q]; k < fptr[q + 1]; ++k) in_tile[fcol[k]] = 0;
      b.push_back(r);
      r0 = r;
    }
    for (uint64_t k = fptr[r]; k < fptr[r + 1]; ++k) in_tile[fcol[k]] = 1;
  }
  b.push_back(m);
  // structure-free matrices: the scan cuts almost every row; keep the grid
  if (b.size() - 1 > fixed.size() - 1 + (fixed.size() - 1) / 2) return fixed;
  return b;
}

}  // namespace

DenseLayout plan_dense(const cbm_b200_cbm_view& v, uint32_t min_count) {
  DenseLayout D;
  const uint32_t m = v.n_rows, n = v.n_cols;
  D.min_count = min_count ? min_count : 3;
  if (const char* e = std::getenv("CBM_B200_DENSE_MIN"))  // dev tool (threshold sweeps)
    D.min_count = std::max(1, std::atoi(e));
  if (m == 0) return D;
  const float* colscale = v.col_scale ? v.col_scale : v.row_scale;  // (normalized)

  // full rows of the represented matrix (parents first)
  std::vector<uint32_t> bfs;
  {
    std::vector<uint64_t> kp(size_t(m) + 1, 0);
    for (uint32_t x = 0; x < m; ++x)
      if (v.parent[x] != kNoItem) ++kp[v.parent[x] + 1];
    std::partial_sum(kp.begin(), kp.end(), kp.begin());
    std::vector<uint32_t> kids(kp.back());
    std::vector<uint64_t> cur(kp.begin(), kp.end() - 1);
    for (uint32_t x = 0; x < m; ++x)
      if (v.parent[x] != kNoItem) kids[cur[v.parent[x]]++] = x;
    bfs.reserve(m);
    for (uint32_t x = 0; x < m; ++x)
      if (v.parent[x] == kNoItem) bfs.push_back(x);
    for (size_t h = 0; h < bfs.size(); ++h)
      for (uint64_t k = kp[bfs[h]]; k < kp[bfs[h] + 1]; ++k) bfs.push_back(kids[k]);
  }
  std::vector<uint64_t> fptr;
  std::vector<uint32_t> fcol;
  if (!reconstruct_full_rows(v, bfs, fptr, fcol)) return D;   // no full-row form
  std::vector<uint32_t>().swap(bfs);

  // Tile boundaries. A tile is <= kDenseRows consecutive rows; a fixed grid
  // of 128 cuts communities in two, and a tile straddling two communities
  // carries both column sets half empty. The greedy scan closes a tile when
  // the next row places under half of its entries on columns the tile already
  // holds (a new community starts); matrices without that structure (the
  // scan would shred them into slivers) keep the fixed grid.
  std::vector<uint32_t> bounds = tile_bounds(m, n, fptr, fcol);
  D.n_tiles = uint32_t(bounds.size() - 1);
  std::vector<TilePlan> plans(D.n_tiles);
  const int threads = int(std::max(1u, std::thread::hardware_concurrency()));
  std::atomic<uint32_t> next{0};
  const uint32_t mc = D.min_count;
  auto worker = [&]() {
    std::vector<uint8_t> cnt(n, 0);      // <= kDenseRows entries per column per tile
    std::vector<uint32_t> pos(n, 0);     // dense column -> chunk slot (+1)
    std::vector<uint32_t> touched, dense;
    for (uint32_t t; (t = next.fetch_add(1)) < D.n_tiles;) {
      TilePlan& P = plans[t];
      const uint32_t r0 = bounds[t], r1 = bounds[t + 1];
      touched.clear();
      for (uint32_t r = r0; r < r1; ++r)
        for (uint64_t k = fptr[r]; k < fptr[r + 1]; ++k) {
          const uint32_t c = fcol[k];
          if (cnt[c]++ == 0) touched.push_back(c);
        }
      dense.clear();
      for (uint32_t c : touched)
        if (cnt[c] >= mc) dense.push_back(c);
      if (dense.size() > size_t(kDenseMaxChunks) * kDenseK) {
        // a tile holding a hub row shares thousands of columns with it: keep
        // the most shared ones (one CTA multiplies a whole unit, so a long
        // unit would serialise the launch), the rest stay cold
        std::stable_sort(dense.begin(), dense.end(),
                         [&](uint32_t a, uint32_t b) { return cnt[a] > cnt[b]; });
        dense.resize(size_t(kDenseMaxChunks) * kDenseK);
      }
      std::sort(dense.begin(), dense.end());
      const uint32_t nch = uint32_t((dense.size() + kDenseK - 1) / kDenseK);
      P.cols.assign(size_t(nch) * kDenseK, 0);
      P.masks.assign(size_t(nch) * kDenseRows, 0);
      for (size_t i = 0; i < dense.size(); ++i) {
        P.cols[i] = dense[i];
        pos[dense[i]] = uint32_t(i) + 1;
      }
      for (size_t i = dense.size(); i < P.cols.size(); ++i) P.cols[i] = dense.back();  // pad
      P.cold_cnt.assign(r1 - r0, 0);
      for (uint32_t r = r0; r < r1; ++r)
        for (uint64_t k = fptr[r]; k < fptr[r + 1]; ++k) {
          const uint32_t c = fcol[k];
          if (pos[c]) {
            const uint32_t i = pos[c] - 1;
            P.masks[size_t(i / kDenseK) * kDenseRows + (r - r0)] |= 1u << (i % kDenseK);
            ++P.dense;
          } else {
            P.cold.push_back(c);
            ++P.cold_cnt[r - r0];
          }
        }
      for (uint32_t c : touched) cnt[c] = 0;
      for (uint32_t c : dense) pos[c] = 0;
    }
  };
  {
    std::vector<std::thread> pool;
    for (int i = 1; i < threads; ++i) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
  }
  std::vector<uint32_t>().swap(fcol);
  std::vector<uint64_t>().swap(fptr);

  // tiles in schedule order (static round-robin over CTAs): the heavy tiles
  // (more than twice the mean chunk count) first, then the rest in row
  // order, so that neighbouring tiles, which share X rows, run at the same
  // time and meet those rows in L2
  std::vector<uint32_t> order(D.n_tiles);
  std::iota(order.begin(), order.end(), 0u);
  {
    uint64_t total = 0;
    for (const auto& P : plans) total += P.cols.size();
    const double heavy = 2.0 * double(total) / double(std::max<uint32_t>(1, D.n_tiles));
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
      const bool ha = double(plans[a].cols.size()) > heavy, hb = double(plans[b].cols.size()) > heavy;
      if (ha != hb) return ha;
      return ha ? plans[a].cols.size() > plans[b].cols.size() : false;
    });
  }
  D.tiles.reserve(size_t(D.n_tiles) * 4);
  for (uint32_t t : order) {
    const TilePlan& P = plans[t];
    const uint32_t r0 = bounds[t];
    D.tiles.push_back(r0);
    D.tiles.push_back(bounds[t + 1] - r0);
    D.tiles.push_back(uint32_t(D.n_chunks));
    D.tiles.push_back(uint32_t(P.cols.size() / kDenseK));
    D.n_chunks += P.cols.size() / kDenseK;
    for (size_t q = 0; q < P.cols.size() / kDenseK; ++q) {
      const uint32_t* cc = P.cols.data() + q * kDenseK;
      D.meta.insert(D.meta.end(), cc, cc + kDenseK);
      for (uint32_t k = 0; k < kDenseK; ++k) {
        const float sc = v.is_normalized ? colscale[cc[k]] : 1.0f;
        uint32_t bits;
        std::memcpy(&bits, &sc, 4);
        D.meta.push_back(bits);
      }
      const uint32_t* mm = P.masks.data() + q * kDenseRows;
      D.meta.insert(D.meta.end(), mm, mm + kDenseRows);
    }
    D.dense_entries += P.dense;
    D.padded_slots += uint64_t(P.cols.size()) * kDenseRows;
  }
  if (D.n_chunks >= 0xFFFFFFFFull) return DenseLayout{};
  // cold rows in row order (tiles cover consecutive rows)
  D.cold_row_ptr.assign(size_t(m) + 1, 0);
  for (uint32_t t = 0; t < D.n_tiles; ++t)
    for (uint32_t i = 0; i < plans[t].cold_cnt.size(); ++i)
      D.cold_row_ptr[size_t(bounds[t]) + i + 1] = plans[t].cold_cnt[i];
  std::partial_sum(D.cold_row_ptr.begin(), D.cold_row_ptr.end(), D.cold_row_ptr.begin());
  D.cold_entries = D.cold_row_ptr[m];
  D.cold_col.resize(D.cold_entries);
  for (uint32_t t = 0; t < D.n_tiles; ++t)
    std::copy(plans[t].cold.begin(), plans[t].cold.end(),
              D.cold_col.begin() + D.cold_row_ptr[bounds[t]]);
  D.cold_val.resize(D.cold_entries);
  const bool norm = v.is_normalized != 0;
  for (uint64_t k = 0; k < D.cold_entries; ++k)
    D.cold_val[k] = norm ? colscale[D.cold_col[k]] : 1.0f;
  D.cold_parent.assign(m, kNoItem);
  D.ok = true;
  return D;
}

}  // namespace cbmb
