#include "tile_layout.hpp"

#include <algorithm>
#include <numeric>

#include "errors.hpp"

namespace cbmb {

namespace {
constexpr uint32_t kVirt = 0xFFFFFFFFu;
constexpr uint32_t kSign = 0x80000000u;

}  // namespace

TileLayout plan_tiles(const cbm_b200_cbm_view& v, uint32_t rows_cap, uint32_t stage_cap,
                      uint32_t num_sms, uint32_t flatten_gain) {
  const uint32_t m = v.n_rows;
  const bool norm = v.is_normalized != 0;
  TileLayout T;
  if (v.n_cols >= (1u << 30)) throw invalid_argument("tiles: too many columns");
  if (rows_cap == 0) {  // ~2 blocks per SM, a power of two in [64, 512]
    const uint64_t want = (uint64_t(m) + 2ull * num_sms - 1) / (2ull * num_sms);
    rows_cap = 64;
    while (rows_cap < 512 && rows_cap < want) rows_cap *= 2;
  }
  if (stage_cap == 0) stage_cap = 600;
  rows_cap = std::max<uint32_t>(rows_cap, 1);
  T.row_cap = rows_cap;
  T.stage_cap = stage_cap;

  // children, BFS order (parents first)
  std::vector<uint32_t> kp(size_t(m) + 1, 0);
  for (uint32_t x = 0; x < m; ++x)
    if (v.parent[x] != kVirt) ++kp[v.parent[x] + 1];
  std::partial_sum(kp.begin(), kp.end(), kp.begin());
  std::vector<uint32_t> kids(kp[m]);
  {
    std::vector<uint32_t> cur(kp.begin(), kp.end() - 1);
    for (uint32_t x = 0; x < m; ++x)
      if (v.parent[x] != kVirt) kids[cur[v.parent[x]]++] = x;
  }
  std::vector<uint32_t> bfs;
  bfs.reserve(m);
  for (uint32_t x = 0; x < m; ++x)
    if (v.parent[x] == kVirt) bfs.push_back(x);
  for (size_t h = 0; h < bfs.size(); ++h)
    for (uint32_t k = kp[bfs[h]]; k < kp[bfs[h] + 1]; ++k) bfs.push_back(kids[k]);

  // rows whose delta row saves fewer than flatten_gain entries over their full
  // row are summed directly (cut from their parent, as plan_layout does)
  std::vector<uint8_t> cut(m, 0);
  if (flatten_gain > 0) {
    std::vector<uint64_t> nA(m, 0);
    for (uint32_t x : bfs) {
      uint64_t plus = 0, minus = 0;
      for (uint64_t k = v.row_ptr[x]; k < v.row_ptr[x + 1]; ++k)
        (v.values[k] < 0.0f ? minus : plus) += 1;
      const uint32_t p = v.parent[x];
      nA[x] = p == kVirt ? plus : nA[p] + plus - minus;
      if (p != kVirt && nA[x] < plus + minus + flatten_gain) {
        cut[x] = 1;
        ++T.n_flat;
      }
    }
  }
  // split trees bigger than rows_cap: children with the largest open subtrees
  // are cut off (each becomes the root of its own piece)
  std::vector<uint32_t> open(m, 1);
  std::vector<std::pair<uint32_t, uint32_t>> ch;
  for (size_t i = m; i-- > 0;) {
    const uint32_t x = bfs[i];
    uint64_t sz = 1;
    ch.clear();
    for (uint32_t k = kp[x]; k < kp[x + 1]; ++k) {
      if (cut[kids[k]]) continue;
      sz += open[kids[k]];
      ch.emplace_back(open[kids[k]], kids[k]);
    }
    if (sz > rows_cap) {
      std::sort(ch.begin(), ch.end(), [](auto a, auto b) {
        return a.first != b.first ? a.first > b.first : a.second < b.second;
      });
      for (auto [s, c] : ch) {
        if (sz <= rows_cap) break;
        cut[c] = 1;
        sz -= s;
        ++T.n_cut;
      }
    }
    open[x] = uint32_t(sz);
  }
  // pieces (rooted at forest roots and cut rows), depth inside the piece
  std::vector<uint32_t> piece(m), pdepth(m, 0);
  for (uint32_t x : bfs) {
    const uint32_t p = v.parent[x];
    if (p == kVirt || cut[x]) {
      piece[x] = x;
      pdepth[x] = 0;
    } else {
      piece[x] = piece[p];
      pdepth[x] = pdepth[p] + 1;
    }
  }
  std::vector<uint32_t> roots;  // piece roots by row id
  for (uint32_t x = 0; x < m; ++x)
    if (piece[x] == x) roots.push_back(x);
  // pack consecutive pieces into blocks of <= rows_cap rows
  std::vector<uint32_t> block_of_piece(m, kVirt);
  std::vector<uint32_t> block_rows_n;
  for (uint32_t r : roots) {
    if (block_rows_n.empty() || block_rows_n.back() + open[r] > rows_cap)
      block_rows_n.push_back(0);
    block_of_piece[r] = uint32_t(block_rows_n.size() - 1);
    block_rows_n.back() += open[r];
  }
  const uint32_t nb = uint32_t(block_rows_n.size());
  // rows of each block: by depth inside the piece, then row id
  std::vector<uint32_t> bptr(size_t(nb) + 1, 0);
  for (uint32_t b = 0; b < nb; ++b) bptr[b + 1] = bptr[b] + block_rows_n[b];
  std::vector<uint32_t> brows(m);
  {
    std::vector<uint32_t> cur(bptr.begin(), bptr.end() - 1);
    for (uint32_t x = 0; x < m; ++x) brows[cur[block_of_piece[piece[x]]]++] = x;
  }
  std::vector<uint32_t> local(m);
  for (uint32_t b = 0; b < nb; ++b) {
    auto* lo = brows.data() + bptr[b];
    auto* hi = brows.data() + bptr[b + 1];
    std::sort(lo, hi, [&](uint32_t a, uint32_t c) {
      return pdepth[a] != pdepth[c] ? pdepth[a] < pdepth[c] : a < c;
    });
    for (auto* q = lo; q < hi; ++q) local[*q] = uint32_t(q - lo);
  }
  // interior rows (an uncut child reads their unscaled row)
  std::vector<uint32_t> slot(m, kTileNone);
  for (uint32_t b = 0; b < nb; ++b)
    for (uint32_t i = bptr[b]; i < bptr[b + 1]; ++i) {
      const uint32_t x = brows[i];
      bool interior = false;
      for (uint32_t k = kp[x]; k < kp[x + 1] && !interior; ++k) interior = !cut[kids[k]];
      if (interior) slot[x] = T.n_interior++;
    }

  // full rows of the cut rows, parents first (reconstruct_rows, builder.cpp:452-490),
  // materialised only along the paths that lead to a cut row
  std::vector<uint8_t> need(cut.begin(), cut.end());
  for (size_t i = m; i-- > 0;) {
    const uint32_t x = bfs[i];
    if (need[x] && v.parent[x] != kVirt) need[v.parent[x]] = 1;
  }
  std::vector<std::vector<uint32_t>> full(m);
  for (uint32_t x : bfs) {
    if (!need[x]) continue;
    const uint32_t p = v.parent[x];
    static const std::vector<uint32_t> kEmpty;
    const std::vector<uint32_t>& base = p == kVirt ? kEmpty : full[p];
    std::vector<uint32_t>& out = full[x];
    uint64_t k = v.row_ptr[x];
    const uint64_t ke = v.row_ptr[x + 1];
    size_t a = 0;
    while (a < base.size() || k < ke) {  // (parent + plus) - minus, ascending
      if (k == ke || (a < base.size() && base[a] < v.col_idx[k])) {
        out.push_back(base[a++]);
      } else if (a == base.size() || v.col_idx[k] < base[a]) {
        if (v.values[k] < 0.0f) throw inconsistent_rows();  // removes a missing column
        out.push_back(v.col_idx[k]);
        ++k;
      } else {
        if (v.values[k] > 0.0f) throw inconsistent_rows();  // adds a present column
        ++a;
        ++k;
      }
    }
  }
  for (uint32_t x = 0; x < m; ++x)
    if (!cut[x]) std::vector<uint32_t>().swap(full[x]);  // keep the cut rows only

  // effective delta rows: the CBM's (column | sign), or the full row for cut rows
  auto row_entries = [&](uint32_t x, std::vector<uint32_t>& out) {
    out.clear();
    if (cut[x]) {
      out.assign(full[x].begin(), full[x].end());
    } else {
      for (uint64_t k = v.row_ptr[x]; k < v.row_ptr[x + 1]; ++k)
        out.push_back(v.col_idx[k] | (v.values[k] < 0.0f ? kSign : 0u));
    }
  };

  // per block: staged columns and the re-laid delta rows
  std::vector<uint32_t> order(nb);
  std::iota(order.begin(), order.end(), 0u);
  std::vector<uint64_t> work(nb, 0);
  for (uint32_t b = 0; b < nb; ++b)
    for (uint32_t i = bptr[b]; i < bptr[b + 1]; ++i) {
      const uint32_t x = brows[i];
      work[b] += 8 + (cut[x] ? full[x].size() : v.row_ptr[x + 1] - v.row_ptr[x]);
    }
  std::stable_sort(order.begin(), order.end(),
                   [&](uint32_t a, uint32_t c) { return work[a] > work[c]; });
  std::vector<uint32_t> cnt(v.n_cols, 0), lidx(v.n_cols, kTileNone), ent, touched, cand;
  T.row.reserve(size_t(m) * 8);
  for (uint32_t b : order) {
    touched.clear();
    for (uint32_t i = bptr[b]; i < bptr[b + 1]; ++i) {
      row_entries(brows[i], ent);
      for (uint32_t e : ent) {
        const uint32_t c = e & ~kSign;
        if (cnt[c]++ == 0) touched.push_back(c);
      }
    }
    cand.clear();
    for (uint32_t c : touched)
      if (cnt[c] >= 2) cand.push_back(c);
    if (cand.size() > stage_cap) {
      std::nth_element(cand.begin(), cand.begin() + stage_cap, cand.end(), [&](uint32_t a, uint32_t c) {
        return cnt[a] != cnt[c] ? cnt[a] > cnt[c] : a < c;
      });
      cand.resize(stage_cap);
    }
    std::sort(cand.begin(), cand.end());
    const uint32_t st0 = uint32_t(T.stage.size());
    for (uint32_t j = 0; j < cand.size(); ++j) {
      lidx[cand[j]] = j;
      T.stage.push_back(cand[j]);
      T.n_staged_cols += 1;
    }
    const uint32_t row0 = uint32_t(T.row.size() / 8);
    uint64_t blk_entries = 0;
    for (uint32_t i = bptr[b]; i < bptr[b + 1]; ++i) {
      const uint32_t x = brows[i];
      row_entries(x, ent);
      while (T.dcol.size() % 4) {  // rows start 16-byte aligned (cp.async of the indices)
        T.dcol.push_back(0);
        if (norm) T.dval.push_back(0.0f);
      }
      const uint64_t beg = T.dcol.size();
      // staged +1 deltas, then staged -1 deltas, each run padded to a multiple
      // of 8 with the block's zero row (no per-delta sign on the tile path)
      uint64_t mpos = 0;
      for (uint32_t sign : {0u, kSign}) {
        for (uint32_t e : ent)
          if ((e & kSign) == sign && lidx[e & ~kSign] != kTileNone) {
            T.dcol.push_back(lidx[e & ~kSign]);
            if (norm) T.dval.push_back(sign ? -v.row_scale[e & ~kSign] : v.row_scale[e & ~kSign]);
          }
        while ((T.dcol.size() - beg) % 8) {
          T.dcol.push_back(uint32_t(cand.size()));
          if (norm) T.dval.push_back(0.0f);
        }
        if (!sign) mpos = T.dcol.size();
      }
      const uint64_t mid = T.dcol.size();
      for (uint32_t e : ent)
        if (lidx[e & ~kSign] == kTileNone) {
          T.dcol.push_back(e);
          if (norm) {
            const float s = v.row_scale[e & ~kSign];
            T.dval.push_back((e & kSign) ? -s : s);
          }
        }
      const uint64_t end = T.dcol.size();
      if (end >= 0xFFFFFFFFull) throw invalid_argument("tiles: more than 2^32-1 deltas");
      for (uint32_t e : ent) T.n_staged_deltas += lidx[e & ~kSign] != kTileNone;
      T.n_entries += ent.size();
      T.max_row_entries = std::max<uint64_t>(T.max_row_entries, ent.size());
      blk_entries += ent.size();
      const uint32_t p = v.parent[x];
      const bool has_parent = p != kVirt && !cut[x];
      const uint32_t r[8] = {uint32_t(beg), uint32_t(mpos), uint32_t(mid), uint32_t(end), x,
                             has_parent ? local[p] : kTileNone,
                             has_parent ? slot[p] : kTileNone, slot[x]};
      T.row.insert(T.row.end(), r, r + 8);
    }
    T.block.insert(T.block.end(), {row0, bptr[b + 1] - bptr[b], st0, uint32_t(cand.size())});
    T.work.push_back(uint32_t(std::min<uint64_t>(work[b], 0xFFFFFFFFull)));
    T.max_block_entries = std::max(T.max_block_entries, blk_entries);
    T.max_rows = std::max(T.max_rows, bptr[b + 1] - bptr[b]);
    T.max_staged = std::max(T.max_staged, uint32_t(cand.size()));
    for (uint32_t c : touched) {
      cnt[c] = 0;
      lidx[c] = kTileNone;
    }
  }
  T.n_blocks = nb;
  T.n_deltas = T.n_entries;
  T.dcol.resize(T.dcol.size() + 8, 0);  // over-read slack of the 16-byte index copies
  if (norm) T.dval.resize(T.dcol.size(), 0.0f);
  return T;
}

}  // namespace cbmb
