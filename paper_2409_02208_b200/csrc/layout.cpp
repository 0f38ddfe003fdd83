#include "layout.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>

#include "cbm_host.hpp"

namespace cbmb {

Layout plan_layout(const cbm_b200_cbm_view& v, bool order_faithful, uint32_t split_threshold,
                   uint32_t chunk) {
  const uint32_t m = v.n_rows;
  Layout L;
  L.n_rows = m;
  L.n_cols = v.n_cols;
  L.normalized = v.is_normalized != 0;
  L.order_faithful = order_faithful;
  if (m >= kInteriorBit) throw invalid_argument("upload: too many rows for the device layout");
  if (v.n_cols >= kSignBit) throw invalid_argument("upload: too many columns for the device layout");
  if (m && (!v.parent || !v.row_ptr)) throw invalid_argument("upload: null array in view");
  if (v.row_ptr && v.row_ptr[0] != 0) throw invalid_argument("csr: row_ptr[0] must be 0");
  const uint64_t nnz = m ? v.row_ptr[m] : 0;
  if (nnz != v.nnz) throw invalid_argument("csr: row_ptr back must equal nnz");
  if (nnz >= 0xFFFFFFFFull) throw invalid_argument("upload: more than 2^32-1 deltas");
  if (nnz && (!v.col_idx || !v.values)) throw invalid_argument("upload: null array in view");
  L.nnz = nnz;
  if (L.normalized) {
    if (v.n_rows != v.n_cols)
      throw invalid_argument("normalized container must be square");
    if (!v.row_scale && m) throw invalid_argument("upload: normalized view without row_scale");
    L.scale.assign(v.row_scale, v.row_scale + m);
    for (float s : L.scale)
      if (!std::isfinite(s) || s <= 0.0f)
        throw invalid_argument("row_scale entries must be positive and finite");
  }
  // delta rows: monotone offsets, strictly increasing in-range columns, value pattern
  for (uint32_t r = 0; r < m; ++r) {
    const uint64_t lo = v.row_ptr[r], hi = v.row_ptr[r + 1];
    if (lo > hi) throw invalid_argument("csr: row_ptr must be non-decreasing");
    L.max_row_deltas = std::max<uint32_t>(L.max_row_deltas, uint32_t(hi - lo));
    for (uint64_t k = lo; k < hi; ++k) {
      const uint32_t c = v.col_idx[k];
      if (c >= v.n_cols)
        throw invalid_argument("csr: column index out of range in row " + std::to_string(r));
      if (k + 1 < hi && c >= v.col_idx[k + 1])
        throw invalid_argument("csr: row " + std::to_string(r) + " is not strictly increasing");
      const float val = v.values[k];
      const float mag = L.normalized ? L.scale[c] : 1.0f;
      if (val != mag && val != -mag)
        throw invalid_argument(L.normalized ? "delta values disagree with the column scales"
                                            : "delta values must be +1 or -1");
    }
  }

  // forest depth, parents first (BFS from the roots)
  std::vector<uint64_t> kid_ptr(size_t(m) + 1, 0);
  for (uint32_t x = 0; x < m; ++x) {
    const uint32_t p = v.parent[x];
    if (p == kVirtual) continue;
    if (p >= m || p == x) throw invalid_argument("chain: bad parent link at row " + std::to_string(x));
    ++kid_ptr[p + 1];
  }
  std::partial_sum(kid_ptr.begin(), kid_ptr.end(), kid_ptr.begin());
  std::vector<uint32_t> kids(kid_ptr.back());
  {
    std::vector<uint64_t> cur(kid_ptr.begin(), kid_ptr.end() - 1);
    for (uint32_t x = 0; x < m; ++x)
      if (v.parent[x] != kVirtual) kids[cur[v.parent[x]]++] = x;
  }
  std::vector<uint32_t> depth(m, kNoItem), bfs;
  bfs.reserve(m);
  for (uint32_t x = 0; x < m; ++x)
    if (v.parent[x] == kVirtual) {
      depth[x] = 0;
      bfs.push_back(x);
    }
  L.n_roots = uint32_t(bfs.size());
  for (size_t h = 0; h < bfs.size(); ++h) {
    const uint32_t u = bfs[h];
    for (uint64_t k = kid_ptr[u]; k < kid_ptr[u + 1]; ++k) {
      depth[kids[k]] = depth[u] + 1;
      bfs.push_back(kids[k]);
    }
  }
  if (bfs.size() != m) throw invalid_argument("chain: parent links contain a cycle");

  // ROW items: by depth, ascending row id inside a level (stable counting sort)
  uint32_t max_depth = 0;
  for (uint32_t x = 0; x < m; ++x) max_depth = std::max(max_depth, depth[x]);
  L.n_levels = m ? max_depth + 1 : 0;
  L.level_ptr.assign(size_t(L.n_levels) + 1, 0);
  for (uint32_t x = 0; x < m; ++x) ++L.level_ptr[depth[x] + 1];
  std::partial_sum(L.level_ptr.begin(), L.level_ptr.end(), L.level_ptr.begin());
  std::vector<uint32_t> rows(m);
  {
    std::vector<uint32_t> cur(L.level_ptr.begin(), L.level_ptr.end() - 1);
    for (uint32_t x = 0; x < m; ++x) rows[cur[depth[x]]++] = x;
  }

  // split plan for long rows
  if (split_threshold == 0) split_threshold = 1024;
  if (chunk == 0) chunk = 512;
  struct Split {
    uint32_t pieces, piece;
  };
  std::vector<Split> sp(m, {1, 0});
  uint64_t n_chunk = 0;
  if (!order_faithful) {
    for (uint32_t i = 0; i < m; ++i) {
      const uint32_t r = rows[i];
      const uint64_t len = v.row_ptr[r + 1] - v.row_ptr[r];
      if (len <= split_threshold) continue;
      const uint64_t piece = std::max<uint64_t>(chunk, (len + 255) / 256);
      const uint32_t pieces = uint32_t((len + piece - 1) / piece);
      if (pieces < 2 || n_chunk + pieces - 1 >= (1u << 24)) continue;
      sp[i] = {pieces, uint32_t(piece)};
      n_chunk += pieces - 1;
    }
  }
  L.n_chunk_items = uint32_t(n_chunk);
  L.n_items = uint32_t(n_chunk) + m;

  std::vector<uint32_t> item_of_row(m);
  for (uint32_t i = 0; i < m; ++i) item_of_row[rows[i]] = uint32_t(n_chunk) + i;
  std::vector<uint8_t> interior(m, 0);
  for (uint32_t x = 0; x < m; ++x)
    if (v.parent[x] != kVirtual) interior[v.parent[x]] = 1;
  std::vector<uint32_t> slot(m, kNoItem);
  for (uint32_t i = 0; i < m; ++i)
    if (interior[rows[i]]) slot[rows[i]] = L.n_interior++;

  L.dptr.assign(size_t(L.n_items) + 1, 0);
  L.dcol.resize(nnz);
  L.meta.assign(size_t(L.n_items) * 4, 0);
  if (L.normalized) L.oslot.assign(L.n_items, kNoItem);
  auto emit = [&](uint32_t row, uint64_t k0, uint64_t k1, uint64_t& o) {
    for (uint64_t k = k0; k < k1; ++k)
      L.dcol[o++] = v.col_idx[k] | (v.values[k] < 0.0f ? kSignBit : 0u);
    (void)row;
  };
  uint64_t o = 0;
  uint32_t t = 0;
  std::vector<uint32_t> first_chunk(m, 0);
  for (uint32_t i = 0; i < m; ++i) {  // CHUNK items: pieces 1.. of split rows
    if (sp[i].pieces < 2) continue;
    const uint32_t r = rows[i];
    const uint64_t lo = v.row_ptr[r], hi = v.row_ptr[r + 1];
    first_chunk[i] = t;
    for (uint32_t q = 1; q < sp[i].pieces; ++q) {
      const uint64_t k0 = lo + uint64_t(q) * sp[i].piece;
      const uint64_t k1 = std::min(hi, k0 + sp[i].piece);
      L.meta[size_t(t) * 4 + 0] = r;
      L.meta[size_t(t) * 4 + 1] = kNoItem;
      emit(r, k0, k1, o);
      L.dptr[++t] = uint32_t(o);
    }
  }
  for (uint32_t i = 0; i < m; ++i) {  // ROW items
    const uint32_t r = rows[i];
    const uint64_t lo = v.row_ptr[r], hi = v.row_ptr[r + 1];
    const uint64_t k1 = sp[i].pieces > 1 ? lo + sp[i].piece : hi;
    emit(r, lo, k1, o);
    uint32_t* mt = &L.meta[size_t(t) * 4];
    const uint32_t p = v.parent[r];
    mt[0] = r | (interior[r] ? kInteriorBit : 0u);
    mt[1] = p == kVirtual ? kNoItem : item_of_row[p];
    mt[2] = p == kVirtual ? 0u : (L.normalized ? slot[p] : p);
    mt[3] = sp[i].pieces > 1 ? ((sp[i].pieces - 1) << 24) | first_chunk[i] : 0u;
    if (L.normalized) L.oslot[t] = slot[r];
    L.dptr[++t] = uint32_t(o);
  }
  return L;
}

}  // namespace cbmb
