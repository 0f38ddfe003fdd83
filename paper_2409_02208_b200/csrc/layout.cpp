#include "layout.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <string>

#include "cbm_host.hpp"

namespace cbmb {

// Full rows (parent + plus - minus, ascending) of every row, parents first
// (reconstruct_rows, builder.cpp:452-490): fptr has m+1 offsets. Returns false,
// without writing past any row, when some delta row is inconsistent with its
// parent's row (a minus column the parent lacks, a plus column it has).
bool reconstruct_full_rows(const cbm_b200_cbm_view& v, const std::vector<uint32_t>& bfs,
                           std::vector<uint64_t>& fptr, std::vector<uint32_t>& fcol) {
  const uint32_t m = v.n_rows;
  std::vector<uint64_t> len(m, 0);
  for (uint32_t x : bfs) {
    uint64_t plus = 0, minus = 0;
    for (uint64_t k = v.row_ptr[x]; k < v.row_ptr[x + 1]; ++k)
      (v.values[k] < 0.0f ? minus : plus) += 1;
    const uint32_t p = v.parent[x];
    const uint64_t base = p == kVirtual ? 0 : len[p];
    if (base + plus < minus || (p == kVirtual && minus)) return false;
    len[x] = base + plus - minus;
  }
  fptr.assign(size_t(m) + 1, 0);
  for (uint32_t x = 0; x < m; ++x) fptr[x + 1] = fptr[x] + len[x];
  fcol.resize(fptr[m]);
  for (uint32_t x : bfs) {
    uint32_t* out = fcol.data() + fptr[x];
    uint32_t* const end = out + len[x];
    const uint32_t p = v.parent[x];
    uint64_t k = v.row_ptr[x];
    const uint64_t ke = v.row_ptr[x + 1];
    const uint32_t* pr = p == kVirtual ? nullptr : fcol.data() + fptr[p];
    const uint32_t* pe = p == kVirtual ? nullptr : pr + len[p];
    while (pr < pe || k < ke) {
      uint32_t c;
      if (k == ke || (pr < pe && *pr < v.col_idx[k])) {
        c = *pr++;                              // parent column kept
      } else if (pr == pe || v.col_idx[k] < *pr) {
        if (v.values[k] < 0.0f) return false;   // removes a column the parent lacks
        c = v.col_idx[k++];                     // added column
      } else {
        if (v.values[k] > 0.0f) return false;   // adds a column the parent has
        ++pr;                                   // removed column
        ++k;
        continue;
      }
      if (out == end) return false;
      *out++ = c;
    }
    if (out != end) return false;
  }
  return true;
}

// load_cbm's structural checks (io.cpp:346-380) on a view, with its messages:
// what plan_layout verifies before it lays anything out. For callers that
// must read the view before a layout exists (hub_layout.cpp).
void validate_view(const cbm_b200_cbm_view& v) {
  const uint32_t m = v.n_rows;
  if (m >= kInteriorBit) throw invalid_argument("upload: too many rows for the device layout");
  if (v.n_cols >= kSignBit) throw invalid_argument("upload: too many columns for the device layout");
  if (m && (!v.parent || !v.row_ptr)) throw invalid_argument("upload: null array in view");
  if (v.row_ptr && v.row_ptr[0] != 0) throw invalid_argument("csr: row_ptr[0] must be 0");
  const uint64_t nnz = m ? v.row_ptr[m] : 0;
  if (nnz != v.nnz) throw invalid_argument("csr: row_ptr back must equal nnz");
  if (nnz >= 0xFFFFFFFFull) throw invalid_argument("upload: more than 2^32-1 deltas");
  if (nnz && (!v.col_idx || !v.values)) throw invalid_argument("upload: null array in view");
  const bool norm = v.is_normalized != 0;
  const float* colscale = v.col_scale ? v.col_scale : v.row_scale;
  if (norm) {
    if (v.n_rows != v.n_cols && !v.col_scale)
      throw invalid_argument("normalized container must be square");
    if (!v.row_scale && m) throw invalid_argument("upload: normalized view without row_scale");
    for (uint32_t r = 0; r < m; ++r)
      if (!std::isfinite(v.row_scale[r]) || v.row_scale[r] <= 0.0f)
        throw invalid_argument("row_scale entries must be positive and finite");
    if (v.col_scale)
      for (uint32_t c = 0; c < v.n_cols; ++c)
        if (!std::isfinite(v.col_scale[c]) || v.col_scale[c] <= 0.0f)
          throw invalid_argument("row_scale entries must be positive and finite");
  }
  for (uint32_t r = 0; r < m; ++r) {
    const uint64_t lo = v.row_ptr[r], hi = v.row_ptr[r + 1];
    if (lo > hi) throw invalid_argument("csr: row_ptr must be non-decreasing");
    if (hi > nnz) throw invalid_argument("csr: row_ptr back must equal nnz");
    for (uint64_t k = lo; k < hi; ++k) {
      const uint32_t c = v.col_idx[k];
      if (c >= v.n_cols)
        throw invalid_argument("csr: column index out of range in row " + std::to_string(r));
      if (k + 1 < hi && c >= v.col_idx[k + 1])
        throw invalid_argument("csr: row " + std::to_string(r) + " is not strictly increasing");
      const float val = v.values[k];
      const float mag = norm ? colscale[c] : 1.0f;
      if (val != mag && val != -mag)
        throw invalid_argument(norm ? "delta values disagree with the column scales"
                                    : "delta values must be +1 or -1");
    }
  }
  for (uint32_t x = 0; x < m; ++x) {
    const uint32_t p = v.parent[x];
    if (p == kVirtual) continue;
    if (p >= m || p == x) throw invalid_argument("chain: bad parent link at row " + std::to_string(x));
  }
  // acyclic: every row reaches a root in at most m steps (path compression by
  // marking rows already known to end at a root)
  std::vector<uint8_t> ok(m, 0);
  std::vector<uint32_t> path;
  for (uint32_t x = 0; x < m; ++x) {
    uint32_t u = x;
    path.clear();
    while (u != kVirtual && !ok[u]) {
      if (path.size() > m) throw invalid_argument("chain: parent links contain a cycle");
      ok[u] = 2;  // on the current path
      path.push_back(u);
      u = v.parent[u];
      if (u != kVirtual && ok[u] == 2) throw invalid_argument("chain: parent links contain a cycle");
    }
    for (uint32_t w : path) ok[w] = 1;
  }
}

Layout plan_layout(const cbm_b200_cbm_view& v, bool order_faithful, uint32_t split_threshold,
                   uint32_t chunk, uint32_t flatten_gain, uint32_t warps_hint) {
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
    if (v.n_rows != v.n_cols && !v.col_scale)
      throw invalid_argument("normalized container must be square");
    if (!v.row_scale && m) throw invalid_argument("upload: normalized view without row_scale");
    L.row_scale.assign(v.row_scale, v.row_scale + m);
    if (v.col_scale) L.scale.assign(v.col_scale, v.col_scale + v.n_cols);
    else L.scale = L.row_scale;
    for (const auto* vec : {&L.scale, &L.row_scale})
      for (float s : *vec)
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

  // ---- effective structure: optionally flatten rows whose parent saves little
  // A row x with full row a_x and delta row D_x costs |D_x| gathers plus a wait
  // on its parent and a parent-row read under the CBM; summed directly it costs
  // |a_x| gathers and no wait. Rows with |a_x| - |D_x| < flatten_gain are
  // summed directly (default mode only: the row VALUE is unchanged, children
  // still read it, only its summation order changes). order_faithful keeps
  // the reference's chain exactly.
  std::vector<uint32_t> eparent(v.parent, v.parent + m);
  std::vector<uint64_t> eptr(size_t(m) + 1, 0);
  std::vector<uint32_t> ecol;
  {
    std::vector<uint8_t> flat(m, 0);
    uint64_t n_flat = 0;
    if (!order_faithful && flatten_gain > 0) {
      std::vector<uint64_t> nA(m, 0);
      for (uint32_t x : bfs) {
        uint64_t plus = 0, minus = 0;
        for (uint64_t k = v.row_ptr[x]; k < v.row_ptr[x + 1]; ++k)
          (v.values[k] < 0.0f ? minus : plus) += 1;
        const uint32_t p = v.parent[x];
        const uint64_t base = p == kVirtual ? 0 : nA[p];
        nA[x] = base + plus >= minus ? base + plus - minus : 0;  // (inconsistent rows: 0)
        const uint64_t dl = plus + minus;
        if (p != kVirtual && nA[x] < dl + flatten_gain) {
          flat[x] = 1;
          ++n_flat;
        }
      }
    }
    L.n_flattened = uint32_t(n_flat);
    std::vector<uint64_t> fptr;  // full rows (only when something is flattened)
    std::vector<uint32_t> fcol;
    if (n_flat && !reconstruct_full_rows(v, bfs, fptr, fcol)) {
      // a delta row that removes a column its parent lacks, or adds one it
      // already has: the reference still multiplies it (U = deltas + U_parent,
      // kernels.cpp:27-53) but it has no full-row form, so nothing is flattened
      // and every row keeps its chain link (exactly the reference's values)
      n_flat = 0;
      L.n_flattened = 0;
      L.inconsistent = true;
    }
    if (n_flat) {
      for (uint32_t x = 0; x < m; ++x)
        if (flat[x]) eparent[x] = kVirtual;
      for (uint32_t x = 0; x < m; ++x)
        eptr[x + 1] = eptr[x] + (flat[x] ? fptr[x + 1] - fptr[x] : v.row_ptr[x + 1] - v.row_ptr[x]);
    } else {
      for (uint32_t x = 0; x < m; ++x) eptr[x + 1] = v.row_ptr[x + 1];
    }
    ecol.resize(eptr[m]);
    for (uint32_t x = 0; x < m; ++x) {
      uint32_t* out = ecol.data() + eptr[x];
      if (n_flat && flat[x]) {
        const uint32_t* fr = fcol.data() + fptr[x];
        for (uint64_t j = 0; j < eptr[x + 1] - eptr[x]; ++j) *out++ = fr[j];
      } else {
        for (uint64_t k = v.row_ptr[x]; k < v.row_ptr[x + 1]; ++k)
          *out++ = v.col_idx[k] | (v.values[k] < 0.0f ? kSignBit : 0u);
      }
    }
    if (n_flat) {  // depths under the effective forest
      std::fill(depth.begin(), depth.end(), kNoItem);
      std::vector<uint64_t> kp(size_t(m) + 1, 0);
      for (uint32_t x = 0; x < m; ++x)
        if (eparent[x] != kVirtual) ++kp[eparent[x] + 1];
      std::partial_sum(kp.begin(), kp.end(), kp.begin());
      std::vector<uint32_t> ks(kp.back());
      std::vector<uint64_t> cur(kp.begin(), kp.end() - 1);
      for (uint32_t x = 0; x < m; ++x)
        if (eparent[x] != kVirtual) ks[cur[eparent[x]]++] = x;
      bfs.clear();
      for (uint32_t x = 0; x < m; ++x)
        if (eparent[x] == kVirtual) {
          depth[x] = 0;
          bfs.push_back(x);
        }
      for (size_t h = 0; h < bfs.size(); ++h) {
        const uint32_t u = bfs[h];
        for (uint64_t k = kp[u]; k < kp[u + 1]; ++k) {
          depth[ks[k]] = depth[u] + 1;
          bfs.push_back(ks[k]);
        }
      }
    }
  }
  L.nnz_effective = eptr[m];
  if (L.nnz_effective >= 0xFFFFFFFFull)  // dcol offsets are 32-bit on the device
    throw invalid_argument("upload: more than 2^32-1 deltas after flattening "
                           "(upload with flatten_gain = 0)");

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

  // split plan for long rows (default mode only)
  // auto: split rows longer than ~1/8 of a warp's share of the deltas (a
  // power of two in [32, 1024]): small matrices need short pieces to spread
  // over the grid, large ones lose more to the partial-sum hand-offs than
  // they gain in balance (tools/probe_split.py: cfg[1] best at 32, cfg[2] and
  // cfg[3] at 256 / 64)
  if (split_threshold == 0) {
    const uint64_t share = L.nnz_effective / std::max<uint32_t>(1, warps_hint) / 8;
    // (up to 1024 on very large matrices: cfg[4] with the hub rows on the tensor
    // cores measures 1-2% better at 1024 / 256-entry pieces than at 256 / 64,
    // profiles/r02t_cfg4_split_chunk_sweep.jsonl; cfg[2]'s share keeps it at 256)
    split_threshold = 32;
    while (split_threshold < 1024 && uint64_t(split_threshold) * 2 <= share) split_threshold *= 2;
  }
  if (chunk == 0) chunk = std::max<uint32_t>(32, split_threshold / 4);
  if (chunk > split_threshold) chunk = split_threshold;
  // Column bands (default mode): when X is far larger than L2, the pieces of
  // the long rows are cut at band boundaries and summed band by band (every
  // long row's piece of band 0, then band 1, ...), so a band of X rows is
  // read from DRAM once and then met in L2 by every long row that references
  // it. Row-major pieces sweep all of X once per long row instead (cfg[4]:
  // 54 GB of DRAM reads per multiply, 10x the compulsory bytes). A band holds
  // 48 MB of 1 KB X row slices; rows too sparse to leave >= 16 entries per
  // band keep plain pieces (still taken in band order of their first column).
  uint32_t band_cols = 0;
  if (!order_faithful) {
    const uint64_t budget = (48ull << 20) / 1024;
    if (const char* e = std::getenv("CBM_B200_BAND_COLS")) band_cols = uint32_t(std::atoll(e));
    else if (uint64_t(v.n_cols) > budget + budget / 3) band_cols = uint32_t(budget);
  }
  const uint32_t n_bands = band_cols ? (v.n_cols + band_cols - 1) / band_cols : 1;
  L.band_cols = band_cols;
  std::vector<uint32_t> pieces(m, 1);  // per ROW position i
  std::vector<uint64_t> cut_ptr(size_t(m) + 1, 0);
  std::vector<uint32_t> cuts;  // piece start offsets inside the split rows (first = 0)
  uint64_t n_leaf = 0;
  if (!order_faithful) {
    for (uint32_t i = 0; i < m; ++i) {
      const uint32_t r = rows[i];
      const uint64_t len = eptr[r + 1] - eptr[r];
      if (len > split_threshold) {
        const uint32_t* e = ecol.data() + eptr[r];
        const bool banded = band_cols && len >= 16ull * n_bands;
        auto band = [&](uint32_t w) { return (w & ~kSignBit) / band_cols; };
        uint32_t start = 0;
        cuts.push_back(0);
        for (uint32_t k = 1; k < len; ++k) {
          bool cut = k - start >= chunk;
          if (!cut && banded && k - start >= 16 && band(e[k]) != band(e[start])) cut = true;
          if (cut) {
            cuts.push_back(k);
            start = k;
          }
        }
        pieces[i] = uint32_t(cuts.size() - cut_ptr[i]);
        n_leaf += pieces[i] - 1;
      }
      cut_ptr[i + 1] = cuts.size();
    }
  }
  // merge tree per split row: level 0 = the row's leaf chunks; a level with
  // more than kFanIn nodes is grouped kFanIn at a time into MERGE nodes.
  uint32_t max_lvls = 0;
  std::vector<uint32_t> nl(m, 0);  // number of levels (incl. leaves) per split row
  for (uint32_t i = 0; i < m; ++i) {
    if (pieces[i] < 2) continue;
    uint32_t n = pieces[i] - 1, k = 1;
    while (n > kFanIn) {
      n = (n + kFanIn - 1) / kFanIn;
      ++k;
    }
    nl[i] = k;
    max_lvls = std::max(max_lvls, k);
  }
  // first item index of each (row, level) block: leaves for all rows first,
  // then merge level 1 for all rows, ...
  std::vector<std::vector<uint32_t>> first_at(max_lvls);
  std::vector<std::vector<uint32_t>> count_at(max_lvls);
  uint64_t t_next = 0;
  for (uint32_t lv = 0; lv < max_lvls; ++lv) {
    first_at[lv].assign(m, kNoItem);
    count_at[lv].assign(m, 0);
    for (uint32_t i = 0; i < m; ++i) {
      if (nl[i] <= lv) continue;
      uint32_t n = pieces[i] - 1;
      for (uint32_t q = 0; q < lv; ++q) n = (n + kFanIn - 1) / kFanIn;
      first_at[lv][i] = uint32_t(t_next);
      count_at[lv][i] = n;
      t_next += n;
    }
  }
  if (t_next + m >= 0x7FFFFFFFull) throw invalid_argument("upload: too many work items");
  L.n_chunk_items = uint32_t(t_next);
  L.n_merge_items = uint32_t(t_next - n_leaf);
  L.n_items = uint32_t(t_next) + m;

  std::vector<uint32_t> item_of_row(m);
  for (uint32_t i = 0; i < m; ++i) item_of_row[rows[i]] = L.n_chunk_items + i;
  std::vector<uint8_t> interior(m, 0);
  for (uint32_t x = 0; x < m; ++x)
    if (eparent[x] != kVirtual) interior[eparent[x]] = 1;
  std::vector<uint32_t> slot(m, kNoItem);
  for (uint32_t i = 0; i < m; ++i)
    if (interior[rows[i]]) slot[rows[i]] = L.n_interior++;

  L.dcol.resize(eptr[m]);
  L.rec.assign(size_t(L.n_items) * 8, 0);
  if (L.normalized) L.srow.assign(L.n_items, 0.0f);
  auto R = [&](uint32_t t) { return &L.rec[size_t(t) * 8]; };
  // delta ranges: items own [beg, end) of dcol, laid out in item order
  std::vector<uint64_t> own_lo(L.n_items, 0), own_hi(L.n_items, 0);
  for (uint32_t t = 0; t < L.n_items; ++t) {
    R(t)[3] = kNoItem;
    R(t)[7] = kNoItem;
  }
  for (uint32_t i = 0; i < m; ++i) {
    const uint32_t r = rows[i];
    const uint64_t lo = eptr[r], hi = eptr[r + 1];
    const uint32_t t_row = L.n_chunk_items + i;
    if (pieces[i] < 2) {
      own_lo[t_row] = lo;
      own_hi[t_row] = hi;
      continue;
    }
    const uint32_t* cq = cuts.data() + cut_ptr[i];
    own_lo[t_row] = lo;  // piece 0 stays with the ROW item
    own_hi[t_row] = lo + cq[1];
    for (uint32_t q = 1; q < pieces[i]; ++q) {
      const uint32_t t = first_at[0][i] + q - 1;
      own_lo[t] = lo + cq[q];
      own_hi[t] = q + 1 < pieces[i] ? lo + cq[q + 1] : hi;
      R(t)[2] = r;
    }
    // merge levels: node j at level lv sums nodes [j*F, min((j+1)*F, n_prev)) of lv-1
    for (uint32_t lv = 1; lv < nl[i]; ++lv) {
      const uint32_t n_prev = count_at[lv - 1][i];
      for (uint32_t j = 0; j < count_at[lv][i]; ++j) {
        const uint32_t t = first_at[lv][i] + j;
        R(t)[2] = r;
        R(t)[5] = first_at[lv - 1][i] + j * kFanIn;
        R(t)[6] = std::min(kFanIn, n_prev - j * kFanIn);
      }
    }
    const uint32_t top = nl[i] - 1;
    R(t_row)[5] = first_at[top][i];
    R(t_row)[6] = count_at[top][i];
  }
  uint64_t o = 0;
  for (uint32_t t = 0; t < L.n_items; ++t) {
    R(t)[0] = uint32_t(o);
    for (uint64_t k = own_lo[t]; k < own_hi[t]; ++k)
      L.dcol[o++] = ecol[k];
    R(t)[1] = uint32_t(o);
  }
  // processing order of the items (schedule.cu): leaf pieces by the band of
  // their first column (stable: row order inside a band), then everything
  // else in item order. Leaf pieces wait on nothing, so every dependency
  // still points to an earlier position.
  if (band_cols && n_leaf) {
    L.order.resize(L.n_items);
    std::iota(L.order.begin(), L.order.end(), 0u);
    std::vector<uint32_t> key(n_leaf);
    for (uint64_t t = 0; t < n_leaf; ++t)
      key[t] = (ecol[own_lo[t]] & ~kSignBit) / band_cols;
    std::stable_sort(L.order.begin(), L.order.begin() + n_leaf,
                     [&](uint32_t a, uint32_t b) { return key[a] < key[b]; });
  }
  L.item_beg.resize(size_t(L.n_items) + 1);
  for (uint32_t t = 0; t < L.n_items; ++t) L.item_beg[t] = R(t)[0];
  L.item_beg[L.n_items] = uint32_t(o);
  for (uint32_t i = 0; i < m; ++i) {  // ROW items
    const uint32_t r = rows[i];
    const uint32_t t = L.n_chunk_items + i;
    const uint32_t p = eparent[r];
    R(t)[2] = r | (interior[r] ? kInteriorBit : 0u);
    R(t)[3] = p == kVirtual ? kNoItem : item_of_row[p];
    R(t)[4] = p == kVirtual ? 0u : (L.normalized ? slot[p] : p);
    if (L.normalized) {
      R(t)[7] = slot[r];
      L.srow[t] = L.row_scale[r];
    }
  }
  return L;
}

}  // namespace cbmb
