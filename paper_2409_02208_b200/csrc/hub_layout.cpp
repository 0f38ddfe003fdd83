// Hub-row panel planner (hub_layout.hpp).
#include "hub_layout.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "cbm_host.hpp"
#include "layout.hpp"

namespace cbmb {

HubPlan plan_hub(const cbm_b200_cbm_view& v, int mode, uint32_t num_sms) {
  HubPlan H;
  const uint32_t m = v.n_rows, n = v.n_cols;
  if (m == 0 || n == 0 || mode == 0) return H;
  // auto: only matrices large enough for a second pipeline to pay
  if (mode < 0 && (m < (1u << 15) || v.nnz < (1ull << 22))) return H;

  // full rows of the represented matrix, parents first
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
  if (!reconstruct_full_rows(v, bfs, fptr, fcol)) return H;
  std::vector<uint32_t>().swap(bfs);
  const uint64_t nnz_full = fptr[m];

  // candidates: the kDenseRows longest rows
  std::vector<uint32_t> cand(m);
  std::iota(cand.begin(), cand.end(), 0u);
  const uint32_t top = std::min<uint32_t>(kDenseRows, m);
  auto len = [&](uint32_t r) { return fptr[r + 1] - fptr[r]; };
  std::partial_sort(cand.begin(), cand.begin() + top, cand.end(), [&](uint32_t a, uint32_t b) {
    return len(a) != len(b) ? len(a) > len(b) : a < b;
  });
  cand.resize(top);
  // Prefix rule: with the k longest rows in the panel the streaming kernel
  // saves their entries (one gathered X row each) and the tensor kernel pays
  // kDenseChunkCost gather-equivalents per chunk of 32 union columns (measured
  // on cfg[3], dense_layout.hpp). A single row never pays (no re-use); the
  // union saturates as rows are added. Take the prefix with the largest gain.
  uint32_t best_k = 0;
  {
    std::vector<uint8_t> seen(n, 0);
    uint64_t uni = 0, ent = 0;
    double best = 0.0;
    for (uint32_t i = 0; i < top; ++i) {
      const uint32_t r = cand[i];
      if (len(r) < (mode > 0 ? 1u : 256u)) break;
      for (uint64_t k = fptr[r]; k < fptr[r + 1]; ++k)
        if (!seen[fcol[k]]) seen[fcol[k]] = 1, ++uni;
      ent += len(r);
      const double gain = double(ent) - kDenseChunkCost * double((uni + kDenseK - 1) / kDenseK);
      if (mode > 0 || gain > best) best = gain, best_k = i + 1;
    }
    if (mode < 0 && best < 0.04 * double(nnz_full)) best_k = 0;
  }
  if (best_k == 0) return H;
  cand.resize(best_k);
  H.rows = cand;

  // union of the hub rows' columns, ascending; chunks of kDenseK
  std::vector<uint32_t> pos(n, 0);  // column -> position in the union (+1)
  for (uint32_t r : H.rows)
    for (uint64_t k = fptr[r]; k < fptr[r + 1]; ++k) pos[fcol[k]] = 1;
  std::vector<uint32_t> uni;
  for (uint32_t c = 0; c < n; ++c)
    if (pos[c]) {
      uni.push_back(c);
      pos[c] = uint32_t(uni.size());
    }
  H.n_chunks = (uni.size() + kDenseK - 1) / kDenseK;
  if (H.n_chunks == 0 || H.n_chunks >= 0x7FFFFFFFull) return H;
  if (mode < 0 && H.n_chunks < 8ull * std::max(1u, num_sms)) return H;
  const float* colscale = v.col_scale ? v.col_scale : v.row_scale;
  const bool norm = v.is_normalized != 0;
  H.meta.assign(size_t(H.n_chunks) * kDenseMetaWords, 0u);
  for (uint64_t q = 0; q < H.n_chunks; ++q) {
    uint32_t* mw = H.meta.data() + q * kDenseMetaWords;
    for (uint32_t k = 0; k < kDenseK; ++k) {
      const uint64_t i = std::min<uint64_t>(q * kDenseK + k, uni.size() - 1);  // pad: a real column
      mw[k] = uni[i];
      const float sc = norm ? colscale[uni[i]] : 1.0f;
      std::memcpy(&mw[kDenseK + k], &sc, 4);
    }
  }
  for (uint32_t i = 0; i < H.rows.size(); ++i) {
    const uint32_t r = H.rows[i];
    for (uint64_t k = fptr[r]; k < fptr[r + 1]; ++k) {
      const uint32_t u = pos[fcol[k]] - 1;
      H.meta[size_t(u / kDenseK) * kDenseMetaWords + 2 * kDenseK + i] |= 1u << (u % kDenseK);
    }
    H.entries += len(r);
  }
  // pieces: consecutive ranges of about kHubPieceChunks chunks. Short on
  // purpose: the tensor cores' fp32 accumulator truncates, and over the ~2,700
  // dependent accumulations of a 340-chunk piece cfg[4]'s hub rows landed
  // 2.5e-5 (normwise) from the exact product; 32-chunk pieces, combined by
  // round-to-nearest adds in a fixed tree, stay ~1e-6 from it
  H.n_pieces = uint32_t((H.n_chunks + kHubPieceChunks - 1) / kHubPieceChunks);
  for (uint32_t p = 0; p < H.n_pieces; ++p) {
    const uint64_t lo = H.n_chunks * p / H.n_pieces, hi = H.n_chunks * (p + 1) / H.n_pieces;
    H.tiles.push_back(p * kDenseRows);
    H.tiles.push_back(kDenseRows);
    H.tiles.push_back(uint32_t(lo));
    H.tiles.push_back(uint32_t(hi - lo));
  }

  // the rest: hub rows emptied, their children summed from their full rows
  std::vector<uint8_t> is_hub(m, 0);
  for (uint32_t r : H.rows) is_hub[r] = 1;
  H.rest_parent.assign(v.parent, v.parent + m);
  H.rest_row_ptr.assign(size_t(m) + 1, 0);
  auto flat = [&](uint32_t x) { return v.parent[x] != kNoItem && is_hub[v.parent[x]]; };
  for (uint32_t x = 0; x < m; ++x) {
    uint64_t l = v.row_ptr[x + 1] - v.row_ptr[x];
    if (is_hub[x]) l = 0;
    else if (flat(x)) l = len(x);
    if (is_hub[x] || flat(x)) H.rest_parent[x] = kNoItem;
    H.rest_row_ptr[x + 1] = H.rest_row_ptr[x] + l;
  }
  H.rest_col.resize(H.rest_row_ptr[m]);
  H.rest_val.resize(H.rest_row_ptr[m]);
  for (uint32_t x = 0; x < m; ++x) {
    uint64_t o = H.rest_row_ptr[x];
    if (is_hub[x]) continue;
    if (flat(x)) {
      for (uint64_t k = fptr[x]; k < fptr[x + 1]; ++k, ++o) {
        H.rest_col[o] = fcol[k];
        H.rest_val[o] = norm ? colscale[fcol[k]] : 1.0f;
      }
    } else {
      const uint64_t l = v.row_ptr[x + 1] - v.row_ptr[x];
      std::copy(v.col_idx + v.row_ptr[x], v.col_idx + v.row_ptr[x] + l, H.rest_col.begin() + o);
      std::copy(v.values + v.row_ptr[x], v.values + v.row_ptr[x] + l, H.rest_val.begin() + o);
    }
  }
  // the hub rows alone
  const uint32_t R = uint32_t(H.rows.size());
  H.hub_parent.assign(R, kNoItem);
  H.hub_row_ptr.assign(size_t(R) + 1, 0);
  for (uint32_t i = 0; i < R; ++i) H.hub_row_ptr[i + 1] = H.hub_row_ptr[i] + len(H.rows[i]);
  H.hub_col.resize(H.hub_row_ptr[R]);
  H.hub_val.resize(H.hub_row_ptr[R]);
  for (uint32_t i = 0; i < R; ++i) {
    uint64_t o = H.hub_row_ptr[i];
    for (uint64_t k = fptr[H.rows[i]]; k < fptr[H.rows[i] + 1]; ++k, ++o) {
      H.hub_col[o] = fcol[k];
      H.hub_val[o] = norm ? colscale[fcol[k]] : 1.0f;
    }
  }
  if (norm)
    for (uint32_t r : H.rows) H.hub_row_scale.push_back(v.row_scale[r]);
  H.on = true;
  return H;
}

}  // namespace cbmb
