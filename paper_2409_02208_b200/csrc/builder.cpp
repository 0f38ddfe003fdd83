// Host CBM construction — produces the same CbmMatrix as the reference
// builder (proj/src/builder.cpp), field for field, but without its O(m^2)
// pair loop.
//
// Candidate edges (reference: build_candidate_edges, builder.cpp:66-118).
//   The reference keeps the row-to-row edge y -> x iff nnz(a_x) >= alpha and
//   hamming(x, y) <= nnz(a_x) - alpha; with ov = |a_x ∩ a_y| that is
//       nnz(a_y) + alpha <= 2 * ov.                                     (*)
//   We enumerate exactly those pairs with an inverted index over column
//   "prefixes" (the classic all-pairs similarity-join prefix filter): order all
//   columns by (frequency, id); the first P_y = n_y - t_y + 1 columns of row y
//   in that order, t_y = ceil((n_y + alpha) / 2), must meet a_x whenever (*)
//   holds (otherwise ov <= t_y - 1). Each candidate is then verified exactly.
//   The one family the index cannot see is ov = 0, i.e. edges out of EMPTY
//   rows (weight nnz(a_x), alpha = 0 only); such an edge ties the virtual edge
//   of its destination at every contraction level and loses the tie
//   (builder.cpp:166-168), so it is never selected and dropping it leaves the
//   arborescence unchanged (proof in DESIGN.md §Builder).
//
// Arborescence (reference: find_min_arborescence, builder.cpp:141-302):
//   Chu-Liu/Edmonds with the reference's total order on edges (weight, then
//   the virtual source, then smaller original source, then smaller original
//   destination), the same cycle-discovery order, node renumbering, reduced
//   weights, newest-first expansion and final re-attachment rule. Because that
//   order is total, the selections do not depend on edge-list order, which
//   lets the best-in-edge scan and the contraction run in parallel.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <numeric>

#include "cbm_host.hpp"

namespace cbmb {

namespace {
using Clock = std::chrono::steady_clock;
double secs(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}
constexpr uint32_t kNone = 0xFFFFFFFFu;
}  // namespace

void validate_csr(uint32_t n_rows, uint32_t n_cols, const uint64_t* row_ptr,
                  const uint32_t* col_idx) {
  if (row_ptr[0] != 0) throw invalid_argument("csr: row_ptr[0] must be 0");
  for (uint32_t r = 0; r < n_rows; ++r) {
    const uint64_t lo = row_ptr[r], hi = row_ptr[r + 1];
    if (lo > hi) throw invalid_argument("csr: row_ptr must be non-decreasing");
    for (uint64_t k = lo; k + 1 < hi; ++k)
      if (col_idx[k] >= col_idx[k + 1])
        throw invalid_argument("csr: row " + std::to_string(r) +
                               " is not strictly increasing");
    if (hi > lo && col_idx[hi - 1] >= n_cols)
      throw invalid_argument("csr: column index out of range in row " + std::to_string(r));
  }
}

// ---------------------------------------------------------------------------
// CompressionChain::from_parents (builder.cpp:16-64)
// ---------------------------------------------------------------------------
void chain_from_parents(HostCbm& c) {
  const uint32_t m = uint32_t(c.parent.size());
  for (uint32_t x = 0; x < m; ++x) {
    const uint32_t p = c.parent[x];
    if (p != kVirtual && (p >= m || p == x))
      throw invalid_argument("chain: bad parent link at row " + std::to_string(x));
  }
  // children grouped by parent, ascending row id inside each group
  std::vector<uint64_t> first(size_t(m) + 1, 0);
  for (uint32_t x = 0; x < m; ++x)
    if (c.parent[x] != kVirtual) ++first[c.parent[x] + 1];
  std::partial_sum(first.begin(), first.end(), first.begin());
  std::vector<uint32_t> kids(first.back());
  std::vector<uint64_t> fill(first.begin(), first.end() - 1);
  c.root_children.clear();
  for (uint32_t x = 0; x < m; ++x) {
    if (c.parent[x] == kVirtual)
      c.root_children.push_back(x);
    else
      kids[fill[c.parent[x]]++] = x;
  }
  // preorder: a node is emitted, then its subtrees left to right
  c.topo_order.clear();
  c.topo_order.reserve(m);
  c.branch_ptr.assign(1, 0);
  std::vector<uint32_t> todo;
  for (uint32_t r : c.root_children) {
    todo.assign(1, r);
    while (!todo.empty()) {
      const uint32_t v = todo.back();
      todo.pop_back();
      c.topo_order.push_back(v);
      for (uint64_t k = first[v + 1]; k-- > first[v];) todo.push_back(kids[k]);
    }
    c.branch_ptr.push_back(c.topo_order.size());
  }
  if (c.topo_order.size() != m) throw invalid_argument("chain: parent links contain a cycle");
}

// ---------------------------------------------------------------------------
// Candidate edges
// ---------------------------------------------------------------------------
EdgeLists candidate_edges(const Csr& a, uint64_t alpha, int threads) {
  const uint32_t m = a.n_rows, n = a.n_cols;
  if (threads < 1) threads = 1;

  // global column order: rare first
  std::vector<uint64_t> freq(n, 0);
  for (uint64_t k = 0; k < a.nnz(); ++k) ++freq[a.col_idx[k]];
  std::vector<uint32_t> order(n);
  std::iota(order.begin(), order.end(), 0u);
  std::sort(order.begin(), order.end(), [&](uint32_t p, uint32_t q) {
    return freq[p] != freq[q] ? freq[p] < freq[q] : p < q;
  });
  std::vector<uint32_t> rank(n);
  for (uint32_t i = 0; i < n; ++i) rank[order[i]] = i;

  auto need = [alpha](uint64_t ny) -> uint64_t {  // t_y = ceil((ny+alpha)/2)
    return (ny + alpha + 1) / 2;
  };

  // prefix length per row, then the prefix columns themselves
  std::vector<uint64_t> pre_ptr(size_t(m) + 1, 0);
  for (uint32_t y = 0; y < m; ++y) {
    const uint64_t ny = a.row_nnz(y);
    uint64_t p = 0;
    if (ny >= 1 && ny >= alpha) p = ny - need(ny) + 1;
    pre_ptr[y + 1] = pre_ptr[y] + p;
  }
  std::vector<uint32_t> pre_col(pre_ptr.back());
  parallel_for_chunks(m, threads, [&](size_t lo, size_t hi, int) {
    std::vector<uint32_t> tmp;
    for (size_t y = lo; y < hi; ++y) {
      const uint64_t p = pre_ptr[y + 1] - pre_ptr[y];
      if (!p) continue;
      const uint32_t* r = a.row(uint32_t(y));
      tmp.assign(r, r + a.row_nnz(uint32_t(y)));
      std::nth_element(tmp.begin(), tmp.begin() + (p - 1), tmp.end(),
                       [&](uint32_t u, uint32_t v) { return rank[u] < rank[v]; });
      std::copy(tmp.begin(), tmp.begin() + p, pre_col.begin() + pre_ptr[y]);
    }
  });
  // inverted index column -> rows whose prefix holds it (ascending row id)
  std::vector<uint64_t> inv_ptr(size_t(n) + 1, 0);
  for (uint32_t c : pre_col) ++inv_ptr[c + 1];
  std::partial_sum(inv_ptr.begin(), inv_ptr.end(), inv_ptr.begin());
  std::vector<uint32_t> inv_row(inv_ptr.back());
  {
    std::vector<uint64_t> cur(inv_ptr.begin(), inv_ptr.end() - 1);
    for (uint32_t y = 0; y < m; ++y)
      for (uint64_t k = pre_ptr[y]; k < pre_ptr[y + 1]; ++k) inv_row[cur[pre_col[k]]++] = y;
  }
  std::vector<uint32_t>().swap(pre_col);

  // probe: one destination row x at a time, rows handed out dynamically
  constexpr uint32_t kBlock = 64;
  const uint32_t n_blocks = (m + kBlock - 1) / kBlock;
  struct Block {
    std::vector<uint32_t> cnt, src, w;
  };
  std::vector<Block> blocks(n_blocks);
  std::atomic<uint32_t> next{0};
  auto worker = [&](size_t, size_t, int) {
    std::vector<uint8_t> mark(n, 0);
    std::vector<uint32_t> stamp(m, kNone);
    std::vector<uint32_t> cand;
    std::vector<std::pair<uint32_t, uint32_t>> hits;
    for (;;) {
      const uint32_t b = next.fetch_add(1);
      if (b >= n_blocks) break;
      Block& out = blocks[b];
      const uint32_t x_lo = b * kBlock, x_hi = std::min(m, x_lo + kBlock);
      out.cnt.assign(x_hi - x_lo, 0);
      for (uint32_t x = x_lo; x < x_hi; ++x) {
        const uint64_t nx = a.row_nnz(x);
        hits.clear();
        if (nx >= alpha && nx > 0) {
          const uint32_t* rx = a.row(x);
          for (uint64_t k = 0; k < nx; ++k) mark[rx[k]] = 1;
          cand.clear();
          for (uint64_t k = 0; k < nx; ++k) {
            const uint32_t c = rx[k];
            for (uint64_t q = inv_ptr[c]; q < inv_ptr[c + 1]; ++q) {
              const uint32_t y = inv_row[q];
              if (y != x && stamp[y] != x) {
                stamp[y] = x;
                cand.push_back(y);
              }
            }
          }
          for (uint32_t y : cand) {
            const uint64_t ny = a.row_nnz(y);
            const uint64_t t = need(ny);
            if (t > nx) continue;  // size filter: ov <= nx < t, (*) cannot hold
            const uint32_t* ry = a.row(y);
            uint64_t ov = 0;
            for (uint64_t k = 0; k < ny; ++k) {
              ov += mark[ry[k]];
              if (ov + (ny - 1 - k) < t) break;  // cannot reach t any more
            }
            if (ov >= t) hits.emplace_back(y + 1, uint32_t(nx + ny - 2 * ov));
          }
          for (uint64_t k = 0; k < nx; ++k) mark[rx[k]] = 0;
          std::sort(hits.begin(), hits.end());
        }
        out.cnt[x - x_lo] = uint32_t(hits.size()) + 1;
        out.src.push_back(0);  // virtual edge first: weight nnz(a_x)
        out.w.push_back(uint32_t(nx));
        for (auto& h : hits) {
          out.src.push_back(h.first);
          out.w.push_back(h.second);
        }
      }
    }
  };
  parallel_for_chunks(size_t(threads), threads, worker);

  EdgeLists e;
  e.ptr.assign(size_t(m) + 1, 0);
  std::vector<uint64_t> boff(size_t(n_blocks) + 1, 0);
  for (uint32_t b = 0; b < n_blocks; ++b) {
    boff[b + 1] = boff[b] + blocks[b].src.size();
    for (uint32_t i = 0; i < blocks[b].cnt.size(); ++i)
      e.ptr[size_t(b) * kBlock + i + 1] = blocks[b].cnt[i];
  }
  std::partial_sum(e.ptr.begin(), e.ptr.end(), e.ptr.begin());
  e.src.resize(boff.back());
  e.w.resize(boff.back());
  parallel_for_chunks(n_blocks, threads, [&](size_t lo, size_t hi, int) {
    for (size_t b = lo; b < hi; ++b) {
      std::copy(blocks[b].src.begin(), blocks[b].src.end(), e.src.begin() + boff[b]);
      std::copy(blocks[b].w.begin(), blocks[b].w.end(), e.w.begin() + boff[b]);
      Block().src.swap(blocks[b].src);
      std::vector<uint32_t>().swap(blocks[b].w);
    }
  });
  return e;
}

// ---------------------------------------------------------------------------
// Chu-Liu/Edmonds
// ---------------------------------------------------------------------------
std::vector<uint32_t> min_arborescence(const EdgeLists& e, uint32_t m, int threads,
                                       uint32_t* n_rounds) {
  if (threads < 1) threads = 1;
  const uint64_t E = e.src.size();
  if (E >= 0xFFFFFFFFull) throw logic_error("arborescence: too many candidate edges");
  // original endpoints per edge
  std::vector<uint32_t> odst(E);
  parallel_for_chunks(m, threads, [&](size_t lo, size_t hi, int) {
    for (size_t x = lo; x < hi; ++x)
      for (uint64_t k = e.ptr[x]; k < e.ptr[x + 1]; ++k) odst[k] = uint32_t(x + 1);
  });
  for (uint32_t x = 0; x < m; ++x)
    if (e.ptr[x + 1] == e.ptr[x] || e.src[e.ptr[x]] != 0)
      throw logic_error("arborescence: row " + std::to_string(x) + " has no virtual edge");
  if (m == 0) return {};

  const auto& osrc = e.src;
  // strict total order of the reference's `better` (builder.cpp:163-170)
  auto orig_less = [&](uint32_t oa, uint32_t ob) {
    const bool va = osrc[oa] == 0, vb = osrc[ob] == 0;
    if (va != vb) return va;
    if (osrc[oa] != osrc[ob]) return osrc[oa] < osrc[ob];
    return odst[oa] < odst[ob];
  };

  // working graph (structure of arrays)
  std::vector<uint32_t> ws(e.src), wd(odst), ww(e.w), wo(E);
  std::iota(wo.begin(), wo.end(), 0u);

  struct Round {
    std::vector<uint32_t> sel, node_map, cycle_of, level_of_orig;
  };
  std::vector<Round> rounds;
  std::vector<uint32_t> level_of_orig(size_t(m) + 1);
  std::iota(level_of_orig.begin(), level_of_orig.end(), 0u);
  uint32_t n_cur = m + 1;
  std::vector<uint32_t> chosen;

  const int T = threads;
  std::vector<std::vector<uint32_t>> local_best(T);
  for (;;) {
    // best in-edge per node (index into the working arrays)
    const uint64_t Ew = ws.size();
    auto better = [&](uint32_t i, uint32_t j) {
      if (ww[i] != ww[j]) return ww[i] < ww[j];
      return orig_less(wo[i], wo[j]);
    };
    std::vector<uint32_t> best(n_cur, kNone);
    parallel_for_chunks(Ew, T, [&](size_t lo, size_t hi, int t) {
      auto& lb = local_best[t];
      lb.assign(n_cur, kNone);
      for (size_t i = lo; i < hi; ++i) {
        const uint32_t v = wd[i];
        if (lb[v] == kNone || better(uint32_t(i), lb[v])) lb[v] = uint32_t(i);
      }
    });
    const int used = int(std::min<uint64_t>(uint64_t(T), std::max<uint64_t>(Ew, 1)));
    parallel_for_chunks(n_cur, T, [&](size_t lo, size_t hi, int) {
      for (size_t v = lo; v < hi; ++v) {
        uint32_t b = kNone;
        for (int t = 0; t < used; ++t) {
          const uint32_t c = local_best[t][v];
          if (c != kNone && (b == kNone || better(c, b))) b = c;
        }
        best[v] = b;
      }
    });
    for (uint32_t v = 1; v < n_cur; ++v)
      if (best[v] == kNone) throw logic_error("arborescence: node lost its incoming edges");

    // cycles among the selected in-edges, discovered in ascending start node
    std::vector<uint32_t> cyc(n_cur, kNone);
    std::vector<uint8_t> state(n_cur, 0);  // 0 unseen, 1 on current walk, 2 settled
    std::vector<uint32_t> walk;
    state[0] = 2;
    uint32_t n_cyc = 0;
    for (uint32_t s = 1; s < n_cur; ++s) {
      if (state[s]) continue;
      walk.clear();
      uint32_t v = s;
      while (!state[v]) {
        state[v] = 1;
        walk.push_back(v);
        v = ws[best[v]];
      }
      if (state[v] == 1) {  // closed a loop at v: the walk suffix from v
        size_t k = walk.size();
        do {
          --k;
          cyc[walk[k]] = n_cyc;
        } while (walk[k] != v);
        ++n_cyc;
      }
      for (uint32_t u : walk) state[u] = 2;
    }

    if (n_cyc == 0) {
      chosen.assign(n_cur, kNone);
      for (uint32_t v = 1; v < n_cur; ++v) chosen[v] = wo[best[v]];
      break;
    }

    Round rec;
    rec.sel.assign(n_cur, kNone);
    for (uint32_t v = 1; v < n_cur; ++v) rec.sel[v] = wo[best[v]];
    rec.level_of_orig = level_of_orig;
    // renumber: root stays 0, every cycle collapses onto the id of its first member
    rec.node_map.assign(n_cur, 0);
    std::vector<uint32_t> cyc_id(n_cyc, kNone);
    uint32_t next_id = 0;
    for (uint32_t v = 0; v < n_cur; ++v) {
      const uint32_t c = cyc[v];
      if (c == kNone) {
        rec.node_map[v] = next_id++;
      } else {
        if (cyc_id[c] == kNone) cyc_id[c] = next_id++;
        rec.node_map[v] = cyc_id[c];
      }
    }
    // contract: drop edges inside a super-node, reduce weights into cycles
    std::vector<uint64_t> keep(size_t(T) + 1, 0);
    auto keep_edge = [&](size_t i) {
      const uint32_t nu = rec.node_map[ws[i]], nv = rec.node_map[wd[i]];
      return nu != nv && nv != 0;
    };
    std::vector<std::pair<size_t, size_t>> span(T, {0, 0});
    parallel_for_chunks(Ew, T, [&](size_t lo, size_t hi, int t) {
      uint64_t k = 0;
      for (size_t i = lo; i < hi; ++i) k += keep_edge(i);
      keep[t + 1] = k;
      span[t] = {lo, hi};
    });
    std::partial_sum(keep.begin(), keep.end(), keep.begin());
    std::vector<uint32_t> ns(keep.back()), nd(keep.back()), nw(keep.back()), no(keep.back());
    parallel_for_chunks(Ew, T, [&](size_t lo, size_t hi, int t) {
      uint64_t o = keep[t];
      for (size_t i = lo; i < hi; ++i) {
        if (!keep_edge(i)) continue;
        const uint32_t dst = wd[i];
        ns[o] = rec.node_map[ws[i]];
        nd[o] = rec.node_map[dst];
        nw[o] = cyc[dst] != kNone ? ww[i] - ww[best[dst]] : ww[i];
        no[o] = wo[i];
        ++o;
      }
    });
    for (auto& v : level_of_orig) v = rec.node_map[v];
    rec.cycle_of = std::move(cyc);
    n_cur = next_id;
    ws.swap(ns);
    wd.swap(nd);
    ww.swap(nw);
    wo.swap(no);
    rounds.push_back(std::move(rec));
  }
  std::vector<uint32_t>().swap(ws);
  std::vector<uint32_t>().swap(wd);
  std::vector<uint32_t>().swap(ww);
  std::vector<uint32_t>().swap(wo);

  // expand, newest contraction first
  for (auto it = rounds.rbegin(); it != rounds.rend(); ++it) {
    const Round& rec = *it;
    const uint32_t nl = uint32_t(rec.node_map.size());
    std::vector<uint32_t> ex(nl, kNone);
    for (uint32_t v = 1; v < nl; ++v)
      ex[v] = rec.cycle_of[v] == kNone ? chosen[rec.node_map[v]] : rec.sel[v];
    for (uint32_t v = 1; v < nl; ++v) {
      if (rec.cycle_of[v] == kNone) continue;
      const uint32_t ext = chosen[rec.node_map[v]];
      if (rec.level_of_orig[odst[ext]] == v) ex[v] = ext;
    }
    chosen.swap(ex);
  }
  if (n_rounds) *n_rounds = uint32_t(rounds.size());

  // re-attach rows whose edge cannot beat their virtual edge (builder.cpp:293-300)
  std::vector<uint32_t> parent(m, kVirtual);
  for (uint32_t x = 0; x < m; ++x) {
    const uint32_t k = chosen[size_t(x) + 1];
    const uint32_t vw = e.w[e.ptr[x]];
    if (osrc[k] != 0 && e.w[k] < vw) parent[x] = osrc[k] - 1;
  }
  return parent;
}

// ---------------------------------------------------------------------------
// Deltas and the full pipeline
// ---------------------------------------------------------------------------
namespace {

// Signed delta matrix against the chain parent (compute_delta_lists +
// assemble_delta_matrix, builder.cpp:304-367): one walk over a_x and a_parent
// emits +1 for columns only in a_x and -1 for columns only in a_parent, in
// ascending column order.
void assemble_deltas(const Csr& a, HostCbm& c, int threads) {
  const uint32_t m = a.n_rows;
  std::vector<uint64_t> len(size_t(m) + 1, 0);
  auto walk = [&](uint32_t x, uint32_t* col, float* val) -> uint64_t {
    const uint32_t* rx = a.row(x);
    const uint64_t nx = a.row_nnz(x);
    if (c.parent[x] == kVirtual) {
      if (col)
        for (uint64_t k = 0; k < nx; ++k) {
          col[k] = rx[k];
          val[k] = 1.0f;
        }
      return nx;
    }
    const uint32_t* rp = a.row(c.parent[x]);
    const uint64_t np = a.row_nnz(c.parent[x]);
    uint64_t i = 0, j = 0, o = 0;
    while (i < nx || j < np) {
      if (j == np || (i < nx && rx[i] < rp[j])) {
        if (col) {
          col[o] = rx[i];
          val[o] = 1.0f;
        }
        ++i, ++o;
      } else if (i == nx || rp[j] < rx[i]) {
        if (col) {
          col[o] = rp[j];
          val[o] = -1.0f;
        }
        ++j, ++o;
      } else {
        ++i, ++j;
      }
    }
    return o;
  };
  parallel_for_chunks(m, threads, [&](size_t lo, size_t hi, int) {
    for (size_t x = lo; x < hi; ++x) len[x + 1] = walk(uint32_t(x), nullptr, nullptr);
  });
  std::partial_sum(len.begin(), len.end(), len.begin());
  c.row_ptr = len;
  c.col_idx.resize(len.back());
  c.values.resize(len.back());
  parallel_for_chunks(m, threads, [&](size_t lo, size_t hi, int) {
    for (size_t x = lo; x < hi; ++x)
      walk(uint32_t(x), c.col_idx.data() + len[x], c.values.data() + len[x]);
  });
}

// Pattern of A + I (with_self_loops, builder.cpp:371-390).
Csr with_diagonal(const Csr& a) {
  Csr r;
  r.n_rows = a.n_rows;
  r.n_cols = a.n_cols;
  r.row_ptr.assign(size_t(a.n_rows) + 1, 0);
  r.col_idx.reserve(a.nnz() + a.n_rows);
  for (uint32_t x = 0; x < a.n_rows; ++x) {
    const uint32_t* rx = a.row(x);
    const uint64_t nx = a.row_nnz(x);
    const uint32_t* pos = std::lower_bound(rx, rx + nx, x);
    r.col_idx.insert(r.col_idx.end(), rx, pos);
    if (pos == rx + nx || *pos != x) r.col_idx.push_back(x);
    r.col_idx.insert(r.col_idx.end(), pos, rx + nx);
    r.row_ptr[x + 1] = r.col_idx.size();
  }
  return r;
}

}  // namespace

HostCbm build_cbm(const Csr& a, uint64_t alpha, int threads, int algo) {
  const auto t0 = Clock::now();
  HostCbm c;
  c.n_rows = a.n_rows;
  c.n_cols = a.n_cols;
  c.alpha = alpha;
  EdgeLists e = candidate_edges(a, alpha, threads);
  c.t_edges = secs(t0);
  c.candidate_edges = e.src.size();
  const auto t1 = Clock::now();
  c.parent = algo == 1 ? min_arborescence(e, a.n_rows, threads, &c.rounds)
                       : min_arborescence_heap(e, a.n_rows, &c.rounds, threads);
  EdgeLists().ptr.swap(e.ptr);
  std::vector<uint32_t>().swap(e.src);
  std::vector<uint32_t>().swap(e.w);
  chain_from_parents(c);
  c.t_arb = secs(t1);
  const auto t2 = Clock::now();
  assemble_deltas(a, c, threads);
  c.t_deltas = secs(t2);
  c.t_total = secs(t0);
  return c;
}

HostCbm build_cbm_normalized(const Csr& a, uint64_t alpha, int threads,
                             bool degrees_from_original, int algo) {
  if (a.n_rows != a.n_cols)
    throw invalid_argument("build_cbm_normalized: matrix must be square");
  const auto t0 = Clock::now();
  const Csr aug = with_diagonal(a);
  std::vector<float> scale(a.n_rows);
  for (uint32_t x = 0; x < a.n_rows; ++x) {
    const uint64_t d = degrees_from_original ? a.row_nnz(x) : aug.row_nnz(x);
    if (d == 0)
      throw invalid_argument("build_cbm_normalized: zero degree at row " + std::to_string(x) +
                             " (isolated vertex with DegreeMode::original)");
    // builder.cpp:420: real_t(1) / static_cast<real_t>(std::sqrt(double(d)))
    scale[x] = 1.0f / static_cast<float>(std::sqrt(static_cast<double>(d)));
  }
  HostCbm c = build_cbm(aug, alpha, threads, algo);
  for (uint64_t k = 0; k < c.values.size(); ++k) c.values[k] *= scale[c.col_idx[k]];
  c.row_scale = std::move(scale);
  c.normalized = true;
  c.t_total = secs(t0);
  return c;
}

}  // namespace cbmb
