// Chu-Liu/Edmonds with mergeable heaps — the same arborescence as the
// reference's round-synchronous contraction (find_min_arborescence,
// proj/src/builder.cpp:141-302), in O(E log E) instead of O(E * rounds).
//
// Why the result is identical:
//  * Edges are compared by the reference's strict total order (reduced weight,
//    virtual source first, smaller original source, smaller original
//    destination), so every "best in-edge" is unique.
//  * Rounds stay synchronous: all cycles among the current best edges are
//    contracted together, then best edges are recomputed. A node that was not
//    contracted keeps its best edge (its in-edges and their reduced weights are
//    unchanged), so only the new super-nodes are re-selected, and any new
//    cycle passes through a new super-node.
//  * Reductions are the reference's: contracting cycle member v subtracts
//    best_weight(v) from every edge whose current destination is v — a lazy
//    add on v's heap. A super-node's candidate set is the union of its members'
//    in-edges minus edges whose source is inside it, exactly the edges the
//    reference keeps (nu != nv).
//  * Expansion: a contracted cycle keeps every member's cycle edge except at
//    the member containing the destination of the edge chosen for the
//    super-node, which takes that edge (builder.cpp:268-288).
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <string>
#include <vector>

#include "cbm_host.hpp"

namespace cbmb {

namespace {

constexpr uint32_t kNil = 0xFFFFFFFFu;

struct Heaps {
  // one leftist-heap node per original edge
  std::vector<int64_t> key, lazy;
  std::vector<uint32_t> left, right;
  std::vector<uint8_t> rank;
  const std::vector<uint32_t>* src;
  const std::vector<uint32_t>* dst;
  std::vector<uint32_t> spine;  // merge scratch

  bool less(uint32_t a, uint32_t b) const {  // a before b (keys already pushed)
    if (key[a] != key[b]) return key[a] < key[b];
    const uint32_t sa = (*src)[a], sb = (*src)[b];
    if ((sa == 0) != (sb == 0)) return sa == 0;
    if (sa != sb) return sa < sb;
    return (*dst)[a] < (*dst)[b];
  }
  void push(uint32_t n) {
    if (n == kNil || lazy[n] == 0) return;
    const int64_t z = lazy[n];
    key[n] += z;
    if (left[n] != kNil) lazy[left[n]] += z;
    if (right[n] != kNil) lazy[right[n]] += z;
    lazy[n] = 0;
  }
  uint8_t rk(uint32_t n) const { return n == kNil ? 0 : rank[n]; }
  // iterative leftist merge along the right spines (scratch: the spine)
  uint32_t merge(uint32_t a, uint32_t b) { return merge_with(a, b, spine); }
  uint32_t merge_with(uint32_t a, uint32_t b, std::vector<uint32_t>& spine) {
    if (a == kNil) return b;
    if (b == kNil) return a;
    spine.clear();
    uint32_t root = kNil;
    while (a != kNil && b != kNil) {
      push(a);
      push(b);
      if (less(b, a)) std::swap(a, b);
      spine.push_back(a);
      if (root == kNil) root = a;
      const uint32_t next = right[a];
      a = next;
    }
    uint32_t tail = a != kNil ? a : b;
    for (size_t i = spine.size(); i-- > 0;) {
      const uint32_t n = spine[i];
      right[n] = tail;
      if (rk(left[n]) < rk(right[n])) std::swap(left[n], right[n]);
      rank[n] = uint8_t(std::min<int>(255, rk(right[n]) + 1));
      tail = n;
    }
    return tail;
  }
  uint32_t pop(uint32_t n) {
    push(n);
    return merge(left[n], right[n]);
  }
};

struct Dsu {
  std::vector<uint32_t> p;
  uint32_t find(uint32_t x) {
    uint32_t r = x;
    while (p[r] != r) r = p[r];
    while (p[x] != r) {
      const uint32_t n = p[x];
      p[x] = r;
      x = n;
    }
    return r;
  }
};

}  // namespace

std::vector<uint32_t> min_arborescence_heap(const EdgeLists& e, uint32_t m, uint32_t* n_rounds,
                                            int threads) {
  if (threads < 1) threads = 1;
  const uint64_t E = e.src.size();
  if (E >= 0xFFFFFFFFull) throw logic_error("arborescence: too many candidate edges");
  for (uint32_t x = 0; x < m; ++x)
    if (e.ptr[x + 1] == e.ptr[x] || e.src[e.ptr[x]] != 0)
      throw logic_error("arborescence: row " + std::to_string(x) + " has no virtual edge");
  if (m == 0) return {};
  std::vector<uint32_t> odst(E);
  parallel_for_chunks(m, threads, [&](size_t lo, size_t hi, int) {
    for (size_t x = lo; x < hi; ++x)
      for (uint64_t k = e.ptr[x]; k < e.ptr[x + 1]; ++k) odst[k] = uint32_t(x + 1);
  });

  Heaps H;
  H.key.resize(E);
  H.lazy.assign(E, 0);
  H.left.assign(E, kNil);
  H.right.assign(E, kNil);
  H.rank.assign(E, 1);
  H.src = &e.src;
  H.dst = &odst;
  for (uint64_t k = 0; k < E; ++k) H.key[k] = e.w[k];

  // node ids: 0 = virtual root, 1..m rows, m+1.. super-nodes (at most m-1 of them)
  const uint32_t cap = 2 * m + 1;
  std::vector<uint32_t> heap(cap, kNil), best(cap, kNil), sup(cap, kNil);
  std::vector<int64_t> bestw(cap, 0);
  Dsu dsu;
  dsu.p.resize(cap);
  std::iota(dsu.p.begin(), dsu.p.end(), 0u);
  // initial heaps: balanced pairwise merging of each row's in-edges (rows
  // own disjoint edge nodes, so they build in parallel)
  parallel_for_chunks(m, threads, [&](size_t lo, size_t hi, int) {
    std::vector<uint32_t> q, spine;
    for (size_t x = lo; x < hi; ++x) {
      q.clear();
      for (uint64_t k = e.ptr[x]; k < e.ptr[x + 1]; ++k) q.push_back(uint32_t(k));
      while (q.size() > 1) {
        size_t o = 0;
        for (size_t i = 0; i + 1 < q.size(); i += 2) q[o++] = H.merge_with(q[i], q[i + 1], spine);
        if (q.size() & 1) q[o++] = q.back();
        q.resize(o);
      }
      heap[x + 1] = q[0];
    }
  });
  // super-node bookkeeping for the expansion: members and their cycle edges
  std::vector<uint32_t> mem_ptr{0}, mem_node, mem_edge;

  std::vector<uint32_t> fresh(m);
  std::iota(fresh.begin(), fresh.end(), 1u);
  std::vector<uint32_t> stamp(cap, 0), onpath(cap, 0);
  uint32_t next_id = m + 1, rounds = 0, walk_id = 0;
  std::vector<uint32_t> path, created;
  for (;;) {
    // best in-edge of every new node: discard edges that became internal
    for (uint32_t v : fresh) {
      uint32_t h = heap[v];
      for (;;) {
        if (h == kNil) throw logic_error("arborescence: node lost its incoming edges");
        H.push(h);
        if (dsu.find(e.src[h]) != v) break;
        h = H.pop(h);
      }
      heap[v] = h;
      best[v] = h;
      bestw[v] = H.key[h];
    }
    // cycles among the best edges; every new cycle passes through a new node
    created.clear();
    ++walk_id;
    for (uint32_t v0 : fresh) {
      if (stamp[v0] == walk_id) continue;
      path.clear();
      uint32_t v = v0;
      while (v != 0 && stamp[v] != walk_id) {
        stamp[v] = walk_id;
        onpath[v] = v0;
        path.push_back(v);
        v = dsu.find(e.src[best[v]]);
      }
      if (v == 0 || onpath[v] != v0) continue;  // reached the root or an older walk
      // contract the cycle v -> ... -> v (the suffix of this walk from v)
      size_t k = path.size();
      while (path[--k] != v) {
      }
      const uint32_t S = next_id++;
      uint32_t hs = kNil;
      for (size_t i = k; i < path.size(); ++i) {
        const uint32_t c = path[i];
        if (heap[c] != kNil) H.lazy[heap[c]] -= bestw[c];
        hs = H.merge(hs, heap[c]);
        heap[c] = kNil;
        dsu.p[c] = S;
        sup[c] = S;
        mem_node.push_back(c);
        mem_edge.push_back(best[c]);
      }
      mem_ptr.push_back(uint32_t(mem_node.size()));
      heap[S] = hs;
      stamp[S] = walk_id;
      onpath[S] = 0;
      created.push_back(S);
    }
    if (created.empty()) break;
    ++rounds;
    fresh = created;
  }
  if (n_rounds) *n_rounds = rounds;

  // expansion, newest super-node first
  std::vector<uint32_t> chosen(next_id, kNil);
  for (uint32_t v = 1; v < next_id; ++v)
    if (dsu.find(v) == v) chosen[v] = best[v];  // top-level nodes
  for (uint32_t S = next_id; S-- > m + 1;) {
    const uint32_t ext = chosen[S];
    uint32_t entry = odst[ext];
    while (sup[entry] != S) entry = sup[entry];
    const uint32_t j = S - (m + 1);
    for (uint32_t q = mem_ptr[j]; q < mem_ptr[j + 1]; ++q)
      chosen[mem_node[q]] = mem_node[q] == entry ? ext : mem_edge[q];
  }
  // re-attach rows whose edge cannot beat their virtual edge (builder.cpp:293-300)
  std::vector<uint32_t> parent(m, kVirtual);
  for (uint32_t x = 0; x < m; ++x) {
    const uint32_t k = chosen[x + 1];
    if (e.src[k] != 0 && e.w[k] < e.w[e.ptr[x]]) parent[x] = e.src[k] - 1;
  }
  return parent;
}

}  // namespace cbmb
