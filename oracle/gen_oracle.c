/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the seeded workload
 * generators, so that bench.py's reference arm and the tests can draw every
 * BASELINE.json config's graph and operand WITHOUT loading the product
 * library (paper_2409_02208_b200/libcbm_b200.so). tests/test_oracle_gen.py
 * pins each one against the product's generators (csrc/graphs.cpp and
 * cbm_b200_gen_dense) on identical seeds: same edges, same bits.
 *
 * Every stream is the reference's UniformRng (prng.hpp:11-28: std::mt19937_64,
 * unit() = (g() >> 11) * 2^-53, below(n) = g() % n), restated in
 * cbm_oracle.c (oracle_rng_*). The graph definitions are the workloads of
 * DESIGN.md §8 (BASELINE.json configs); CSR assembly follows
 * CsrBinaryMatrix::from_coo (csr.cpp:44-66): rows sorted, duplicates merged.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint64_t mt[312];
  int idx;
} oracle_rng;
void oracle_rng_seed(oracle_rng* r, uint64_t seed);
uint64_t oracle_rng_bits(oracle_rng* r);
double oracle_rng_unit(oracle_rng* r);

static uint64_t below(oracle_rng* r, uint64_t n) { return n ? oracle_rng_bits(r) % n : 0; }

/* growable edge list of (row, col) pairs, both directions */
typedef struct {
  uint32_t* u;
  uint32_t* v;
  uint64_t n, cap;
} edges;

static int push(edges* e, uint32_t a, uint32_t b) {
  if (e->n + 2 > e->cap) {
    uint64_t cap = e->cap ? e->cap * 2 : 1024;
    uint32_t* nu = realloc(e->u, cap * 4);
    if (!nu) return -1;
    e->u = nu;
    uint32_t* nv = realloc(e->v, cap * 4);
    if (!nv) return -1;
    e->v = nv;
    e->cap = cap;
  }
  e->u[e->n] = a;
  e->v[e->n++] = b;
  e->u[e->n] = b;
  e->v[e->n++] = a;
  return 0;
}

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}

/* Result of a generator: CSR arrays owned by the library, freed with
 * oracle_graph_free. */
typedef struct {
  uint32_t n_rows, n_cols;
  uint64_t nnz;
  uint64_t* row_ptr;
  uint32_t* col_idx;
} oracle_graph;

/* sort + dedup rows [lo, hi) of the bucketed columns */
typedef struct {
  uint32_t* cols;
  const uint64_t* cnt;
  uint64_t* keep;
  uint32_t lo, hi;
} sort_job;

static void* sort_rows(void* arg) {
  sort_job* j = arg;
  for (uint32_t r = j->lo; r < j->hi; ++r) {
    uint32_t* b = j->cols + j->cnt[r];
    const uint64_t len = j->cnt[r + 1] - j->cnt[r];
    if (len > 1) qsort(b, len, 4, cmp_u32);
    uint64_t w = 0;
    for (uint64_t i = 0; i < len; ++i)
      if (i == 0 || b[i] != b[i - 1]) b[w++] = b[i];
    j->keep[r] = w;
  }
  return NULL;
}

/* counting sort by row, then sort + dedup each row (threads over row ranges) */
static int assemble(edges* e, uint32_t n, oracle_graph* g) {
  uint64_t* cnt = calloc((size_t)n + 1, 8);
  uint32_t* cols = malloc((e->n ? e->n : 1) * 4);
  if (!cnt || !cols) return -1;
  for (uint64_t i = 0; i < e->n; ++i) ++cnt[e->u[i] + 1];
  for (uint32_t r = 0; r < n; ++r) cnt[r + 1] += cnt[r];
  {
    uint64_t* cur = malloc(((size_t)n + 1) * 8);
    if (!cur) return -1;
    memcpy(cur, cnt, ((size_t)n + 1) * 8);
    for (uint64_t i = 0; i < e->n; ++i) cols[cur[e->u[i]]++] = e->v[i];
    free(cur);
  }
  free(e->u);
  free(e->v);
  e->u = e->v = NULL;
  uint64_t* keep = malloc(((size_t)n + 1) * 8);
  if (!keep) return -1;
  {
    enum { kThreads = 16 };
    pthread_t th[kThreads];
    sort_job jobs[kThreads];
    int started[kThreads] = {0};
    for (int t = 0; t < kThreads; ++t) {
      jobs[t].cols = cols;
      jobs[t].cnt = cnt;
      jobs[t].keep = keep;
      jobs[t].lo = (uint32_t)((uint64_t)n * t / kThreads);
      jobs[t].hi = (uint32_t)((uint64_t)n * (t + 1) / kThreads);
      started[t] = pthread_create(&th[t], NULL, sort_rows, &jobs[t]) == 0;
      if (!started[t]) sort_rows(&jobs[t]);
    }
    for (int t = 0; t < kThreads; ++t)
      if (started[t]) pthread_join(th[t], NULL);
  }
  g->row_ptr = malloc(((size_t)n + 1) * 8);
  if (!g->row_ptr) return -1;
  g->row_ptr[0] = 0;
  for (uint32_t r = 0; r < n; ++r) g->row_ptr[r + 1] = g->row_ptr[r] + keep[r];
  g->nnz = g->row_ptr[n];
  g->col_idx = malloc((g->nnz ? g->nnz : 1) * 4);
  if (!g->col_idx) return -1;
  for (uint32_t r = 0; r < n; ++r)
    memcpy(g->col_idx + g->row_ptr[r], cols + cnt[r], keep[r] * 4);
  free(keep);
  free(cols);
  free(cnt);
  g->n_rows = g->n_cols = n;
  return 0;
}

/* Planted communities: intra pairs (community, i < j) as Bernoulli draws in
 * order; inter pairs by geometric skipping over the row-major sequence of all
 * pairs i < j, landings inside a community ignored. */
static int gen_community(const double* p, uint64_t seed, oracle_graph* g) {
  const uint32_t n = (uint32_t)p[0], size = (uint32_t)p[1];
  const double p_in = p[2], p_out = p[3];
  oracle_rng r;
  oracle_rng_seed(&r, seed);
  edges e = {0};
  for (uint32_t c0 = 0; c0 < n; c0 += size) {
    const uint32_t c1 = c0 + size < n ? c0 + size : n;
    for (uint32_t i = c0; i < c1; ++i)
      for (uint32_t j = i + 1; j < c1; ++j)
        if (oracle_rng_unit(&r) < p_in && push(&e, i, j)) return -1;
  }
  if (p_out > 0 && n > 1) {
    const double lq = log1p(-p_out);
    uint64_t i = 0, j = 0;
    for (;;) {
      const double u = oracle_rng_unit(&r);
      uint64_t step = (uint64_t)floor(log1p(-u) / lq) + 1;
      while (i < (uint64_t)n - 1) {
        const uint64_t room = ((uint64_t)n - 1) - j;
        if (step <= room) {
          j += step;
          break;
        }
        step -= room;
        ++i;
        j = i;
      }
      if (i >= (uint64_t)n - 1) break;
      if (i / size != j / size && push(&e, (uint32_t)i, (uint32_t)j)) return -1;
    }
  }
  return assemble(&e, n, g);
}

/* adjacency lists for the preferential-attachment generator */
typedef struct {
  uint32_t* a;
  uint32_t n, cap;
} alist;

static int apush(alist* l, uint32_t v) {
  if (l->n == l->cap) {
    uint32_t cap = l->cap ? l->cap * 2 : 8;
    uint32_t* na = realloc(l->a, (size_t)cap * 4);
    if (!na) return -1;
    l->a = na;
    l->cap = cap;
  }
  l->a[l->n++] = v;
  return 0;
}

static int linked(const alist* adj, uint32_t u, uint32_t v) {
  const alist* l = adj[u].n < adj[v].n ? &adj[u] : &adj[v];
  const uint32_t w = adj[u].n < adj[v].n ? v : u;
  for (uint32_t i = 0; i < l->n; ++i)
    if (l->a[i] == w) return 1;
  return 0;
}

/* Preferential attachment (m edges per new node to endpoints drawn from the
 * pool of all edge endpoints) with Holme–Kim triangle closing; seed triangle
 * on nodes 0..m. */
static int gen_pa_triangle(const double* p, uint64_t seed, oracle_graph* g) {
  const uint32_t n = (uint32_t)p[0], m = (uint32_t)p[1];
  const double pt = p[2];
  oracle_rng r;
  oracle_rng_seed(&r, seed);
  alist* adj = calloc(n ? n : 1, sizeof(alist));
  alist pool = {0};
  if (!adj) return -1;
#define LINK(U, V)                                                        \
  do {                                                                    \
    if (apush(&adj[U], V) || apush(&adj[V], U) || apush(&pool, U) ||      \
        apush(&pool, V))                                                  \
      return -1;                                                          \
  } while (0)
  const uint32_t s = n < m + 1 ? n : m + 1;
  for (uint32_t i = 0; i < s; ++i)
    for (uint32_t j = i + 1; j < s; ++j) LINK(i, j);
  for (uint32_t v = s; v < n; ++v) {
    uint32_t made = 0, guard = 0;
    while (made < m && guard++ < 64 * m) {
      const uint32_t t = pool.a[below(&r, pool.n)];
      if (t == v || linked(adj, v, t)) continue;
      LINK(v, t);
      ++made;
      if (oracle_rng_unit(&r) < pt) {
        for (int tries = 0; tries < 8; ++tries) {
          const uint32_t u = adj[t].a[below(&r, adj[t].n)];
          if (u != v && !linked(adj, v, u)) {
            LINK(v, u);
            break;
          }
        }
      }
    }
  }
#undef LINK
  edges e = {0};
  for (uint32_t u = 0; u < n; ++u)
    for (uint32_t k = 0; k < adj[u].n; ++k) {
      /* one direction per adjacency entry (both lists hold the edge) */
      if (e.n + 1 > e.cap) {
        uint64_t cap = e.cap ? e.cap * 2 : 1024;
        e.u = realloc(e.u, cap * 4);
        e.v = realloc(e.v, cap * 4);
        if (!e.u || !e.v) return -1;
        e.cap = cap;
      }
      e.u[e.n] = u;
      e.v[e.n++] = adj[u].a[k];
    }
  for (uint32_t u = 0; u < n; ++u) free(adj[u].a);
  free(adj);
  free(pool.a);
  return assemble(&e, n, g);
}

/* Clique overlay: popularity rank r (1-based) has weight r^-s; ranks map to
 * node ids through a seeded Fisher–Yates permutation; each group draws its size
 * uniformly in [k_min, k_max], then that many distinct members by inverse-CDF
 * sampling (duplicates redrawn), and adds the clique. */
static int gen_clique_overlay(const double* p, uint64_t seed, oracle_graph* g) {
  const uint32_t n = (uint32_t)p[0];
  const uint64_t groups = (uint64_t)p[1];
  const uint32_t kmin = (uint32_t)p[2], kmax = (uint32_t)p[3];
  const double s = p[4];
  oracle_rng r;
  oracle_rng_seed(&r, seed);
  uint32_t* perm = malloc((size_t)(n ? n : 1) * 4);
  double* cdf = malloc((size_t)(n ? n : 1) * 8);
  if (!perm || !cdf) return -1;
  for (uint32_t i = 0; i < n; ++i) perm[i] = i;
  for (uint32_t i = n; i > 1; --i) {
    const uint32_t k = (uint32_t)below(&r, i);
    const uint32_t t = perm[i - 1];
    perm[i - 1] = perm[k];
    perm[k] = t;
  }
  double acc = 0;
  for (uint32_t q = 0; q < n; ++q) {
    acc += pow((double)(q + 1), -s);
    cdf[q] = acc;
  }
  for (uint32_t q = 0; q < n; ++q) cdf[q] /= acc;
  edges e = {0};
  uint32_t mem[64];
  for (uint64_t gi = 0; gi < groups; ++gi) {
    const uint32_t k = kmin + (uint32_t)below(&r, kmax - kmin + 1);
    if (k > 64) return -1;
    uint32_t have = 0;
    while (have < k) {
      const double u = oracle_rng_unit(&r);
      /* upper_bound: first index with cdf > u */
      uint32_t lo = 0, hi = n;
      while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (cdf[mid] > u) hi = mid;
        else lo = mid + 1;
      }
      uint32_t q = lo >= n ? n - 1 : lo;
      const uint32_t node = perm[q];
      int dup = 0;
      for (uint32_t t = 0; t < have; ++t) dup |= mem[t] == node;
      if (!dup) mem[have++] = node;
    }
    for (uint32_t a = 0; a < k; ++a)
      for (uint32_t b = a + 1; b < k; ++b)
        if (push(&e, mem[a], mem[b])) return -1;
  }
  free(perm);
  free(cdf);
  return assemble(&e, n, g);
}

/* kind: 0 community {n, size, p_in, p_out}; 1 pa_triangle {n, m, p};
 * 2 clique_overlay {n, groups, k_min, k_max, s}. Returns 0 on success. */
int oracle_gen_graph(int kind, const double* params, uint64_t seed, oracle_graph* out) {
  memset(out, 0, sizeof(*out));
  switch (kind) {
    case 0: return gen_community(params, seed, out);
    case 1: return gen_pa_triangle(params, seed, out);
    case 2: return gen_clique_overlay(params, seed, out);
    default: return -2;
  }
}

void oracle_graph_free(oracle_graph* g) {
  free(g->row_ptr);
  free(g->col_idx);
  memset(g, 0, sizeof(*g));
}

/* Dense operands: kind 1 = integers below(hi-lo+1)+lo, 2 = N(0,1) by
 * Box–Muller over two unit() draws (computed in double, rounded to f32),
 * 3 = Glorot-uniform for a rows x cols (fan_in x fan_out) weight. (Kind 0,
 * random_dense, is oracle_random_dense in cbm_oracle.c.) */
int oracle_gen_dense(int kind, uint64_t rows, uint64_t cols, double lo, double hi,
                     uint64_t seed, float* out) {
  oracle_rng r;
  oracle_rng_seed(&r, seed);
  const uint64_t n = rows * cols;
  if (kind == 1) {
    const int64_t a = (int64_t)lo, b = (int64_t)hi;
    if (b < a) return -1;
    for (uint64_t i = 0; i < n; ++i)
      out[i] = (float)((int64_t)below(&r, (uint64_t)(b - a + 1)) + a);
  } else if (kind == 2) {
    for (uint64_t i = 0; i < n; i += 2) {
      const double u1 = oracle_rng_unit(&r), u2 = oracle_rng_unit(&r);
      const double rad = sqrt(-2.0 * log1p(-u1));
      const double th = 6.283185307179586 * u2;
      out[i] = (float)(rad * cos(th));
      if (i + 1 < n) out[i + 1] = (float)(rad * sin(th));
    }
  } else if (kind == 3) {
    const double b = sqrt(6.0 / (double)(rows + cols));
    for (uint64_t i = 0; i < n; ++i) out[i] = (float)(-b + 2.0 * b * oracle_rng_unit(&r));
  } else {
    return -1;
  }
  return 0;
}
