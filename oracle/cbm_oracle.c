/*
 * TEST INFRASTRUCTURE ONLY — the parity oracle. Never linked into, or called
 * by, the product path (paper_2409_02208_b200/). Only tests/, smoke() and the
 * cpu_baseline leg of bench.py load it, as the checker.
 *
 * Plain-C restatement of the reference CBM multiply in its f32 build
 * (proj/include/cbm/types.hpp:8-12 with CBM_SINGLE_PRECISION). Pinned against
 * the reference itself (oracle/_ref/libcbmref.so, built by oracle/Makefile from
 * the reference sources) and against tests/golden/*.npz in
 * tests/test_oracle.py. Compiled with -ffp-contract=off: the reference's
 * object code has no FMA (x86-64 baseline, SSE mulps/addps), so each product
 * is rounded before the add.
 *
 * Numeric contract restated here:
 *   stage 1  (kernels.cpp:27-36)  U[i,j] = fl(...fl(fl(+0 + fl(v0*X[c0,j])) + fl(v1*X[c1,j]))...)
 *                                 deltas of row i taken in ascending storage order
 *   stage 2  (kernels.cpp:42-53)  U[x,j] = fl(U[x,j] + U[parent(x),j]) in topo order
 *                                 (children read the UNSCALED parent)
 *   stage 3  (kernels.cpp:54-60)  Y[x,j] = fl(U[x,j] * row_scale[x])   (normalized only)
 */
#include <stdint.h>
#include <string.h>

#define VIRTUAL_PARENT 0xFFFFFFFFu /* kVirtualParent, types.hpp:19 */

/* spmm_into (kernels.cpp:105-123). topo must list parents before children
 * (CompressionChain::topo_order, builder.cpp:44-61); any such order gives the
 * same bits because each row's update reads only its own parent. */
void oracle_spmm(uint32_t m, uint32_t d, const uint32_t* parent,
                 const uint32_t* topo, const uint64_t* row_ptr,
                 const uint32_t* col_idx, const float* values,
                 const float* row_scale, int normalized, const float* x,
                 uint64_t ldx, float* y, uint64_t ldy) {
  /* stage 1: y_i = delta_i * X, ascending k, +0 start */
  for (uint32_t i = 0; i < m; ++i) {
    float* out = y + (uint64_t)i * ldy;
    for (uint32_t j = 0; j < d; ++j) out[j] = 0.0f;
    for (uint64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      const float v = values[k];
      const float* in = x + (uint64_t)col_idx[k] * ldx;
      for (uint32_t j = 0; j < d; ++j) {
        const float prod = v * in[j];
        out[j] = out[j] + prod;
      }
    }
  }
  /* stage 2: y_x += y_parent along topo order */
  for (uint32_t t = 0; t < m; ++t) {
    const uint32_t r = topo[t];
    const uint32_t p = parent[r];
    if (p == VIRTUAL_PARENT) continue;
    float* dst = y + (uint64_t)r * ldy;
    const float* src = y + (uint64_t)p * ldy;
    for (uint32_t j = 0; j < d; ++j) dst[j] = dst[j] + src[j];
  }
  /* stage 3: deferred row scaling */
  if (normalized) {
    for (uint32_t i = 0; i < m; ++i) {
      float* out = y + (uint64_t)i * ldy;
      const float s = row_scale[i];
      for (uint32_t j = 0; j < d; ++j) out[j] = out[j] * s;
    }
  }
}

/* csr_spmm_into (kernels.cpp:152-168): per row, ascending k, +0 start. */
void oracle_csr_spmm(uint32_t m, uint32_t d, const uint64_t* row_ptr,
                     const uint32_t* col_idx, const float* values,
                     const float* x, uint64_t ldx, float* y, uint64_t ldy) {
  for (uint32_t i = 0; i < m; ++i) {
    float* out = y + (uint64_t)i * ldy;
    for (uint32_t j = 0; j < d; ++j) out[j] = 0.0f;
    for (uint64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      const float v = values[k];
      const float* in = x + (uint64_t)col_idx[k] * ldx;
      for (uint32_t j = 0; j < d; ++j) {
        const float prod = v * in[j];
        out[j] = out[j] + prod;
      }
    }
  }
}

/* Reference GEMM (dense.cpp:31-49): c[i,:] += a[i,j] * b[j,:] over ascending j,
 * zero lhs entries skipped; products rounded before the add. */
void oracle_dense_matmul(uint32_t m, uint32_t k, uint32_t n, const float* a,
                         const float* b, float* c) {
  memset(c, 0, sizeof(float) * (size_t)m * n);
  for (uint32_t i = 0; i < m; ++i) {
    float* out = c + (uint64_t)i * n;
    for (uint32_t j = 0; j < k; ++j) {
      const float v = a[(uint64_t)i * k + j];
      if (v == 0.0f) continue;
      const float* in = b + (uint64_t)j * n;
      for (uint32_t q = 0; q < n; ++q) {
        const float prod = v * in[q];
        out[q] = out[q] + prod;
      }
    }
  }
}

/* ------------------------------------------------------------------------
 * UniformRng (prng.hpp:11-28): std::mt19937_64 with the standard parameters,
 * unit() = (g() >> 11) * 2^-53, below(n) = g() % n. Restated so tests can
 * regenerate the reference's seeded instances without the reference.
 * ---------------------------------------------------------------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
} oracle_rng;

void oracle_rng_seed(oracle_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) +
               (uint64_t)i;
  r->idx = 312;
}

uint64_t oracle_rng_bits(oracle_rng* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (r->mt[i] & 0xFFFFFFFF80000000ULL) |
                         (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = r->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = v;
    }
    r->idx = 0;
  }
  uint64_t z = r->mt[r->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

double oracle_rng_unit(oracle_rng* r) {
  return (double)(oracle_rng_bits(r) >> 11) * 0x1.0p-53;
}

/* random_dense (dense.cpp:56-62): row-major, v = (float)(lo + (hi-lo)*unit()) */
void oracle_random_dense(uint32_t rows, uint32_t cols, double lo, double hi,
                         uint64_t seed, float* out) {
  oracle_rng r;
  oracle_rng_seed(&r, seed);
  for (uint64_t i = 0; i < (uint64_t)rows * cols; ++i)
    out[i] = (float)(lo + (hi - lo) * oracle_rng_unit(&r));
}

/* random_binary (oracles.hpp:167-175): row-major Bernoulli sweep. Writes the
 * CSR pattern; row_ptr has rows+1 entries, col_idx capacity rows*cols.
 * Returns nnz. */
uint64_t oracle_random_binary(uint32_t rows, uint32_t cols, double density,
                              uint64_t seed, uint64_t* row_ptr,
                              uint32_t* col_idx) {
  oracle_rng r;
  oracle_rng_seed(&r, seed);
  uint64_t nnz = 0;
  row_ptr[0] = 0;
  for (uint32_t i = 0; i < rows; ++i) {
    for (uint32_t j = 0; j < cols; ++j)
      if (oracle_rng_unit(&r) < density) col_idx[nnz++] = j;
    row_ptr[i + 1] = nnz;
  }
  return nnz;
}

/* Exact-as-possible product for parity judging: y = A x (or
 * S (A + I) S x with s = row_scale when scale != NULL) over a CSR pattern,
 * every product and sum in double. Used where the reference's own f32
 * sequential sums drift (rows with ~1e6 entries): the test then requires the
 * device result within the tolerance of THIS product and reports how far the
 * reference itself is from it. add_identity: include the diagonal entry of
 * each row if the pattern lacks it (normalized_adjacency_csr, gcn.cpp:48-89). */
void oracle_csr_spmm_f64(uint32_t m, uint32_t d, const uint64_t* row_ptr,
                         const uint32_t* col_idx, const float* scale, int add_identity,
                         const float* x, uint64_t ldx, double* y, uint64_t ldy) {
  for (uint32_t r = 0; r < m; ++r) {
    double* yr = y + (uint64_t)r * ldy;
    for (uint32_t j = 0; j < d; ++j) yr[j] = 0.0;
    int has_diag = 0;
    for (uint64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
      const uint32_t c = col_idx[k];
      has_diag |= c == r;
      const double sc = scale ? (double)scale[c] : 1.0;
      const float* xc = x + (uint64_t)c * ldx;
      for (uint32_t j = 0; j < d; ++j) yr[j] += sc * (double)xc[j];
    }
    if (add_identity && !has_diag) {
      const double sc = scale ? (double)scale[r] : 1.0;
      const float* xc = x + (uint64_t)r * ldx;
      for (uint32_t j = 0; j < d; ++j) yr[j] += sc * (double)xc[j];
    }
    if (scale) {
      const double sr = (double)scale[r];
      for (uint32_t j = 0; j < d; ++j) yr[j] *= sr;
    }
  }
}
