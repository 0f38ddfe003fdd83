// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C entry points over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile with -DCBM_SINGLE_PRECISION into
// oracle/_ref/libcbmref.so). Python reaches them through oracle/ref.py (ctypes)
// to (a) pin the C restatement in oracle/cbm_oracle.c, (b) generate the golden
// fixtures under tests/golden/, and (c) time the reference CPU path for
// bench.py's cpu_baseline leg and `--impl reference`.
//
// Every function maps 1:1 onto a reference call site:
//   ref_build_cbm / ref_build_cbm_normalized  -> proj/src/builder.cpp:394,406
//   ref_spmm / ref_spmv / ref_spmm_sequential -> proj/src/kernels.cpp:105,70,131
//   ref_csr_spmm                              -> proj/src/kernels.cpp:152 (+ gcn.cpp:48 / csr.cpp:84)
//   ref_gcn_forward                           -> proj/src/gcn.cpp:22
//   generators                                -> proj/tests/oracles.hpp:167-237
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "cbm/builder.hpp"
#include "cbm/csr.hpp"
#include "cbm/dense.hpp"
#include "cbm/gcn.hpp"
#include "cbm/io.hpp"
#include "cbm/kernels.hpp"
#include "oracles.hpp"

static_assert(sizeof(cbm::real_t) == 4, "oracle must be the f32 build");

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

cbm::DenseMatrix dense_from(const float* p, uint32_t rows, uint32_t cols) {
  return cbm::DenseMatrix(rows, cols,
                          std::vector<float>(p, p + size_t(rows) * cols));
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int ref_real_bytes() { return int(sizeof(cbm::real_t)); }
int ref_hw_threads() { return int(std::thread::hardware_concurrency()); }

// ---------------------------------------------------------------- CSR
void* ref_csr_from_arrays(uint32_t rows, uint32_t cols, const uint64_t* rp,
                          const uint32_t* ci) {
  cbm::CsrBinaryMatrix* out = nullptr;
  guard([&] {
    std::vector<uint64_t> r(rp, rp + rows + 1);
    std::vector<uint32_t> c(ci, ci + r.back());
    out = new cbm::CsrBinaryMatrix(rows, cols, std::move(r), std::move(c));
  });
  return out;
}
void* ref_gen_random_binary(uint32_t rows, uint32_t cols, double density,
                            uint64_t seed) {
  return new cbm::CsrBinaryMatrix(
      cbm::test::random_binary(rows, cols, density, seed));
}
void* ref_gen_block_graph(uint32_t blocks, uint32_t copies, uint32_t nnz) {
  return new cbm::CsrBinaryMatrix(cbm::test::block_graph(blocks, copies, nnz));
}
void* ref_gen_community_graph(uint32_t comms, uint32_t size, uint32_t base,
                              uint32_t noise, uint64_t seed) {
  return new cbm::CsrBinaryMatrix(
      cbm::test::community_graph(comms, size, base, noise, seed));
}
void* ref_gen_citation_graph(uint32_t nodes, uint64_t edges, uint64_t seed) {
  return new cbm::CsrBinaryMatrix(
      cbm::test::citation_graph(nodes, edges, seed));
}
void ref_csr_dims(void* h, uint32_t* rows, uint32_t* cols, uint64_t* nnz) {
  auto* a = static_cast<cbm::CsrBinaryMatrix*>(h);
  *rows = a->n_rows;
  *cols = a->n_cols;
  *nnz = a->nnz();
}
void ref_csr_export(void* h, uint64_t* rp, uint32_t* ci) {
  auto* a = static_cast<cbm::CsrBinaryMatrix*>(h);
  std::memcpy(rp, a->row_ptr.data(), a->row_ptr.size() * 8);
  std::memcpy(ci, a->col_idx.data(), a->col_idx.size() * 4);
}
void ref_csr_free(void* h) { delete static_cast<cbm::CsrBinaryMatrix*>(h); }

// ---------------------------------------------------------------- CBM
void* ref_build_cbm(void* csr, uint64_t alpha, int threads, int normalized) {
  cbm::CbmMatrix* out = nullptr;
  guard([&] {
    const auto& a = *static_cast<cbm::CsrBinaryMatrix*>(csr);
    out = new cbm::CbmMatrix(normalized
                                 ? cbm::build_cbm_normalized(a, alpha, threads)
                                 : cbm::build_cbm(a, alpha, threads));
  });
  return out;
}

// Wraps externally built arrays into the reference's own CbmMatrix through its
// validating constructors (CompressionChain::from_parents, CsrRealMatrix ctor).
void* ref_cbm_from_arrays(uint32_t m, uint32_t n, uint64_t alpha,
                          int normalized, const uint32_t* parent,
                          const uint64_t* rp, const uint32_t* ci,
                          const float* vals, const float* scale) {
  cbm::CbmMatrix* out = nullptr;
  guard([&] {
    auto c = std::make_unique<cbm::CbmMatrix>();
    c->n_rows = m;
    c->n_cols = n;
    c->alpha = alpha;
    c->is_normalized = normalized != 0;
    c->chain = cbm::CompressionChain::from_parents(
        std::vector<uint32_t>(parent, parent + m));
    std::vector<uint64_t> r(rp, rp + m + 1);
    const uint64_t nnz = r.back();
    c->delta_matrix = cbm::CsrRealMatrix(
        m, n, std::move(r), std::vector<uint32_t>(ci, ci + nnz),
        std::vector<float>(vals, vals + nnz));
    if (normalized) c->row_scale.assign(scale, scale + m);
    out = c.release();
  });
  return out;
}

void ref_cbm_dims(void* h, uint32_t* m, uint32_t* n, uint64_t* nnz,
                  uint64_t* alpha, int* normalized, uint64_t* n_roots) {
  auto* c = static_cast<cbm::CbmMatrix*>(h);
  *m = c->n_rows;
  *n = c->n_cols;
  *nnz = c->delta_matrix.nnz();
  *alpha = c->alpha;
  *normalized = c->is_normalized ? 1 : 0;
  *n_roots = c->chain.root_children.size();
}
void ref_cbm_export(void* h, uint32_t* parent, uint32_t* topo,
                    uint64_t* branch_ptr, uint64_t* rp, uint32_t* ci,
                    float* vals, float* scale) {
  auto* c = static_cast<cbm::CbmMatrix*>(h);
  const auto& ch = c->chain;
  std::memcpy(parent, ch.parent.data(), ch.parent.size() * 4);
  std::memcpy(topo, ch.topo_order.data(), ch.topo_order.size() * 4);
  std::memcpy(branch_ptr, ch.branch_ptr.data(), ch.branch_ptr.size() * 8);
  const auto& d = c->delta_matrix;
  std::memcpy(rp, d.row_ptr.data(), d.row_ptr.size() * 8);
  std::memcpy(ci, d.col_idx.data(), d.col_idx.size() * 4);
  std::memcpy(vals, d.values.data(), d.values.size() * 4);
  if (c->is_normalized && scale)
    std::memcpy(scale, c->row_scale.data(), c->row_scale.size() * 4);
}
void ref_cbm_free(void* h) { delete static_cast<cbm::CbmMatrix*>(h); }

void ref_count_ops(void* h, uint64_t* mult, uint64_t* upd) {
  const auto ops = cbm::count_scalar_ops(*static_cast<cbm::CbmMatrix*>(h));
  *mult = ops.multiply_adds;
  *upd = ops.update_adds;
}
uint64_t ref_memory_footprint(void* h) {
  return cbm::memory_footprint(*static_cast<cbm::CbmMatrix*>(h));
}

// Pattern replay (builder.cpp:452): row_ptr has m+1 entries, col_idx is
// written only when non-null (call twice: sizes first).
uint64_t ref_reconstruct_rows(void* h, uint64_t* rp, uint32_t* ci) {
  const auto a = cbm::reconstruct_rows(*static_cast<cbm::CbmMatrix*>(h));
  if (rp) std::memcpy(rp, a.row_ptr.data(), a.row_ptr.size() * 8);
  if (ci) std::memcpy(ci, a.col_idx.data(), a.col_idx.size() * 4);
  return a.nnz();
}

int ref_save_cbm(void* h, const char* path) {
  return guard([&] { cbm::save_cbm(*static_cast<cbm::CbmMatrix*>(h), path); });
}
void* ref_load_cbm(const char* path) {
  cbm::CbmMatrix* out = nullptr;
  guard([&] { out = new cbm::CbmMatrix(cbm::load_cbm(path)); });
  return out;
}

// ---------------------------------------------------------------- kernels
int ref_spmm(void* h, const float* x, uint32_t rows, uint32_t cols, float* y,
             int threads) {
  return guard([&] {
    const auto& c = *static_cast<cbm::CbmMatrix*>(h);
    const auto b = dense_from(x, rows, cols);
    cbm::DenseMatrix out(c.n_rows, cols);
    cbm::spmm_into(c, b, out, threads);
    std::memcpy(y, out.data.data(), out.data.size() * 4);
  });
}
int ref_spmv(void* h, const float* x, uint32_t rows, float* y, int threads) {
  return guard([&] {
    const auto& c = *static_cast<cbm::CbmMatrix*>(h);
    const auto v = dense_from(x, rows, 1);
    const auto out = cbm::spmv(c, v, threads);
    std::memcpy(y, out.data.data(), out.data.size() * 4);
  });
}
int ref_spmm_sequential(void* h, const float* x, uint32_t rows, uint32_t cols,
                        float* y) {
  return guard([&] {
    const auto& c = *static_cast<cbm::CbmMatrix*>(h);
    const auto out =
        cbm::spmm_sequential_reference(c, dense_from(x, rows, cols));
    std::memcpy(y, out.data.data(), out.data.size() * 4);
  });
}

// CSR baseline: to_real(A) (csr.cpp:84) or normalized_adjacency_csr(A)
// (gcn.cpp:48), then csr_spmm_into (kernels.cpp:152).
void* ref_csr_real(void* csr, int normalized) {
  cbm::CsrRealMatrix* out = nullptr;
  guard([&] {
    const auto& a = *static_cast<cbm::CsrBinaryMatrix*>(csr);
    out = new cbm::CsrRealMatrix(normalized ? cbm::normalized_adjacency_csr(a)
                                            : cbm::to_real(a));
  });
  return out;
}
void ref_csr_real_free(void* h) { delete static_cast<cbm::CsrRealMatrix*>(h); }
int ref_csr_spmm(void* real, const float* x, uint32_t rows, uint32_t cols,
                 float* y, int threads) {
  return guard([&] {
    const auto& a = *static_cast<cbm::CsrRealMatrix*>(real);
    const auto b = dense_from(x, rows, cols);
    cbm::DenseMatrix out(a.n_rows, cols);
    cbm::csr_spmm_into(a, b, out, threads);
    std::memcpy(y, out.data.data(), out.data.size() * 4);
  });
}

// Timing, following cmd_spmm_bench's time_runs (cbm_main.cpp:116-122): one
// untimed warm-up, then the mean over `runs` calls. Operands are built once
// outside the timed region, exactly as the CLI does. Returns seconds/call
// (negative on error). kind 0 = CBM spmm_into, 1 = CSR csr_spmm_into.
double ref_time(int kind, void* h, const float* x, uint32_t rows,
                uint32_t cols, int threads, int runs, double min_seconds,
                int* runs_done) {
  double result = -1.0;
  guard([&] {
    const auto b = dense_from(x, rows, cols);
    if (kind == 2) {  // spmv_into (kernels.cpp:70-97), cols == 1
      const auto& c = *static_cast<cbm::CbmMatrix*>(h);
      cbm::DenseMatrix out(c.n_rows, 1);
      cbm::spmv_into(c, b, out, threads);
      const auto t0 = Clock::now();
      int r = 0;
      while (r < runs || since(t0) < min_seconds) {
        cbm::spmv_into(c, b, out, threads);
        ++r;
      }
      result = since(t0) / r;
      *runs_done = r;
    } else if (kind == 0) {
      const auto& c = *static_cast<cbm::CbmMatrix*>(h);
      cbm::DenseMatrix out(c.n_rows, cols);
      cbm::spmm_into(c, b, out, threads);
      const auto t0 = Clock::now();
      int r = 0;
      while (r < runs || since(t0) < min_seconds) {
        cbm::spmm_into(c, b, out, threads);
        ++r;
      }
      result = since(t0) / r;
      *runs_done = r;
    } else {
      const auto& a = *static_cast<cbm::CsrRealMatrix*>(h);
      cbm::DenseMatrix out(a.n_rows, cols);
      cbm::csr_spmm_into(a, b, out, threads);
      const auto t0 = Clock::now();
      int r = 0;
      while (r < runs || since(t0) < min_seconds) {
        cbm::csr_spmm_into(a, b, out, threads);
        ++r;
      }
      result = since(t0) / r;
      *runs_done = r;
    }
  });
  return result;
}

// ---------------------------------------------------------------- dense / GCN
void ref_random_dense(uint32_t rows, uint32_t cols, double lo, double hi,
                      uint64_t seed, float* out) {
  const auto m = cbm::random_dense(rows, cols, lo, hi, seed);
  std::memcpy(out, m.data.data(), m.data.size() * 4);
}
void ref_gcn_seeded(uint32_t f, uint32_t h, uint32_t c, uint64_t seed,
                    float* w0, float* w1) {
  const auto m = cbm::GcnModel::seeded(f, h, c, seed);
  std::memcpy(w0, m.w0.data.data(), m.w0.data.size() * 4);
  std::memcpy(w1, m.w1.data.data(), m.w1.data.size() * 4);
}
int ref_gcn_forward(void* h, const float* x, uint32_t n, uint32_t f,
                    const float* w0, uint32_t hid, const float* w1,
                    uint32_t classes, float* out, int threads) {
  return guard([&] {
    const auto& adj = *static_cast<cbm::CbmMatrix*>(h);
    cbm::GcnModel m;
    m.w0 = dense_from(w0, f, hid);
    m.w1 = dense_from(w1, hid, classes);
    const auto y = cbm::gcn_forward(adj, dense_from(x, n, f), m, threads);
    std::memcpy(out, y.data.data(), y.data.size() * 4);
  });
}
int ref_gcn_forward_csr(void* real, const float* x, uint32_t n, uint32_t f,
                        const float* w0, uint32_t hid, const float* w1,
                        uint32_t classes, float* out, int threads) {
  return guard([&] {
    const auto& adj = *static_cast<cbm::CsrRealMatrix*>(real);
    cbm::GcnModel m;
    m.w0 = dense_from(w0, f, hid);
    m.w1 = dense_from(w1, hid, classes);
    const auto y = cbm::gcn_forward_csr(adj, dense_from(x, n, f), m, threads);
    std::memcpy(out, y.data.data(), y.data.size() * 4);
  });
}

}  // extern "C"
