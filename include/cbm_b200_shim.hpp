// cbm_b200_shim.hpp — reference-side C++ adapter (header-only).
//
// A maintainer of the reference library (/root/reference/proj) adds this
// header next to proj/include/cbm/kernels.hpp to route the hot path to the
// B200 library while keeping the reference signatures and error behaviour:
//
//   reference (proj/include/cbm/kernels.hpp:26-44)   here
//   DenseMatrix spmm(const CbmMatrix&, ...)          cbm::b200::spmm
//   void spmm_into(const CbmMatrix&, ..., out, ...)  cbm::b200::spmm_into
//   DenseMatrix spmv(...) / void spmv_into(...)      cbm::b200::spmv / spmv_into
//
// The CbmMatrix is uploaded once per object (DeviceCbm) and reused; the
// `threads` argument is accepted and ignored (the GPU grid replaces
// parallel_chunks, proj/include/cbm/parallel.hpp:13-32). EINVAL from the C ABI
// becomes std::invalid_argument with the reference's own message
// (kernels.cpp:11-14,72-76,107-109); any other failure becomes
// std::runtime_error. Requires the f32 build (CBM_SINGLE_PRECISION), the
// element type of the device path.
#pragma once

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "cbm/builder.hpp"
#include "cbm/dense.hpp"
#include "cbm_b200.h"

namespace cbm::b200 {

static_assert(sizeof(real_t) == 4, "the B200 path multiplies in f32 (CBM_SINGLE_PRECISION)");

inline void check(int rc) {
  if (rc == CBM_B200_OK) return;
  if (rc == CBM_B200_EINVAL) throw std::invalid_argument(cbm_b200_last_error());
  throw std::runtime_error(std::string("cbm_b200: ") + cbm_b200_last_error());
}

inline cbm_b200_cbm_view view_of(const CbmMatrix& c) {
  cbm_b200_cbm_view v{};
  v.n_rows = c.n_rows;
  v.n_cols = c.n_cols;
  v.nnz = c.delta_matrix.nnz();
  v.alpha = c.alpha;
  v.is_normalized = c.is_normalized ? 1 : 0;
  v.parent = c.chain.parent.data();
  v.topo_order = c.chain.topo_order.data();
  v.row_ptr = c.delta_matrix.row_ptr.data();
  v.col_idx = c.delta_matrix.col_idx.data();
  v.values = c.delta_matrix.values.data();
  v.row_scale = c.is_normalized ? c.row_scale.data() : nullptr;
  return v;
}

// The uploaded operator (the device counterpart of holding a CbmMatrix). As a
// drop-in it defaults to the order-faithful mode: results are bit-identical
// to cbm::spmm_into for any X. order_faithful = false selects the faster mode
// (split / flattened rows; bit-exact on integer X, <= 1e-5 normwise otherwise).
class DeviceCbm {
 public:
  explicit DeviceCbm(const CbmMatrix& c, int device = -1, bool order_faithful = true) {
    cbm_b200_options opt;
    cbm_b200_default_options(&opt);
    opt.device = device;
    opt.order_faithful = order_faithful ? 1 : 0;
    const cbm_b200_cbm_view v = view_of(c);
    cbm_b200_matrix* h = nullptr;
    check(cbm_b200_upload(&v, &opt, &h));
    h_.reset(h);
    rows_ = c.n_rows;
    cols_ = c.n_cols;
  }
  cbm_b200_matrix* handle() const { return h_.get(); }
  index_t n_rows() const { return rows_; }
  index_t n_cols() const { return cols_; }

 private:
  struct Free {
    void operator()(cbm_b200_matrix* h) const { cbm_b200_free(h); }
  };
  std::unique_ptr<cbm_b200_matrix, Free> h_;
  index_t rows_ = 0, cols_ = 0;
};

// spmm_into (kernels.hpp:36-39): host DenseMatrix in, host DenseMatrix out.
inline void spmm_into(const DeviceCbm& c, const DenseMatrix& b, DenseMatrix& out,
                      int /*threads*/ = 1) {
  check(cbm_b200_spmm_host(c.handle(), b.data.data(), b.n_rows, b.n_cols, out.data.data(),
                           out.n_rows, out.n_cols, nullptr));
}

inline DenseMatrix spmm(const DeviceCbm& c, const DenseMatrix& b, int threads = 1) {
  if (c.n_cols() != b.n_rows) throw std::invalid_argument("spmm: inner dimensions differ");
  DenseMatrix out(c.n_rows(), b.n_cols);
  spmm_into(c, b, out, threads);
  return out;
}

// spmv_into / spmv (kernels.hpp:28-44). The host path goes through the same
// kernel at width 1 after the reference's own shape checks.
inline void spmv_into(const DeviceCbm& c, const DenseMatrix& v, DenseMatrix& out,
                      int /*threads*/ = 1) {
  if (c.n_cols() != v.n_rows) throw std::invalid_argument("spmv: inner dimensions differ");
  if (v.n_cols != 1) throw std::invalid_argument("spmv: operand must be a single column");
  if (out.n_rows != c.n_rows() || out.n_cols != 1)
    throw std::invalid_argument("spmv: output must be n_rows x 1");
  check(cbm_b200_spmm_host(c.handle(), v.data.data(), v.n_rows, 1, out.data.data(), out.n_rows,
                           1, nullptr));
}

inline DenseMatrix spmv(const DeviceCbm& c, const DenseMatrix& v, int threads = 1) {
  DenseMatrix out(c.n_rows(), 1);
  spmv_into(c, v, out, threads);
  return out;
}

// Column-sharded spmm_into over several devices: one DeviceCbm
// of the same CbmMatrix per device; slab k of the columns runs on shards[k].
// Bit-identical to the single-device result.
inline void spmm_sharded_into(const std::vector<const DeviceCbm*>& shards, const DenseMatrix& b,
                              DenseMatrix& out) {
  std::vector<cbm_b200_matrix*> hs;
  for (const DeviceCbm* d : shards) hs.push_back(d->handle());
  check(cbm_b200_spmm_sharded(hs.data(), int32_t(hs.size()), b.data.data(), b.n_rows, b.n_cols,
                              out.data.data(), out.n_rows, out.n_cols));
}

// One-shot overloads with the reference's exact signatures: upload, multiply.
inline void spmm_into(const CbmMatrix& c, const DenseMatrix& b, DenseMatrix& out,
                      int threads = 1) {
  spmm_into(DeviceCbm(c), b, out, threads);
}
inline DenseMatrix spmm(const CbmMatrix& c, const DenseMatrix& b, int threads = 1) {
  return spmm(DeviceCbm(c), b, threads);
}

}  // namespace cbm::b200
