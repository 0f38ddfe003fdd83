// extern "C" boundary (include/cbm_b200.h). Exceptions never cross it: each
// entry point maps them onto a status code plus a thread-local message, the
// way the reference raises std::invalid_argument / std::logic_error.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/cbm_b200.h"
#include "cbm_host.hpp"
#include "dense_layout.hpp"
#include "hub_layout.hpp"
#include "device.hpp"
#include "layout.hpp"

struct cbm_b200_host_cbm {
  cbmb::HostCbm c;
};
struct cbm_b200_matrix {
  cbmb::DeviceMatrix* d;
};
struct cbm_b200_csr {
  cbmb::Csr a;
};

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    g_err.clear();
    f();
    return CBM_B200_OK;
  } catch (const cbmb::invalid_argument& e) {
    g_err = e.what();
    return CBM_B200_EINVAL;
  } catch (const cbmb::logic_error& e) {
    g_err = e.what();
    return CBM_B200_ELOGIC;
  } catch (const cbmb::format_error& e) {
    g_err = e.what();
    return CBM_B200_EFORMAT;
  } catch (const cbmb::cuda_error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return CBM_B200_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CBM_B200_ELOGIC;
  }
}

void need(bool ok, const char* msg) {
  if (!ok) throw cbmb::invalid_argument(msg);
}

// Shape checks of kernels.cpp:11-14,107-109 (messages verbatim).
void check_spmm_shapes(const cbmb::Layout& L, int64_t x_rows, int64_t x_cols, int64_t y_rows,
                       int64_t y_cols, const char* who) {
  if (x_rows != int64_t(L.n_cols))
    throw cbmb::invalid_argument(std::string(who) + ": inner dimensions differ");
  if (y_rows != int64_t(L.n_rows) || y_cols != x_cols)
    throw cbmb::invalid_argument(std::string(who) + ": output has the wrong shape");
  if (x_cols < 0 || x_cols > 0x7FFFFFFF)
    throw cbmb::invalid_argument(std::string(who) + ": bad column count");
}

// Options check + device upload of a borrowed view (throws).
cbm_b200_matrix* upload_view(const cbm_b200_cbm_view& view, const cbm_b200_options* opt) {
  const cbm_b200_cbm_view* c = &view;
  cbm_b200_options o;
  cbm_b200_default_options(&o);
  if (opt) o = *opt;
  need(o.kernel == 0 || o.kernel == 1, "upload: options.kernel must be 0 (auto) or 1 (scalar)");
  need(o.max_segments >= 0 && o.max_segments <= 4, "upload: options.max_segments must be 0..4");
  need(o.tile >= -1 && o.tile <= 1, "upload: options.tile must be -1, 0 or 1");
  need(o.dense >= -1 && o.dense <= 1, "upload: options.dense must be -1, 0 or 1");
  need(o.tile_vec == 0 || o.tile_vec == 1 || o.tile_vec == 2 || o.tile_vec == 4,
       "upload: options.tile_vec must be 0, 1, 2 or 4");
  auto* h = new cbm_b200_matrix{nullptr};
  try {
    h->d = cbmb::device_upload(*c, o);
  } catch (...) {
    delete h;
    throw;
  }
  return h;
}
}  // namespace

extern "C" {

const char* cbm_b200_last_error(void) { return g_err.c_str(); }

// ------------------------------------------------------------------ builder
int cbm_b200_build(const cbm_b200_csr_view* a, uint64_t alpha, int32_t normalized,
                   int32_t degree_mode, int32_t threads, cbm_b200_host_cbm** out) {
  return cbm_b200_build_ex(a, alpha, normalized, degree_mode, threads, 0, out);
}

int cbm_b200_build_ex(const cbm_b200_csr_view* a, uint64_t alpha, int32_t normalized,
                      int32_t degree_mode, int32_t threads, int32_t algo,
                      cbm_b200_host_cbm** out) {
  return guard([&] {
    need(a && out, "build: null argument");
    *out = nullptr;
    need(a->row_ptr != nullptr, "build: null row_ptr");
    cbmb::validate_csr(a->n_rows, a->n_cols, a->row_ptr, a->col_idx);
    cbmb::Csr csr;
    csr.n_rows = a->n_rows;
    csr.n_cols = a->n_cols;
    csr.row_ptr.assign(a->row_ptr, a->row_ptr + size_t(a->n_rows) + 1);
    csr.col_idx.assign(a->col_idx, a->col_idx + csr.row_ptr.back());
    const int t = threads > 0 ? threads : 1;
    auto* h = new cbm_b200_host_cbm;
    try {
      h->c = normalized ? cbmb::build_cbm_normalized(csr, alpha, t, degree_mode == 1, algo)
                        : cbmb::build_cbm(csr, alpha, t, algo);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int cbm_b200_host_view(const cbm_b200_host_cbm* h, cbm_b200_cbm_view* v) {
  return guard([&] {
    need(h && v, "host_view: null argument");
    const auto& c = h->c;
    v->n_rows = c.n_rows;
    v->n_cols = c.n_cols;
    v->nnz = c.row_ptr.back();
    v->alpha = c.alpha;
    v->is_normalized = c.normalized ? 1 : 0;
    v->parent = c.parent.data();
    v->topo_order = c.topo_order.data();
    v->row_ptr = c.row_ptr.data();
    v->col_idx = c.col_idx.data();
    v->values = c.values.data();
    v->row_scale = c.normalized ? c.row_scale.data() : nullptr;
    v->col_scale = nullptr;
  });
}

int cbm_b200_host_branches(const cbm_b200_host_cbm* h, const uint64_t** bp, uint64_t* nb) {
  return guard([&] {
    need(h && bp && nb, "host_branches: null argument");
    *bp = h->c.branch_ptr.data();
    *nb = h->c.root_children.size();
  });
}

int cbm_b200_host_stats(const cbm_b200_host_cbm* h, cbm_b200_build_stats* s) {
  return guard([&] {
    need(h && s, "host_stats: null argument");
    s->t_edges = h->c.t_edges;
    s->t_arborescence = h->c.t_arb;
    s->t_deltas = h->c.t_deltas;
    s->t_total = h->c.t_total;
    s->candidate_edges = h->c.candidate_edges;
    s->rounds = h->c.rounds;
  });
}

void cbm_b200_host_free(cbm_b200_host_cbm* h) { delete h; }

int cbm_b200_load_cbm1(const char* path, cbm_b200_host_cbm** out) {
  return guard([&] {
    need(path && out, "load_cbm1: null argument");
    *out = nullptr;
    auto* h = new cbm_b200_host_cbm;
    try {
      h->c = cbmb::load_cbm1(path);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int cbm_b200_save_cbm1(const cbm_b200_cbm_view* v, const char* path) {
  return guard([&] {
    need(v && path, "save_cbm1: null argument");
    need(!(v->is_normalized && v->col_scale),
         "save_cbm1: a row block of a normalized matrix is not a CBM1 container");
    cbmb::HostCbm c;
    c.n_rows = v->n_rows;
    c.n_cols = v->n_cols;
    c.alpha = v->alpha;
    c.normalized = v->is_normalized != 0;
    c.parent.assign(v->parent, v->parent + v->n_rows);
    cbmb::chain_from_parents(c);  // topo order as the reference stores it
    c.row_ptr.assign(v->row_ptr, v->row_ptr + size_t(v->n_rows) + 1);
    c.col_idx.assign(v->col_idx, v->col_idx + v->nnz);
    c.values.assign(v->values, v->values + v->nnz);
    if (c.normalized) c.row_scale.assign(v->row_scale, v->row_scale + v->n_rows);
    cbmb::save_cbm1(c, path);
  });
}

int cbm_b200_count_ops(const cbm_b200_cbm_view* c, uint64_t* mult, uint64_t* upd) {
  return guard([&] {
    need(c && mult && upd, "count_ops: null argument");
    *mult = c->nnz;
    uint64_t non_virtual = 0;
    for (uint32_t x = 0; x < c->n_rows; ++x) non_virtual += c->parent[x] != cbmb::kVirtual;
    *upd = non_virtual;
  });
}

// ------------------------------------------------------------------ device
void cbm_b200_default_options(cbm_b200_options* o) {
  if (!o) return;
  o->device = -1;
  o->order_faithful = 0;
  o->split_threshold = 0;
  o->chunk = 0;
  o->prescale = -1;
  o->kernel = 0;
  o->max_segments = 0;
  o->flatten_gain = -1;
  o->prefetch = 0;
  o->tile = -1;
  o->tile_rows = 0;
  o->tile_stage = 0;
  o->tile_vec = 0;
  o->dense = -1;
  o->dense_min = 0;
  o->hub = -1;
}

int cbm_b200_upload(const cbm_b200_cbm_view* c, const cbm_b200_options* opt,
                    cbm_b200_matrix** out) {
  return guard([&] {
    need(c && out, "upload: null argument");
    *out = nullptr;
    *out = upload_view(*c, opt);
  });
}

int cbm_b200_upload_cbm1(const char* path, const cbm_b200_options* opt,
                         cbm_b200_matrix** out) {
  return guard([&] {
    need(path && out, "upload_cbm1: null argument");
    *out = nullptr;
    const cbmb::HostCbm c = cbmb::load_cbm1(path);   // mapped, validated by all host threads
    cbm_b200_cbm_view v{c.n_rows, c.n_cols, c.row_ptr.back(), c.alpha, c.normalized ? 1 : 0,
                        c.parent.data(), c.topo_order.data(), c.row_ptr.data(),
                        c.col_idx.data(), c.values.data(),
                        c.normalized ? c.row_scale.data() : nullptr, nullptr};
    *out = upload_view(v, opt);
  });
}

void cbm_b200_free(cbm_b200_matrix* h) {
  if (!h) return;
  cbmb::device_free(h->d);
  delete h;
}

int cbm_b200_reserve(cbm_b200_matrix* h, int64_t d_max) {
  return guard([&] {
    need(h && d_max >= 0, "reserve: bad argument");
    std::lock_guard<std::mutex> lk(h->d->mu);
    cbmb::device_reserve(h->d, uint64_t(d_max), nullptr);
  });
}

int cbm_b200_reserve_on(cbm_b200_matrix* h, int64_t d_max, void* stream) {
  return guard([&] {
    need(h && d_max >= 0, "reserve: bad argument");
    std::lock_guard<std::mutex> lk(h->d->mu);
    cbmb::device_reserve(h->d, uint64_t(d_max), stream);
  });
}

int cbm_b200_spmm(cbm_b200_matrix* h, const float* x, int64_t x_rows, int64_t x_cols,
                  int64_t ldx, float* y, int64_t y_rows, int64_t y_cols, int64_t ldy,
                  void* stream) {
  return guard([&] {
    need(h != nullptr, "spmm: null handle");
    check_spmm_shapes(h->d->info, x_rows, x_cols, y_rows, y_cols, "spmm");
    need(ldx >= x_cols && ldy >= y_cols, "spmm: leading dimension smaller than the width");
    need(ldx < (int64_t(1) << 30), "spmm: leading dimension of X must be below 2^30");
    need((x || x_rows * x_cols == 0) && (y || y_rows * y_cols == 0), "spmm: null data");
    std::lock_guard<std::mutex> lk(h->d->mu);
    cbmb::device_spmm(h->d, x, ldx, uint32_t(x_cols), y, ldy, stream);
  });
}

int cbm_b200_spmm_ex(cbm_b200_matrix* h, const float* x, int64_t x_rows, int64_t x_cols,
                     int64_t ldx, float* y, int64_t y_rows, int64_t y_cols, int64_t ldy,
                     uint32_t flags, void* stream) {
  return guard([&] {
    need(h != nullptr, "spmm: null handle");
    need((flags & ~CBM_B200_RELU) == 0, "spmm: unknown flags");
    check_spmm_shapes(h->d->info, x_rows, x_cols, y_rows, y_cols, "spmm");
    need(ldx >= x_cols && ldy >= y_cols, "spmm: leading dimension smaller than the width");
    need(ldx < (int64_t(1) << 30), "spmm: leading dimension of X must be below 2^30");
    need((x || x_rows * x_cols == 0) && (y || y_rows * y_cols == 0), "spmm: null data");
    std::lock_guard<std::mutex> lk(h->d->mu);
    cbmb::device_spmm(h->d, x, ldx, uint32_t(x_cols), y, ldy, stream,
                      (flags & CBM_B200_RELU) != 0);
  });
}

int cbm_b200_spmm_host(cbm_b200_matrix* h, const float* x, int64_t x_rows, int64_t x_cols,
                       float* y, int64_t y_rows, int64_t y_cols, void* stream) {
  return guard([&] {
    need(h != nullptr, "spmm: null handle");
    check_spmm_shapes(h->d->info, x_rows, x_cols, y_rows, y_cols, "spmm");
    need((x || x_rows * x_cols == 0) && (y || y_rows * y_cols == 0), "spmm: null data");
    std::lock_guard<std::mutex> lk(h->d->mu);
    cbmb::device_spmm_host(h->d, x, x_cols, uint32_t(x_cols), y, y_cols, stream);
  });
}

int cbm_b200_column_slab(int64_t d, int32_t world, int32_t rank, int64_t* lo, int64_t* hi) {
  return guard([&] {
    need(lo && hi && d >= 0 && world >= 1 && rank >= 0 && rank < world,
         "column_slab: bad rank/world");
    // contiguous, balanced in units of 4 columns (16-byte rows for LDG.128)
    const int64_t units = (d + 3) / 4;
    *lo = std::min<int64_t>(d, units * rank / world * 4);
    *hi = std::max<int64_t>(*lo, std::min<int64_t>(d, units * (rank + 1) / world * 4));
  });
}

int cbm_b200_spmm_sharded(cbm_b200_matrix* const* handles, int32_t n_handles, const float* x,
                          int64_t x_rows, int64_t x_cols, float* y, int64_t y_rows,
                          int64_t y_cols) {
  return guard([&] {
    need(handles && n_handles >= 1, "spmm_sharded: no handles");
    for (int32_t k = 0; k < n_handles; ++k) {
      need(handles[k] != nullptr, "spmm_sharded: null handle");
      for (int32_t j = 0; j < k; ++j)
        need(handles[j] != handles[k], "spmm_sharded: a handle appears twice");
    }
    const auto& L0 = handles[0]->d->info;
    for (int32_t k = 1; k < n_handles; ++k) {
      const auto& L = handles[k]->d->info;
      need(L.n_rows == L0.n_rows && L.n_cols == L0.n_cols && L.normalized == L0.normalized &&
               L.nnz == L0.nnz,
           "spmm_sharded: handles hold different matrices");
    }
    check_spmm_shapes(L0, x_rows, x_cols, y_rows, y_cols, "spmm");
    need((x || x_rows * x_cols == 0) && (y || y_rows * y_cols == 0), "spmm: null data");
    // lock every handle (distinct, in address order), queue every slab, then wait:
    // the devices' copies and kernels run concurrently
    std::vector<cbm_b200_matrix*> order(handles, handles + n_handles);
    std::sort(order.begin(), order.end());
    std::vector<std::unique_lock<std::mutex>> locks;
    for (auto* h : order) locks.emplace_back(h->d->mu);
    std::vector<int32_t> queued;
    for (int32_t k = 0; k < n_handles; ++k) {
      int64_t lo = 0, hi = 0;
      cbm_b200_column_slab(x_cols, n_handles, k, &lo, &hi);
      if (hi == lo) continue;
      cbmb::device_spmm_host(handles[k]->d, x + lo, x_cols, uint32_t(hi - lo), y + lo, y_cols,
                             nullptr, /*wait=*/false);
      queued.push_back(k);
    }
    for (int32_t k : queued) cbmb::device_spmm_host_wait(handles[k]->d, nullptr);
  });
}

int cbm_b200_spmv(cbm_b200_matrix* h, const float* v, int64_t v_rows, int64_t v_cols, float* u,
                  int64_t u_rows, int64_t u_cols, void* stream) {
  return guard([&] {
    need(h != nullptr, "spmv: null handle");
    const auto& L = h->d->info;
    // kernels.cpp:72-76
    if (v_rows != int64_t(L.n_cols)) throw cbmb::invalid_argument("spmv: inner dimensions differ");
    if (v_cols != 1) throw cbmb::invalid_argument("spmv: operand must be a single column");
    if (u_rows != int64_t(L.n_rows) || u_cols != 1)
      throw cbmb::invalid_argument("spmv: output must be n_rows x 1");
    std::lock_guard<std::mutex> lk(h->d->mu);
    cbmb::device_spmm(h->d, v, 1, 1, u, 1, stream);
  });
}

int cbm_b200_dense_matmul(const float* a, int64_t m, int64_t k, const float* b, int64_t n,
                          float* c, void* stream) {
  return guard([&] {
    need(m >= 0 && k >= 0 && n >= 0 && m < (1ll << 32) && k < (1ll << 32) && n < (1ll << 32),
         "dense_matmul: bad shape");
    need((a || m * k == 0) && (b || k * n == 0) && (c || m * n == 0), "dense_matmul: null data");
    cbmb::device_dense_matmul(a, uint32_t(m), uint32_t(k), b, uint32_t(n), c, stream);
  });
}

int cbm_b200_gemm_parts(const float* const* a_parts, const int64_t* part_k, int32_t n_parts,
                        int64_t m, const float* b, int64_t n, float* const* outs, int32_t n_outs,
                        int64_t ldc, int32_t ordered, void* stream) {
  return guard([&] {
    need(a_parts && part_k && outs && n_parts >= 1 && n_parts <= int32_t(cbmb::kMaxParts) &&
             n_outs >= 1 && n_outs <= int32_t(cbmb::kMaxParts),
         "gemm_parts: 1..8 parts and outputs");
    need(m >= 0 && n >= 0 && ldc >= n && m < (int64_t(1) << 31) && n < (int64_t(1) << 31),
         "gemm_parts: bad shape");
    uint32_t pk[cbmb::kMaxParts];
    int64_t k = 0;
    for (int32_t p = 0; p < n_parts; ++p) {
      need(part_k[p] >= 0 && (a_parts[p] || part_k[p] * m == 0), "gemm_parts: bad part");
      if (!ordered) need(part_k[p] % 4 == 0 || p == n_parts - 1,
                         "gemm_parts: part widths must be multiples of 4 (column_slab)");
      pk[p] = uint32_t(part_k[p]);
      k += part_k[p];
    }
    need(k < (int64_t(1) << 31) && (b || k * n == 0), "gemm_parts: bad shape");
    for (int32_t o = 0; o < n_outs; ++o) need(outs[o] || m * n == 0, "gemm_parts: null output");
    cbmb::device_gemm_parts(a_parts, pk, uint32_t(n_parts), uint32_t(m), b, uint32_t(n), outs,
                            uint32_t(n_outs), uint32_t(ldc), ordered != 0, stream);
  });
}

int cbm_b200_ipc_handle(const void* dptr, unsigned char* handle64, uint64_t* offset) {
  return guard([&] {
    need(dptr && handle64 && offset, "ipc: null argument");
    cbmb::ipc_handle(dptr, handle64, offset);
  });
}

int cbm_b200_ipc_open(const unsigned char* handle64, int32_t device, void** dptr) {
  return guard([&] {
    need(handle64 && dptr, "ipc: null argument");
    *dptr = cbmb::ipc_open(handle64, device);
  });
}

int cbm_b200_ipc_close(void* dptr) {
  return guard([&] {
    need(dptr != nullptr, "ipc: null argument");
    cbmb::ipc_close(dptr);
  });
}

int cbm_b200_gcn_forward(cbm_b200_matrix* h, const float* x, int64_t n, int64_t f,
                         const float* w0, int64_t hid, const float* w1, int64_t classes,
                         float* out, void* stream) {
  return guard([&] {
    need(h != nullptr, "gcn_forward: null handle");
    const auto& L = h->d->info;
    // gcn.cpp:24-27
    if (!L.normalized) throw cbmb::invalid_argument("gcn_forward: adjacency must be normalized");
    if (n != int64_t(L.n_cols))
      throw cbmb::invalid_argument("gcn_forward: feature rows must match nodes");
    need(f > 0 && hid > 0 && classes > 0, "gcn_forward: empty weight shape");
    need(x && w0 && w1 && out, "gcn_forward: null data");
    std::lock_guard<std::mutex> lk(h->d->mu);
    cbmb::device_gcn_forward(h->d, x, uint32_t(n), uint32_t(f), w0, uint32_t(hid), w1,
                             uint32_t(classes), out, stream);
  });
}

int cbm_b200_get_info(const cbm_b200_matrix* h, cbm_b200_info* o) {
  return guard([&] {
    need(h && o, "info: null argument");
    const auto& L = h->d->info;
    o->n_rows = L.n_rows;
    o->n_cols = L.n_cols;
    o->nnz_delta = h->d->hub_on ? h->d->hub_nnz : L.nnz;   // (the uploaded CBM's count)
    o->nnz_effective = L.nnz_effective;
    o->n_flattened = L.n_flattened;
    o->n_levels = L.n_levels;
    o->n_roots = L.n_roots;
    o->n_interior = L.n_interior;
    o->n_items = L.n_items;
    o->n_chunk_items = L.n_chunk_items;
    o->max_row_deltas = L.max_row_deltas;
    o->device_bytes = h->d->device_bytes;
    o->launches_per_call = h->d->last_launches;
    o->is_normalized = L.normalized ? 1 : 0;
    o->order_faithful = L.order_faithful ? 1 : 0;
    const auto& T = h->d->tile;
    o->tile_active = h->d->tile_on ? 1 : 0;
    o->tile_blocks = T.n_blocks;
    o->tile_max_rows = T.max_rows;
    o->tile_max_staged = T.max_staged;
    o->tile_cut_rows = T.n_cut;
    o->tile_deltas = T.n_deltas;
    o->tile_staged_deltas = T.n_staged_deltas;
    o->tile_staged_rows = T.n_staged_cols;
    const auto& D = h->d->dense;
    o->dense_active = h->d->dense_on ? 1 : 0;
    o->dense_tiles = D.n_tiles;
    o->dense_chunks = D.n_chunks;
    o->dense_entries = D.dense_entries;
    o->cold_entries = D.cold_entries;
    o->hub_active = h->d->hub_on ? 1 : 0;
    o->hub_rows = h->d->hub_n_rows;
    o->hub_entries = h->d->hub_entries;
    o->hub_chunks = h->d->hub_chunks;
  });
}

// Host-only plan of the dense-block layout (no device needed): what an upload
// with dense = 1 would multiply on the tensor cores. stats: tiles, chunks,
// dense entries, cold entries, padded slots, max tile rows.
int cbm_b200_plan_dense(const cbm_b200_cbm_view* c, uint32_t dense_min, uint64_t stats[6]) {
  return guard([&] {
    need(c && stats, "plan_dense: null argument");
    (void)cbmb::plan_layout(*c, true, 0, 0, 0, 148 * 20);  // validates like load_cbm
    const cbmb::DenseLayout D = cbmb::plan_dense(*c, dense_min);
    need(D.ok, "plan_dense: delta rows inconsistent with their parents");
    uint64_t max_rows = 0;
    for (uint32_t t = 0; t < D.n_tiles; ++t) max_rows = std::max<uint64_t>(max_rows, D.tiles[4 * t + 1]);
    stats[0] = D.n_tiles;
    stats[1] = D.n_chunks;
    stats[2] = D.dense_entries;
    stats[3] = D.cold_entries;
    stats[4] = D.padded_slots;
    stats[5] = max_rows;
  });
}

// Host-only: the hub-row panel an upload with hub = mode would build
// (hub_layout.hpp). stats: active, rows, entries, chunks, pieces, rest deltas.
int cbm_b200_plan_hub(const cbm_b200_cbm_view* c, int32_t mode, uint64_t stats[6]) {
  return guard([&] {
    need(c && stats, "plan_hub: null argument");
    cbmb::validate_view(*c);
    const cbmb::HubPlan H = cbmb::plan_hub(*c, mode, 148);
    stats[0] = H.on ? 1 : 0;
    stats[1] = H.rows.size();
    stats[2] = H.entries;
    stats[3] = H.n_chunks;
    stats[4] = H.n_pieces;
    stats[5] = H.on ? H.rest_row_ptr.back() : c->nnz;
  });
}

// ------------------------------------------------------------------ workloads
int cbm_b200_gen_graph(const char* kind, const double* params, int32_t n_params, uint64_t seed,
                       cbm_b200_csr** out) {
  return guard([&] {
    need(kind && out && (params || n_params == 0), "gen_graph: null argument");
    *out = nullptr;
    std::vector<double> p(params, params + n_params);
    auto* h = new cbm_b200_csr;
    try {
      h->a = cbmb::gen_graph(kind, p, seed);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int cbm_b200_csr_get(const cbm_b200_csr* a, cbm_b200_csr_view* v) {
  return guard([&] {
    need(a && v, "csr_get: null argument");
    v->n_rows = a->a.n_rows;
    v->n_cols = a->a.n_cols;
    v->row_ptr = a->a.row_ptr.data();
    v->col_idx = a->a.col_idx.data();
  });
}

void cbm_b200_csr_free(cbm_b200_csr* a) { delete a; }

int cbm_b200_gen_dense(int32_t kind, uint64_t rows, uint64_t cols, double lo, double hi,
                       uint64_t seed, float* out) {
  return guard([&] {
    need(out || rows * cols == 0, "gen_dense: null output");
    cbmb::Rng rng(seed);
    const uint64_t n = rows * cols;
    switch (kind) {
      case 0:  // random_dense (dense.cpp:56-62)
        for (uint64_t i = 0; i < n; ++i) out[i] = float(lo + (hi - lo) * rng.unit());
        break;
      case 1: {  // integers in [lo, hi]
        const int64_t a = int64_t(lo), b = int64_t(hi);
        need(b >= a, "gen_dense: empty integer range");
        for (uint64_t i = 0; i < n; ++i) out[i] = float(int64_t(rng.below(uint64_t(b - a + 1))) + a);
        break;
      }
      case 2:  // N(0,1), Box–Muller over two unit() draws, double then f32
        for (uint64_t i = 0; i < n; i += 2) {
          const double u1 = rng.unit(), u2 = rng.unit();
          const double r = std::sqrt(-2.0 * std::log1p(-u1));
          const double th = 6.283185307179586 * u2;
          out[i] = float(r * std::cos(th));
          if (i + 1 < n) out[i + 1] = float(r * std::sin(th));
        }
        break;
      case 3: {  // Glorot-uniform for a rows x cols (fan_in x fan_out) weight
        const double b = std::sqrt(6.0 / double(rows + cols));
        for (uint64_t i = 0; i < n; ++i) out[i] = float(-b + 2.0 * b * rng.unit());
        break;
      }
      default:
        throw cbmb::invalid_argument("gen_dense: unknown kind");
    }
  });
}

}  // extern "C"
