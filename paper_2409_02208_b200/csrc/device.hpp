// Device-resident CBM operator (host-side handle; implementation in
// cbm_kernels.cu).
#pragma once

#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "errors.hpp"
#include "layout.hpp"
#include "dense_layout.hpp"
#include "hub_layout.hpp"
#include "tile_layout.hpp"

namespace cbmb {

inline constexpr uint32_t kHostChunks = 8;  // column chunks of the host-buffer pipeline

struct DeviceMatrix {
  int device = 0;
  int num_sms = 148;
  int l2_bytes = 126 << 20;
  Layout info;  // sizes only after upload (host vectors released)
  cbm_b200_options opt{};
  // structure (immutable)
  uint32_t* dcol = nullptr;
  float* dval = nullptr;  // normalized: signed delta values in dcol order
  uint32_t* rec = nullptr;
  float* srow = nullptr;
  float* scale = nullptr;
  uint64_t device_bytes = 0;
  // tiled path (tile_layout.hpp): sizes in `tile` (host vectors released)
  bool tile_on = false;
  TileLayout tile;
  uint32_t* tdcol = nullptr;
  float* tdval = nullptr;
  uint32_t* trow = nullptr;
  uint32_t* tblock = nullptr;
  uint32_t* tstage = nullptr;
  std::map<uint64_t, uint32_t> tile_main;  // (W, slabs) -> full-width units of the launch
  // dense-block path (dense_layout.hpp): sizes in `dense` (host vectors
  // released); the cold entries are their own streaming-kernel operator
  bool dense_on = false;
  DenseLayout dense;
  uint32_t* dtiles = nullptr;
  uint32_t* dmeta = nullptr;
  struct DeviceMatrix* cold = nullptr;
  // hub-row panel (hub_layout.hpp): this operator's own layout is then the
  // matrix WITHOUT its hub rows; the panel adds them after the multiply
  bool hub_on = false;
  uint32_t hub_n_rows = 0, hub_pieces = 0;
  uint64_t hub_entries = 0, hub_chunks = 0;
  uint64_t hub_nnz = 0;          // deltas of the uploaded CBM (info: the view's own count)
  uint32_t* htiles = nullptr;    // per piece: piece * 128, 128, first chunk, chunks
  uint32_t* hmeta = nullptr;     // chunk records (dense_layout.hpp)
  uint32_t* hrows = nullptr;     // the hub rows' ids
  float* hsrow = nullptr;        // normalized: their row scales
  struct DeviceMatrix* hub_op = nullptr;  // the hub rows alone (X narrower than the tensor path)
  // per-call workspace, one per stream (concurrent calls on distinct streams
  // never share flags or scratch); grown on demand, or by cbm_b200_reserve
  struct Workspace {
    uint32_t* flags = nullptr;
    uint64_t flags_cap = 0;      // entries
    float* partial = nullptr;
    uint64_t partial_cap = 0;    // floats
    float* interior = nullptr;
    uint64_t interior_cap = 0;
    float* tinterior = nullptr;  // tiled path: unscaled rows with children
    uint64_t tinterior_cap = 0;
    float* xs = nullptr;         // pre-scaled operand (normalized, prescale on)
    uint64_t xs_cap = 0;
    float* gcn_h = nullptr;      // GCN hidden activations (2 x n x hid)
    uint64_t gcn_h_cap = 0;
    float* hub_part = nullptr;   // hub panel: per piece, 128 partial rows
    uint64_t hub_part_cap = 0;
    uint32_t epoch = 0;          // ready-flag stamp of the last call
  };
  std::map<void*, Workspace> ws;
  float* xstage = nullptr;       // host-API staging
  uint64_t xstage_cap = 0;
  float* ystage = nullptr;
  uint64_t ystage_cap = 0;
  // host-API pipeline: copy-in / copy-out streams and chunk events
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev[1 + 2 * kHostChunks] = {};
  // end of the last host call's copy-out: the shared staging buffers are free
  // again (the next call's copy-in, whatever stream it comes from, waits on it)
  cudaEvent_t ev_done = nullptr;
  // static ticket -> warp schedules (cbm_kernel), one per (warps, slabs)
  struct Schedule {
    void* trec = nullptr;    // ticket stream: per warp, its records in increasing order
    uint32_t wstride = 0;    // records per warp region
  };
  std::map<uint64_t, Schedule> schedules;
  std::vector<uint32_t> item_dep;  // per item: parent item (ppos), first partial, count
  uint32_t last_launches = 0;
  std::mutex mu;
};

DeviceMatrix* device_upload(const cbm_b200_cbm_view& v, const cbm_b200_options& opt);
void device_free(DeviceMatrix* h);
void device_reserve(DeviceMatrix* h, uint64_t d, void* stream);
// Y = A X; x/y are device pointers; d = columns. Shapes already validated.
// base (optional, n_rows x d, leading dimension ldbase; may alias y): added to
// every row's unscaled sum before the row scale (the dense-block path's
// tensor-core part under the cold entries).
void device_spmm(DeviceMatrix* h, const float* x, int64_t ldx, uint32_t d, float* y,
                 int64_t ldy, void* stream, bool relu = false, const float* base = nullptr,
                 int64_t ldbase = 0);
inline constexpr uint32_t kDenseMinD = 32;  // narrower X stays on the streaming kernel
void dense_spmm(DeviceMatrix* h, const float* x, int64_t ldx, uint32_t d, float* y,
                int64_t ldy, cudaStream_t s);
// Y[hub rows] = (A X)[hub rows]: the panel's units on the dense-block kernel,
// then the fixed-order reduction of their partials (row scale / ReLU applied).
void hub_spmm(DeviceMatrix* h, const float* x, int64_t ldx, uint32_t d, float* y, int64_t ldy,
              bool relu, float*& part, uint64_t& part_cap, cudaStream_t s);
// out[rows[i], :] = src[i, :] (the narrow-X form of the panel: rows from hub_op)
void hub_scatter(const float* src, uint32_t ld, const uint32_t* rows, uint32_t n, uint32_t d,
                 float* y, int64_t ldy, cudaStream_t s);
void device_dense_matmul(const float* a, uint32_t m, uint32_t k, const float* b, uint32_t n,
                         float* c, void* stream);
void device_fast_matmul(const float* a, uint32_t m, uint32_t k, const float* b, uint32_t n,
                        float* c, void* stream);
// C = [A_0 | ... | A_{P-1}] B written to every outs[o] (leading dimension ldc);
// A_p is m x part_k[p] row-major and may live on another device (CUDA IPC).
inline constexpr uint32_t kMaxParts = 8;
void device_gemm_parts(const float* const* a_parts, const uint32_t* part_k, uint32_t n_parts,
                       uint32_t m, const float* b, uint32_t n, float* const* outs,
                       uint32_t n_outs, uint32_t ldc, bool ordered, void* stream);
void ipc_handle(const void* dptr, unsigned char* out64, uint64_t* offset);
void* ipc_open(const unsigned char* in64, int device);
void ipc_close(void* dptr);
void device_gcn_forward(DeviceMatrix* h, const float* x, uint32_t n, uint32_t f,
                        const float* w0, uint32_t hid, const float* w1, uint32_t classes,
                        float* out, void* stream);
// Host buffers (row-major, leading dimensions ldx/ldy in floats): column
// chunks of X in, multiply, Y out, copies overlapped on the handle's copy
// streams. wait = false leaves the work queued (device_spmm_host_wait).
void device_spmm_host(DeviceMatrix* h, const float* x, int64_t ldx, uint32_t d, float* y,
                      int64_t ldy, void* stream, bool wait = true);
void device_spmm_host_wait(DeviceMatrix* h, void* stream);
// tiled path (tile_kernel.cu): slab vector width for a call (0 = not usable)
uint32_t tile_pick_vec(const DeviceMatrix* h, uint32_t d, const float* x, int64_t ldx,
                       const float* y, int64_t ldy);
void tile_spmm(DeviceMatrix* h, uint32_t V, const float* x, int64_t ldx, uint32_t d, float* y,
               int64_t ldy, float* interior, uint32_t dpad, bool relu, cudaStream_t s);

}  // namespace cbmb
