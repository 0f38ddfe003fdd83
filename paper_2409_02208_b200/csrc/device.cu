// The device operator's host side: upload (validation, layout, device
// arrays), workspace reservation, release, and the host-buffer entry point
// (column chunks of X and Y overlapped with the multiply on copy streams).
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <utility>
#include <vector>

#include "cuda_common.hpp"

namespace cbmb {

namespace {

// Hub-row panel (hub_layout.hpp): the operator is uploaded WITHOUT its hub
// rows (the plan's rest view, through the ordinary upload: streaming, tiled or
// dense-block as that view deserves) and carries the panel beside it.
DeviceMatrix* upload_with_hub(const cbm_b200_cbm_view& v, const cbm_b200_options& opt,
                              HubPlan& H) {
  cbm_b200_options ro = opt;
  ro.hub = 0;
  cbm_b200_cbm_view rv{v.n_rows, v.n_cols, H.rest_row_ptr.back(), v.alpha, v.is_normalized,
                       H.rest_parent.data(), nullptr, H.rest_row_ptr.data(), H.rest_col.data(),
                       H.rest_val.data(), v.row_scale, v.col_scale};
  DeviceMatrix* h = device_upload(rv, ro);
  try {
    H.rest_parent = {};
    H.rest_row_ptr = {};
    H.rest_col = {};
    H.rest_val = {};
    auto put = [&](auto*& dst, const auto& vec, const char* what) {
      using E = typename std::remove_reference_t<decltype(vec)>::value_type;
      ck(cudaMalloc(&dst, std::max<size_t>(vec.size(), 1) * sizeof(E)), what);
      if (!vec.empty()) ck(cudaMemcpy(dst, vec.data(), vec.size() * sizeof(E),
                                      cudaMemcpyHostToDevice), what);
      h->device_bytes += vec.size() * sizeof(E);
    };
    put(h->htiles, H.tiles, "upload hub pieces");
    put(h->hmeta, H.meta, "upload hub chunk records");
    put(h->hrows, H.rows, "upload hub rows");
    if (v.is_normalized) put(h->hsrow, H.hub_row_scale, "upload hub row scales");
    h->hub_n_rows = uint32_t(H.rows.size());
    h->hub_pieces = H.n_pieces;
    h->hub_entries = H.entries;
    h->hub_chunks = H.n_chunks;
    h->hub_nnz = v.nnz;
    // the hub rows alone, for X narrower than the tensor path takes
    const float* colscale = v.col_scale ? v.col_scale : v.row_scale;
    cbm_b200_cbm_view hv{h->hub_n_rows, v.n_cols, H.hub_row_ptr.back(), v.alpha, v.is_normalized,
                         H.hub_parent.data(), nullptr, H.hub_row_ptr.data(), H.hub_col.data(),
                         H.hub_val.data(), H.hub_row_scale.data(), colscale};
    cbm_b200_options ho = ro;
    ho.tile = 0;
    ho.dense = 0;
    ho.flatten_gain = 0;
    h->hub_op = device_upload(hv, ho);
    h->device_bytes += h->hub_op->device_bytes;
    h->opt.hub = opt.hub;
    h->hub_on = true;
  } catch (...) {
    device_free(h);
    throw;
  }
  return h;
}

}  // namespace

DeviceMatrix* device_upload(const cbm_b200_cbm_view& v, const cbm_b200_options& opt) {
  // validate + plan on the host first: malformed input is EINVAL, never a CUDA error
  const uint32_t gain = opt.flatten_gain < 0 ? 16u : uint32_t(opt.flatten_gain);
  // resident warps for the auto split: ~20 per SM (the multiply's occupancy);
  // without a device the upload fails after validation anyway
  int sms = 148, cur = 0;
  if (cudaGetDevice(&cur) == cudaSuccess &&
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount,
                             opt.device >= 0 ? opt.device : cur) != cudaSuccess)
    sms = 148;
  cudaGetLastError();  // a failed probe must not leak into later error checks
  if (!opt.order_faithful && opt.hub != 0 && opt.tile != 1 && opt.dense != 1 && v.n_rows > 0 &&
      (opt.hub > 0 || (v.n_rows >= (1u << 15) && v.nnz >= (1ull << 22)))) {
    validate_view(v);
    HubPlan H = plan_hub(v, opt.hub, uint32_t(sms));
    if (opt.hub > 0 && !H.on)
      throw invalid_argument("upload: the hub-row panel needs delta rows consistent with "
                             "their parents' rows");
    if (H.on) return upload_with_hub(v, opt, H);
  }
  Layout L = plan_layout(v, opt.order_faithful != 0, opt.split_threshold, opt.chunk, gain,
                         uint32_t(sms) * 20);
  auto* h = new DeviceMatrix;
  try {
    int dev = opt.device;
    if (dev < 0) ck(cudaGetDevice(&dev), "cudaGetDevice");
    ck(cudaSetDevice(dev), "cudaSetDevice");
    h->device = dev;
    h->opt = opt;
    ck(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    ck(cudaDeviceGetAttribute(&h->l2_bytes, cudaDevAttrL2CacheSize, dev), "attr");
    auto put = [&](auto*& dst, const auto& vec, const char* what) {
      using E = typename std::remove_reference_t<decltype(vec)>::value_type;
      const size_t bytes = std::max<size_t>(vec.size(), 1) * sizeof(E);
      ck(cudaMalloc(&dst, bytes), what);
      if (!vec.empty()) ck(cudaMemcpy(dst, vec.data(), vec.size() * sizeof(E),
                                      cudaMemcpyHostToDevice), what);
      h->device_bytes += vec.size() * sizeof(E);
    };
    put(h->dcol, L.dcol, "upload dcol");
    put(h->rec, L.rec, "upload rec");
    if (L.normalized) {
      put(h->srow, L.srow, "upload srow");
      put(h->scale, L.scale, "upload scale");
      // the signed delta values in dcol order (bit-identical to the CBM's
      // values: +-row_scale[col], validated by plan_layout)
      std::vector<float> dval(L.dcol.size());
      for (size_t k = 0; k < dval.size(); ++k) {
        const float sc = L.scale[L.dcol[k] & 0x7FFFFFFFu];
        dval[k] = (L.dcol[k] >> 31) ? -sc : sc;
      }
      put(h->dval, dval, "upload dval");
    }
    // dense-block path (default mode): the tensor cores take the columns each
    // 128-row tile shares, a streaming operator the rest
    if (!L.order_faithful && (opt.dense == 1 || (opt.dense == -1 && opt.tile != 1)) &&
        v.n_rows > 0) {
      DenseLayout D = plan_dense(v, opt.dense_min);
      if (opt.dense == 1 && !D.ok)
        throw invalid_argument("upload: the dense-block path needs delta rows consistent "
                               "with their parents' rows");
      // cost in gather-equivalents (one X row per gathered entry): measured on
      // cfg[3] (profiles/r02_dense_*), a chunk of the dense kernel costs about
      // as much as 150 gathers of the streaming kernel; the cold entries are
      // gathered on top, the streaming kernel alone gathers every effective entry
      const double dense_cost = double(D.cold_entries) + kDenseChunkCost * double(D.n_chunks);
      // (and enough chunks to fill the SMs: two launches and a persistent
      // pipeline do not pay on small matrices, cfg[0]: 23.6 vs 13.3 us tiled)
      h->dense_on = D.ok && (opt.dense == 1 ||
                             (dense_cost < 0.85 * double(L.nnz_effective) &&
                              D.n_chunks >= 8ull * uint64_t(std::max(1, h->num_sms))));
      if (h->dense_on) {
        put(h->dtiles, D.tiles, "upload dense tiles");
        put(h->dmeta, D.meta, "upload dense chunk records");
        cbm_b200_cbm_view cv{v.n_rows, v.n_cols, D.cold_entries, v.alpha, v.is_normalized,
                             D.cold_parent.data(), nullptr, D.cold_row_ptr.data(),
                             D.cold_col.data(), D.cold_val.data(), v.row_scale, v.col_scale};
        cbm_b200_options co = opt;
        co.order_faithful = 0;
        co.tile = 0;
        co.dense = 0;
        co.flatten_gain = 0;
        if (const char* e = std::getenv("CBM_B200_COLD_SEGS")) co.max_segments = std::atoi(e);  // dev A/B
        h->cold = device_upload(cv, co);
        h->device_bytes += h->cold->device_bytes;
      }
      D.tiles = {};
      D.meta = {};
      D.cold_parent = {};
      D.cold_row_ptr = {};
      D.cold_col = {};
      D.cold_val = {};
      h->dense = std::move(D);
    }
    // tiled path (default mode): planned here, kept only when it pays
    // (the tiled kernel scales rows and staged columns from one array: square only)
    if (!L.order_faithful && opt.tile != 0 && v.n_rows > 0 && !h->dense_on &&
        !(L.normalized && v.col_scale)) {
      TileLayout T;
      bool planned = true;
      try {
        T = plan_tiles(v, opt.tile_rows, opt.tile_stage, uint32_t(h->num_sms), gain);
      } catch (const inconsistent_rows&) {
        if (opt.tile == 1) throw;  // forced: EINVAL; auto: the streaming kernel takes it
        planned = false;
      }
      if (planned) {
      const double frac = T.n_deltas ? double(T.n_staged_deltas) / double(T.n_deltas) : 0.0;
      const double reuse = T.n_staged_cols ? double(T.n_staged_deltas) / double(T.n_staged_cols) : 0.0;
      // a row is summed by one warp and a block by one CTA: auto mode also
      // refuses layouts whose longest row or heaviest block would dominate
      // the launch (hub rows of power-law graphs)
      const double per_sm = double(T.n_entries) / double(std::max(1, h->num_sms));
      const bool balanced = double(T.max_row_entries) <= std::max(4096.0, 0.25 * per_sm) &&
                            double(T.max_block_entries) <= std::max(65536.0, 2.0 * per_sm);
      h->tile_on = opt.tile == 1 ||
                   (frac >= kTileMinStagedFrac && reuse >= kTileMinReuse && balanced);
      if (h->tile_on) {
        put(h->tdcol, T.dcol, "upload tile dcol");
        if (L.normalized) put(h->tdval, T.dval, "upload tile dval");
        put(h->trow, T.row, "upload tile rows");
        put(h->tblock, T.block, "upload tile blocks");
        put(h->tstage, T.stage, "upload tile stage");
      }
      T.dcol = {};
      T.dval = {};
      T.row = {};
      T.block = {};
      T.stage = {};  // (T.work stays: it sizes the split of the last wave)
      h->tile = std::move(T);
      }
    }
    int coop = 0;
    ck(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev), "attr");
    if (!coop) throw cuda_error("device lacks cooperative launch", CBM_B200_ECUDA);
    // keep only sizes on the host
    L.dcol = {};
    h->item_dep.resize(size_t(L.n_items) * 3);  // for the ticket schedule
    for (uint32_t t = 0; t < L.n_items; ++t) {
      h->item_dep[size_t(t) * 3] = L.rec[size_t(t) * 8 + 3];
      h->item_dep[size_t(t) * 3 + 1] = L.rec[size_t(t) * 8 + 5];
      h->item_dep[size_t(t) * 3 + 2] = L.rec[size_t(t) * 8 + 6];
    }
    L.rec = {};  // item_beg and item_dep stay: they drive the ticket schedule
    L.srow = {};
    L.scale = {};
    L.row_scale = {};
    h->info = std::move(L);
  } catch (...) {
    device_free(h);
    throw;
  }
  return h;
}

void device_free(DeviceMatrix* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->s_in) {
    cudaStreamDestroy(h->s_in);
    cudaStreamDestroy(h->s_out);
    for (auto e : h->ev) cudaEventDestroy(e);
    cudaEventDestroy(h->ev_done);
  }
  for (auto& kv : h->schedules) cudaFree(kv.second.trec);
  for (auto& kv : h->ws)
    for (void* p : {(void*)kv.second.flags, (void*)kv.second.partial, (void*)kv.second.interior,
                    (void*)kv.second.xs, (void*)kv.second.gcn_h})
      if (p) cudaFree(p);
  for (auto& kv : h->ws)
    if (kv.second.tinterior) cudaFree(kv.second.tinterior);
  if (h->cold) device_free(h->cold);
  if (h->hub_op) device_free(h->hub_op);
  for (auto& kv : h->ws)
    if (kv.second.hub_part) cudaFree(kv.second.hub_part);
  for (void* p : {(void*)h->dtiles, (void*)h->dmeta, (void*)h->htiles, (void*)h->hmeta,
                  (void*)h->hrows, (void*)h->hsrow})
    if (p) cudaFree(p);
  for (void* p : {(void*)h->dcol, (void*)h->dval, (void*)h->rec, (void*)h->srow, (void*)h->scale,
                  (void*)h->xstage, (void*)h->ystage, (void*)h->tdcol, (void*)h->tdval,
                  (void*)h->trow, (void*)h->tblock, (void*)h->tstage})
    if (p) cudaFree(p);
  delete h;
}

void device_reserve(DeviceMatrix* h, uint64_t d, void* stream) {
  const Layout& L = h->info;
  const uint64_t dpad = (d + 3) & ~uint64_t(3);
  const uint64_t slabs = (d + 31) / 32;  // worst case (V = 1)
  ck(cudaSetDevice(h->device), "cudaSetDevice");
  auto& ws = h->ws[stream];
  if (uint64_t(L.n_items) * slabs > ws.flags_cap) {
    grow(ws.flags, ws.flags_cap, uint64_t(L.n_items) * slabs, "workspace flags");
    // on the stream the workspace serves (the kernel that spins on these flags
    // runs there; a legacy-stream memset would not be ordered before it on a
    // non-blocking or per-thread stream)
    ck(cudaMemsetAsync(ws.flags, 0, ws.flags_cap * sizeof(uint32_t),
                       static_cast<cudaStream_t>(stream)), "flags memset");
    ws.epoch = 0;
  }
  grow(ws.partial, ws.partial_cap, uint64_t(L.n_chunk_items) * dpad, "workspace partial");
  if (L.normalized) grow(ws.interior, ws.interior_cap, uint64_t(L.n_interior) * dpad,
                         "workspace interior");
  if (h->tile_on) grow(ws.tinterior, ws.tinterior_cap, uint64_t(h->tile.n_interior) * dpad,
                       "workspace tile interior");
  if (h->cold) device_reserve(h->cold, d, stream);
  if (h->hub_on) {
    if (d >= kDenseMinD) {
      uint64_t rows = 0;
      for (uint32_t n = h->hub_pieces; n > 1; n = (n + kHubFanIn - 1) / kHubFanIn)
        rows += uint64_t(n) * kDenseRows;
      rows = std::max<uint64_t>(rows, uint64_t(h->hub_pieces) * kDenseRows);
      grow(ws.hub_part, ws.hub_part_cap, rows * dpad, "workspace hub partials");
    } else {
      device_reserve(h->hub_op, d, stream);
    }
  }
}

// Host-buffer entry point. Columns are independent (kernels.cpp:27-62), so X
// and Y move in column chunks on three streams: H2D of chunk k+1 and D2H of
// chunk k-1 run while chunk k multiplies, and the two copy directions overlap
// on the full-duplex PCIe link. One chunk when the operand is small.
void device_spmm_host(DeviceMatrix* h, const float* x, int64_t ldx, uint32_t d, float* y,
                      int64_t ldy, void* stream, bool wait) {
  const Layout& L = h->info;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ck(cudaSetDevice(h->device), "cudaSetDevice");
  const uint32_t dpad = (d + 3) & ~3u;
  grow(h->xstage, h->xstage_cap, uint64_t(L.n_cols) * dpad, "staging X");
  grow(h->ystage, h->ystage_cap, uint64_t(L.n_rows) * dpad, "staging Y");
  if (!h->s_in) {
    ck(cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking), "stream");
    for (auto& e : h->ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&h->ev_done, cudaEventDisableTiming), "event");
    ck(cudaEventRecord(h->ev_done, h->s_out), "event");
  }
  const uint64_t bytes = (uint64_t(L.n_cols) + L.n_rows) * d * sizeof(float);
  // Column chunks (16-byte aligned): the first chunk's H2D and the last
  // chunk's D2H cannot overlap anything, so for d >= 512 those two are narrow
  // (d/8) and the middle is cut in three (tools/probe_e2e.py: uniform x4
  // 1109 us, x8 1151 us on cfg[1]); rows narrower than 64 floats slow the 2D
  // copies, so narrower operands take uniform 64-column chunks.
  std::vector<std::pair<uint32_t, uint32_t>> parts;  // (first column, width)
  auto r4 = [](uint32_t v) { return (v + 3) & ~3u; };
  uint32_t chunks = 1;
  if (bytes >= (8u << 20) && d >= 128) chunks = d >= 256 ? 5 : 2;
  if (const char* e = std::getenv("CBM_B200_HOST_CHUNKS"))  // dev tool: uniform chunks
    chunks = std::max<uint32_t>(1, std::min<uint32_t>({kHostChunks, uint32_t(std::atoi(e)), d}));
  if (const char* e = std::getenv("CBM_B200_HOST_WIDTHS")) {  // dev tool: explicit widths
    uint32_t c0 = 0;
    for (const char* q = e; *q && c0 < d;) {
      const uint32_t w = std::min<uint32_t>(uint32_t(std::strtoul(q, const_cast<char**>(&q), 10)), d - c0);
      if (w == 0) break;
      parts.emplace_back(c0, w);
      c0 += w;
      if (*q == ',') ++q;
    }
    if (c0 < d) parts.emplace_back(c0, d - c0);
    if (parts.size() > kHostChunks) throw invalid_argument("CBM_B200_HOST_WIDTHS: too many chunks");
  } else if (chunks == 5 && !std::getenv("CBM_B200_HOST_CHUNKS") && d >= 512) {
    const uint32_t edge = r4(d / 8), rest = d - 2 * edge, mid = r4((rest + 2) / 3);
    uint32_t c0 = 0;
    const uint32_t m3 = (rest - 2 * mid) & ~3u;  // every chunk starts 16-byte aligned
    for (uint32_t w : {edge, mid, mid, m3, d - edge - 2 * mid - m3}) {
      parts.emplace_back(c0, w);
      c0 += w;
    }
  } else {
    // 256 <= d < 512: uniform chunks of 64 columns. Strided 2-D copies of rows
    // narrower than 64 floats run well below the link rate (cfg[4], 2.5 GB each
    // way: 32/64/64/64/32 81.8 ms, 4 x 64 64.7 ms, 8 x 32 90.2 ms; the floor
    // for fully overlapped copies is 53.5 ms: profiles/r02l_e2e_sweep.txt)
    if (chunks == 5 && !std::getenv("CBM_B200_HOST_CHUNKS")) chunks = std::min(kHostChunks, (d + 63) / 64);
    const uint32_t cw = r4((d + chunks - 1) / chunks);
    for (uint32_t c0 = 0; c0 < d; c0 += cw) parts.emplace_back(c0, std::min(cw, d - c0));
  }
  // ev[0]: caller's prior work on s; ev[1+k]: X chunk k landed; ev[1+C+k]: Y chunk k ready
  ck(cudaEventRecord(h->ev[0], s), "event");
  ck(cudaStreamWaitEvent(h->s_in, h->ev[0], 0), "wait");
  ck(cudaStreamWaitEvent(h->s_out, h->ev[0], 0), "wait");
  // xstage/ystage are shared by every caller stream: the previous call's
  // kernel has read xstage and its copy-out has drained ystage before this
  // call's copy-in starts (the kernels below wait on the copy-in, so their
  // ystage writes are ordered after it too)
  ck(cudaStreamWaitEvent(h->s_in, h->ev_done, 0), "wait");
  for (size_t k = 0; k < parts.size(); ++k) {
    const auto [c0, w] = parts[k];
    ck(cudaMemcpy2DAsync(h->xstage + c0, dpad * sizeof(float), x + c0, ldx * sizeof(float),
                         w * sizeof(float), L.n_cols, cudaMemcpyHostToDevice, h->s_in),
       "H2D X");
    ck(cudaEventRecord(h->ev[1 + k], h->s_in), "event");
  }
  uint32_t launches = 0;
  for (size_t k = 0; k < parts.size(); ++k) {
    const auto [c0, w] = parts[k];
    ck(cudaStreamWaitEvent(s, h->ev[1 + k], 0), "wait");
    device_spmm(h, h->xstage + c0, dpad, w, h->ystage + c0, dpad, stream, false);
    launches += h->last_launches;
    ck(cudaEventRecord(h->ev[1 + kHostChunks + k], s), "event");
    ck(cudaStreamWaitEvent(h->s_out, h->ev[1 + kHostChunks + k], 0), "wait");
    ck(cudaMemcpy2DAsync(y + c0, ldy * sizeof(float), h->ystage + c0, dpad * sizeof(float),
                         w * sizeof(float), L.n_rows, cudaMemcpyDeviceToHost, h->s_out),
       "D2H Y");
  }
  h->last_launches = launches;  // kernels launched by this call (one per chunk)
  // the caller's stream resumes after the last copy-out
  ck(cudaEventRecord(h->ev_done, h->s_out), "event");
  ck(cudaStreamWaitEvent(s, h->ev_done, 0), "wait");
  if (wait) device_spmm_host_wait(h, stream);
}

void device_spmm_host_wait(DeviceMatrix* h, void* stream) {
  ck(cudaSetDevice(h->device), "cudaSetDevice");
  ck(cudaStreamSynchronize(h->s_out), "spmm_host synchronize");
  ck(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "spmm_host synchronize");
}

}  // namespace cbmb
