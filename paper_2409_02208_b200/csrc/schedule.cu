// Static list schedule of the multiply's tickets and the per-warp ticket
// stream it is uploaded as (DESIGN.md §6 Schedule).
#include <algorithm>
#include <utility>
#include <vector>

#include "cuda_common.hpp"

namespace cbmb {

namespace {
// Gathers each warp's ticket records into its region of the ticket stream.
__global__ void build_ticket_stream(const uint4* __restrict__ rec, const float* __restrict__ srow,
                                    const uint32_t* __restrict__ list,
                                    const uint32_t* __restrict__ wstart, uint32_t n_items,
                                    uint32_t warps, uint32_t stride, uint64_t n_rec,
                                    TRec* __restrict__ out) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n_rec;
       k += (uint64_t)gridDim.x * blockDim.x) {
    TRec r{};
    const uint64_t w = k / stride, i = k - w * stride;
    if (w < warps) {
      const uint32_t lo = wstart[w], n = wstart[w + 1] - lo;
      if (i < n) {
        const uint32_t T = list[lo + i];
        const uint32_t sl = T / n_items, t = T - sl * n_items;
        const uint4 a = rec[2 * (size_t)t], b = rec[2 * (size_t)t + 1];
        r = TRec{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w,
                 t, sl, srow ? __float_as_uint(srow[t]) : 0u, 0u};
      }
      if (i == 0) r.nw = n;
    }
    out[k] = r;
  }
}

}  // namespace

// Static list schedule of the tickets over the resident warps (cbm_kernel).
// Tickets are taken in processing order (slab-major, then Layout::order: item
// order, with the long rows' leaf pieces band by band) and each goes to the warp that an estimated
// clock frees first (ties: lowest warp), starting no earlier than its
// parent / partial producers are estimated to finish; cost ~ per-ticket
// overhead + deltas + partial rows + parent row. Every warp's list follows
// the processing order and every wait targets an earlier position, which is
// all the deadlock argument needs (the earliest unfinished ticket is always
// being worked on). Balancing by work instead of
// round-robin by count removes the tail where warps holding several 32-delta
// chunks finish long after the rest.
const DeviceMatrix::Schedule& schedule_for(DeviceMatrix* h, uint32_t warps, uint32_t slabs,
                                           cudaStream_t s) {
  const uint64_t key = (uint64_t(warps) << 32) | slabs;
  auto it = h->schedules.find(key);
  if (it != h->schedules.end()) return it->second;
  const Layout& L = h->info;
  const uint32_t n = L.n_items;
  const uint64_t total = uint64_t(n) * slabs;
#ifndef CBM_TICKET_COST
#define CBM_TICKET_COST 4.0f
#endif
  constexpr float kTicket = CBM_TICKET_COST;  // epilogue / record overhead in delta-equivalents
  std::vector<uint32_t> owner(total);
  std::vector<uint32_t> count(size_t(warps) + 1, 0);
  std::vector<float> fin(n);
  using Slot = std::pair<float, uint32_t>;
  std::vector<Slot> heap;
  heap.reserve(warps);
  for (uint32_t w = 0; w < warps; ++w) heap.emplace_back(0.0f, w);
  auto later = [](const Slot& a, const Slot& b) { return a > b; };  // min-heap
  std::make_heap(heap.begin(), heap.end(), later);
  for (uint32_t sl = 0; sl < slabs; ++sl) {
    for (uint32_t idx = 0; idx < n; ++idx) {
      const uint32_t t = L.order.empty() ? idx : L.order[idx];
      std::pop_heap(heap.begin(), heap.end(), later);
      Slot& top = heap.back();
      const uint32_t* dp = &h->item_dep[size_t(t) * 3];
      float start = top.first;
      float cost = kTicket + float(L.item_beg[t + 1] - L.item_beg[t]) + float(dp[2]);
      if (dp[0] != kNoItem) {
        start = std::max(start, fin[dp[0]]);
        cost += 1.0f;
      }
      for (uint32_t j = 0; j < dp[2]; ++j) start = std::max(start, fin[dp[1] + j]);
      fin[t] = start + cost;
      top.first = fin[t];
      owner[uint64_t(sl) * n + t] = top.second;
      ++count[top.second + 1];
      std::push_heap(heap.begin(), heap.end(), later);
    }
  }
  uint32_t most = 0;
  for (uint32_t w = 0; w < warps; ++w) {
    most = std::max(most, count[w + 1]);
    count[w + 1] += count[w];
  }
  std::vector<uint32_t> list(total);
  {
    std::vector<uint32_t> pos(count.begin(), count.end() - 1);
    for (uint32_t sl = 0; sl < slabs; ++sl)
      for (uint32_t idx = 0; idx < n; ++idx) {  // each warp's list in processing order
        const uint64_t T = uint64_t(sl) * n + (L.order.empty() ? idx : L.order[idx]);
        list[pos[owner[T]]++] = uint32_t(T);
      }
  }
  // the ticket stream: warp w's records at [w * stride, w * stride + count_w),
  // zero records after them and 64 more after the last region
  DeviceMatrix::Schedule sc;
  sc.wstride = std::max<uint32_t>(32, (most + 31) & ~31u);
  const uint64_t n_rec = uint64_t(warps) * sc.wstride + kRecWin;
  uint32_t *d_list = nullptr, *d_start = nullptr;
  try {
    ck(cudaMalloc(&sc.trec, n_rec * sizeof(TRec)), "schedule");
    ck(cudaMalloc(&d_list, std::max<uint64_t>(total, 1) * sizeof(uint32_t)), "schedule");
    ck(cudaMalloc(&d_start, count.size() * sizeof(uint32_t)), "schedule");
    ck(cudaMemcpyAsync(d_list, list.data(), total * sizeof(uint32_t), cudaMemcpyHostToDevice, s),
       "schedule upload");
    ck(cudaMemcpyAsync(d_start, count.data(), count.size() * sizeof(uint32_t),
                       cudaMemcpyHostToDevice, s),
       "schedule upload");
    const int grid = int(std::min<uint64_t>((n_rec + 255) / 256, uint64_t(h->num_sms) * 32));
    build_ticket_stream<<<grid, 256, 0, s>>>(reinterpret_cast<const uint4*>(h->rec), h->srow,
                                             d_list, d_start, L.n_items, warps, sc.wstride,
                                             n_rec, reinterpret_cast<TRec*>(sc.trec));
    ck(cudaGetLastError(), "schedule build");
    ck(cudaStreamSynchronize(s), "schedule build");  // the host vectors go out of scope
  } catch (...) {
    if (sc.trec) cudaFree(sc.trec);
    cudaFree(d_list);
    cudaFree(d_start);
    throw;
  }
  cudaFree(d_list);
  cudaFree(d_start);
  return h->schedules.emplace(key, sc).first->second;
}

}  // namespace cbmb
