// Host/device pieces shared by the CUDA translation units of the library:
// error mapping, workspace growth, the ticket record of the ticket stream
// and the schedule builder (schedule.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "device.hpp"

namespace cbmb {

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    const int code = (e == cudaErrorMemoryAllocation) ? CBM_B200_ENOMEM : CBM_B200_ECUDA;
    throw cuda_error(std::string(what) + ": " + cudaGetErrorString(e), code);
  }
}

// Grow a device buffer to at least `need` elements (contents not kept).
template <typename T>
void grow(T*& ptr, uint64_t& cap, uint64_t need, const char* what) {
  if (need <= cap) return;
  if (ptr) ck(cudaFree(ptr), "cudaFree");
  ptr = nullptr;
  cap = 0;
  ck(cudaMalloc(&ptr, std::max<uint64_t>(need, 1) * sizeof(T)), what);
  cap = need;
}

constexpr uint32_t kRecWin = 64;  // ticket records staged per warp (two groups of 32)

// One ticket's record (3 x 16 bytes), as stored in the warp's region of the
// ticket stream and staged in shared memory: the item's layout record, the
// ticket's item and column slab, the row scale, and (first record of a region
// only) the warp's ticket count.
struct alignas(16) TRec {
  uint32_t beg, end, rowk, ppos;
  uint32_t psrc, first, cnt, slot;
  uint32_t item, slab, srow, nw;
};

// The ticket stream for (resident warps, slabs), built once and cached on the
// handle (DESIGN.md §6 Schedule).
const DeviceMatrix::Schedule& schedule_for(DeviceMatrix* h, uint32_t warps, uint32_t slabs,
                                           cudaStream_t s);

}  // namespace cbmb
