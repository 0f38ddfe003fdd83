// Tiled CBM multiply (DESIGN.md §6 "Tiled path"; layout in tile_layout.hpp).
//
// One CTA per (row block, column slab of W = 32*V floats). The CTA
//   1. copies its block's row records into shared memory and the block's
//      STAGED X rows (the columns its deltas reference at least twice) into a
//      shared-memory tile, pre-multiplied by the column scale when the matrix is
//      normalized (the reference's per-product rounding, fl(s_c * x));
//   2. sums the block's rows, claimed in order by its warps (a shared-memory
//      counter). Per row: staged deltas from the tile (LDS), cold deltas from
//      L2 (issued before the staged loop so their latency hides behind it),
//      then the parent's unscaled row (kernels.cpp:52, parent inside the block:
//      a shared-memory flag; the wait always targets an earlier row of the same
//      CTA), then the row scale (kernels.cpp:57-58) and the optional ReLU.
// Blocks never wait on each other, so this is an ordinary launch.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <queue>
#include <vector>

#include "cuda_common.hpp"

namespace cbmb {

namespace {

constexpr uint32_t kLocalMask = 0x7FFFFFFFu;
constexpr uint32_t kNone = 0xFFFFFFFFu;
#ifndef CBM_TILE_IDXCAP
#define CBM_TILE_IDXCAP 224
#endif
constexpr uint32_t kIdxCap = CBM_TILE_IDXCAP;  // row indices per buffer (two per warp)

struct TileParams {
  const uint32_t* __restrict__ dcol;
  const float* __restrict__ dval;
  const uint4* __restrict__ rows;    // 2 x uint4 per tile row
  const uint4* __restrict__ blocks;  // row0, nrows, st0, nst
  const uint32_t* __restrict__ stage;
  const float* __restrict__ scale;   // normalized: per row / column
  const float* __restrict__ x;
  long long ldx;
  float* y;
  long long ldy;
  float* interior;  // unscaled rows with children, stride dpad
  uint32_t dpad, d, n_slabs, relu;
  uint32_t max_staged, max_rows;
  uint32_t n_main;            // full-width units; the rest are split in two
  unsigned long long* trace;  // dev tool (CBM_B200_TILE_TRACE): 4 x u64 per unit, else null
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                     __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 f4sub(float4 a, float4 b) {
  return make_float4(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y), __fsub_rn(a.z, b.z),
                     __fsub_rn(a.w, b.w));
}
__device__ __forceinline__ float4 f4fma(float4 x, float s, float4 a) {  // a + s*x, one rounding
  return make_float4(__fmaf_rn(x.x, s, a.x), __fmaf_rn(x.y, s, a.y), __fmaf_rn(x.z, s, a.z),
                     __fmaf_rn(x.w, s, a.w));
}
__device__ __forceinline__ float4 f4mul(float4 a, float s) {
  return make_float4(__fmul_rn(a.x, s), __fmul_rn(a.y, s), __fmul_rn(a.z, s), __fmul_rn(a.w, s));
}
__device__ __forceinline__ float relu1(float v) { return v < 0.0f ? 0.0f : v; }  // dense.cpp:51-54
__device__ __forceinline__ float4 f4relu(float4 v) {
  return make_float4(relu1(v.x), relu1(v.y), relu1(v.z), relu1(v.w));
}
__device__ __forceinline__ float4 f4shfl_xor(float4 v, int m) {
  return make_float4(__shfl_xor_sync(0xFFFFFFFFu, v.x, m), __shfl_xor_sync(0xFFFFFFFFu, v.y, m),
                     __shfl_xor_sync(0xFFFFFFFFu, v.z, m), __shfl_xor_sync(0xFFFFFFFFu, v.w, m));
}
// +1.0f or -1.0f from a sign bit (fma(x, +-1, acc) == fl(acc +- x) exactly)
__device__ __forceinline__ float unit_sign(uint32_t e) {
  return __uint_as_float((e & 0x80000000u) | 0x3F800000u);
}

__device__ __forceinline__ uint32_t smem_addr(const void* q) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(q));
}
// cp.async of 16 bytes; src_bytes 0 writes zeros
__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src),
               "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// D consecutive row indices from shared memory (SMEM) or global memory
template <int D, bool SMEM>
__device__ __forceinline__ void load_idx(const uint32_t* q, uint32_t (&e)[D]) {
  if constexpr (D == 8) {
    const uint4 a = SMEM ? *reinterpret_cast<const uint4*>(q) : __ldg(reinterpret_cast<const uint4*>(q));
    const uint4 b = SMEM ? *reinterpret_cast<const uint4*>(q + 4)
                         : __ldg(reinterpret_cast<const uint4*>(q + 4));
    e[0] = a.x; e[1] = a.y; e[2] = a.z; e[3] = a.w; e[4] = b.x; e[5] = b.y; e[6] = b.z; e[7] = b.w;
  } else if constexpr (D == 4) {
    const uint4 a = SMEM ? *reinterpret_cast<const uint4*>(q) : __ldg(reinterpret_cast<const uint4*>(q));
    e[0] = a.x; e[1] = a.y; e[2] = a.z; e[3] = a.w;
  } else {
    const uint2 a = SMEM ? *reinterpret_cast<const uint2*>(q) : __ldg(reinterpret_cast<const uint2*>(q));
    e[0] = a.x; e[1] = a.y;
  }
}

// acc +-= the staged rows of entries [k0, k1) (a multiple of 8 long): 16
// entries per step (two index vectors, 2*D tile reads in flight per lane)
#ifndef CBM_TILE_STEP
#define CBM_TILE_STEP 8
#endif
template <int H, bool SMEM, bool NEG>
__device__ __forceinline__ void staged_run(const uint32_t* ix, uint32_t k0, uint32_t k1,
                                           const float* xl, uint32_t g, float4& acc) {
  constexpr int D = 8 / H;
  constexpr uint32_t kW = 128u / H;
  uint32_t k = k0;
#pragma unroll 1
  for (; CBM_TILE_STEP == 16 && k + 16 <= k1; k += 16) {
    uint32_t e[D], f[D];
    load_idx<D, SMEM>(ix + k + g * D, e);
    load_idx<D, SMEM>(ix + k + 8 + g * D, f);
    float4 v[2 * D];
#pragma unroll
    for (int q = 0; q < D; ++q) v[q] = *reinterpret_cast<const float4*>(xl + e[q] * kW);
#pragma unroll
    for (int q = 0; q < D; ++q) v[D + q] = *reinterpret_cast<const float4*>(xl + f[q] * kW);
#pragma unroll
    for (int q = 0; q < 2 * D; ++q) acc = NEG ? f4sub(acc, v[q]) : f4add(acc, v[q]);
  }
#pragma unroll 1
  for (; k < k1; k += 8) {
    uint32_t e[D];
    load_idx<D, SMEM>(ix + k + g * D, e);
    float4 v[D];
#pragma unroll
    for (int q = 0; q < D; ++q) v[q] = *reinterpret_cast<const float4*>(xl + e[q] * kW);
#pragma unroll
    for (int q = 0; q < D; ++q) acc = NEG ? f4sub(acc, v[q]) : f4add(acc, v[q]);
  }
}

// One row's delta sum for this lane's group (H lane groups of 32/H lanes x 4
// floats; group g takes deltas g*D .. g*D+D-1 of every 8). Indices come from
// `ix` (shared-memory buffer, or global memory for rows longer than a buffer).
template <int H, bool NORM, bool SMEM>
__device__ __forceinline__ float4 row_sum(const TileParams& p, const uint32_t* ix, uint32_t npos,
                                          uint32_t nsk, uint32_t ncold, uint32_t mid,
                                          const float* xl, uint32_t g, bool act, long long col) {
  constexpr int D = 8 / H;
  constexpr uint32_t kW = 128u / H;  // floats per slab
#ifndef CBM_TILE_CPG
#define CBM_TILE_CPG 4
#endif
  constexpr int CPG = CBM_TILE_CPG;  // cold deltas per group per batch
  const int lane = threadIdx.x & 31;
  // first batch of cold deltas: group g takes entries g, g+H, ... (loads in
  // flight during the staged loop)
  const uint32_t nc = min(uint32_t(CPG * H), ncold);
  float cvv = 0.0f;
  if constexpr (NORM) {
    if (uint32_t(lane) < nc) cvv = __ldg(p.dval + mid + lane);
  }
  float4 cv[CPG];
  uint32_t ce[CPG];
#pragma unroll
  for (int q = 0; q < CPG; ++q) {
    const uint32_t c = g + uint32_t(H * q);
    ce[q] = c < nc ? (SMEM ? ix[nsk + c] : __ldg(ix + nsk + c)) : 0u;
    cv[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c < nc && act)
      cv[q] = __ldg(reinterpret_cast<const float4*>(p.x + (long long)(ce[q] & kLocalMask) * p.ldx + col));
  }
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  staged_run<H, SMEM, false>(ix, 0, npos, xl, g, acc);
  staged_run<H, SMEM, true>(ix, npos, nsk, xl, g, acc);
#pragma unroll
  for (int q = 0; q < CPG; ++q) {
    const uint32_t c = g + uint32_t(H * q);
    float s = unit_sign(ce[q]);
    if constexpr (NORM) s = __shfl_sync(0xFFFFFFFFu, cvv, int(c & 31u));
    if (c < nc) acc = f4fma(cv[q], s, acc);
  }
  // remaining cold deltas (rows with more than CPG*H)
  for (uint32_t k0 = CPG * H; k0 < ncold; k0 += CPG * H) {
    const uint32_t n2 = min(uint32_t(CPG * H), ncold - k0);
    if constexpr (NORM) {
      cvv = 0.0f;
      if (uint32_t(lane) < n2) cvv = __ldg(p.dval + mid + k0 + lane);
    }
#pragma unroll
    for (int q = 0; q < CPG; ++q) {
      const uint32_t c = g + uint32_t(H * q);
      ce[q] = c < n2 ? (SMEM ? ix[nsk + k0 + c] : __ldg(ix + nsk + k0 + c)) : 0u;
      cv[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (c < n2 && act)
        cv[q] = __ldg(reinterpret_cast<const float4*>(p.x + (long long)(ce[q] & kLocalMask) * p.ldx + col));
    }
#pragma unroll
    for (int q = 0; q < CPG; ++q) {
      const uint32_t c = g + uint32_t(H * q);
      float s = unit_sign(ce[q]);
      if constexpr (NORM) s = __shfl_sync(0xFFFFFFFFu, cvv, int(c & 31u));
      if (c < n2) acc = f4fma(cv[q], s, acc);
    }
  }
  // combine the lane groups (fixed tree: the same bits on every group)
#pragma unroll
  for (int off = 32 / H; off < 32; off *= 2) acc = f4add(acc, f4shfl_xor(acc, off));
  return acc;
}

// One (row block, column slab) unit: slab columns [col0, col0 + 128/H).
template <int H, bool NORM, int NT>
__device__ __forceinline__ void tile_unit(const TileParams& p, uint32_t blk, uint32_t col0,
                                          unsigned char* smem, uint32_t unit) {
  constexpr uint32_t LG = 32u / H;  // lanes per group
  constexpr uint32_t kW = 4u * LG;  // floats per slab
  constexpr int kWarps = NT / 32;
  const uint4 B = p.blocks[blk];
  const uint32_t row0 = B.x, nrows = B.y, st0 = B.z, nst = B.w;
  float* xs = reinterpret_cast<float*>(smem);
  uint4* recs = reinterpret_cast<uint4*>(smem + size_t(p.max_staged + 1) * kW * sizeof(float));
  volatile uint32_t* flags = reinterpret_cast<volatile uint32_t*>(recs + 2 * p.max_rows);
  uint32_t* counter = const_cast<uint32_t*>(flags + p.max_rows);
  uint32_t* idxbuf = counter + 4 + ((p.max_rows & 3u) ? 4u - (p.max_rows & 3u) : 0u);
  float* ssc = reinterpret_cast<float*>(idxbuf + kWarps * 2 * kIdxCap);  // staged scales
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned long long t0 = p.trace ? gtimer() : 0ull;

  // ---- stage: row records, flags, the staged X rows (+ a zero row at nst)
  for (uint32_t i = tid; i < 2 * nrows; i += NT) cp_async16(recs + i, p.rows + 2ull * row0 + i, 16);
  for (uint32_t i = tid; i < nrows; i += NT) flags[i] = 0u;
  if (tid == 0) *counter = 0u;
  if constexpr (NORM) {
    for (uint32_t s = tid; s < nst; s += NT) ssc[s] = __ldg(p.scale + __ldg(p.stage + st0 + s));
  }
  {
    const uint32_t items = (nst + 1) * LG;
    constexpr int kU = 8;
    for (uint32_t i0 = tid; i0 < items; i0 += kU * NT) {
      uint32_t cols[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t s = (i0 + u * NT) / LG;
        cols[u] = s < nst ? __ldg(p.stage + st0 + s) : 0u;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t i = i0 + u * NT;
        if (i >= items) break;
        const uint32_t s = i / LG, c = col0 + (i % LG) * 4;
        const bool real = s < nst && c < p.d;
        cp_async16(xs + size_t(s) * kW + (i % LG) * 4,
                   real ? p.x + (long long)cols[u] * p.ldx + c : p.x, real ? 16u : 0u);
      }
    }
  }
  cp_commit();
  cp_wait<0>();
  __syncthreads();
  if constexpr (NORM) {  // the reference's products fl(s_c * x) (kernels.cpp:30-35)
    for (uint32_t i = tid; i < nst * LG; i += NT) {
      float4* q = reinterpret_cast<float4*>(xs + size_t(i / LG) * kW + (i % LG) * 4);
      *q = f4mul(*q, ssc[i / LG]);
    }
    __syncthreads();
  }

  const unsigned long long t1 = p.trace ? gtimer() : 0ull;
  const uint32_t g = uint32_t(lane) / LG, gl = uint32_t(lane) % LG;
  const uint32_t colu = col0 + gl * 4;
  const bool act = colu < p.d;
  const long long col = colu;
  const float* xl = xs + gl * 4;
  uint32_t* ib = idxbuf + warp * 2 * kIdxCap;
  auto claim = [&]() {
    uint32_t j = 0;
    if (lane == 0) j = atomicAdd(counter, 1u);
    return __shfl_sync(0xFFFFFFFFu, j, 0);
  };
  // copy row j's indices into buf (16 bytes per lane-op; beg is 16-byte aligned)
  auto fetch = [&](uint32_t j, uint32_t* buf) {
    if (j < nrows) {
      const uint4 r0 = recs[2 * j];
      const uint32_t n4 = min((r0.w - r0.x + 3u) >> 2, kIdxCap / 4u);
      for (uint32_t q = lane; q < n4; q += 32) cp_async16(buf + 4 * q, p.dcol + r0.x + 4 * q, 16);
    }
    cp_commit();
  };
  uint32_t j = claim(), b = 0;
  fetch(j, ib);
  while (j < nrows) {
    const uint32_t jn = claim();
    fetch(jn, ib + (b ^ 1u) * kIdxCap);
    cp_wait<1>();
    __syncwarp();
    const uint32_t* buf = ib + b * kIdxCap;
    const uint4 r0 = recs[2 * j], r1 = recs[2 * j + 1];
    const uint32_t beg = r0.x, npos = r0.y - beg, nsk = r0.z - beg, ncold = r0.w - r0.z;
    const uint32_t row = r1.x, plocal = r1.y, psrc = r1.z, own = r1.w;
    const bool lead = g == 0 && act;  // lanes of group 0 finish the row
    float srow = 1.0f;
    if constexpr (NORM) srow = __ldg(p.scale + row);
    // parent already published: fetch its row now, under the delta sums
    bool have_parent = false;
    float4 pv = make_float4(0.f, 0.f, 0.f, 0.f);
    if (plocal != kNone && flags[plocal] != 0u) {
      __threadfence_block();
      if (lead) pv = __ldcg(reinterpret_cast<const float4*>(p.interior + (size_t)psrc * p.dpad + col));
      have_parent = true;
    }
    float4 acc;
    if (nsk + ncold <= kIdxCap)
      acc = row_sum<H, NORM, true>(p, buf, npos, nsk, ncold, r0.z, xl, g, act, col);
    else
      acc = row_sum<H, NORM, false>(p, p.dcol + beg, npos, nsk, ncold, r0.z, xl, g, act, col);
    // parent (unscaled), then publish this row's unscaled value for its children
    if (plocal != kNone) {
      if (!have_parent) {
        while (flags[plocal] == 0u) __nanosleep(32);
        __threadfence_block();
        if (lead) pv = __ldcg(reinterpret_cast<const float4*>(p.interior + (size_t)psrc * p.dpad + col));
      }
      acc = f4add(acc, pv);
    }
    if (own != kNone) {
      if (lead) *reinterpret_cast<float4*>(p.interior + (size_t)own * p.dpad + col) = acc;
      __threadfence_block();
      __syncwarp();
      if (lane == 0) flags[j] = 1u;
    }
    float4 yv = acc;
    if constexpr (NORM) yv = f4mul(acc, srow);
    if (p.relu) yv = f4relu(yv);
    if (lead) *reinterpret_cast<float4*>(p.y + (long long)row * p.ldy + col) = yv;
    __syncwarp();  // every lane is done with buf before it is refilled
    j = jn;
    b ^= 1u;
  }
  cp_wait<0>();
  if (p.trace) {
    __syncthreads();
    if (tid == 0) {
      uint32_t sm;
      asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
      unsigned long long* o = p.trace + 4 * (size_t)unit;
      o[0] = sm;
      o[1] = t0;
      o[2] = t1;
      o[3] = gtimer();
    }
  }
}

// Units [0, n_main) are (block, slab of 128/H columns), block-major. The
// remaining (block, slab) pairs of that order are each split into two units of
// half the width, so the last wave is made of smaller pieces (tile_spmm picks
// n_main by simulating the dispatch).
template <int H, bool NORM, int NT>
__global__ void __launch_bounds__(NT, (NT <= 256 ? 2 : 1)) tile_kernel(const TileParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t u = blockIdx.x;
  if constexpr (H < 4) {
    if (u >= p.n_main) {
      const uint32_t v = u - p.n_main, w = p.n_main + v / 2;
      const uint32_t blk = w / p.n_slabs, slab = w - blk * p.n_slabs;
      tile_unit<2 * H, NORM, NT>(p, blk, slab * (128u / H) + (v & 1u) * (64u / H), smem, u);
      return;
    }
  }
  const uint32_t blk = u / p.n_slabs, slab = u - blk * p.n_slabs;
  tile_unit<H, NORM, NT>(p, blk, slab * (128u / H), smem, u);
}

#ifndef CBM_TILE_THREADS
#define CBM_TILE_THREADS 768
#endif

template <int H, bool NORM>
void launch_tile(const TileParams& p, uint32_t units, size_t smem, int device, cudaStream_t s) {
  constexpr int NT = CBM_TILE_THREADS;
  // the dynamic shared-memory attribute belongs to each device's context
  static std::atomic<uint64_t> set_on{0};
  const uint64_t bit = 1ull << (device & 63);
  if (!(set_on.load(std::memory_order_acquire) & bit)) {
    ck(cudaFuncSetAttribute(tile_kernel<H, NORM, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            227 * 1024),
       "tile smem attribute");
    set_on.fetch_or(bit, std::memory_order_acq_rel);
  }
  tile_kernel<H, NORM, NT><<<units, NT, smem, s>>>(p);
}

}  // namespace

size_t tile_smem_bytes(const DeviceMatrix* h, uint32_t W) {
  const auto& t = h->tile;
  const size_t flags = (size_t(t.max_rows) + 3) / 4 * 16;
  return size_t(t.max_staged + 1) * W * sizeof(float) + size_t(t.max_rows) * 32 + flags + 16 +
         size_t(CBM_TILE_THREADS / 32) * 2 * kIdxCap * sizeof(uint32_t) +
         (h->info.normalized ? size_t(t.max_staged + 1) * sizeof(float) : 0);
}

// Slab width W (floats) for a call: 16-byte aligned rows (d, ldx, ldy multiples
// of 4), the tile must fit in shared memory; the widest W that still gives
// every SM a unit (tile_vec forces W = 32 * tile_vec). 0 = not usable.
uint32_t tile_pick_vec(const DeviceMatrix* h, uint32_t d, const float* x, int64_t ldx,
                       const float* y, int64_t ldy) {
  auto al = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) % 16) == 0; };
  if (d % 4 || ldx % 4 || ldy % 4 || !al(x) || !al(y)) return 0;
  const size_t cap = 227 * 1024;
  auto ok = [&](uint32_t W) { return tile_smem_bytes(h, W) <= cap; };
  if (h->opt.tile_vec == 1 || h->opt.tile_vec == 2 || h->opt.tile_vec == 4)
    return ok(32u * h->opt.tile_vec) ? 32u * uint32_t(h->opt.tile_vec) : 0u;
  uint32_t best = 0;
  for (uint32_t W : {32u, 64u, 128u}) {
    if (!ok(W) || (W > 32 && d < W)) continue;
    const uint64_t units = uint64_t(h->tile.n_blocks) * ((d + W - 1) / W);
    if (best == 0 || units >= uint64_t(h->num_sms)) best = W;
  }
  return best;
}

// Full-width units of a launch (tile_kernel): the last (block, slab) pairs are
// split into two half-width units when that shortens the last wave. The CTA
// dispatch (one CTA per SM: 24 warps x ~80 registers) is simulated on the
// blocks' work estimates; a half unit is costed at 0.62 of a full one.
uint32_t tile_pick_main(DeviceMatrix* h, uint32_t W, uint32_t n_slabs) {
  const uint64_t key = (uint64_t(W) << 32) | n_slabs;
  auto it = h->tile_main.find(key);
  if (it != h->tile_main.end()) return it->second;
  const auto& wk = h->tile.work;
  const uint64_t T = uint64_t(wk.size()) * n_slabs;
  const uint32_t S = uint32_t(std::max(1, h->num_sms));
  uint64_t best_x = 0;
  double best = -1.0;
  if (W > 32 && !std::getenv("CBM_B200_TILE_NOSPLIT")) {
    const uint64_t cand[] = {0, S / 4, S / 2, S * 3 / 4, S, S * 3 / 2, uint64_t(S) * 2,
                             uint64_t(S) * 3};
    for (uint64_t x : cand) {
      if (x > T) continue;
      std::priority_queue<double, std::vector<double>, std::greater<double>> q;
      for (uint32_t i = 0; i < S; ++i) q.push(0.0);
      auto put = [&](double w) {
        const double t0 = q.top();
        q.pop();
        q.push(t0 + w);
      };
      for (uint64_t u = 0; u < T - x; ++u) put(double(wk[u / n_slabs]));
      for (uint64_t u = T - x; u < T; ++u) {
        put(0.62 * wk[u / n_slabs]);
        put(0.62 * wk[u / n_slabs]);
      }
      double mk = 0.0;
      while (!q.empty()) {
        mk = std::max(mk, q.top());
        q.pop();
      }
      if (best < 0.0 || mk < best * 0.999) {
        best = mk;
        best_x = x;
      }
    }
  }
  if (const char* e = std::getenv("CBM_B200_TILE_SPLIT"))  // test hook: split the last x pairs
    if (W > 32) best_x = std::min<uint64_t>(T, std::strtoull(e, nullptr, 10));
  const uint32_t n_main = uint32_t(T - best_x);
  h->tile_main[key] = n_main;
  return n_main;
}

void tile_spmm(DeviceMatrix* h, uint32_t W, const float* x, int64_t ldx, uint32_t d, float* y,
               int64_t ldy, float* interior, uint32_t dpad, bool relu, cudaStream_t s) {
  const auto& t = h->tile;
  TileParams p;
  p.dcol = h->tdcol;
  p.dval = h->tdval;
  p.rows = reinterpret_cast<const uint4*>(h->trow);
  p.blocks = reinterpret_cast<const uint4*>(h->tblock);
  p.stage = h->tstage;
  p.scale = h->scale;
  p.x = x;
  p.ldx = ldx;
  p.y = y;
  p.ldy = ldy;
  p.interior = interior;
  p.dpad = dpad;
  p.d = d;
  p.n_slabs = (d + W - 1) / W;
  p.relu = relu ? 1u : 0u;
  p.max_staged = t.max_staged;
  p.max_rows = t.max_rows;
  const uint64_t pairs = uint64_t(t.n_blocks) * p.n_slabs;
  if (pairs == 0) return;
  p.n_main = tile_pick_main(h, W, p.n_slabs);
  const uint64_t units = p.n_main + 2 * (pairs - p.n_main);
  if (units >= 0x7FFFFFFFull) throw invalid_argument("spmm: too many tile units");
  const size_t smem = tile_smem_bytes(h, W);
  const bool norm = h->info.normalized;
  // dev tool: CBM_B200_TILE_TRACE=<file> appends (sm, start, staged, end) per unit
  const char* trace_path = std::getenv("CBM_B200_TILE_TRACE");
  p.trace = nullptr;
  if (trace_path) {
    ck(cudaMalloc(&p.trace, units * 32), "trace");
    ck(cudaMemsetAsync(p.trace, 0, units * 32, s), "trace");
  }
  if (W == 128) norm ? launch_tile<1, true>(p, uint32_t(units), smem, h->device, s)
                     : launch_tile<1, false>(p, uint32_t(units), smem, h->device, s);
  else if (W == 64) norm ? launch_tile<2, true>(p, uint32_t(units), smem, h->device, s)
                         : launch_tile<2, false>(p, uint32_t(units), smem, h->device, s);
  else norm ? launch_tile<4, true>(p, uint32_t(units), smem, h->device, s)
            : launch_tile<4, false>(p, uint32_t(units), smem, h->device, s);
  ck(cudaGetLastError(), "tile_kernel launch");
  if (p.trace) {
    std::vector<unsigned long long> t(units * 4);
    ck(cudaStreamSynchronize(s), "trace");
    ck(cudaMemcpy(t.data(), p.trace, units * 32, cudaMemcpyDeviceToHost), "trace");
    cudaFree(p.trace);
    if (FILE* f = std::fopen(trace_path, "a")) {
      std::fprintf(f, "call units=%llu W=%u\n", (unsigned long long)units, W);
      for (uint64_t u = 0; u < units; ++u)
        std::fprintf(f, "%llu %llu %llu %llu %llu\n", (unsigned long long)u, t[4 * u], t[4 * u + 1],
                     t[4 * u + 2], t[4 * u + 3]);
      std::fclose(f);
    }
  }
}

}  // namespace cbmb
