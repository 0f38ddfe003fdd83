// sm_100a kernels of the CBM multiply.
//
// One persistent, dependency-driven kernel computes the reference's three
// stages (proj/src/kernels.cpp:27-62) in a single pass over the work items of
// layout.hpp:
//   stage 1  delta sum        acc = ((+0 (+) v0*x0) (+) v1*x1) ...   ascending k
//   stage 2  parent add       acc = acc (+) U[parent]                (unscaled parent)
//   stage 3  row scale        Y   = acc (*) s_row                    (normalized)
// with every (+)/(*) an explicitly rounded __fadd_rn/__fsub_rn/__fmul_rn (the
// reference's object code has no FMA).
//
// Schedule. A ticket is (column slab, item), ordered slab-major then item
// order (CHUNK, MERGE, then ROW items by tree depth). The grid is launched
// cooperatively (every warp co-resident) and each warp walks a host-built
// list of tickets (schedule_for: list scheduling by estimated work): no claim
// counter, no atomics. A warp finishes its tickets in increasing order and
// every wait (parent row, split-row partials) targets a smaller ticket, so the
// smallest unfinished ticket is always being worked on and its inputs are
// complete: no deadlock.
//
// Streaming. Each warp walks its ticket sequence with two cursors. The issue
// cursor keeps D X-row segments in flight with cp.async (LDGSTS): every lane
// copies its own V floats of the row into its own slice of a shared-memory
// slot and later reads exactly those bytes back, so a lane-private
// cp.async.wait_group is the only synchronisation. The consume cursor adds
// slot after slot into the accumulator in delta order and runs each item's
// epilogue (partials, parent, stores, flag) as it passes the item's end, while
// the issue cursor is already fetching the next items' rows. Ticket records
// and column-index windows are prefetched a group / a ticket ahead.
// (Bulk async copies were measured and rejected for these row sizes: one
// lane's copies serialise at ~350 ns each — profiles/r01_ubench_gather.txt.)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <string>

#include "cuda_common.hpp"

namespace cbmb {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kThreads = 256;  // 8 warps per CTA


// ---------------------------------------------------------------- vectors
template <int V>
struct Vec;
template <>
struct Vec<1> {
  using T = float;
  static __device__ __forceinline__ T zero() { return 0.0f; }
  static __device__ __forceinline__ T ldg(const float* p) { return __ldg(p); }
  static __device__ __forceinline__ T ldcg(const float* p) { return __ldcg(p); }
  static __device__ __forceinline__ T ldcs(const float* p) { return __ldcs(p); }
  static __device__ __forceinline__ void st(float* p, T v) { *p = v; }
  static __device__ __forceinline__ void stcs(float* p, T v) { __stcs(p, v); }
  static __device__ __forceinline__ T add(T a, T b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ T sub(T a, T b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ T mul(T a, float s) { return __fmul_rn(a, s); }
};
template <>
struct Vec<2> {
  using T = float2;
  static __device__ __forceinline__ T zero() { return make_float2(0.f, 0.f); }
  static __device__ __forceinline__ T ldg(const float* p) {
    return __ldg(reinterpret_cast<const float2*>(p));
  }
  static __device__ __forceinline__ T ldcg(const float* p) {
    return __ldcg(reinterpret_cast<const float2*>(p));
  }
  static __device__ __forceinline__ void st(float* p, T v) { *reinterpret_cast<float2*>(p) = v; }
  static __device__ __forceinline__ T ldcs(const float* p) {
    return __ldcs(reinterpret_cast<const float2*>(p));
  }
  static __device__ __forceinline__ void stcs(float* p, T v) {
    __stcs(reinterpret_cast<float2*>(p), v);
  }
  static __device__ __forceinline__ T add(T a, T b) {
    return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y));
  }
  static __device__ __forceinline__ T sub(T a, T b) {
    return make_float2(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y));
  }
  static __device__ __forceinline__ T mul(T a, float s) {
    return make_float2(__fmul_rn(a.x, s), __fmul_rn(a.y, s));
  }
};
template <>
struct Vec<4> {
  using T = float4;
  static __device__ __forceinline__ T zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
  static __device__ __forceinline__ T ldg(const float* p) {
    return __ldg(reinterpret_cast<const float4*>(p));
  }
  static __device__ __forceinline__ T ldcg(const float* p) {
    return __ldcg(reinterpret_cast<const float4*>(p));
  }
  static __device__ __forceinline__ void st(float* p, T v) { *reinterpret_cast<float4*>(p) = v; }
  static __device__ __forceinline__ T ldcs(const float* p) {
    return __ldcs(reinterpret_cast<const float4*>(p));
  }
  static __device__ __forceinline__ void stcs(float* p, T v) {
    __stcs(reinterpret_cast<float4*>(p), v);
  }
  static __device__ __forceinline__ T add(T a, T b) {
    return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                       __fadd_rn(a.w, b.w));
  }
  static __device__ __forceinline__ T sub(T a, T b) {
    return make_float4(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y), __fsub_rn(a.z, b.z),
                       __fsub_rn(a.w, b.w));
  }
  static __device__ __forceinline__ T mul(T a, float s) {
    return make_float4(__fmul_rn(a.x, s), __fmul_rn(a.y, s), __fmul_rn(a.z, s),
                       __fmul_rn(a.w, s));
  }
};

// ---------------------------------------------------------------- flags
// Every lane's row stores, then the warp barrier (memory ordering among the
// participating lanes), then lane 0's release store at gpu scope, which is
// cumulative over the stores it has observed: the split-K semaphore pattern
// (barrier, then one thread's fence.acq_rel + store). No per-lane
// fence.sc.gpu: that was a second full MEMBAR (+ L1 invalidate) per publish,
// ~5% of cfg[2]'s stall samples.
__device__ __forceinline__ void publish(uint32_t* f, uint32_t epoch) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0)
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* f) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
  return v;
}

__device__ __forceinline__ void await(const uint32_t* f, uint32_t epoch) {
  if ((threadIdx.x & 31) == 0) {
    while (ld_acquire(f) != epoch) __nanosleep(128);
  }
  __syncwarp();
  (void)ld_acquire(f);  // every lane orders its own subsequent loads
}

struct Params {
  const uint32_t* __restrict__ dcol;
  const float* __restrict__ dval;     // per delta: +-row_scale[col] (normalized), dcol order
  const float* __restrict__ scale;    // per column scale (normalized, per-delta products)
  const float* __restrict__ x;
  long long ldx;
  float* y;
  long long ldy;
  float* partial;   // CHUNK / MERGE partial sums, stride dpad
  float* interior;  // unscaled interior rows (normalized), stride dpad
  uint32_t* flags;
  const uint4* __restrict__ trec;  // per warp: wstride ticket records (3 x uint4), in order
  uint32_t wstride;                 // records per warp region
  uint32_t n_items, n_chunk, d, dpad;
  uint32_t total_tickets, total_warps, epoch;
  uint32_t cta_stride;  // CTAs per residency round (grid / CTAs per SM)
  uint32_t relu;        // fused ReLU on Y (relu_inplace, dense.cpp:51-54) for the GCN
  uint32_t faithful;    // order-faithful mode (spmv: sequential adds)
  uint64_t prefetch_bytes;  // > 0: X is one contiguous block of this size, pulled into L2 first
  unsigned long long* trace;  // dev tool (CBM_B200_TRACE): 4 x u64 per warp, else null
  uint32_t ldx32;             // ldx in floats (< 2^30): 32x32->64 address multiply
  uint32_t ldxb;              // ldx in bytes (< 2^32): one IMAD.WIDE per gathered row
  const float* base;          // optional addend per output row (unscaled), may alias y
  long long ldbase;
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Every warp streams its share of a contiguous X into L2 with bulk prefetches
// (sequential HBM reads at full bandwidth instead of first-touch random misses
// on the gather path). Used when X fits comfortably in L2.
__device__ __forceinline__ void prefetch_x(const Params& p, uint32_t w) {
  if (p.prefetch_bytes == 0 || (threadIdx.x & 31) != 0) return;
  const uint64_t share = ((p.prefetch_bytes + p.total_warps - 1) / p.total_warps + 15) & ~15ull;
  const uint64_t lo = share * w;
  if (lo >= p.prefetch_bytes) return;
  const uint64_t hi = lo + share < p.prefetch_bytes ? lo + share : p.prefetch_bytes;
  const char* base = reinterpret_cast<const char*>(p.x);
  for (uint64_t o = lo; o < hi; o += 32768) {
    const uint32_t n = uint32_t((hi - o < 32768 ? hi - o : 32768) & ~15ull);
    if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + o), "r"(n) : "memory");
  }
}

// acc += partial[first], partial[first+1], ... in order. The producers' ready
// flags are checked 32 at a time (one lane each), then the partial rows are
// streamed with PF loads in flight. U segments of 32*V floats per lane.
template <int V, int U, int PF>
__device__ __forceinline__ void add_partials(const Params& p, const uint32_t* flag_base,
                                             uint32_t first, uint32_t cnt, uint32_t col,
                                             typename Vec<V>::T (&acc)[U]) {
  using W = Vec<V>;
  const int lane = threadIdx.x & 31;
  for (uint32_t b0 = 0; b0 < cnt; b0 += 32) {
    const uint32_t nb = min(32u, cnt - b0);
    if (uint32_t(lane) < nb) {
      const uint32_t* f = flag_base + first + b0 + lane;
      while (ld_acquire(f) != p.epoch) __nanosleep(128);
    }
    __syncwarp();
#pragma unroll 1
    for (uint32_t j = 0; j < nb; j += PF) {
      typename W::T v[PF][U];
#pragma unroll
      for (int q = 0; q < PF; ++q)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t c = col + uint32_t(u) * 32u * V;
          v[q][u] = (j + q < nb && c < p.d)
                        ? W::ldcg(p.partial + (size_t)(first + b0 + j + q) * p.dpad + c)
                        : W::zero();
        }
#pragma unroll
      for (int q = 0; q < PF; ++q)
        if (j + q < nb) {
#pragma unroll
          for (int u = 0; u < U; ++u) acc[u] = W::add(acc[u], v[q][u]);
        }
    }
  }
}

// cp.async (LDGSTS) helpers: each lane copies its own V floats of an X row
// into its own slice of a shared-memory slot (16 B: through L2 only, L1 reuse
// measured nil).
// Predicated form: `on` = false copies nothing and zero-fills the lane's slot
// (src-size 0), so a ring group is always written in full without a branch.
template <int V>
__device__ __forceinline__ void cp_async_n(float* dst, const float* src, uint32_t n) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  if constexpr (V == 4)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(d), "l"(src), "n"(V * 4),
                 "r"(n)
                 : "memory");
}
template <int V>
__device__ __forceinline__ void cp_async_z(float* dst, const float* src, bool on) {
  cp_async_n<V>(dst, src, on ? uint32_t(V * 4) : 0u);
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// Copies of one ring slot at the matrix's column edge: out-of-range segments
// copy nothing (and point at a valid address). Not inlined, so the common
// full-width path stays a straight line instead of being if-converted.
template <int V, int U, uint32_t kSeg>
__device__ __noinline__ void edge_copies(float* slot, const float* src, const float* any,
                                         uint32_t imask, bool on) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const bool ok = on && ((imask >> u) & 1u);
    cp_async_z<V>(slot + u * 32 * V, ok ? src + u * kSeg : any, ok);
  }
}

// Wait until at most n (<= N) of the most recently committed groups are pending.
template <int N>
__device__ __forceinline__ void cp_wait_upto(uint32_t n) {
  if constexpr (N == 0) {
    cp_wait<0>();
  } else {
    if (n >= uint32_t(N)) cp_wait<N>();
    else cp_wait_upto<N - 1>(n);
  }
}
// relu_inplace (dense.cpp:51-54): v < 0 -> +0, everything else (-0.0 too) kept
__device__ __forceinline__ float relu1(float v) { return v < 0.0f ? 0.0f : v; }
template <int V>
__device__ __forceinline__ typename Vec<V>::T relu_v(typename Vec<V>::T v) {
  if constexpr (V == 4) return make_float4(relu1(v.x), relu1(v.y), relu1(v.z), relu1(v.w));
  else if constexpr (V == 2) return make_float2(relu1(v.x), relu1(v.y));
  else return relu1(v);
}
// n consecutive floats from shared memory (16-byte aligned for n >= 4)
template <int N>
__device__ __forceinline__ void load_vals(const float* p, float (&o)[N]) {
  if constexpr (N % 4 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 4) {
      const float4 a = *reinterpret_cast<const float4*>(p + i);
      o[i] = a.x; o[i + 1] = a.y; o[i + 2] = a.z; o[i + 3] = a.w;
    }
  } else if constexpr (N == 2) {
    const float2 a = *reinterpret_cast<const float2*>(p);
    o[0] = a.x; o[1] = a.y;
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) o[i] = p[i];
  }
}
template <int V>
__device__ __forceinline__ typename Vec<V>::T lds(const float* p) {
  if constexpr (V == 4) return *reinterpret_cast<const float4*>(p);
  else if constexpr (V == 2) return *reinterpret_cast<const float2*>(p);
  else return *p;
}

template <int V>
__device__ __forceinline__ typename Vec<V>::T xor_sign(typename Vec<V>::T v, uint32_t m) {
  if constexpr (V == 4) {
    return make_float4(__int_as_float(__float_as_int(v.x) ^ m), __int_as_float(__float_as_int(v.y) ^ m),
                       __int_as_float(__float_as_int(v.z) ^ m), __int_as_float(__float_as_int(v.w) ^ m));
  } else if constexpr (V == 2) {
    return make_float2(__int_as_float(__float_as_int(v.x) ^ m), __int_as_float(__float_as_int(v.y) ^ m));
  } else {
    return __int_as_float(__float_as_int(v) ^ m);
  }
}

// acc (+) (+-v) in one instruction per element: fma(v, +-1, acc) forms the
// exact product +-v and rounds the sum once, i.e. exactly fl(acc + v) or
// fl(acc - v) (signed zeros included) -- the reference's stage-1 step for a
// +-1 delta value (kernels.cpp:30-35).
template <int V>
__device__ __forceinline__ typename Vec<V>::T shfl_xor_v(typename Vec<V>::T v, uint32_t off) {
  if constexpr (V == 4) {
    return make_float4(__shfl_xor_sync(kFull, v.x, off), __shfl_xor_sync(kFull, v.y, off),
                       __shfl_xor_sync(kFull, v.z, off), __shfl_xor_sync(kFull, v.w, off));
  } else if constexpr (V == 2) {
    return make_float2(__shfl_xor_sync(kFull, v.x, off), __shfl_xor_sync(kFull, v.y, off));
  } else {
    return __shfl_xor_sync(kFull, v, off);
  }
}

template <int V>
__device__ __forceinline__ typename Vec<V>::T fma_sign(typename Vec<V>::T acc,
                                                       typename Vec<V>::T v, float sg) {
  if constexpr (V == 4) {
    return make_float4(__fmaf_rn(v.x, sg, acc.x), __fmaf_rn(v.y, sg, acc.y),
                       __fmaf_rn(v.z, sg, acc.z), __fmaf_rn(v.w, sg, acc.w));
  } else if constexpr (V == 2) {
    return make_float2(__fmaf_rn(v.x, sg, acc.x), __fmaf_rn(v.y, sg, acc.y));
  } else {
    return __fmaf_rn(v, sg, acc);
  }
}

constexpr int kWarpsPerCta = 4;
// Ring geometry (measured defaults; overridable for A/B builds, `make alt`):
// D slots per warp ring by segments per ticket, B slots per ring group.
#ifndef CBM_D_U4
#define CBM_D_U4 4
#endif
#ifndef CBM_D_U2
#define CBM_D_U2 8
#endif
#ifndef CBM_D_U1
#define CBM_D_U1 16
#endif
#ifndef CBM_B_U4
#define CBM_B_U4 2
#endif
#ifndef CBM_B_U2
#define CBM_B_U2 4
#endif
#ifndef CBM_B_U1
#define CBM_B_U1 8
#endif
#ifndef CBM_D_H2  // lane groups of 16 lanes (d <= 64)
#define CBM_D_H2 16
#endif
#ifndef CBM_B_H2
#define CBM_B_H2 8
#endif


// Record window per warp for the multiply kernel (a power of two <= kRecWin).
#ifndef CBM_RECWIN_U4
#define CBM_RECWIN_U4 64
#endif
// 5 CTAs per SM (<= 96 registers): shared memory allows 5 at 45.5 KB per CTA.
// Unbounded, the 4-segment normalized variants took 97 registers and the
// one-segment ones 110, both dropping to 4 CTAs (16 warps) per SM.
#ifndef CBM_MINB
#define CBM_MINB 5
#endif
#define CBM_LAUNCH_BOUNDS(U) __launch_bounds__(kWarpsPerCta * 32, CBM_MINB)
#ifndef CBM_RECWIN_U2
#define CBM_RECWIN_U2 64
#endif
#ifndef CBM_RECWIN_U1
#define CBM_RECWIN_U1 64
#endif
template <int U>
constexpr uint32_t rec_window() {
  return U == 4 ? CBM_RECWIN_U4 : (U == 2 ? CBM_RECWIN_U2 : CBM_RECWIN_U1);
}

template <int V, int U, int D, int H = 1>
struct alignas(16) WarpSmem {
  float ring[D][U][32 * V];      // slot s, segment u, lane l: [s][u][l*V, l*V+V)
  TRec rec[rec_window<U>()];     // warp-sequence tickets [g, g+RW), slot i & (RW-1)
  float val[D * H > 32 ? D * H : 32];  // signed delta values: lane group h, slot s at [h*D + s]
};

// Stage the records of warp-sequence tickets [i0, i0+RW/2) into a window of
// RW records. Regions are padded (zero records past a warp's count, 64 more
// after the last region), so the loads need no bound: one dependent hop from
// the kernel start to the records.
template <uint32_t RW = kRecWin, class SM>
__device__ __forceinline__ void stage_recs(const Params& p, SM& sm, uint32_t w, uint32_t i0) {
  const uint32_t lane = threadIdx.x & 31;
  if (lane >= RW / 2) return;
  const uint32_t i = i0 + lane;
  const uint4* src = p.trec + 3 * ((size_t)w * p.wstride + i);
  uint4* dst = reinterpret_cast<uint4*>(&sm.rec[i & (RW - 1)]);
  const uint4 a = __ldg(src), b = __ldg(src + 1), c = __ldg(src + 2);
  dst[0] = a;
  dst[1] = b;
  dst[2] = c;
}

// SC: how a delta value enters stage 1.
//   0  +-1 (binary, or normalized with a pre-scaled X): fma(x, +-1, acc), exact
//   1  +-s_c, order-faithful: fl(acc + fl(+-s_c * x)), the reference's two roundings
//   2  +-s_c, default mode: fma(x, +-s_c, acc), one rounding (within tolerance)
// H: deltas per warp instruction. H = 1: the 32 lanes span one X row segment.
//   H = 2 / 4 (narrow X, default mode only): the warp splits into H lane
//   groups, each takes every H-th delta of the ticket, and the H partial sums
//   are combined once per ticket by a fixed shuffle tree (summation order
//   changes; integer sums stay exact).
template <int V, int U, int D, bool NORM, int SC, int H = 1>
__global__ void CBM_LAUNCH_BOUNDS(U) cbm_kernel(const Params p) {
  using W = Vec<V>;
  using T4 = typename W::T;
  static_assert(H == 1 || (U == 1 && SC != 1), "lane groups: one segment, default mode");
  constexpr uint32_t kLanes = 32u / H;    // lanes per delta
  constexpr uint32_t kSeg = kLanes * V;   // floats of one segment (one LDGSTS per lane)
  constexpr uint32_t kSlab = kSeg * U;    // floats per ticket
  constexpr int PFp = U >= 4 ? 2 : (U == 2 ? 4 : 8);
  static_assert((D & (D - 1)) == 0, "ring depth must be a power of two");
  // deltas per ring group: copies are issued, committed and awaited B at a
  // time (a group never spans two tickets; its unused slots stay idle)
  constexpr int B = H >= 8 ? 32 / H : (H == 4 ? 4 : (H == 2 ? CBM_B_H2 : (U == 4 ? CBM_B_U4 : (U == 2 ? CBM_B_U2 : CBM_B_U1))));
  static_assert(D % B == 0, "whole ring groups");
  constexpr int G = D / B;  // groups in flight
  constexpr uint32_t kGroup = uint32_t(B) * H;  // deltas per ring group
  static_assert(32 % kGroup == 0, "a ring group never spans two index windows");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  constexpr uint32_t RW = rec_window<U>();  // staged records (two halves)
  constexpr uint32_t kHalf = RW / 2;
  const uint32_t hl = uint32_t(lane) / kLanes;          // lane group
  const uint32_t jv = (uint32_t(lane) % kLanes) * V;    // column offset in a segment
  using SM = WarpSmem<V, U, D, H>;
  SM& sm = reinterpret_cast<SM*>(smem_raw)[threadIdx.x >> 5];
  // warp -> position in the round-robin: CTAs b, b+G, b+2G, ... (G = p.cta_stride,
  // one per SM) share an SM, so consecutive tickets (adjacent rows, similar
  // delta columns) land on one SM and reuse its L1
  const uint32_t cta = blockIdx.x, wi = threadIdx.x >> 5;
  const uint32_t w = (cta % p.cta_stride) * (p.total_warps / p.cta_stride) +
                     (cta / p.cta_stride) * kWarpsPerCta + wi;
  if (w >= p.total_warps) return;
  const unsigned long long t_start = p.trace ? globaltimer() : 0ull;
  prefetch_x(p, w);
  uint32_t g = 0;  // staged records cover warp-sequence tickets [g, g + 64)
  stage_recs<RW>(p, sm, w, 0);
  __syncwarp();
  const uint32_t n_w = sm.rec[0].nw;  // this warp's tickets (increasing ticket order)
  if (n_w == 0) return;
  if (n_w > kHalf) {  // (most warps of small matrices fit one half: less start-up traffic)
    stage_recs<RW>(p, sm, w, kHalf);
    __syncwarp();
  }
  auto R = [&](uint32_t i) -> const TRec& { return sm.rec[i & (RW - 1)]; };
  // 32 column words (and values) of a delta block: lane j holds delta k0 + j
  struct Wd {
    uint32_t c;
    float v;
  };
  auto fetch = [&](uint32_t k0, uint32_t end) -> Wd {
    Wd r{0u, 0.0f};
    if (k0 + lane < end) {
      r.c = __ldg(p.dcol + k0 + lane);
      if constexpr (SC != 0) r.v = __ldg(p.dval + k0 + lane);
    }
    return r;
  };
  // first block of ticket i (empty past the end / outside the staged records)
  auto window = [&](uint32_t i) -> Wd {
    if (i >= n_w || i >= g + RW) return Wd{0u, 0.0f};
    const TRec& r = R(i);
    return fetch(r.beg, r.end);
  };

  // ---- issue cursor: ticket ii, offset iq inside it. win = window of ii,
  // wn1 / wn2 = windows of ii+1 / ii+2 (fetched two tickets ahead)
  uint32_t ii = 0, iq = 0, ibeg = 0, ilen = 0, icol = 0, imask = 0;
  const char* ixb = reinterpret_cast<const char*>(p.x);  // this ticket's column slab of X row 0
  bool ifull = true;  // warp-uniform: every segment of every lane inside the matrix
  Wd win = window(0), wn1 = window(1), wn2 = window(2), wlong{0u, 0.0f};
  uint32_t iseq = 0;     // ring slots issued (B per group)
  uint32_t icommit = 0;  // ring groups committed; the consumer's k-th group is the k-th
  uint32_t cgroup = 0;   // groups consumed
  bool iblocked = false;
  auto load_ticket = [&]() {  // cursor fields of ticket ii (window already in win)
    iq = 0;
    const TRec& r = R(ii);
    ibeg = r.beg;
    ilen = r.end - r.beg;
    icol = r.slab * kSlab + jv;
    ixb = reinterpret_cast<const char*>(p.x + icol);
    imask = 0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (icol + uint32_t(u) * kSeg < p.d) imask |= 1u << u;
    ifull = __all_sync(kFull, imask == (1u << U) - 1u);
    wlong = fetch(ibeg + 32, r.end);
  };
  // step to the next ticket with deltas, shifting the window prefetch;
  // block while the ticket two ahead is outside the staged records
  auto next_ticket = [&]() {
    for (;;) {
      if (ii + 1 >= n_w) {
        ii = n_w;
        return;
      }
      if (ii + 3 >= g + RW && ii + 3 < n_w) {
        iblocked = true;  // resume after the record window slides
        return;
      }
      ++ii;
      win = wn1;
      wn1 = wn2;
      wn2 = window(ii + 2);
      if (R(ii).end != R(ii).beg) {
        load_ticket();
        return;
      }
    }
  };
  auto issue_group = [&]() {
    if (!iblocked && ii < n_w) {
      const uint32_t n = min(kGroup, ilen - iq);
      const uint32_t s0 = iseq & (D - 1);  // a multiple of B
      // all B column words first (no shuffle under a branch), then B
      // predicated copies: slots past the ticket's end are zero-filled with
      // value 0, so the consumer adds exact zeros there (acc is never -0)
      // slot s0 + b holds deltas b*H + h of the group, lane group h each.
      // The window is kept rotated so that lane q holds the group's delta q
      // (shifted down by kGroup after each group): the shuffles below take
      // immediate lane indices (H = 1) and the values need no shuffle at all.
      uint32_t cwb[B];
#pragma unroll
      for (int b = 0; b < B; ++b) cwb[b] = __shfl_sync(kFull, win.c, uint32_t(b) * H + hl);
      // the deltas' signed values (the reference's values[k], kernels.cpp:33):
      // lane q < kGroup stores its delta q = b * H + h at val[h * D + s0 + b],
      // so the consumer reads a group's B values of its lane group with one or
      // two broadcast LDS
      {
        const uint32_t q = uint32_t(lane);
        float val;
        if constexpr (SC != 0) val = win.v;
        else val = __int_as_float(0x3F800000u | (win.c & 0x80000000u));
        if (q < kGroup) sm.val[(q % H) * D + s0 + q / H] = q < n ? val : 0.0f;
      }
      if (ifull) {  // straight-line copies: one size for all segments, immediate
        // segment offsets, one IMAD.WIDE per row address (byte pitch < 2^32)
#pragma unroll
        for (int b = 0; b < B; ++b) {
          // past the ticket's end the word is another delta of this window or
          // 0 (fetch, or a lane the rotation left in place): a valid row either
          // way, and nothing is read (size 0)
          const bool on = uint32_t(b) * H + hl < n;
          const uint32_t c = cwb[b] & 0x7FFFFFFFu;
          const float* src = reinterpret_cast<const float*>(ixb + (uint64_t)c * p.ldxb);
          const uint32_t sz = on ? uint32_t(V * 4) : 0u;
#pragma unroll
          for (int u = 0; u < U; ++u) cp_async_n<V>(&sm.ring[s0 + b][u][lane * V], src + u * kSeg, sz);
        }
      } else {
#pragma unroll
        for (int b = 0; b < B; ++b) {
          const bool on = uint32_t(b) * H + hl < n;
          const uint32_t c = on ? (cwb[b] & 0x7FFFFFFFu) : 0u;
          const float* src = reinterpret_cast<const float*>(ixb + (uint64_t)c * p.ldxb);
          if constexpr (U == 1 && H == 1) {  // the matrix edge: a real call keeps
            // the one-segment hot path unpredicated (A/B: cfg[2] 921 -> 838 us; with
            // lane groups the call costs more than it saves, cfg[0] 20.5 -> 22.5 us)
            edge_copies<V, U, kSeg>(&sm.ring[s0 + b][0][lane * V], src, p.x, imask, on);
          } else {  // (inline for U > 1: a call there costs more than the predication)
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const bool ok = on && ((imask >> u) & 1u);
              cp_async_z<V>(&sm.ring[s0 + b][u][lane * V], ok ? src + u * kSeg : p.x, ok);
            }
          }
        }
      }
      iseq += B;
      iq += n;
      if (iq == ilen) {
        next_ticket();
      } else if ((iq & 31) == 0) {  // next 32-delta block of a long ticket
        win = wlong;
        wlong = fetch(ibeg + iq + 32, ibeg + ilen);
      } else {  // rotate: the next group's deltas to lanes 0 .. kGroup-1
        win.c = __shfl_down_sync(kFull, win.c, kGroup);
        if constexpr (SC != 0) win.v = __shfl_down_sync(kFull, win.v, kGroup);
      }
      cp_commit();  // only real groups are committed: group k is the consumer's k-th
      ++icommit;
    }
  };
  // keep G groups in flight (after a consumed group, and when the issue
  // cursor resumes after waiting for the record window to slide)
  auto refill = [&]() {
    while (icommit - cgroup < uint32_t(G) && !iblocked && ii < n_w) issue_group();
  };

  if (R(0).end != R(0).beg) load_ticket();
  else next_ticket();
  refill();
  __syncwarp();  // the first groups' values are in sm.val

  uint32_t cseq = 0;  // deltas consumed
#pragma unroll 1
  for (uint32_t ci = 0; ci < n_w; ++ci) {
    if (ci - g == kHalf) {  // slide the record window by one half
      __syncwarp();
      stage_recs<RW>(p, sm, w, g + RW);
      g += kHalf;
      __syncwarp();
      if (iblocked) {
        iblocked = false;
        next_ticket();
        refill();
        __syncwarp();
      }
    }
    const uint32_t k_ci = ci & (RW - 1);
    const TRec r = sm.rec[k_ci];
    const uint32_t slab = r.slab, t = r.item;
    const uint32_t col = slab * kSlab + jv;
    const bool writer = H == 1 || hl == 0;  // lane groups hold equal rows after the combine
    T4 acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = W::zero();
    // one ring group (B slots) per wait: all B shared-memory reads are in
    // flight before the adds, which stay in delta order. Segments outside the
    // matrix read stale ring bytes into accumulators that are never stored.
#pragma unroll 1
    for (uint32_t k = r.beg; k < r.end; k += kGroup) {
      // this group was committed (the issue cursor is never behind the
      // consumer: it only stops at a record-window edge the consumer reaches
      // first); wait until its copies have landed
      if (icommit <= cgroup) __trap();
      cp_wait_upto<G - 1>(icommit - 1 - cgroup);
      const uint32_t s0 = cseq & (D - 1);
      if constexpr (G == 1) __syncwarp();  // (G >= 2: a barrier already follows the issue)
      float sc[B];
      load_vals<B>(&sm.val[hl * D + s0], sc);  // +-1 or +-s_c
      T4 v[B][U];
#pragma unroll
      for (int b = 0; b < B; ++b) {
#pragma unroll
        for (int u = 0; u < U; ++u) v[b][u] = lds<V>(&sm.ring[s0 + b][u][lane * V]);
      }
#pragma unroll
      for (int b = 0; b < B; ++b) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if constexpr (SC == 1) acc[u] = W::add(acc[u], W::mul(v[b][u], sc[b]));
          else acc[u] = fma_sign<V>(acc[u], v[b][u], sc[b]);
        }
      }
      cseq += B;
      ++cgroup;
      __syncwarp();  // the group's slots are fully read before their refill
      refill();
    }
    if constexpr (H > 1) {  // combine the lane groups: a fixed tree, equal bits everywhere
#pragma unroll
      for (uint32_t off = kLanes; off < 32u; off *= 2u)
        acc[0] = W::add(acc[0], shfl_xor_v<V>(acc[0], off));
    }
    // ---- epilogue: partials, then CHUNK/MERGE publish or ROW stage 2 + 3
    uint32_t* flag_base = p.flags + (size_t)slab * p.n_items;
    if (r.cnt) add_partials<V, U, PFp>(p, flag_base, r.first, r.cnt, col, acc);
    if (t < p.n_chunk) {
      float* dst = p.partial + (size_t)t * p.dpad;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (writer && col + uint32_t(u) * kSeg < p.d) W::st(dst + col + u * kSeg, acc[u]);
      publish(flag_base + t, p.epoch);
      continue;
    }
    if (r.ppos != 0xFFFFFFFFu) {  // + unscaled parent row
      await(flag_base + r.ppos, p.epoch);
      const float* src =
          NORM ? p.interior + (size_t)r.psrc * p.dpad : p.y + (long long)r.psrc * p.ldy;
      T4 pv[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        pv[u] = col + uint32_t(u) * kSeg < p.d ? W::ldcg(src + col + u * kSeg) : W::zero();
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u] = W::add(acc[u], pv[u]);
    }
    const uint32_t row = r.rowk & 0x7FFFFFFFu;
    if (p.base) {  // + the row's dense-block (tensor-core) sum, read before Y is written
      const float* src = p.base + (long long)row * p.ldbase;
      T4 bv[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        bv[u] = col + uint32_t(u) * kSeg < p.d ? W::ldcs(src + col + u * kSeg) : W::zero();
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u] = W::add(acc[u], bv[u]);
    }
    const bool is_parent = (r.rowk >> 31) != 0;
    float* yrow = p.y + (long long)row * p.ldy;
    if constexpr (NORM) {
      if (is_parent) {  // children read the unscaled row from scratch
        float* dst = p.interior + (size_t)r.slot * p.dpad;
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (writer && col + uint32_t(u) * kSeg < p.d) W::st(dst + col + u * kSeg, acc[u]);
        publish(flag_base + t, p.epoch);
      }
      const float sr = __uint_as_float(r.srow);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (writer && col + uint32_t(u) * kSeg < p.d) {
          T4 yv = W::mul(acc[u], sr);
          if (p.relu) yv = relu_v<V>(yv);
          // (dense-block path: Y is final here and X should keep its L2 lines)
          if (p.base) W::stcs(yrow + col + u * kSeg, yv);
          else W::st(yrow + col + u * kSeg, yv);
        }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (writer && col + uint32_t(u) * kSeg < p.d) {
          if (p.base) W::stcs(yrow + col + u * kSeg, p.relu ? relu_v<V>(acc[u]) : acc[u]);
          else W::st(yrow + col + u * kSeg, p.relu ? relu_v<V>(acc[u]) : acc[u]);
        }
      if (is_parent) publish(flag_base + t, p.epoch);
    }
  }
  cp_wait<0>();  // no copy may target shared memory after exit
  if (p.trace && lane == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    unsigned long long* o = p.trace + 4 * (size_t)w;
    o[0] = t_start;
    o[1] = 0ull;  // (first-data stamp removed from the hot loop)
    o[2] = globaltimer();
    o[3] = (unsigned long long)smid | ((unsigned long long)n_w << 16) |
           ((unsigned long long)cseq << 32);
  }
}

// ------------------------------------------------------------------ spmv
// d = 1 (spmv_into / spmv, kernels.cpp:70-103). A column of width one leaves
// 31 lanes idle in cbm_kernel, so here the 32 lanes take 32 consecutive
// deltas of a ticket at once: column word, value and the gathered x element
// are loaded in parallel. Order-faithful: the products are added to the
// accumulator one by one in delta order (shuffled from their lanes, every
// lane carrying the same accumulator), exactly as the reference. Default:
// each lane accumulates its deltas (fma), then a fixed butterfly reduction.
// Same tickets, schedule, flags, partials and epilogue as cbm_kernel.
struct alignas(16) SpmvSmem {
  TRec rec[kRecWin];
};

template <bool NORM, int SC>
__global__ void __launch_bounds__(kWarpsPerCta * 32) cbm_spmv_kernel(const Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  SpmvSmem& sm = reinterpret_cast<SpmvSmem*>(smem_raw)[threadIdx.x >> 5];
  const uint32_t cta = blockIdx.x, wi = threadIdx.x >> 5;
  const uint32_t w = (cta % p.cta_stride) * (p.total_warps / p.cta_stride) +
                     (cta / p.cta_stride) * kWarpsPerCta + wi;
  if (w >= p.total_warps) return;
  uint32_t g = 0;
  stage_recs(p, sm, w, 0);
  stage_recs(p, sm, w, 32);
  __syncwarp();
  const uint32_t n_w = sm.rec[0].nw;
  if (n_w == 0) return;
  const bool faithful = SC == 1 || p.faithful;
#pragma unroll 1
  for (uint32_t ci = 0; ci < n_w; ++ci) {
    if (ci - g == 32) {
      __syncwarp();
      stage_recs(p, sm, w, g + kRecWin);
      g += 32;
      __syncwarp();
    }
    const TRec r = sm.rec[ci & (kRecWin - 1)];
    const uint32_t t = r.item;
    float acc = 0.0f;   // faithful: the running sum (same on every lane)
    float part = 0.0f;  // default: this lane's partial sum
#pragma unroll 1
    // batches of K blocks of 32 deltas: all K index loads, then all K
    // gathers are in flight together (two latencies per batch, not per block)
    constexpr int K = 8;
#pragma unroll 1
    for (uint32_t k0 = r.beg; k0 < r.end; k0 += 32 * K) {
      uint32_t cw[K];
      float val[K], xv[K];
#pragma unroll
      for (int q = 0; q < K; ++q) {
        const uint32_t k = k0 + 32u * q + lane;
        const bool on = k < r.end;
        cw[q] = on ? __ldg(p.dcol + k) : 0u;
        if constexpr (SC != 0) val[q] = on ? __ldg(p.dval + k) : 0.0f;
      }
#pragma unroll
      for (int q = 0; q < K; ++q) {
        const bool on = k0 + 32u * q + lane < r.end;
        xv[q] = on ? __ldg(p.x + (uint64_t)(cw[q] & 0x7FFFFFFFu) * p.ldx32) : 0.0f;
        if constexpr (SC == 0) val[q] = on ? __int_as_float(0x3F800000u | (cw[q] & 0x80000000u)) : 0.0f;
      }
#pragma unroll
      for (int q = 0; q < K; ++q) {
        const uint32_t kb = k0 + 32u * q;
        if (kb >= r.end) break;
        if (faithful) {
          // fl(v * x): exact for +-1 (a sign flip), the reference's rounded
          // product for +-s_c; then ascending adds (kernels.cpp:18-24)
          const float prod = __fmul_rn(val[q], xv[q]);
          const uint32_t n = min(32u, r.end - kb);
          for (uint32_t j = 0; j < n; ++j) acc = __fadd_rn(acc, __shfl_sync(kFull, prod, j));
        } else {
          part = __fmaf_rn(xv[q], val[q], part);  // idle lanes add 0 * 0
        }
      }
    }
    if (!faithful) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part = __fadd_rn(part, __shfl_xor_sync(kFull, part, o));
      acc = part;
    }
    // ---- epilogue (cbm_kernel's, one column)
    const uint32_t* flag_base = p.flags;
    if (r.cnt) {  // + partial sums in order
      for (uint32_t b0 = 0; b0 < r.cnt; b0 += 32) {
        const uint32_t nb = min(32u, r.cnt - b0);
        float pv = 0.0f;
        if (uint32_t(lane) < nb) {
          const uint32_t* f = flag_base + r.first + b0 + lane;
          while (ld_acquire(f) != p.epoch) __nanosleep(128);
          pv = __ldcg(p.partial + (size_t)(r.first + b0 + lane) * p.dpad);
        }
        for (uint32_t j = 0; j < nb; ++j) acc = __fadd_rn(acc, __shfl_sync(kFull, pv, j));
      }
    }
    if (t < p.n_chunk) {
      if (lane == 0) p.partial[(size_t)t * p.dpad] = acc;
      publish(p.flags + t, p.epoch);
      continue;
    }
    if (r.ppos != 0xFFFFFFFFu) {  // + unscaled parent (kernels.cpp:84-90)
      await(flag_base + r.ppos, p.epoch);
      const float* src =
          NORM ? p.interior + (size_t)r.psrc * p.dpad : p.y + (long long)r.psrc * p.ldy;
      acc = __fadd_rn(acc, __ldcg(src));
    }
    const uint32_t row = r.rowk & 0x7FFFFFFFu;
    const bool is_parent = (r.rowk >> 31) != 0;
    if constexpr (NORM) {
      if (is_parent) {
        if (lane == 0) p.interior[(size_t)r.slot * p.dpad] = acc;
        publish(p.flags + t, p.epoch);
      }
      float yv = __fmul_rn(acc, __uint_as_float(r.srow));
      if (p.relu) yv = relu1(yv);
      if (lane == 0) p.y[(long long)row * p.ldy] = yv;
    } else {
      if (lane == 0) p.y[(long long)row * p.ldy] = p.relu ? relu1(acc) : acc;
      if (is_parent) publish(p.flags + t, p.epoch);
    }
  }
}

// xs[c, :] = row_scale[c] (*) x[c, :] — the bit-identical products of the
// normalized stage 1 (fl(+-s*x) = +-fl(s*x)), formed once per call.
__global__ void prescale_kernel(const float* __restrict__ x, long long ldx,
                                const float* __restrict__ scale, uint32_t rows, uint32_t d,
                                float* __restrict__ xs, uint32_t dpad) {
  const uint64_t total = (uint64_t)rows * d;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = uint32_t(i / d), c = uint32_t(i - (uint64_t)r * d);
    xs[(uint64_t)r * dpad + c] = __fmul_rn(__ldg(scale + r), __ldg(x + (long long)r * ldx + c));
  }
}

// relu_inplace (dense.cpp:51-54) on a column slab of Y: the binary streaming
// kernel's children read their parent's row from Y itself, so a fused ReLU
// would feed them clipped parents; binary multiplies with ReLU clip afterwards.
__global__ void relu_kernel(float* __restrict__ y, long long ldy, uint32_t rows, uint32_t d) {
  const uint64_t total = (uint64_t)rows * d;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = uint32_t(i / d), c = uint32_t(i - (uint64_t)r * d);
    float* q = y + (long long)r * ldy + c;
    const float v = *q;
    if (v < 0.0f) *q = 0.0f;
  }
}

// Cooperative launch: one full residency wave (all warps co-resident), no
// more warps than tickets.
// Per (kernel instance, device): the dynamic shared-memory attribute is set
// and the occupancy queried once on every device the kernel runs on (0 = not
// yet; the attribute belongs to the device's context).
constexpr int kMaxDevices = 64;
using DeviceSlots = std::atomic<int>[kMaxDevices];

void launch_coop(const void* kernel, size_t smem, DeviceSlots& slots, Params& p,
                 uint64_t tickets, uint32_t slabs, DeviceMatrix* h, cudaStream_t s) {
  if (h->device < 0 || h->device >= kMaxDevices) throw invalid_argument("spmm: device ordinal");
  int bps = slots[h->device].load(std::memory_order_acquire);
  if (bps == 0) {
    ck(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
       "smem attribute");
    int b = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kWarpsPerCta * 32, smem),
       "occupancy");
    bps = std::max(1, b);
    slots[h->device].store(bps, std::memory_order_release);
  }
  // cooperative launch: one full residency wave, never more warps than tickets
  constexpr uint64_t wpb = kWarpsPerCta;
  const uint64_t cap = uint64_t(h->num_sms) * bps * wpb;
  const uint64_t warps = std::max<uint64_t>(1, std::min(cap, tickets));
  int grid = int((warps + wpb - 1) / wpb);
  // SM-local mapping needs grid = cta_stride * CTAs-per-SM exactly
  const int per_sm = std::max(1, (grid + h->num_sms - 1) / h->num_sms);
  p.cta_stride = uint32_t((grid + per_sm - 1) / per_sm);
  grid = int(p.cta_stride) * per_sm;
  if (uint64_t(grid) > uint64_t(h->num_sms) * bps) {  // rounding overflowed a wave
    p.cta_stride = uint32_t(grid / per_sm);
    grid = int(p.cta_stride) * per_sm;
  }
  p.total_warps = uint32_t(grid * wpb);
  const auto& sc = schedule_for(h, p.total_warps, slabs, s);
  p.trec = reinterpret_cast<const uint4*>(sc.trec);
  p.wstride = sc.wstride;
  void* args[] = {&p};
  ck(cudaLaunchCooperativeKernel(kernel, dim3(grid), dim3(kWarpsPerCta * 32), args, smem, s),
     "cbm_kernel cooperative launch");
}

template <int V, int U, int D, bool NORM, int SC, int H = 1>
void launch_one(Params& p, uint64_t tickets, uint32_t slabs, DeviceMatrix* h, cudaStream_t s) {
  static DeviceSlots slots;  // per template instance and device
  launch_coop(reinterpret_cast<const void*>(&cbm_kernel<V, U, D, NORM, SC, H>),
              kWarpsPerCta * sizeof(WarpSmem<V, U, D, H>), slots, p, tickets, slabs, h, s);
}

template <bool NORM, int SC>
void launch_spmv(Params& p, uint64_t tickets, DeviceMatrix* h, cudaStream_t s) {
  static DeviceSlots slots;
  launch_coop(reinterpret_cast<const void*>(&cbm_spmv_kernel<NORM, SC>),
              kWarpsPerCta * sizeof(SpmvSmem), slots, p, tickets, 1, h, s);
}

template <int V, int U, int D>
void run_kernel(Params& p, uint64_t tickets, uint32_t slabs, bool norm, bool scl,
                DeviceMatrix* h, cudaStream_t s) {
  if (!norm) launch_one<V, U, D, false, 0>(p, tickets, slabs, h, s);
  else if (!scl) launch_one<V, U, D, true, 0>(p, tickets, slabs, h, s);
  else if (h->info.order_faithful) launch_one<V, U, D, true, 1>(p, tickets, slabs, h, s);
  else launch_one<V, U, D, true, 2>(p, tickets, slabs, h, s);
}

// Narrow X in the default mode: H deltas per warp instruction (V = 4, U = 1).
// H = 8 / 16 (d <= 16 / 8, e.g. the slabs of 4-8 column-sharded ranks): a
// ring group is a whole 32-delta window (B = 32 / H), two groups in flight.
template <int H>
void run_groups(Params& p, uint64_t tickets, uint32_t slabs, bool norm, bool scl,
                DeviceMatrix* h, cudaStream_t s) {
  constexpr int D = H == 2 ? CBM_D_H2 : (H == 16 ? 4 : 8);
  if (!norm) launch_one<4, 1, D, false, 0, H>(p, tickets, slabs, h, s);
  else if (!scl) launch_one<4, 1, D, true, 0, H>(p, tickets, slabs, h, s);
  else launch_one<4, 1, D, true, 2, H>(p, tickets, slabs, h, s);
}


}  // namespace

namespace {
uint32_t pick_vec(uint32_t d, const float* x, int64_t ldx, const float* y, int64_t ldy) {
  auto al = [](const void* p, unsigned b) { return (reinterpret_cast<uintptr_t>(p) % b) == 0; };
  if (d > 32 && d % 4 == 0 && ldx % 4 == 0 && ldy % 4 == 0 && al(x, 16) && al(y, 16)) return 4;
  if (d > 16 && d % 2 == 0 && ldx % 2 == 0 && ldy % 2 == 0 && al(x, 8) && al(y, 8)) return 2;
  return 1;
}
}  // namespace

namespace {
void spmm_rest(DeviceMatrix* h, const float* x, int64_t ldx, uint32_t d, float* y, int64_t ldy,
               void* stream, bool relu, const float* base, int64_t ldbase);
}

void device_spmm(DeviceMatrix* h, const float* x, int64_t ldx, uint32_t d, float* y,
                 int64_t ldy, void* stream, bool relu, const float* base, int64_t ldbase) {
  spmm_rest(h, x, ldx, d, y, ldy, stream, relu, base, ldbase);
  if (!h->hub_on || h->info.n_rows == 0 || d == 0) return;
  // hub-row panel: this operator's layout leaves the hub rows empty (zeros in
  // Y so far); their rows come from the tensor cores, or, for X narrower than
  // that path takes, from the hub rows' own streaming operator
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint32_t launches = h->last_launches;
  if (d >= kDenseMinD) {
    if (ldx >= (int64_t(1) << 30))
      throw invalid_argument("spmm: leading dimension of X must be below 2^30");
    auto& ws = h->ws[stream];
    h->last_launches = launches + 1;  // the panel's tensor kernel; hub_spmm adds its reductions
    hub_spmm(h, x, ldx, d, y, ldy, relu, ws.hub_part, ws.hub_part_cap, s);
  } else {
    const uint32_t dpad = (d + 3) & ~3u;
    auto& ws = h->ws[stream];
    grow(ws.hub_part, ws.hub_part_cap, uint64_t(h->hub_n_rows) * dpad, "workspace hub rows");
    device_spmm(h->hub_op, x, ldx, d, ws.hub_part, dpad, stream, relu);
    hub_scatter(ws.hub_part, dpad, h->hrows, h->hub_n_rows, d, y, ldy, s);
    h->last_launches = launches + h->hub_op->last_launches + 1;
  }
}

namespace {
void spmm_rest(DeviceMatrix* h, const float* x, int64_t ldx, uint32_t d, float* y, int64_t ldy,
               void* stream, bool relu, const float* base, int64_t ldbase) {
  const Layout& L = h->info;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  h->last_launches = 0;
  if (L.n_rows == 0 || d == 0) return;
  if (ldx >= (int64_t(1) << 31)) throw invalid_argument("spmm: leading dimension too large");
  ck(cudaSetDevice(h->device), "cudaSetDevice");
  if (h->dense_on && d >= kDenseMinD && !base) {
    // dense-block path: the tensor cores write the shared-column part of
    // every row (unscaled) into Y, the streaming kernel adds the cold
    // entries to it in place and applies the row scale / ReLU
    if (ldx >= (int64_t(1) << 30))
      throw invalid_argument("spmm: leading dimension of X must be below 2^30");
    uint32_t dbg = 0;  // dev timing only (CBM_B200_DENSE_DBG): 16 no cold kernel, 32 no dense kernel
    if (const char* e = std::getenv("CBM_B200_DENSE_DBG")) dbg = uint32_t(std::atoi(e));
    if (!(dbg & 32)) dense_spmm(h, x, ldx, d, y, ldy, s);
    if (!(dbg & 16)) device_spmm(h->cold, x, ldx, d, y, ldy, stream, relu, y, ldy);
    h->last_launches = 1 + h->cold->last_launches;
    return;
  }
  device_reserve(h, d, stream);
  auto& ws = h->ws[stream];
  const uint32_t dpad = (d + 3) & ~3u;
  // tiled path (tile_kernel.cu): community-structured matrices, d >= 32
  if (h->tile_on && d >= 32 && !base) {
    if (const uint32_t tv = tile_pick_vec(h, d, x, ldx, y, ldy)) {
      tile_spmm(h, tv, x, ldx, d, y, ldy, ws.tinterior, dpad, relu, s);
      h->last_launches = 1;
      return;
    }
  }
  bool prescale = false;
  if (L.normalized) {
    if (h->opt.prescale > 0) prescale = true;
    // auto: in the order-faithful mode the per-delta FMUL costs nnz*d ALU ops
    // and pre-scaling an extra 8*n*d bytes of HBM traffic; the
    // default mode fuses the product into the FMA, so there is nothing to save
    else if (h->opt.prescale < 0)
      prescale = L.order_faithful && L.nnz_effective > 48ull * L.n_cols;
  }
  const float* xin = x;
  int64_t ldin = ldx;
  if (prescale) {
    grow(ws.xs, ws.xs_cap, uint64_t(L.n_cols) * dpad, "workspace prescale");
    const uint64_t total = uint64_t(L.n_cols) * d;
    const int grid = int(std::min<uint64_t>((total + 255) / 256, uint64_t(h->num_sms) * 16));
    prescale_kernel<<<grid, 256, 0, s>>>(x, ldx, h->scale, L.n_cols, d, ws.xs, dpad);
    ck(cudaGetLastError(), "prescale launch");
    ++h->last_launches;
    xin = ws.xs;
    ldin = dpad;
  }
  // lanes x V floats per column slab: V = 4 (LDG.128) when rows are 16-byte
  // aligned multiples, else 2 or 1; kernel option 1 forces scalar lanes
  const uint32_t V = h->opt.kernel == 1 ? 1u : pick_vec(d, xin, ldin, y, ldy);
  // segments of 32*V columns per ticket: wide X shares one ticket's record,
  // indices and epilogue across up to 4 segments ...
  const uint32_t segs = (d + 32 * V - 1) / (32 * V);
  uint32_t U = segs >= 4 ? 4 : (segs >= 2 ? 2 : 1);
  if (h->opt.max_segments == 1 || h->opt.max_segments == 2)
    U = std::min<uint32_t>(U, uint32_t(h->opt.max_segments));
  // (narrower slabs that fit X in L2 were measured slower on cfg[2]/cfg[3]:
  // the extra per-ticket work outweighs the L2 misses they remove)
  // narrow X in the default mode: H lane groups of 32/H lanes, one delta each
  // per warp instruction (d <= 64, rows 16-byte aligned)
  uint32_t H = 1;
#ifndef CBM_NO_LANE_GROUPS
  if (!L.order_faithful && h->opt.kernel == 0 && d >= 4 && d <= 64 && d % 4 == 0 &&
      ldin % 4 == 0 && ldy % 4 == 0 && (reinterpret_cast<uintptr_t>(xin) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(y) & 15) == 0)
    H = d <= 8 ? 16 : (d <= 16 ? 8 : (d <= 32 ? 4 : 2));
#endif
  const uint32_t lanes_v = (H > 1 ? 4u : V) * (32 / H) * (H > 1 ? 1u : U);  // floats per slab
  const uint32_t n_slabs = (d + lanes_v - 1) / lanes_v;
  if (++ws.epoch == 0) {  // wrapped: re-zero the flags
    ck(cudaMemsetAsync(ws.flags, 0, ws.flags_cap * sizeof(uint32_t), s), "flags memset");
    ws.epoch = 1;
  }
  Params p;
  p.base = base;
  p.ldbase = ldbase;
  p.dcol = h->dcol;
  p.dval = h->dval;
  p.scale = h->scale;
  p.x = xin;
  p.ldx = ldin;
  p.y = y;
  p.ldy = ldy;
  p.partial = ws.partial;
  p.interior = ws.interior;
  p.flags = ws.flags;
  p.n_items = L.n_items;
  p.n_chunk = L.n_chunk_items;
  p.d = d;
  p.dpad = dpad;
  const uint64_t tickets = uint64_t(L.n_items) * n_slabs;
  if (tickets >= 0x7FFFFFFFull) throw invalid_argument("spmm: too many work tickets");
  p.total_tickets = uint32_t(tickets);
  p.epoch = ws.epoch;
  // binary streaming kernel: children read parents from Y, so the ReLU runs
  // after the multiply (relu_kernel below); normalized parents come from scratch
  const bool relu_after = relu && !L.normalized;
  p.relu = relu && !relu_after ? 1u : 0u;
  // pull a small, contiguous X into L2 ahead of the gathers
  const uint64_t xbytes = uint64_t(L.n_cols) * d * sizeof(float);
  p.prefetch_bytes = (h->opt.prefetch != 0 && uint64_t(ldin) == d && xbytes >= (1u << 20) &&
                      xbytes <= uint64_t(h->l2_bytes) / 2 &&
                      (reinterpret_cast<uintptr_t>(xin) & 15) == 0)
                         ? (xbytes & ~15ull)
                         : 0;

  const bool norm = L.normalized, scl = L.normalized && !prescale;
  // dev tool: CBM_B200_TRACE=<file> appends per-warp timestamps of every call
  const char* trace_path = std::getenv("CBM_B200_TRACE");
  unsigned long long* trace = nullptr;
  const size_t trace_n = size_t(h->num_sms) * 64 * 4;
  p.trace = nullptr;
  if (trace_path) {
    ck(cudaMalloc(&trace, trace_n * 8), "trace");
    ck(cudaMemsetAsync(trace, 0, trace_n * 8, s), "trace");
    p.trace = trace;
  }
  p.faithful = L.order_faithful ? 1u : 0u;
  p.ldx32 = uint32_t(ldin);
  // every caller (C ABI, host pipeline, GCN, prescale) lands here: the byte
  // pitch of one gathered row must fit 32 bits
  if (uint64_t(ldin) >= (uint64_t(1) << 30))
    throw invalid_argument("spmm: leading dimension of X must be below 2^30");
  p.ldxb = uint32_t(ldin) * 4u;
  if (H > 1) {
    if (H == 2) run_groups<2>(p, tickets, n_slabs, norm, scl, h, s);
    else if (H == 4) run_groups<4>(p, tickets, n_slabs, norm, scl, h, s);
    else if (H == 8) run_groups<8>(p, tickets, n_slabs, norm, scl, h, s);
    else run_groups<16>(p, tickets, n_slabs, norm, scl, h, s);
  } else if (d == 1) {  // spmv: lanes over deltas
    if (!norm) launch_spmv<false, 0>(p, tickets, h, s);
    else if (!scl) launch_spmv<true, 0>(p, tickets, h, s);
    else if (L.order_faithful) launch_spmv<true, 1>(p, tickets, h, s);
    else launch_spmv<true, 2>(p, tickets, h, s);
  } else if (V == 4) {
    if (U == 4) run_kernel<4, 4, CBM_D_U4>(p, tickets, n_slabs, norm, scl, h, s);
    else if (U == 2) run_kernel<4, 2, CBM_D_U2>(p, tickets, n_slabs, norm, scl, h, s);
    else run_kernel<4, 1, CBM_D_U1>(p, tickets, n_slabs, norm, scl, h, s);
  } else if (V == 2) {
    if (U == 4) run_kernel<2, 4, 8>(p, tickets, n_slabs, norm, scl, h, s);
    else if (U == 2) run_kernel<2, 2, 8>(p, tickets, n_slabs, norm, scl, h, s);
    else run_kernel<2, 1, 16>(p, tickets, n_slabs, norm, scl, h, s);
  } else {
    if (U == 4) run_kernel<1, 4, 16>(p, tickets, n_slabs, norm, scl, h, s);
    else if (U == 2) run_kernel<1, 2, 16>(p, tickets, n_slabs, norm, scl, h, s);
    else run_kernel<1, 1, 16>(p, tickets, n_slabs, norm, scl, h, s);
  }
  ck(cudaGetLastError(), "cbm_kernel launch");
  ++h->last_launches;
  if (relu_after) {
    const uint64_t total = uint64_t(L.n_rows) * d;
    const int grid = int(std::min<uint64_t>((total + 255) / 256, uint64_t(h->num_sms) * 16));
    relu_kernel<<<grid, 256, 0, s>>>(y, ldy, L.n_rows, d);
    ck(cudaGetLastError(), "relu launch");
    ++h->last_launches;
  }
  if (trace) {
    std::vector<unsigned long long> t(trace_n);
    ck(cudaStreamSynchronize(s), "trace");
    ck(cudaMemcpy(t.data(), trace, trace_n * 8, cudaMemcpyDeviceToHost), "trace");
    cudaFree(trace);
    if (FILE* f = std::fopen(trace_path, "a")) {
      std::fprintf(f, "call warps=%u tickets=%llu\n", p.total_warps, (unsigned long long)tickets);
      for (uint32_t w = 0; w < p.total_warps; ++w)
        std::fprintf(f, "%u %llu %llu %llu %llu\n", w, t[4 * w], t[4 * w + 1], t[4 * w + 2],
                     t[4 * w + 3]);
      std::fclose(f);
    }
  }
}

}  // namespace

}  // namespace cbmb
