// sm_100a kernels of the CBM multiply.
//
// One persistent, dependency-driven kernel computes the reference's three
// stages (proj/src/kernels.cpp:27-62) in a single pass over the work items of
// layout.hpp:
//   stage 1  delta sum        acc = ((+0 (+) v0*x0) (+) v1*x1) ...   ascending k
//   stage 2  parent add       acc = acc (+) U[parent]                (unscaled parent)
//   stage 3  row scale        Y   = acc (*) s_row                    (normalized)
// with every (+)/(*) an explicitly rounded __fadd_rn/__fsub_rn/__fmul_rn (the
// reference's object code has no FMA). Warps claim tickets (slab, item) from a
// global counter in slab-major, level order; a ROW item whose parent (or whose
// split chunks) are not finished yet spins on a per-item ready flag. Tickets
// are only ever claimed by running warps and every wait targets an earlier
// ticket, so the smallest unfinished ticket always makes progress: no
// deadlock for any grid size or residency.
//
// Lanes cover a column slab of 32*V floats (V = 4: 128-bit loads of X rows);
// a row's delta column indices are fetched 32 at a time with one coalesced load
// and broadcast with shuffles; PF X-row slabs are in flight per warp.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <string>

#include "device.hpp"

namespace cbmb {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kThreads = 256;  // 8 warps per CTA

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    const int code = (e == cudaErrorMemoryAllocation) ? CBM_B200_ENOMEM : CBM_B200_ECUDA;
    throw cuda_error(std::string(what) + ": " + cudaGetErrorString(e), code);
  }
}

// ---------------------------------------------------------------- vectors
template <int V>
struct Vec;
template <>
struct Vec<1> {
  using T = float;
  static __device__ __forceinline__ T zero() { return 0.0f; }
  static __device__ __forceinline__ T ldg(const float* p) { return __ldg(p); }
  static __device__ __forceinline__ T ldcg(const float* p) { return __ldcg(p); }
  static __device__ __forceinline__ void st(float* p, T v) { *p = v; }
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
__device__ __forceinline__ void publish(uint32_t* f, uint32_t epoch) {
  __threadfence();  // each lane's row stores before the flag (gpu scope)
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
    while (ld_acquire(f) != epoch) __nanosleep(32);
  }
  __syncwarp();
  (void)ld_acquire(f);  // every lane orders its own subsequent loads
}

struct Params {
  const uint32_t* __restrict__ dptr;
  const uint32_t* __restrict__ dcol;
  const uint4* __restrict__ meta;
  const uint32_t* __restrict__ pcnt;
  const uint32_t* __restrict__ oslot;
  const float* __restrict__ scale;
  const float* __restrict__ x;
  long long ldx;
  float* y;
  long long ldy;
  float* partial;   // CHUNK partial sums, stride dpad
  float* interior;  // unscaled interior rows (normalized), stride dpad
  uint32_t* flags;
  uint32_t* counters;
  uint32_t n_items, n_chunk, d, dpad;
  uint32_t total_tickets, batch, total_warps, epoch;
};

// Per lane: U vectors of V floats at columns col0 + u*32*V (each u is one
// fully coalesced 32*V*4-byte segment of an X row).
template <int V, int U>
struct Acc {
  typename Vec<V>::T v[U];
};

// Stage 1 for one item: delta sum over dcol[beg, end) into acc, deltas in
// storage (ascending column) order, PF deltas x U segments in flight.
template <int V, int U, int PF, bool SCALE>
__device__ __forceinline__ void delta_sum(const Params& p, uint32_t beg, uint32_t end,
                                          uint32_t col0, Acc<V, U>& acc) {
  using W = Vec<V>;
  const int lane = threadIdx.x & 31;
  for (uint32_t k0 = beg; k0 < end; k0 += 32) {
    const uint32_t n = min(32u, end - k0);
    const uint32_t myc = lane < n ? __ldg(p.dcol + k0 + lane) : 0u;
    float mys = 0.0f;
    if constexpr (SCALE) mys = lane < n ? __ldg(p.scale + (myc & 0x7FFFFFFFu)) : 0.0f;
#pragma unroll 1
    for (uint32_t j = 0; j < n; j += PF) {
      typename W::T xv[PF][U];
      uint32_t cq[PF];
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        cq[q] = __shfl_sync(kFull, myc, (j + q) & 31);
        const float* row = p.x + (long long)(cq[q] & 0x7FFFFFFFu) * p.ldx;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t c = col0 + uint32_t(u) * 32u * V;
          xv[q][u] = (j + q < n && c < p.d) ? W::ldg(row + c) : W::zero();
        }
      }
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        float s = 0.0f;
        if constexpr (SCALE) s = __shfl_sync(kFull, mys, (j + q) & 31);
        if (j + q < n) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            typename W::T v = xv[q][u];
            if constexpr (SCALE) v = W::mul(v, s);
            acc.v[u] = (cq[q] & 0x80000000u) ? W::sub(acc.v[u], v) : W::add(acc.v[u], v);
          }
        }
      }
    }
  }
}

template <int V, int U>
__device__ __forceinline__ void add_row(Acc<V, U>& acc, const float* src, uint32_t col0,
                                        uint32_t d) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t c = col0 + uint32_t(u) * 32u * V;
    if (c < d) acc.v[u] = Vec<V>::add(acc.v[u], Vec<V>::ldcg(src + c));
  }
}

template <int V, int U>
__device__ __forceinline__ void store_row(const Acc<V, U>& acc, float* dst, uint32_t col0,
                                          uint32_t d) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t c = col0 + uint32_t(u) * 32u * V;
    if (c < d) Vec<V>::st(dst + c, acc.v[u]);
  }
}

template <int V, int U>
__device__ __forceinline__ void store_row_scaled(const Acc<V, U>& acc, float* dst, uint32_t col0,
                                                 uint32_t d, float s) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t c = col0 + uint32_t(u) * 32u * V;
    if (c < d) Vec<V>::st(dst + c, Vec<V>::mul(acc.v[u], s));
  }
}

// acc += partial[first], partial[first+1], ... in order. The producers' ready
// flags are checked 32 at a time (one lane each), then the partial rows are
// streamed with PF x U loads in flight.
template <int V, int U, int PF>
__device__ __forceinline__ void add_partials(const Params& p, const uint32_t* flag_base,
                                             uint32_t first, uint32_t cnt, uint32_t col0,
                                             Acc<V, U>& acc) {
  using W = Vec<V>;
  const int lane = threadIdx.x & 31;
  for (uint32_t b0 = 0; b0 < cnt; b0 += 32) {
    const uint32_t nb = min(32u, cnt - b0);
    if (uint32_t(lane) < nb) {
      const uint32_t* f = flag_base + first + b0 + lane;
      while (ld_acquire(f) != p.epoch) __nanosleep(32);
    }
    __syncwarp();
#pragma unroll 1
    for (uint32_t j = 0; j < nb; j += PF) {
      typename W::T xv[PF][U];
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        const float* src = p.partial + (size_t)(first + b0 + j + q) * p.dpad;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t c = col0 + uint32_t(u) * 32u * V;
          xv[q][u] = (j + q < nb && c < p.d) ? W::ldcg(src + c) : W::zero();
        }
      }
#pragma unroll
      for (int q = 0; q < PF; ++q)
        if (j + q < nb) {
#pragma unroll
          for (int u = 0; u < U; ++u) acc.v[u] = W::add(acc.v[u], xv[q][u]);
        }
    }
  }
}

// One ticket = one item over a column slab of 32*V*U columns. Tickets are
// claimed in batches; the batch's dptr/meta are fetched with one
// lane-parallel load and broadcast with shuffles.
template <int V, int U, int PF, bool NORM, bool SCALE>
__global__ void __launch_bounds__(kThreads) cbm_fused_kernel(const Params p) {
  using W = Vec<V>;
  constexpr uint32_t kSlab = 32u * V * U;
  const int lane = threadIdx.x & 31;
  for (;;) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(p.counters, p.batch);
    base = __shfl_sync(kFull, base, 0);
    if (base >= p.total_tickets) break;
    const uint32_t nb = min(p.batch, p.total_tickets - base);
    uint32_t my_beg = 0, my_end = 0, my_slot = 0, my_cnt = 0;
    uint4 my_meta = make_uint4(0u, 0xFFFFFFFFu, 0u, 0u);
    if (uint32_t(lane) < nb) {
      const uint32_t T = base + lane;
      const uint32_t t = T - (T / p.n_items) * p.n_items;
      my_beg = __ldg(p.dptr + t);
      my_end = __ldg(p.dptr + t + 1);
      my_meta = __ldg(p.meta + t);
      my_cnt = __ldg(p.pcnt + t);
      if constexpr (NORM) my_slot = __ldg(p.oslot + t);
    }
    for (uint32_t i = 0; i < nb; ++i) {
      const uint32_t T = base + i;
      const uint32_t slab = T / p.n_items;
      const uint32_t t = T - slab * p.n_items;
      const uint32_t col0 = slab * kSlab + uint32_t(lane) * V;
      const uint32_t beg = __shfl_sync(kFull, my_beg, i);
      const uint32_t end = __shfl_sync(kFull, my_end, i);
      const uint32_t first = __shfl_sync(kFull, my_meta.w, i);
      const uint32_t cnt = __shfl_sync(kFull, my_cnt, i);
      Acc<V, U> acc;
#pragma unroll
      for (int u = 0; u < U; ++u) acc.v[u] = W::zero();
      delta_sum<V, U, PF, SCALE>(p, beg, end, col0, acc);
      uint32_t* flag_base = p.flags + (size_t)slab * p.n_items;
      if (cnt) add_partials<V, U, PF>(p, flag_base, first, cnt, col0, acc);
      if (t < p.n_chunk) {  // CHUNK / MERGE item: publish the partial sum
        store_row(acc, p.partial + (size_t)t * p.dpad, col0, p.d);
        publish(flag_base + t, p.epoch);
        continue;
      }
      const uint32_t mrow = __shfl_sync(kFull, my_meta.x, i);
      const uint32_t ppos = __shfl_sync(kFull, my_meta.y, i);
      const uint32_t psrc = __shfl_sync(kFull, my_meta.z, i);
      if (ppos != 0xFFFFFFFFu) {  // stage 2: + unscaled parent row
        await(flag_base + ppos, p.epoch);
        const float* src = NORM ? p.interior + (size_t)psrc * p.dpad
                                : p.y + (long long)psrc * p.ldy;
        add_row(acc, src, col0, p.d);
      }
      const uint32_t row = mrow & 0x7FFFFFFFu;
      const bool is_parent = (mrow >> 31) != 0;
      if constexpr (NORM) {
        if (is_parent) {  // children read the unscaled row from scratch
          const uint32_t slot = __shfl_sync(kFull, my_slot, i);
          store_row(acc, p.interior + (size_t)slot * p.dpad, col0, p.d);
          publish(flag_base + t, p.epoch);
        }
        store_row_scaled(acc, p.y + (long long)row * p.ldy, col0, p.d, __ldg(p.scale + row));
      } else {
        store_row(acc, p.y + (long long)row * p.ldy, col0, p.d);
        if (is_parent) publish(flag_base + t, p.epoch);
      }
    }
  }
  // self-resetting ticket counter: the last warp out rearms it
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(p.counters + 1, 1u) == p.total_warps - 1) {
      p.counters[0] = 0;
      p.counters[1] = 0;
      __threadfence();
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

template <int V, int U, int PF, bool NORM, bool SCALE>
int blocks_per_sm() {
  static int cached = -1;  // per template instance
  if (cached < 0) {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, cbm_fused_kernel<V, U, PF, NORM, SCALE>,
                                                  kThreads, 0);
    cached = std::max(1, b);
  }
  return cached;
}

// Persistent grid: at most one full residency wave, never more warps than
// tickets; ~4 ticket batches per warp keep the claim counter cool.
template <int V, int U, int PF, bool NORM, bool SCALE>
void launch_one(Params& p, uint64_t tickets, int num_sms, cudaStream_t s) {
  constexpr uint64_t wpb = kThreads / 32;
  const uint64_t cap = uint64_t(num_sms) * blocks_per_sm<V, U, PF, NORM, SCALE>() * wpb;
  const uint64_t warps = std::max<uint64_t>(1, std::min(cap, tickets));
  const int grid = int((warps + wpb - 1) / wpb);
  p.total_warps = uint32_t(grid * wpb);
  p.batch = uint32_t(std::clamp<uint64_t>(tickets / (uint64_t(p.total_warps) * 2), 1, 16));
  cbm_fused_kernel<V, U, PF, NORM, SCALE><<<grid, kThreads, 0, s>>>(p);
}

template <int V, int U>
void run_fused(Params& p, uint64_t tickets, bool norm, bool scl, int num_sms, cudaStream_t s) {
  constexpr int PF = (32 / (V * U)) < 2 ? 2 : ((32 / (V * U)) > 16 ? 16 : (32 / (V * U)));
  if (!norm) launch_one<V, U, PF, false, false>(p, tickets, num_sms, s);
  else if (scl) launch_one<V, U, PF, true, true>(p, tickets, num_sms, s);
  else launch_one<V, U, PF, true, false>(p, tickets, num_sms, s);
}

template <int V>
void run_fused_u(uint32_t U, Params& p, uint64_t tickets, bool norm, bool scl, int num_sms,
                 cudaStream_t s) {
  if (U == 4) run_fused<V, 4>(p, tickets, norm, scl, num_sms, s);
  else if (U == 2) run_fused<V, 2>(p, tickets, norm, scl, num_sms, s);
  else run_fused<V, 1>(p, tickets, norm, scl, num_sms, s);
}

template <typename T>
void grow(T*& ptr, uint64_t& cap, uint64_t need, const char* what) {
  if (need <= cap) return;
  if (ptr) ck(cudaFree(ptr), "cudaFree");
  ptr = nullptr;
  cap = 0;
  ck(cudaMalloc(&ptr, std::max<uint64_t>(need, 1) * sizeof(T)), what);
  cap = need;
}

}  // namespace

DeviceMatrix* device_upload(const cbm_b200_cbm_view& v, const cbm_b200_options& opt) {
  // validate + plan on the host first: malformed input is EINVAL, never a CUDA error
  Layout L = plan_layout(v, opt.order_faithful != 0, opt.split_threshold, opt.chunk);
  auto* h = new DeviceMatrix;
  try {
    int dev = opt.device;
    if (dev < 0) ck(cudaGetDevice(&dev), "cudaGetDevice");
    ck(cudaSetDevice(dev), "cudaSetDevice");
    h->device = dev;
    h->opt = opt;
    ck(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    auto put = [&](auto*& dst, const auto& vec, const char* what) {
      using E = typename std::remove_reference_t<decltype(vec)>::value_type;
      const size_t bytes = std::max<size_t>(vec.size(), 1) * sizeof(E);
      ck(cudaMalloc(&dst, bytes), what);
      if (!vec.empty()) ck(cudaMemcpy(dst, vec.data(), vec.size() * sizeof(E),
                                      cudaMemcpyHostToDevice), what);
      h->device_bytes += vec.size() * sizeof(E);
    };
    put(h->dptr, L.dptr, "upload dptr");
    put(h->dcol, L.dcol, "upload dcol");
    put(h->meta, L.meta, "upload meta");
    put(h->pcnt, L.pcnt, "upload pcnt");
    if (L.normalized) {
      put(h->oslot, L.oslot, "upload oslot");
      put(h->scale, L.scale, "upload scale");
    }
    ck(cudaMalloc(&h->counters, 2 * sizeof(uint32_t)), "counters");
    ck(cudaMemset(h->counters, 0, 2 * sizeof(uint32_t)), "counters");
    // keep only sizes on the host
    L.dptr = {};
    L.dcol = {};
    L.meta = {};
    L.pcnt = {};
    L.oslot = {};
    L.scale = {};
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
  for (void* p : {(void*)h->dptr, (void*)h->dcol, (void*)h->meta, (void*)h->pcnt, (void*)h->oslot,
                  (void*)h->scale, (void*)h->counters, (void*)h->flags, (void*)h->partial,
                  (void*)h->interior, (void*)h->xs, (void*)h->xstage, (void*)h->ystage})
    if (p) cudaFree(p);
  delete h;
}

namespace {
uint32_t pick_vec(uint32_t d, const float* x, int64_t ldx, const float* y, int64_t ldy) {
  auto al = [](const void* p, unsigned b) { return (reinterpret_cast<uintptr_t>(p) % b) == 0; };
  if (d > 64 && d % 4 == 0 && ldx % 4 == 0 && ldy % 4 == 0 && al(x, 16) && al(y, 16)) return 4;
  if (d > 32 && d % 2 == 0 && ldx % 2 == 0 && ldy % 2 == 0 && al(x, 8) && al(y, 8)) return 2;
  return 1;
}
}  // namespace

void device_reserve(DeviceMatrix* h, uint64_t d) {
  const Layout& L = h->info;
  const uint64_t dpad = (d + 3) & ~uint64_t(3);
  const uint64_t slabs = (d + 31) / 32;  // worst case (V = 1)
  ck(cudaSetDevice(h->device), "cudaSetDevice");
  if (uint64_t(L.n_items) * slabs > h->flags_cap) {
    grow(h->flags, h->flags_cap, uint64_t(L.n_items) * slabs, "workspace flags");
    ck(cudaMemset(h->flags, 0, h->flags_cap * sizeof(uint32_t)), "flags memset");
    h->epoch = 0;
  }
  grow(h->partial, h->partial_cap, uint64_t(L.n_chunk_items) * dpad, "workspace partial");
  if (L.normalized) grow(h->interior, h->interior_cap, uint64_t(L.n_interior) * dpad,
                         "workspace interior");
}

void device_spmm(DeviceMatrix* h, const float* x, int64_t ldx, uint32_t d, float* y,
                 int64_t ldy, void* stream) {
  const Layout& L = h->info;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  h->last_launches = 0;
  if (L.n_rows == 0 || d == 0) return;
  ck(cudaSetDevice(h->device), "cudaSetDevice");
  device_reserve(h, d);
  const uint32_t dpad = (d + 3) & ~3u;
  bool prescale = false;
  if (L.normalized) {
    if (h->opt.prescale > 0) prescale = true;
    // auto: the per-delta FMUL costs nnz*d ALU ops; pre-scaling costs an
    // extra 8*n*d bytes of HBM traffic (prescale).
    else if (h->opt.prescale < 0) prescale = L.nnz > 48ull * L.n_cols;
  }
  const float* xin = x;
  int64_t ldin = ldx;
  if (prescale) {
    grow(h->xs, h->xs_cap, uint64_t(L.n_cols) * dpad, "workspace prescale");
    const uint64_t total = uint64_t(L.n_cols) * d;
    const int grid = int(std::min<uint64_t>((total + 255) / 256, uint64_t(h->num_sms) * 16));
    prescale_kernel<<<grid, 256, 0, s>>>(x, ldx, h->scale, L.n_cols, d, h->xs, dpad);
    ck(cudaGetLastError(), "prescale launch");
    ++h->last_launches;
    xin = h->xs;
    ldin = dpad;
  }
  const uint32_t V = pick_vec(d, xin, ldin, y, ldy);
  // columns per ticket: up to 4 segments of 32*V columns (<= 512 floats)
  const uint32_t segs = (d + 32 * V - 1) / (32 * V);
  const uint32_t U = segs >= 3 ? 4 : segs;
  const uint32_t n_slabs = (d + 32 * V * U - 1) / (32 * V * U);
  if (++h->epoch == 0) {  // wrapped: re-zero the flags
    ck(cudaMemsetAsync(h->flags, 0, h->flags_cap * sizeof(uint32_t), s), "flags memset");
    h->epoch = 1;
  }
  Params p;
  p.dptr = h->dptr;
  p.dcol = h->dcol;
  p.meta = reinterpret_cast<const uint4*>(h->meta);
  p.pcnt = h->pcnt;
  p.oslot = h->oslot;
  p.scale = h->scale;
  p.x = xin;
  p.ldx = ldin;
  p.y = y;
  p.ldy = ldy;
  p.partial = h->partial;
  p.interior = h->interior;
  p.flags = h->flags;
  p.counters = h->counters;
  p.n_items = L.n_items;
  p.n_chunk = L.n_chunk_items;
  p.d = d;
  p.dpad = dpad;
  const uint64_t tickets = uint64_t(L.n_items) * n_slabs;
  if (tickets >= 0x7FFFFFFFull) throw invalid_argument("spmm: too many work tickets");
  p.total_tickets = uint32_t(tickets);
  p.epoch = h->epoch;

  const bool norm = L.normalized, scl = L.normalized && !prescale;
  if (V == 4) run_fused_u<4>(U, p, tickets, norm, scl, h->num_sms, s);
  else if (V == 2) run_fused_u<2>(U, p, tickets, norm, scl, h->num_sms, s);
  else run_fused_u<1>(U, p, tickets, norm, scl, h->num_sms, s);
  ck(cudaGetLastError(), "cbm_fused launch");
  ++h->last_launches;
}

void device_spmm_host(DeviceMatrix* h, const float* x, uint32_t d, float* y, void* stream) {
  const Layout& L = h->info;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ck(cudaSetDevice(h->device), "cudaSetDevice");
  const uint32_t dpad = (d + 3) & ~3u;
  grow(h->xstage, h->xstage_cap, uint64_t(L.n_cols) * dpad, "staging X");
  grow(h->ystage, h->ystage_cap, uint64_t(L.n_rows) * dpad, "staging Y");
  const size_t xb = size_t(L.n_cols) * d * sizeof(float);
  const size_t yb = size_t(L.n_rows) * d * sizeof(float);
  if (d == dpad) {
    if (xb) ck(cudaMemcpyAsync(h->xstage, x, xb, cudaMemcpyHostToDevice, s), "H2D X");
  } else if (xb) {
    ck(cudaMemcpy2DAsync(h->xstage, dpad * sizeof(float), x, d * sizeof(float),
                         d * sizeof(float), L.n_cols, cudaMemcpyHostToDevice, s), "H2D X");
  }
  device_spmm(h, h->xstage, dpad, d, h->ystage, dpad, stream);
  if (d == dpad) {
    if (yb) ck(cudaMemcpyAsync(y, h->ystage, yb, cudaMemcpyDeviceToHost, s), "D2H Y");
  } else if (yb) {
    ck(cudaMemcpy2DAsync(y, d * sizeof(float), h->ystage, dpad * sizeof(float),
                         d * sizeof(float), L.n_rows, cudaMemcpyDeviceToHost, s), "D2H Y");
  }
  ck(cudaStreamSynchronize(s), "spmm_host synchronize");
}

}  // namespace cbmb
