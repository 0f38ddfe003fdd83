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

// Stage 1 for one item: delta sum over dcol[beg, end) into acc.
template <int V, int PF, bool SCALE>
__device__ __forceinline__ void delta_sum(const Params& p, uint32_t beg, uint32_t end,
                                          uint32_t col, bool active, typename Vec<V>::T& acc) {
  using W = Vec<V>;
  const int lane = threadIdx.x & 31;
  for (uint32_t k0 = beg; k0 < end; k0 += 32) {
    const uint32_t n = min(32u, end - k0);
    const uint32_t myc = lane < n ? __ldg(p.dcol + k0 + lane) : 0u;
    float mys = 0.0f;
    if constexpr (SCALE) mys = lane < n ? __ldg(p.scale + (myc & 0x7FFFFFFFu)) : 0.0f;
#pragma unroll 1
    for (uint32_t j = 0; j < n; j += PF) {
      typename W::T xv[PF];
      uint32_t cq[PF];
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        cq[q] = __shfl_sync(kFull, myc, (j + q) & 31);
        xv[q] = W::zero();
        if (j + q < n && active)
          xv[q] = W::ldg(p.x + (long long)(cq[q] & 0x7FFFFFFFu) * p.ldx + col);
      }
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        typename W::T v = xv[q];
        if constexpr (SCALE) v = W::mul(v, __shfl_sync(kFull, mys, (j + q) & 31));
        if (j + q < n) acc = (cq[q] & 0x80000000u) ? W::sub(acc, v) : W::add(acc, v);
      }
    }
  }
}

template <int V, int PF, bool NORM, bool SCALE>
__global__ void __launch_bounds__(kThreads) cbm_fused_kernel(const Params p) {
  using W = Vec<V>;
  const int lane = threadIdx.x & 31;
  for (;;) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(p.counters, p.batch);
    base = __shfl_sync(kFull, base, 0);
    if (base >= p.total_tickets) break;
    const uint32_t lim = min(base + p.batch, p.total_tickets);
    for (uint32_t T = base; T < lim; ++T) {
      const uint32_t slab = T / p.n_items;
      const uint32_t t = T - slab * p.n_items;
      const uint32_t col = slab * (32u * V) + uint32_t(lane) * V;
      const bool active = col < p.d;
      typename W::T acc = W::zero();
      delta_sum<V, PF, SCALE>(p, p.dptr[t], p.dptr[t + 1], col, active, acc);
      uint32_t* flag_base = p.flags + (size_t)slab * p.n_items;
      if (t < p.n_chunk) {  // CHUNK item: publish the partial sum
        if (active) W::st(p.partial + (size_t)t * p.dpad + col, acc);
        publish(flag_base + t, p.epoch);
        continue;
      }
      const uint4 mt = p.meta[t];
      const uint32_t extra = mt.w >> 24;
      if (extra) {  // remaining chunks of a split row, in order
        const uint32_t first = mt.w & 0xFFFFFFu;
        for (uint32_t i = 0; i < extra; ++i) {
          await(flag_base + first + i, p.epoch);
          if (active) acc = W::add(acc, W::ldcg(p.partial + (size_t)(first + i) * p.dpad + col));
        }
      }
      if (mt.y != 0xFFFFFFFFu) {  // stage 2: + unscaled parent row
        await(flag_base + mt.y, p.epoch);
        const float* src = NORM ? p.interior + (size_t)mt.z * p.dpad
                                : p.y + (long long)mt.z * p.ldy;
        if (active) acc = W::add(acc, W::ldcg(src + col));
      }
      const uint32_t row = mt.x & 0x7FFFFFFFu;
      const bool is_parent = (mt.x >> 31) != 0;
      if (active) {
        if constexpr (NORM) {
          if (is_parent) W::st(p.interior + (size_t)p.oslot[t] * p.dpad + col, acc);
          W::st(p.y + (long long)row * p.ldy + col, W::mul(acc, __ldg(p.scale + row)));
        } else {
          W::st(p.y + (long long)row * p.ldy + col, acc);
        }
      }
      if (is_parent) publish(flag_base + t, p.epoch);
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

template <int V, int PF, bool NORM, bool SCALE>
int blocks_per_sm() {
  static int cached = -1;  // per template instance
  if (cached < 0) {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, cbm_fused_kernel<V, PF, NORM, SCALE>,
                                                  kThreads, 0);
    cached = std::max(1, b);
  }
  return cached;
}

// Persistent grid: at most one full residency wave, never more warps than
// tickets; ~6 ticket batches per warp keep the claim counter cool.
template <int V, int PF, bool NORM, bool SCALE>
void launch_one(Params& p, uint64_t tickets, int num_sms, cudaStream_t s) {
  constexpr uint64_t wpb = kThreads / 32;
  const uint64_t cap = uint64_t(num_sms) * blocks_per_sm<V, PF, NORM, SCALE>() * wpb;
  const uint64_t warps = std::max<uint64_t>(1, std::min(cap, tickets));
  const int grid = int((warps + wpb - 1) / wpb);
  p.total_warps = uint32_t(grid * wpb);
  p.batch = uint32_t(std::clamp<uint64_t>(tickets / (uint64_t(p.total_warps) * 6), 1, 8));
  cbm_fused_kernel<V, PF, NORM, SCALE><<<grid, kThreads, 0, s>>>(p);
}

template <int V, int PF>
void run_fused(Params& p, uint64_t tickets, bool norm, bool scl, int num_sms, cudaStream_t s) {
  if (!norm) launch_one<V, PF, false, false>(p, tickets, num_sms, s);
  else if (scl) launch_one<V, PF, true, true>(p, tickets, num_sms, s);
  else launch_one<V, PF, true, false>(p, tickets, num_sms, s);
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
  for (void* p : {(void*)h->dptr, (void*)h->dcol, (void*)h->meta, (void*)h->oslot,
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
  const uint32_t slab_w = 32 * V;
  const uint32_t n_slabs = (d + slab_w - 1) / slab_w;
  if (++h->epoch == 0) {  // wrapped: re-zero the flags
    ck(cudaMemsetAsync(h->flags, 0, h->flags_cap * sizeof(uint32_t), s), "flags memset");
    h->epoch = 1;
  }
  Params p;
  p.dptr = h->dptr;
  p.dcol = h->dcol;
  p.meta = reinterpret_cast<const uint4*>(h->meta);
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
  if (tickets >= 0xFFFFFFFFull) throw invalid_argument("spmm: too many work tickets");
  p.total_tickets = uint32_t(tickets);
  p.epoch = h->epoch;

  const bool norm = L.normalized, scl = L.normalized && !prescale;
  if (V == 4) run_fused<4, 8>(p, tickets, norm, scl, h->num_sms, s);
  else if (V == 2) run_fused<2, 16>(p, tickets, norm, scl, h->num_sms, s);
  else run_fused<1, 16>(p, tickets, norm, scl, h->num_sms, s);
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
