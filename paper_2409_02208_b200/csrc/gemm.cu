// Reference-order dense GEMM (dense.cpp:31-49) and the GCN forward
// (gcn.cpp:22-33) built from it and the CBM multiply.
#include <cstring>

#include "cuda_common.hpp"

namespace cbmb {

namespace {

// A as column parts [A_0 | A_1 | ...] (A_p: m x k_p row-major, ld k_p, possibly
// another device's memory opened through CUDA IPC), C written to every output
// (each m x n with leading dimension ldc): the all-gather before `. W1` and the
// result's gather fused into one GEMM.
struct Parts {
  const float* a[kMaxParts];
  uint32_t koff[kMaxParts + 1];  // global k offset of each part
  uint32_t n_parts;
  float* out[kMaxParts];
  uint32_t n_out;
  uint32_t ldc;
};

template <bool MULTI>
__device__ __forceinline__ float load_a(const Parts& P, uint32_t row, uint32_t kk) {
  if constexpr (!MULTI) return __ldg(P.a[0] + (size_t)row * P.koff[1] + kk);
  uint32_t p = 0;
  while (p + 1 < P.n_parts && kk >= P.koff[p + 1]) ++p;
  const uint32_t kp = P.koff[p + 1] - P.koff[p];
  return P.a[p][(size_t)row * kp + (kk - P.koff[p])];
}

template <bool MULTI>
__device__ __forceinline__ void store_c(const Parts& P, uint32_t i, uint32_t cc, float v) {
  if constexpr (!MULTI) {
    P.out[0][(size_t)i * P.ldc + cc] = v;
    return;
  }
  for (uint32_t o = 0; o < P.n_out; ++o) P.out[o][(size_t)i * P.ldc + cc] = v;
}

// 128 x 128 output tile per CTA, 8 x 8 per thread, k staged 8 at a time (A
// transposed in shared memory).
//   ORDERED: dense_matmul (dense.cpp:31-49) bit for bit. Every entry sums
//     fl(a*b) in ascending k with separate rounding (FMUL then FADD). The
//     reference skips zero lhs entries (dense.cpp:42); adding fl(0*b) = +-0
//     instead leaves the sum unchanged (it starts at +0 and can never become
//     -0), unless b is not finite, so a k-step whose B rows hold an inf or
//     NaN takes the per-entry skip (block-uniform branch).
//   !ORDERED (default-mode GCN, north_star tolerance): FFMA.
// Part widths are multiples of 4 (column_slab), so a 4-wide k group never
// straddles two parts.
constexpr int kFB = 128, kFK = 8;
template <bool MULTI, bool ORDERED>
__global__ void __launch_bounds__(256, 2) tiled_gemm_kernel(const Parts P,
                                                            const float* __restrict__ b,
                                                            uint32_t m, uint32_t k, uint32_t n) {
  __shared__ __align__(16) float as[kFK][kFB];
  __shared__ __align__(16) float bs[kFK][kFB];
  const uint32_t t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const uint32_t row0 = blockIdx.y * kFB, col0 = blockIdx.x * kFB;
  float acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[r][q] = 0.0f;
  const uint32_t ar = t >> 1, ak = (t & 1) * 4;   // A tile: row ar, k ak..ak+3
  const uint32_t bk = t >> 5, bc = (t & 31) * 4;  // B tile: k bk, cols bc..bc+3
  for (uint32_t k0 = 0; k0 < k; k0 += kFK) {
    float av[4], bv[4];
    bool nonfinite = false;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t kk = k0 + ak + i;
      av[i] = (row0 + ar < m && kk < k) ? load_a<MULTI>(P, row0 + ar, kk) : 0.0f;
      const uint32_t cc = col0 + bc + i;
      bv[i] = (k0 + bk < k && cc < n) ? __ldg(b + (size_t)(k0 + bk) * n + cc) : 0.0f;
      nonfinite |= !isfinite(bv[i]);
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) as[ak + i][ar] = av[i];
    *reinterpret_cast<float4*>(&bs[bk][bc]) = make_float4(bv[0], bv[1], bv[2], bv[3]);
    const bool exact_skip = __syncthreads_or(ORDERED && nonfinite) != 0;
    const uint32_t kn = min(uint32_t(kFK), k - k0);
    if (!exact_skip) {
#pragma unroll
      for (int kk = 0; kk < kFK; ++kk) {
        if (ORDERED && uint32_t(kk) >= kn) break;  // (zero padding is harmless for FFMA)
        const float4 a0 = *reinterpret_cast<const float4*>(&as[kk][ty * 4]);
        const float4 a1 = *reinterpret_cast<const float4*>(&as[kk][64 + ty * 4]);
        const float4 b0 = *reinterpret_cast<const float4*>(&bs[kk][tx * 4]);
        const float4 b1 = *reinterpret_cast<const float4*>(&bs[kk][64 + tx * 4]);
        const float ar8[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float br8[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int q = 0; q < 8; ++q)
            acc[r][q] = ORDERED ? __fadd_rn(acc[r][q], __fmul_rn(ar8[r], br8[q]))
                                : __fmaf_rn(ar8[r], br8[q], acc[r][q]);
      }
    } else {
      for (uint32_t kk = 0; kk < kn; ++kk) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const float a = as[kk][r < 4 ? ty * 4 + r : 64 + ty * 4 + r - 4];
          if (a == 0.0f) continue;  // dense.cpp:42
#pragma unroll
          for (int q = 0; q < 8; ++q)
            acc[r][q] = __fadd_rn(acc[r][q],
                                  __fmul_rn(a, bs[kk][q < 4 ? tx * 4 + q : 64 + tx * 4 + q - 4]));
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const uint32_t i = row0 + (r < 4 ? ty * 4 + r : 64 + ty * 4 + r - 4);
    if (i >= m) continue;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t cc = col0 + (q < 4 ? tx * 4 + q : 64 + tx * 4 + q - 4);
      if (cc < n) store_c<MULTI>(P, i, cc, acc[r][q]);
    }
  }
}

Parts one_part(const float* a, uint32_t k, float* c, uint32_t n) {
  Parts P{};
  P.a[0] = a;
  P.koff[0] = 0;
  P.koff[1] = k;
  P.n_parts = 1;
  P.out[0] = c;
  P.n_out = 1;
  P.ldc = n;
  return P;
}

void launch_gemm(const Parts& P, uint32_t m, uint32_t k, const float* b, uint32_t n,
                 bool ordered, cudaStream_t s) {
  if (m == 0 || n == 0) return;
  const bool multi = P.n_parts > 1 || P.n_out > 1;
  const dim3 grid((n + kFB - 1) / kFB, (m + kFB - 1) / kFB);
  if (ordered) {
    if (multi) tiled_gemm_kernel<true, true><<<grid, 256, 0, s>>>(P, b, m, k, n);
    else tiled_gemm_kernel<false, true><<<grid, 256, 0, s>>>(P, b, m, k, n);
  } else {
    if (multi) tiled_gemm_kernel<true, false><<<grid, 256, 0, s>>>(P, b, m, k, n);
    else tiled_gemm_kernel<false, false><<<grid, 256, 0, s>>>(P, b, m, k, n);
  }
  ck(cudaGetLastError(), "gemm launch");
}
}  // namespace

void device_fast_matmul(const float* a, uint32_t m, uint32_t k, const float* b, uint32_t n,
                        float* c, void* stream) {
  launch_gemm(one_part(a, k, c, n), m, k, b, n, false, static_cast<cudaStream_t>(stream));
}

void device_dense_matmul(const float* a, uint32_t m, uint32_t k, const float* b, uint32_t n,
                         float* c, void* stream) {
  launch_gemm(one_part(a, k, c, n), m, k, b, n, true, static_cast<cudaStream_t>(stream));
}

void device_gemm_parts(const float* const* a_parts, const uint32_t* part_k, uint32_t n_parts,
                       uint32_t m, const float* b, uint32_t n, float* const* outs,
                       uint32_t n_outs, uint32_t ldc, bool ordered, void* stream) {
  if (n_parts < 1 || n_parts > kMaxParts || n_outs < 1 || n_outs > kMaxParts)
    throw invalid_argument("gemm_parts: 1..8 parts and outputs");
  Parts P{};
  uint32_t k = 0;
  for (uint32_t p = 0; p < n_parts; ++p) {
    P.a[p] = a_parts[p];
    P.koff[p] = k;
    k += part_k[p];
  }
  P.koff[n_parts] = k;
  P.n_parts = n_parts;
  for (uint32_t o = 0; o < n_outs; ++o) P.out[o] = outs[o];
  P.n_out = n_outs;
  P.ldc = ldc;
  launch_gemm(P, m, k, b, n, ordered, static_cast<cudaStream_t>(stream));
}

// CUDA IPC between the ranks of one node (one process per GPU): a rank
// exports a device buffer, its peers map it and read / write it over NVLink.
void ipc_handle(const void* dptr, unsigned char* out64, uint64_t* offset) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  // the handle names the whole allocation: find its base (a caching allocator
  // hands out pieces of larger allocations) through the driver entry point
  using range_fn = int (*)(unsigned long long*, size_t*, unsigned long long);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  ck(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q),
     "cudaGetDriverEntryPoint");
  if (!fn || q != cudaDriverEntryPointSuccess)
    throw cuda_error("cuMemGetAddressRange unavailable", CBM_B200_ECUDA);
  unsigned long long base = 0;
  size_t size = 0;
  if (reinterpret_cast<range_fn>(fn)(&base, &size, reinterpret_cast<unsigned long long>(dptr)) != 0)
    throw cuda_error("cuMemGetAddressRange failed", CBM_B200_ECUDA);
  cudaIpcMemHandle_t hnd;
  ck(cudaIpcGetMemHandle(&hnd, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle");
  std::memcpy(out64, &hnd, 64);
  *offset = reinterpret_cast<unsigned long long>(dptr) - base;
}

void* ipc_open(const unsigned char* in64, int device) {
  cudaIpcMemHandle_t hnd;
  std::memcpy(&hnd, in64, 64);
  if (device >= 0) ck(cudaSetDevice(device), "cudaSetDevice");
  void* p = nullptr;
  ck(cudaIpcOpenMemHandle(&p, hnd, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  return p;
}

void ipc_close(void* dptr) { ck(cudaIpcCloseMemHandle(dptr), "cudaIpcCloseMemHandle"); }

// gcn_forward (gcn.cpp:22-33): X W0 -> A_hat . -> relu -> A_hat . -> . W1, the
// ReLU fused into the first product's epilogue. Device pointers throughout.
void device_gcn_forward(DeviceMatrix* h, const float* x, uint32_t n, uint32_t f,
                        const float* w0, uint32_t hid, const float* w1, uint32_t classes,
                        float* out, void* stream) {
  ck(cudaSetDevice(h->device), "cudaSetDevice");
  const uint32_t hp = (hid + 3) & ~3u;
  auto& ws = h->ws[stream];
  grow(ws.gcn_h, ws.gcn_h_cap, uint64_t(n) * hp * 2, "gcn workspace");
  float* h0 = ws.gcn_h;
  float* h1 = ws.gcn_h + uint64_t(n) * hp;
  uint32_t launches = 0;
  // order-faithful handles keep the reference's GEMM arithmetic (bit-identical
  // gcn_forward); the default mode uses the FFMA GEMM (north_star tolerance)
  auto gemm = h->info.order_faithful ? device_dense_matmul : device_fast_matmul;
  gemm(x, n, f, w0, hid, h0, stream);  // packed n x hid
  ++launches;
  device_spmm(h, h0, hid, hid, h1, hid, stream, /*relu=*/true);
  launches += h->last_launches;
  device_spmm(h, h1, hid, hid, h0, hid, stream, /*relu=*/false);
  launches += h->last_launches;
  gemm(h0, n, hid, w1, classes, out, stream);
  h->last_launches = launches + 1;
}

}  // namespace cbmb
