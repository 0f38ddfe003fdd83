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

// dense_matmul (dense.cpp:31-49) with the reference's exact arithmetic:
// c[i,q] = sum over ascending j with a[i,j] != 0 of fl(a[i,j] * b[j,q]),
// each product rounded before the add, starting from +0. A CTA computes a
// 32-row x 128-column tile; b is staged through shared memory 32 rows of j at
// a time; the zero test is warp-uniform (a warp shares its row).
constexpr int kGemmRows = 32, kGemmCols = 128, kGemmK = 32;
template <bool MULTI>
__global__ void __launch_bounds__(256) ordered_gemm_kernel(const Parts P,
                                                           const float* __restrict__ b,
                                                           uint32_t m, uint32_t k, uint32_t n) {
  __shared__ float bs[kGemmK][kGemmCols];
  __shared__ float as[kGemmRows][kGemmK + 1];
  const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 lanes x 8 warps
  const uint32_t row0 = blockIdx.y * kGemmRows, col0 = blockIdx.x * kGemmCols;
  float acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[r][q] = 0.0f;
  for (uint32_t j0 = 0; j0 < k; j0 += kGemmK) {
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < kGemmK * kGemmCols; e += 256) {
      const uint32_t jj = e / kGemmCols, cc = e % kGemmCols;
      bs[jj][cc] = (j0 + jj < k && col0 + cc < n) ? b[(size_t)(j0 + jj) * n + col0 + cc] : 0.0f;
    }
    for (uint32_t e = threadIdx.x; e < kGemmRows * kGemmK; e += 256) {
      const uint32_t rr = e / kGemmK, jj = e % kGemmK;
      as[rr][jj] = (row0 + rr < m && j0 + jj < k) ? load_a<MULTI>(P, row0 + rr, j0 + jj) : 0.0f;
    }
    __syncthreads();
    const uint32_t jn = min(uint32_t(kGemmK), k - j0);
    for (uint32_t jj = 0; jj < jn; ++jj) {
      float bv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) bv[q] = bs[jj][tx + 32 * q];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const float av = as[ty + 8 * r][jj];
        if (av != 0.0f) {  // dense.cpp:42 skips zero lhs entries
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[r][q] = __fadd_rn(acc[r][q], __fmul_rn(av, bv[q]));
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint32_t i = row0 + ty + 8 * r;
    if (i >= m) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t cc = col0 + tx + 32 * q;
      if (cc < n) store_c<MULTI>(P, i, cc, acc[r][q]);
    }
  }
}

// Default-mode GEMM of the GCN (within the north_star tolerance, not bit-exact):
// FFMA, 128 x 128 output tile per CTA, 8 x 8 per thread, k staged 8 at a time
// (A transposed in shared memory). Finite operands assumed: a zero lhs entry
// contributes fma(0, b, acc) = acc like dense.cpp:42's skip. Part widths are
// multiples of 4 (column_slab), so a 4-wide k group never straddles two parts.
constexpr int kFB = 128, kFK = 8;
template <bool MULTI>
__global__ void __launch_bounds__(256, 2) fast_gemm_kernel(const Parts P,
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
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t kk = k0 + ak + i;
      av[i] = (row0 + ar < m && kk < k) ? load_a<MULTI>(P, row0 + ar, kk) : 0.0f;
      const uint32_t cc = col0 + bc + i;
      bv[i] = (k0 + bk < k && cc < n) ? __ldg(b + (size_t)(k0 + bk) * n + cc) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) as[ak + i][ar] = av[i];
    *reinterpret_cast<float4*>(&bs[bk][bc]) = make_float4(bv[0], bv[1], bv[2], bv[3]);
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kFK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&as[kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&as[kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&bs[kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&bs[kk][64 + tx * 4]);
      const float ar8[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float br8[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[r][q] = __fmaf_rn(ar8[r], br8[q], acc[r][q]);
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
  if (ordered) {
    const dim3 grid((n + kGemmCols - 1) / kGemmCols, (m + kGemmRows - 1) / kGemmRows);
    if (multi) ordered_gemm_kernel<true><<<grid, 256, 0, s>>>(P, b, m, k, n);
    else ordered_gemm_kernel<false><<<grid, 256, 0, s>>>(P, b, m, k, n);
  } else {
    const dim3 grid((n + kFB - 1) / kFB, (m + kFB - 1) / kFB);
    if (multi) fast_gemm_kernel<true><<<grid, 256, 0, s>>>(P, b, m, k, n);
    else fast_gemm_kernel<false><<<grid, 256, 0, s>>>(P, b, m, k, n);
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
