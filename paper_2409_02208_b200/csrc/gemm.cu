// Reference-order dense GEMM (dense.cpp:31-49) and the GCN forward
// (gcn.cpp:22-33) built from it and the CBM multiply.
#include "cuda_common.hpp"

namespace cbmb {

namespace {
// dense_matmul (dense.cpp:31-49) with the reference's exact arithmetic:
// c[i,q] = sum over ascending j with a[i,j] != 0 of fl(a[i,j] * b[j,q]),
// each product rounded before the add, starting from +0. A CTA computes a
// 32-row x 128-column tile; b is staged through shared memory 32 rows of j at
// a time; the zero test is warp-uniform (a warp shares its row).
constexpr int kGemmRows = 32, kGemmCols = 128, kGemmK = 32;
__global__ void __launch_bounds__(256) ordered_gemm_kernel(const float* __restrict__ a,
                                                           const float* __restrict__ b,
                                                           float* __restrict__ c, uint32_t m,
                                                           uint32_t k, uint32_t n) {
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
      as[rr][jj] = (row0 + rr < m && j0 + jj < k) ? a[(size_t)(row0 + rr) * k + j0 + jj] : 0.0f;
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
      if (cc < n) c[(size_t)i * n + cc] = acc[r][q];
    }
  }
}

// Default-mode GEMM of the GCN (within the north_star tolerance, not bit-exact):
// FFMA, 128 x 128 output tile per CTA, 8 x 8 per thread, k staged 8 at a time
// (A transposed in shared memory). Finite operands assumed: a zero lhs entry
// contributes fma(0, b, acc) = acc like dense.cpp:42's skip.
constexpr int kFB = 128, kFK = 8;
__global__ void __launch_bounds__(256, 2) fast_gemm_kernel(const float* __restrict__ a,
                                                           const float* __restrict__ b,
                                                           float* __restrict__ c, uint32_t m,
                                                           uint32_t k, uint32_t n) {
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
      av[i] = (row0 + ar < m && kk < k) ? __ldg(a + (size_t)(row0 + ar) * k + kk) : 0.0f;
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
      if (cc < n) c[(size_t)i * n + cc] = acc[r][q];
    }
  }
}
}  // namespace

void device_fast_matmul(const float* a, uint32_t m, uint32_t k, const float* b, uint32_t n,
                        float* c, void* stream) {
  if (m == 0 || n == 0) return;
  const dim3 grid((n + kFB - 1) / kFB, (m + kFB - 1) / kFB);
  fast_gemm_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(a, b, c, m, k, n);
  ck(cudaGetLastError(), "fast_gemm launch");
}

void device_dense_matmul(const float* a, uint32_t m, uint32_t k, const float* b, uint32_t n,
                         float* c, void* stream) {
  if (m == 0 || n == 0) return;
  const dim3 grid((n + kGemmCols - 1) / kGemmCols, (m + kGemmRows - 1) / kGemmRows);
  ordered_gemm_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(a, b, c, m, k, n);
  ck(cudaGetLastError(), "ordered_gemm launch");
}

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
