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
}  // namespace

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
  device_dense_matmul(x, n, f, w0, hid, h0, stream);  // packed n x hid
  ++launches;
  device_spmm(h, h0, hid, hid, h1, hid, stream, /*relu=*/true);
  launches += h->last_launches;
  device_spmm(h, h1, hid, hid, h0, hid, stream, /*relu=*/false);
  launches += h->last_launches;
  device_dense_matmul(h0, n, hid, w1, classes, out, stream);
  h->last_launches = launches + 1;
}

}  // namespace cbmb
