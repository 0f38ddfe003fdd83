// Dev probe (not product code): the bf16 form of the dense-block product.
//   A (M=128 x K=64) in TMEM as packed bf16 pairs (lane = row; column j holds
//   K elements 2j (low half) and 2j+1 (high half)), three terms b1+b2+b3 = x
//   (exact 8+8+8-bit split of an fp32 value), B (N x 64, K-major, 0/1 in bf16)
//   in shared memory with the 128-byte swizzle,
//   tcgen05.mma.cta_group::1.kind::f16 (bf16 x bf16 -> f32), 4 K-steps of 16.
// Checks: integer X exact; N(0,1)-like X against the f64 sum.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_probe_bf16 tools/umma_probe_bf16.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                \
    }                                                                          \
  } while (0)

constexpr int M = 128, K = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sw128_kmajor_desc(uint32_t saddr) {
  return uint64_t((saddr & 0x3FFFF) >> 4) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

// x = b1 + b2 + b3 exactly: each term the top 8 significant bits of what is left
__device__ __forceinline__ void split3(float x, uint32_t& h1, uint32_t& h2, uint32_t& h3) {
  const uint32_t u1 = __float_as_uint(x) & 0xFFFF0000u;
  const float r1 = __fsub_rn(x, __uint_as_float(u1));
  const uint32_t u2 = __float_as_uint(r1) & 0xFFFF0000u;
  const float r2 = __fsub_rn(r1, __uint_as_float(u2));
  h1 = u1 >> 16;
  h2 = u2 >> 16;
  h3 = __float_as_uint(r2) >> 16;   // <= 8 significant bits left: exact
}

template <int N>
__global__ void probe(const float* a, const unsigned char* b, float* d) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* bs = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // B: row n (N rows of 64 bf16 = 128 B), 16-byte chunk j stored at chunk j ^ (n & 7)
  for (int i = tid; i < N * 8; i += blockDim.x) {
    const int n = i / 8, j = i % 8;
    uint32_t w[4];
    for (int e = 0; e < 4; ++e) {
      const uint32_t lo = b[n * K + 8 * j + 2 * e] ? 0x3F80u : 0u;
      const uint32_t hi = b[n * K + 8 * j + 2 * e + 1] ? 0x3F80u : 0u;
      w[e] = lo | (hi << 16);
    }
    unsigned char* dst = bs + (n >> 3) * 1024 + (n & 7) * 128 + ((j ^ (n & 7)) << 4);
    *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tmem_base;
  // A terms: term t at columns [256 + 32 t, 256 + 32 t + 32)
  {
    const int m = 32 * warp + lane;
    uint32_t t1[32], t2[32], t3[32];
    for (int j = 0; j < 32; ++j) {
      uint32_t a1, a2, a3, c1, c2, c3;
      split3(a[m * K + 2 * j], a1, a2, a3);
      split3(a[m * K + 2 * j + 1], c1, c2, c3);
      t1[j] = a1 | (c1 << 16);
      t2[j] = a2 | (c2 << 16);
      t3[j] = a3 | (c3 << 16);
    }
    const uint32_t addr = tb + ((uint32_t(32 * warp)) << 16) + 256;
#define ST32(off, r)                                                                             \
  asm volatile(                                                                                  \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, " \
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "    \
      "%28, %29, %30, %31, %32};" ::"r"(addr + off),                                             \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),    \
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),          \
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),        \
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),        \
      "r"(r[29]), "r"(r[30]), "r"(r[31]))
    ST32(0, t1);
    ST32(32, t2);
    ST32(64, t3);
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    // D f32, A bf16, B bf16, both K-major
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) |
                           (uint32_t(M >> 4) << 24);
    for (int term = 0; term < 3; ++term)
      for (int ks = 0; ks < K / 16; ++ks) {
        const uint32_t ta = tb + 256 + 32 * term + 8 * ks;   // 8 packed columns per K-step
        const uint64_t bd = sw128_kmajor_desc(smem_u32(bs)) + 2 * ks;
        const uint32_t acc = (term | ks) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tb),
            "r"(ta), "l"(bd), "r"(idesc), "r"(acc));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
  }
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(smem_u32(&bar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t r[32];
    const uint32_t addr = tb + ((uint32_t(32 * warp)) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 32; ++j) d[(32 * warp + lane) * N + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

template <int N>
int run(bool integers) {
  std::vector<float> a(M * K), d(M * N);
  std::vector<unsigned char> b(N * K);
  std::vector<double> want(M * N, 0.0);
  srand(integers ? 1 : 2);
  for (auto& v : a)
    v = integers ? float(rand() % 17 - 8)
                 : float((rand() / double(RAND_MAX) - 0.5) * 6.0 * std::exp((rand() % 9) - 4.0));
  for (auto& v : b) v = (unsigned char)(rand() % 5 != 0);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += double(a[m * K + k]) * b[n * K + k];
      want[m * N + n] = s;
    }
  float *da, *dd;
  unsigned char* db;
  CK(cudaMalloc(&da, a.size() * 4));
  CK(cudaMalloc(&db, b.size()));
  CK(cudaMalloc(&dd, d.size() * 4));
  CK(cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dd, 0, d.size() * 4));
  const int smem = N * 128 + 1024;
  CK(cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe<N><<<1, 128, smem>>>(da, db, dd);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  double worst = 0, scale = 0;
  for (int i = 0; i < M * N; ++i) scale = std::fmax(scale, std::fabs(want[i]));
  for (int i = 0; i < M * N; ++i) {
    const double e = std::fabs(double(d[i]) - want[i]);
    worst = std::fmax(worst, e);
    if (integers ? e != 0.0 : e > 1e-6 * scale) {
      if (bad < 6) printf("  mismatch m=%d n=%d got %.9g want %.9g\n", i / N, i % N, d[i], want[i]);
      ++bad;
    }
  }
  printf("umma_probe_bf16 N=%d %s: %d mismatches, max|err|/max|want| = %.3g\n", N,
         integers ? "integer X (exact)" : "float X (3-term split)", bad, worst / scale);
  cudaFree(da);
  cudaFree(db);
  cudaFree(dd);
  return bad != 0;
}

int main() {
  int rc = 0;
  rc |= run<128>(true);
  rc |= run<128>(false);
  rc |= run<256>(true);
  rc |= run<256>(false);
  return rc;
}
