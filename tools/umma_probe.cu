// Dev probe (not product code): validates the tcgen05 building blocks the
// dense-block kernel uses, on one CTA:
//   A (M=128 x K) written into TMEM with tcgen05.st (lane = row, one 32-bit
//   column per tf32 element), B (N x K, K-major) in shared memory with the
//   128-byte swizzle, tcgen05.mma.cta_group::1.kind::tf32 D[tmem] += A.B^T,
//   tcgen05.commit -> mbarrier, tcgen05.ld of D.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_probe tools/umma_probe.cu
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

constexpr int M = 128, N = 128, K = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t sw128_kmajor_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr & 0x3FFFF) >> 4);          // start address
  d |= uint64_t(1) << 16;                          // LBO (ignored for swizzled K-major)
  d |= uint64_t(1024 >> 4) << 32;                  // SBO: 8-row core-matrix groups
  d |= uint64_t(1) << 46;                          // version (sm_100)
  d |= uint64_t(2) << 61;                          // SWIZZLE_128B
  return d;
}

__global__ void probe(const float* a, const float* b, float* d, int variant) {
  __shared__ __align__(1024) float bs[N * K];  // 128 rows x 128 B
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // B: row n, 16-byte chunk j (4 floats) stored at chunk (j ^ (n & 7))
  for (int i = tid; i < N * (K / 4); i += blockDim.x) {
    const int n = i / (K / 4), j = i % (K / 4);
    float4 v = *reinterpret_cast<const float4*>(b + n * K + j * 4);
    char* dst = reinterpret_cast<char*>(bs) + (n >> 3) * 1024 + (n & 7) * 128 + ((j ^ (n & 7)) << 4);
    *reinterpret_cast<float4*>(dst) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tmem_base;
  // A: thread = row m = 32*warp + lane, columns [256, 256+K) of its lane
  {
    uint32_t r[32];
    for (int k = 0; k < 32; ++k) r[k] = __float_as_uint(a[(32 * warp + lane) * K + k]);
    const uint32_t addr = tb + ((uint32_t(32 * warp)) << 16) + 256;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31, %32};" ::"r"(addr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
        "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
        "r"(r[29]), "r"(r[30]), "r"(r[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) |
                           (uint32_t(M >> 4) << 24);
    for (int ks = 0; ks < K / 8; ++ks) {
      const uint32_t ta = tb + 256 + 8 * ks;       // A: 8 tf32 columns per K-step
      const uint64_t bd = sw128_kmajor_desc(smem_u32(bs) + 32 * ks);
      const uint32_t acc = ks > 0 ? 1u : 0u;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tb),
          "r"(ta), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
  }
  // wait for the MMA
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

int main() {
  std::vector<float> a(M * K), b(N * K), d(M * N), want(M * N, 0.f);
  srand(1);
  for (auto& v : a) v = float(rand() % 17 - 8);
  for (auto& v : b) v = float(rand() % 2);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      float s = 0;
      for (int k = 0; k < K; ++k) s += a[m * K + k] * b[n * K + k];
      want[m * N + n] = s;
    }
  float *da, *db, *dd;
  CK(cudaMalloc(&da, a.size() * 4));
  CK(cudaMalloc(&db, b.size() * 4));
  CK(cudaMalloc(&dd, d.size() * 4));
  CK(cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(dd, 0, d.size() * 4));
  probe<<<1, 128>>>(da, db, dd, 0);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int i = 0; i < M * N; ++i)
    if (d[i] != want[i]) {
      if (bad < 10) printf("mismatch m=%d n=%d got %g want %g\n", i / N, i % N, d[i], want[i]);
      ++bad;
    }
  printf("umma_probe tf32 A-in-TMEM M=%d N=%d K=%d: %d mismatches\n", M, N, K, bad);
  return bad != 0;
}
